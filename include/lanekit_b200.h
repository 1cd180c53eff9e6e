/*
 * lanekit_b200.h — C-ABI drop-in for stages 5–12 of lanekit's run_pipeline
 * (grey frame + dense disparity in, lane positions + per-stage hooks out),
 * executed by hand-written sm_100a CUDA kernels.
 *
 * Reference interface replaced (all paths under /root/reference/proj/include/lanekit/):
 *   - lanekit::PipelineConfig            config.hpp:16-46      -> lk_config
 *   - lanekit::validate_config           config.hpp:124-152    -> lk_validate_config
 *   - lanekit::run_pipeline, stages 5-12 pipeline.hpp:184-270  -> lk_run_batch
 *     (the disparity map is injected instead of being produced by stages 1-4)
 *   - lanekit::PipelineReport            pipeline.hpp:30-66    -> lk_frame_report
 *   - lanekit::PipelineResult members    pipeline.hpp:69-99    -> lk_get_stage (per-stage hooks)
 *   - lanekit::StageTiming / run_stage   pipeline.hpp:24-28,138-150 -> lk_stage_times
 *   - lanekit::StageError                common.hpp:18-24      -> per-frame status/failed_stage/msg
 *   - lanekit::gen_scene                 synth.hpp:103-200     -> lk_synth_scene (test-kit input generator)
 *
 * Conventions: no exceptions cross this boundary; every entry point returns
 * an lk_status; lk_last_error() describes the most recent failure on the
 * calling thread. A context owns its device buffers, stream and CUDA graphs;
 * one context per host thread (thread-compatible, not internally locked).
 * Frames are independent: a frame that fails a stage reports that stage in
 * its lk_frame_report and never aborts the rest of the batch.
 */
#ifndef LANEKIT_B200_H
#define LANEKIT_B200_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define LK_ABI_VERSION 1
#define LK_MAX_INLINE_LANES 16

typedef enum lk_status {
    LK_OK = 0,
    LK_ERR_INVALID_ARGUMENT = 1, /* bad pointer / size / frame index            */
    LK_ERR_CONFIG = 2,           /* validate_config rejected the config          */
    LK_ERR_CUDA = 3,             /* CUDA runtime error (see lk_last_error)       */
    LK_ERR_NO_DEVICE = 4,        /* no sm_100 device / extension not usable      */
    LK_ERR_FRAME = 5,            /* at least one frame failed a stage            */
    LK_ERR_UNAVAILABLE = 6       /* hook not captured (enable LK_FLAG_HOOKS)     */
} lk_status;

/* Mirrors lanekit::PipelineConfig field for field (config.hpp:16-46), same
 * defaults (lk_config_default). Stereo-only fields (rho, tau, tr_lrc,
 * sigma_floor) are validated for drop-in fidelity but unused on this path.
 * tr_lpv = NaN means "auto" (config.hpp:40). */
typedef struct lk_config {
    int32_t rho;
    int32_t tau;
    int32_t d_max;
    int32_t tr_lrc;
    double sigma_floor;
    double lambda_y;
    double tr_y;
    double eps_y;
    double varpi;
    double sigma_s;
    double sigma_r;
    int32_t bf_window;
    int32_t chi;
    double sobel_threshold;
    double rho_vote;
    double lambda_x;
    double tr_x;
    double eps_x;
    double sigma_g;
    int32_t nu;
    int32_t varsigma;
    double lambda_g;
    double xi;
    double tr_lpv;
    int32_t min_lane_sep;
    int32_t paper_sign;
    uint64_t rng_seed;
    int32_t threads; /* CLI-level knob (config.hpp:45); results never depend on it */
    int32_t _pad0;
} lk_config;

/* Per-frame message ids; lk_frame_message() renders the reference's text,
 * "stage N (name): msg" (pipeline.hpp:138-150). */
typedef enum lk_msg {
    LK_MSG_NONE = 0,
    LK_MSG_EMPTY_INPUT = 1,          /* stage 1: empty input image                         */
    LK_MSG_NO_ROAD_EVIDENCE = 2,     /* stage 6: pipeline.hpp:189-190                      */
    LK_MSG_RANSAC_FEW_POINTS = 3,    /* stage 7/11: ransac.hpp:41-42                       */
    LK_MSG_RANSAC_NO_FIT = 4,        /* stage 7/11: ransac.hpp:90                          */
    LK_MSG_SINGULAR_VPY = 5,         /* stage 7: road_profile.hpp:223-225 (err_row)        */
    LK_MSG_SOBEL_TOO_SMALL = 6,      /* stage 10: preprocess.hpp:69                        */
    LK_MSG_NO_EDGE_EVIDENCE = 7,     /* stage 11: pipeline.hpp:238-239                     */
    LK_MSG_M1_TOO_SMALL = 8,         /* stage 12: lanes.hpp:68                             */
    LK_MSG_BAD_DIMENSIONS = 9        /* stage 1: grey/disparity sizes differ               */
} lk_msg;

/* Mirrors lanekit::PipelineReport (pipeline.hpp:30-66) minus the stage
 * timings (see lk_stage_times). Every field is 8 bytes wide so the record
 * has one layout on host and device. */
typedef struct lk_frame_report {
    int64_t status;            /* 0 = ok, else LK_ERR_FRAME                          */
    int64_t failed_stage;      /* 0, or the reference's stage number (1, 5..12)      */
    int64_t msg;               /* lk_msg                                             */
    int64_t err_row;           /* row for LK_MSG_SINGULAR_VPY                        */
    int64_t width;
    int64_t height;
    uint64_t rng_seed;
    int64_t valid_disparities; /* non-zero disparities of the injected map           */
    int64_t vpath_has_evidence;
    double vpath_energy;
    double beta[3];
    int64_t beta_iterations;
    double beta_inlier_fraction;
    int64_t beta_degraded;
    int64_t beta_inlier_count;
    int64_t horizon;
    int64_t horizon_in_range;
    int64_t road_mask_pixels;
    int64_t edge_pixels;
    int64_t vpx_votes;
    int64_t vpx_skipped;
    int64_t upath_has_evidence;
    double upath_energy;
    double gamma[5];
    double gamma_kappa;
    double gamma_v_normalizer;
    int64_t gamma_iterations;
    double gamma_inlier_fraction;
    int64_t gamma_degraded;
    int64_t gamma_inlier_count;
    double tr_lpv_used;
    int64_t lane_count;        /* full count; first LK_MAX_INLINE_LANES inline below */
    int64_t lane_bottom_col[LK_MAX_INLINE_LANES];
    double lane_energy[LK_MAX_INLINE_LANES];
    /* Certificate of the lane decisions (not a reference field; 0 from the
     * CPU checkers): the number of integer decisions whose outcome the GPU's
     * libdevice atan2 / exp (<= 2 ulp from glibc) could have flipped, i.e. the
     * w_g gates within 1e-12 of pi/6 and the lane-minimum / threshold /
     * order comparisons within their propagated error bounds. 0 means the
     * lane columns and polyline lengths equal the reference's exactly. */
    int64_t uncertain;
} lk_frame_report;

/* Per-stage hooks: the PipelineResult members (pipeline.hpp:69-99). Layouts:
 *   VDISPARITY   int32 [H][d_max+1]                       (VDisparityHist.count)
 *   VPATH        int32 [d_max+1][2]  (d, v) in stage order (DpPath.points)
 *   BETA_INLIERS int32 [n][2]        (d, v)
 *   VPY          f64  [H]           VPY_SINGULAR u8 [H]
 *   MASK         u8   [H][W]                    (hooks flag)
 *   SMOOTHED     f64  [H][W]
 *   GX/GY/MAG/THETA f64 [H][W]                  (hooks flag)
 *   EDGES        lk_edge [n]         row-major order (EdgeSet.pixels)
 *   VOTES        lk_vote [n]         (SparseVpxMap.votes)
 *   VPX_ACC      f64  [H-horizon][ext_cols]     (hooks flag)
 *   UPATH        int32 [H-horizon][2] (ext col, v) in stage order
 *   GAMMA_INLIERS int32 [n][2]       (u, v)
 *   VPX          f64  [H]
 *   M0           f64  [H][W]                    (hooks flag)
 *   M1           f64  [H][W]
 *   ENERGY       f64  [ext_cols]
 *   LANES        lk_lane [lane_count]
 *   POLYLINES    f64 [lane_count][H-horizon]  track u per row v_top..v_max, NaN = truncated
 */
typedef enum lk_stage {
    LK_STAGE_VDISPARITY = 0,
    LK_STAGE_VPATH = 1,
    LK_STAGE_BETA_INLIERS = 2,
    LK_STAGE_VPY = 3,
    LK_STAGE_VPY_SINGULAR = 4,
    LK_STAGE_MASK = 5,
    LK_STAGE_SMOOTHED = 6,
    LK_STAGE_GX = 7,
    LK_STAGE_GY = 8,
    LK_STAGE_MAG = 9,
    LK_STAGE_THETA = 10,
    LK_STAGE_EDGES = 11,
    LK_STAGE_VOTES = 12,
    LK_STAGE_VPX_ACC = 13,
    LK_STAGE_UPATH = 14,
    LK_STAGE_GAMMA_INLIERS = 15,
    LK_STAGE_VPX = 16,
    LK_STAGE_M0 = 17,
    LK_STAGE_M1 = 18,
    LK_STAGE_ENERGY = 19,
    LK_STAGE_LANES = 20,
    LK_STAGE_POLYLINES = 21,
    /* stereo contexts (LK_FLAG_STEREO): PipelineResult members of stages 1-4 */
    LK_STAGE_STATS_MU = 22,    /* f64 [H][W] stats_left.mu (0 on the border)      */
    LK_STAGE_STATS_SIGMA = 23, /* f64 [H][W] stats_left.sigma                     */
    LK_STAGE_DISP_LEFT = 24,   /* u8 [H][W] match_srp, left reference             */
    LK_STAGE_DISP_RIGHT = 25,  /* u8 [H][W] match_srp, right reference            */
    LK_STAGE_DISPARITY = 26,   /* u8 [H][W] lrc_check result (input of stage 5)   */
    LK_STAGE_COUNT = 27
} lk_stage;

typedef struct lk_edge {   /* lanekit::EdgePixel (preprocess.hpp:92-95) */
    int32_t u, v;
    double gx, gy, theta;
} lk_edge;

typedef struct lk_vote {   /* lanekit::SparseVpxMap::Vote (vanish.hpp:35-38) */
    int32_t u_e, v_e, col;
} lk_vote;

typedef struct lk_lane {   /* lanekit::Lane (lanes.hpp:131-135) minus the polyline */
    int32_t bottom_col;
    int32_t n_points;      /* non-NaN rows of the track = polyline length */
    double energy;
} lk_lane;

/* Context flags. */
#define LK_FLAG_HOOKS 1u   /* also materialise mask, gx/gy/mag/theta, accumulator, m0 */
#define LK_FLAG_NO_GRAPH 2u /* launch kernels directly instead of replaying a CUDA graph */
#define LK_FLAG_STEREO 8u  /* also run stages 1-4 (stereo.hpp): stereo pair in, the whole
                              * run_pipeline (pipeline.hpp:118-270); needs d_max <= 255 and
                              * a block radius rho of 1..5 */
#define LK_FLAG_EXACT 4u    /* exact bilateral on every pixel even without hooks (the
                               default throughput path computes it exactly only around
                               edge candidates; outputs are identical either way) */

typedef struct lk_ctx lk_ctx;

/* Where lk_run_batch's input pointers live. */
typedef enum lk_mem { LK_MEM_HOST = 0, LK_MEM_DEVICE = 1 } lk_mem;

void lk_config_default(lk_config* cfg);
lk_status lk_validate_config(const lk_config* cfg);
const char* lk_last_error(void);
int lk_abi_version(void);
const char* lk_stage_name(int stage); /* 1..12, pipeline.hpp:101-116 */
/* Renders "stage N (name): msg" for a failed frame into buf. */
lk_status lk_frame_message(const lk_frame_report* rep, char* buf, size_t len);

lk_status lk_create(lk_ctx** out, int device, const lk_config* cfg, int width, int height,
                    int max_batch, uint32_t flags);
lk_status lk_destroy(lk_ctx* ctx);

/* Runs stages 5-12 on n frames. grey: u8 [n][H][W], value k means k/255.0
 * (image_io.hpp:147); disparity: u8 [n][H][W] (0 = invalid). reports may be
 * NULL. Returns LK_ERR_FRAME when some frame failed (details per report). */
lk_status lk_run_batch(lk_ctx* ctx, const uint8_t* grey, const uint8_t* disparity, int n,
                       lk_mem where, lk_frame_report* reports);

/* Device-resident variant for throughput runs: the frames are already in
 * the context's input buffers (lk_device_inputs), results stay on the device
 * until lk_fetch_reports. Asynchronous on the context stream. */
lk_status lk_device_inputs(lk_ctx* ctx, uint8_t** grey, uint8_t** disparity);
lk_status lk_enqueue(lk_ctx* ctx, int n);

/* Streaming host-fed batches: batch k+1's host-to-device copy (a copy stream,
 * two input slots) overlaps batch k's kernels. lk_submit_batch queues the copy
 * of grey/disparity (u8 [n][H][W], pinned: lk_host_alloc), the pipeline and the
 * read-back of the n reports into `reports` (pinned; may be NULL), and returns
 * without waiting. Up to two batches are in flight: a third submit first waits
 * for the oldest. lk_wait_batch waits for the oldest submitted batch and
 * returns its status (LK_ERR_FRAME when one of its frames failed). The host
 * buffers of a batch must stay untouched until it has been waited for. */
lk_status lk_submit_batch(lk_ctx* ctx, const uint8_t* grey, const uint8_t* disparity, int n,
                          lk_frame_report* reports);
/* The same stream of stereo pairs (LK_FLAG_STEREO contexts): left/right u8
 * [n][H][W] in, stages 1-12 (run_pipeline, pipeline.hpp:118-270) per batch. */
lk_status lk_submit_stereo_batch(lk_ctx* ctx, const uint8_t* left, const uint8_t* right, int n,
                                 lk_frame_report* reports);
/* Device-resident stream (BASELINE config 5): the pipeline over the frames
 * already in the input buffers (lk_device_inputs), and the asynchronous
 * read-back of their n reports into `reports` (pinned; may be NULL), queued
 * like lk_submit_batch (at most two in flight; lk_wait_batch). */
lk_status lk_submit_resident(lk_ctx* ctx, int n, lk_frame_report* reports);
lk_status lk_wait_batch(lk_ctx* ctx);
lk_status lk_fetch_reports(lk_ctx* ctx, lk_frame_report* reports, int n);
lk_status lk_synchronize(lk_ctx* ctx);
void* lk_stream(lk_ctx* ctx); /* cudaStream_t of the context */

/* Copies hook `stage` of batch frame `frame` into dst (capacity bytes);
 * *needed receives the full size in bytes. dst may be NULL to query. */
lk_status lk_get_stage(lk_ctx* ctx, int frame, int stage, void* dst, size_t capacity,
                       size_t* needed);

/* Device milliseconds of the last batch per pipeline stage 5..12 (ms[5..12]),
 * from CUDA events recorded on the context stream around each stage's kernels
 * (event-record nodes inside the CUDA graph); ms[0] is the whole batch.
 * Stage 8 (road mask) is fused into stage 10's Sobel pass and reads ~0.
 * A captured batch runs as up to LK_BRANCHES (env, default 4) concurrent
 * frame ranges; the events time the first range (lk_timed_frames frames)
 * while the others overlap it. ms[0] is then that range's span. */
lk_status lk_stage_times(lk_ctx* ctx, float ms[13]);

/* Frames of the last batch covered by lk_stage_times. */
int lk_timed_frames(lk_ctx* ctx);

/* ---- stereo pair in (LK_FLAG_STEREO contexts): run_pipeline itself.
 * lanekit::run_pipeline(left, right, cfg)      pipeline.hpp:118-270 -> lk_run_stereo_batch
 *   stage 1 precompute_stats                   stereo.hpp:39-60     (both images)
 *   stages 2/3 match_srp, left / right ref     stereo.hpp:157-196
 *   stage 4 lrc_check                          stereo.hpp:263-276   -> the stage-5 disparity
 * left/right: u8 [n][H][W] (k means k/255.0, image_io.hpp:147). Reports as lk_run_batch;
 * lk_stage_times then also fills ms[1..4] (the two SRP views run as one launch: ms[3] ~ 0). */
lk_status lk_run_stereo_batch(lk_ctx* ctx, const uint8_t* left, const uint8_t* right, int n,
                              lk_mem where, lk_frame_report* reports);
/* Device buffers [max_batch][H][W] for the left / right grey of lk_enqueue_stereo. */
lk_status lk_stereo_inputs(lk_ctx* ctx, uint8_t** left, uint8_t** right);
/* Enqueues stages 1-12 on frames already in the stereo input buffers (asynchronous). */
lk_status lk_enqueue_stereo(lk_ctx* ctx, int n);

/* Measured FP64 add+mul issue rate of this device (ops/s), for rooflines. */
lk_status lk_measure_fp64(int device, double* ops_per_s);

/* Number of kernel launches one lk_run_batch / lk_enqueue issues (all
 * branches of the last batch size, else of max_batch). */
int lk_launches_per_batch(lk_ctx* ctx);

/* Largest |approximate - exact| smoothed value over the last batch: verifies
 * the fast path's error bound (2.5e-5) by also running the exact bilateral on
 * every pixel. LK_ERR_UNAVAILABLE when the context uses the exact path. */
lk_status lk_fast_path_error(lk_ctx* ctx, double* max_abs_error);

/* Host-to-device bytes the context has copied so far (host-fed inputs). On
 * the streaming fast path (lk_submit_batch, no LK_FLAG_HOOKS) a batch's grey
 * is copied only from row min_f(horizon_f - 1 - rho) down, per frame chunk
 * (LK_ROAD_CHUNKS, default 2): the chunk's disparity is copied first, stages
 * 5-7 of the chunk run on a side stream, and the call waits for them (the
 * previous batch keeps computing) before queuing the grey rows stages 8-12
 * read (the mask is empty above the horizon, preprocess.hpp:18).
 * After a batch whose rows above the horizons were < 15 % of its grey (a
 * high-resolution frame with a high horizon), whole frames are copied without
 * waiting, re-probing every 16th batch. LK_ROAD_COPY=0 in the environment at
 * lk_create always copies whole frames. */
lk_status lk_h2d_bytes(lk_ctx* ctx, unsigned long long* bytes);

/* Page-locked host buffers for host-fed (end-to-end) runs. */
lk_status lk_host_alloc(void** ptr, size_t bytes);
lk_status lk_host_free(void* ptr);

/* sizeof of lk_config, lk_frame_report, lk_scene_params, lk_edge, lk_vote,
 * lk_lane (in that order) — lets bindings verify their struct layouts. */
void lk_abi_sizes(size_t out[6]);

/* ---- synthetic input generator: restates lanekit::gen_scene (synth.hpp:103-200)
 * and extends it with obstacles and a pitch change (stress config). Output is
 * the 8-bit quantisation lround(x*255) clamped (image_io.hpp:184-193). */
typedef struct lk_scene_params {
    int32_t width, height;
    double beta[3];
    double gamma[5];
    int32_t d_max;
    int32_t n_lanes;
    double lane_bottoms[8];
    double lane_width;
    double lane_brightness;
    double road_base;
    double sky_level;
    double texture_amplitude;
    double noise_sigma;
    uint64_t rng_seed;
    /* extensions (not in the reference): obstacles and a pitch change */
    int32_t n_obstacles;
    int32_t pitch_row;        /* < 0: none; else the profile becomes linear above it */
    double pitch_jump;        /* relative slope jump at pitch_row                      */
    int32_t obstacle_box[4][4]; /* u0, v0, u1, v1 inclusive                            */
    int32_t obstacle_disp[4];
} lk_scene_params;

void lk_scene_default(lk_scene_params* p); /* SceneParams defaults (synth.hpp:62-80) */
/* grey_l/grey_r/disparity: u8 [H][W] (any may be NULL); returns LK_ERR_INVALID_ARGUMENT
 * with lk_last_error() set to the reference's "scene: ..." message on bad params. */
lk_status lk_synth_scene(const lk_scene_params* p, uint8_t* grey_l, uint8_t* grey_r,
                         uint8_t* disparity, int32_t* horizon);
/* n scenes in parallel on host threads: params[i] -> frame i. */
lk_status lk_synth_batch(const lk_scene_params* params, int n, uint8_t* grey, uint8_t* disparity,
                         int threads);
/* Same, with the right view too (any output may be NULL). */
lk_status lk_synth_stereo_batch(const lk_scene_params* params, int n, uint8_t* left,
                                uint8_t* right, uint8_t* disparity, int threads);

#ifdef __cplusplus
}
#endif
#endif /* LANEKIT_B200_H */
