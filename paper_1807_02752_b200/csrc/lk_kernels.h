// lk_kernels.h — host-visible launch plan for the stage kernels.
#pragma once

#include <cuda_runtime.h>

#include "lk_device.cuh"

namespace lkg {

constexpr int K1_ROWS = 32;             // rows per v-disparity CTA
constexpr int BF_TW = 32, BF_TH = 8;    // bilateral tile (generic window)
constexpr int BT_W = 64, BT_H = 16, BT_R = 4;  // bilateral tile (11x11), outputs per thread
constexpr int BT_TRI_N = 128;           // max distinct values per tile for the smem sub-table
constexpr int K4_THREADS = 512;         // V_px CTA (2 per SM)
#ifndef GAMMA_NW
#define GAMMA_NW 8                      // RANSAC-gamma warps = speculative iterations per round
#endif
constexpr int K4_VOTE_CAP = 8192;       // edges whose vote columns are staged in smem
constexpr int BT_CHUNK = 32;            // u-path backtrack: stages per window
constexpr int BT_SPAN = 5 * BT_CHUNK;   // max drift inside a window (|offset| <= 5)
constexpr int M_TW = 128;               // m0/m1 tile width
constexpr int SB_TW = 128, SB_TH = 16;  // Sobel tile; SB_TW is the edge-list segment width
constexpr int SB_PPT = SB_TH / 2;       // fast-path Sobel pixels per thread (256 threads)

// 11x11 spatial weights exp(-ds*inv_s2), passed by value (constant bank)
struct WsParam {
    double w[121];
};

// Certified pre-screen (k_prescreen): constants of the bound |s - b| <= E on
// the gap between the bilateral s and the 11x11 box mean b,
// each rounded so the bound stays an upper bound.
struct PrescreenParam {
    float kappa;     // inv_r2 = 1 / sigma_r^2 (range exponent per unit dr^2), rounded up
    float inv_wmin;  // 1 / (smallest spatial weight of the window), rounded up
    float ew;        // inv_wmin - 1, rounded up
    float fmax;      // sup over 0 < x <= 1 of (1 - exp(-kappa x^2)) / x, rounded up
    float c1;        // 1 / (121 * 255), rounded up
    float c2;        // 1 / (121 * 255^2), rounded up
    float s_star_lo; // largest float <= the exact Sobel threshold s*
};

// Need-list bilateral (k_bilateral_need): the spatial factor of every tap
// (j-major) as float; the range factors come from a shared (R, R*delta) table.
struct NeedBfParam {
    float S[121];
};

struct LaunchPlan {
    WsParam ws;
    PrescreenParam ps;
    NeedBfParam nbf;
    int need_ctas;            // persistent k_bilateral_need CTAs
    int fast_width;           // frame width (k_prescreen's block shape)
    int fast_front;           // certified fast bilateral + exact refinement (lk_fastpath.cu)
    int refine_ctas, decide_ctas;  // per-frame grids of k_refine_exact / k_sobel_decide
    int32_t* vhistT;          // [B][D1][H] transposed v-disparity for the v-path DP
    size_t vdisp_smem;        // k_vdisparity: barrier + histogram rows + staged bytes
    size_t vpath_smem;
    int vpath_choice_smem;    // choices of the v-path DP kept in shared memory
    size_t road_smem;
    size_t bf_smem;
    size_t bt_smem;
    int bt_mode;              // bilateral table path (see k_bilateral_tile)
    size_t vanish_smem;
    int upath_sp;             // u-path DP states per thread (0 = strided fallback)
    int upath_nt;             // u-path DP threads per CTA (512 or 1024)
    size_t gamma_smem;
    size_t m_smem;
    int m_tile_h;
    int collect_blocks;
    size_t select_smem;
    int sort_cap;
};

// Enqueues stages 5-12 for n frames on stream s. stage_ev (13 events, may
// be null) are recorded at the stage boundaries: [0] start, [k] end of stage k.
cudaError_t launch_pipeline(const Dev& d, const LaunchPlan& lp, int n, cudaStream_t s,
                            cudaEvent_t* stage_ev, bool mark_start = true);
// Stages 1-4 (lk_stereo.cu): events [0] start, [1] stats, [2]/[3] both SRP views, [4] LRC.
cudaError_t launch_stereo(const Dev& d, int n, cudaStream_t s, cudaEvent_t* stage_ev);
cudaError_t configure_stereo(const Dev& d);
size_t stereo_smem(const Dev& d);
int stereo_launches();
cudaError_t configure_kernels(const LaunchPlan& lp);
int vdisparity_rows(int W, int D1);
size_t vdisparity_smem(int W, int D1);
cudaError_t configure_fastpath(int W);
size_t prescreen_smem(int W, int nt);
int prescreen_threads(int W);
int need_bilateral_ctas(int sm_count);
void launch_fast_bilateral(const Dev& d, const LaunchPlan& lp, int n, cudaStream_t s, int all = 0);
void launch_sobel_refine(const Dev& d, const LaunchPlan& lp, int n, cudaStream_t s);
void launch_exact_bilateral(const Dev& d, const LaunchPlan& lp, int n, cudaStream_t s);
// stages 5-7 into d's (scratch) buffers + each frame's first grey row read downstream
cudaError_t launch_road_front(const Dev& d, const LaunchPlan& lp, int n, int* rows, cudaStream_t s);
cudaError_t fast_error(const Dev& d, int n, cudaStream_t s, double* out_dev);
int launches_per_batch(const Dev& d, const LaunchPlan& lp);

}  // namespace lkg
