// ref_wrapper.cpp — TEST INFRASTRUCTURE ONLY.
//
// Compiles the UNMODIFIED reference headers from /root/reference (never
// copied into this repo) and composes stages 5-12 exactly as
// pipeline.hpp:184-270 does, with the disparity map injected in place of
// stages 1-4 (the reference has no from-disparity entry point). Eigen3 is
// replaced by oracle/eigen_standin. Output: oracle/_ref/liblk_ref.so with the
// same C API as the restatement (prefix lkref_) so tests compare the two
// bit for bit, and bench.py's reference arm times this build.
#include <atomic>
#include <cmath>
#include <cstring>
#include <string>
#include <thread>
#include <vector>

#include "lanekit/config.hpp"
#include "lanekit/lanes.hpp"
#include "lanekit/preprocess.hpp"
#include "lanekit/road_profile.hpp"
#include "lanekit/stereo.hpp"
#include "lanekit/synth.hpp"
#include "lanekit/vanish.hpp"
#include "lk_oracle.hpp"

using namespace lanekit;

namespace {

int msg_of(const std::string& what) {
    if (what.find("fewer points") != std::string::npos) return LK_MSG_RANSAC_FEW_POINTS;
    if (what.find("no sample produced") != std::string::npos) return LK_MSG_RANSAC_NO_FIT;
    if (what.find("singular V_py") != std::string::npos) return LK_MSG_SINGULAR_VPY;
    if (what.find("sobel") != std::string::npos) return LK_MSG_SOBEL_TOO_SMALL;
    if (what.find("m1:") != std::string::npos) return LK_MSG_M1_TOO_SMALL;
    return -1;
}

struct StageFail {
    int stage;
    int msg;
    int row;
};

void compute_frame(const uint8_t* grey, const uint8_t* dispu8, int W, int H,
                   const lk_config& c, orc::Result& r) {
    r = orc::Result{};
    lk_frame_report& rep = r.rep;
    rep.width = W;
    rep.height = H;
    rep.rng_seed = c.rng_seed;
    r.W = W;
    r.H = H;

    PipelineConfig cfg;
    cfg.rho = c.rho;
    cfg.tau = c.tau;
    cfg.d_max = c.d_max;
    cfg.tr_lrc = c.tr_lrc;
    cfg.sigma_floor = c.sigma_floor;
    cfg.lambda_y = c.lambda_y;
    cfg.tr_y = c.tr_y;
    cfg.eps_y = c.eps_y;
    cfg.varpi = c.varpi;
    cfg.sigma_s = c.sigma_s;
    cfg.sigma_r = c.sigma_r;
    cfg.bf_window = c.bf_window;
    cfg.sobel_threshold = c.sobel_threshold;
    cfg.chi = c.chi;
    cfg.rho_vote = c.rho_vote;
    cfg.lambda_x = c.lambda_x;
    cfg.tr_x = c.tr_x;
    cfg.eps_x = c.eps_x;
    cfg.sigma_g = c.sigma_g;
    cfg.nu = c.nu;
    cfg.varsigma = c.varsigma;
    cfg.lambda_g = c.lambda_g;
    cfg.xi = c.xi;
    cfg.tr_lpv = c.tr_lpv;
    cfg.min_lane_sep = c.min_lane_sep;
    cfg.rng_seed = c.rng_seed;
    cfg.paper_sign = c.paper_sign != 0;
    cfg.threads = c.threads > 0 ? c.threads : 1;  // the reference's own intra-frame threading

    int stage = 1;
    auto run_stage = [&](int n, auto&& body) {  // pipeline.hpp:138-150
        stage = n;
        try {
            body();
        } catch (const StageFail&) {
            throw;
        } catch (const Error& e) {
            throw StageFail{n, msg_of(e.what()), 0};
        }
    };
    try {
        if (W <= 0 || H <= 0) throw StageFail{1, LK_MSG_EMPTY_INPUT, 0};
        GrayImage left(W, H, 0);
        for (size_t i = 0; i < left.data.size(); ++i) left.data[i] = grey[i] / 255.0;
        DisparityMap disparity(W, H, 0);
        long valid = 0;
        for (size_t i = 0; i < disparity.data.size(); ++i) {
            disparity.data[i] = dispu8[i];
            valid += dispu8[i] != 0;
        }
        rep.valid_disparities = valid;

        VDisparityHist vd;
        DpPath vpath, upath;
        BetaResult beta;
        RoadProfile road;
        Mask mask;
        GrayImage smoothed, m0, m1;
        GradientField grad;
        EdgeSet edges;
        SparseVpxMap sp;
        DenseVpxAccumulator acc;
        GammaResult gamma;
        VpProfile vp;
        EnergyHistogram energy;
        LaneSet lanes;

        run_stage(5, [&] { vd = build_vdisparity(disparity, cfg.d_max); });
        r.D1 = cfg.d_max + 1;
        r.vdisp = vd.count;
        run_stage(6, [&] {
            vpath = dp_extract_vpath(vd, cfg.lambda_y, cfg.paper_sign);
            rep.vpath_has_evidence = vpath.has_evidence;
            rep.vpath_energy = vpath.energy;
            r.vpath = vpath.points;
            if (!vpath.has_evidence) throw StageFail{6, LK_MSG_NO_ROAD_EVIDENCE, 0};
        });
        run_stage(7, [&] {
            RansacConfig rc;
            rc.tolerance = cfg.tr_y;
            rc.inlier_fraction = cfg.eps_y;
            rc.sample_size = 3;
            rc.max_iterations = 200;
            rc.rng_seed = cfg.rng_seed;
            beta = ransac_beta(vpath, rc);
            for (int k = 0; k < 3; ++k) rep.beta[k] = beta.beta[k];
            rep.beta_iterations = beta.iterations;
            rep.beta_inlier_fraction = beta.inlier_fraction;
            rep.beta_degraded = beta.degraded;
            rep.beta_inlier_count = static_cast<int64_t>(beta.inliers.size());
            r.beta_inliers = beta.inliers;
            const auto hz = horizon_row(beta.beta, H);
            rep.horizon = hz.row;
            rep.horizon_in_range = hz.in_range;
            const VpyProfile vpy = vpy_profile(beta.beta, H);
            r.vpy = vpy.value;
            r.vpy_singular = vpy.singular;
            for (int v = hz.row; v < H; ++v)
                if (vpy.singular[v]) throw StageFail{7, LK_MSG_SINGULAR_VPY, v};
            road = make_road_profile(beta.beta, H);
        });
        run_stage(8, [&] {
            mask = road_mask(disparity, road, cfg.varpi);
            long n = 0;
            for (uint8_t m : mask.data) n += m != 0;
            rep.road_mask_pixels = n;
            r.mask = mask.data;
        });
        run_stage(9, [&] {
            smoothed = bilateral_filter(left, cfg.sigma_s, cfg.sigma_r, (cfg.bf_window - 1) / 2,
                                        cfg.threads);
            r.smoothed = smoothed.data;
        });
        run_stage(10, [&] {
            grad = sobel_gradients(smoothed);
            edges = edge_map(grad, cfg.sobel_threshold / Real(255), mask);
            rep.edge_pixels = static_cast<int64_t>(edges.pixels.size());
            r.gx = grad.gx.data;
            r.gy = grad.gy.data;
            r.mag = grad.magnitude.data;
            r.theta = grad.theta.data;
            for (const auto& e : edges.pixels) r.edges.push_back({e.u, e.v, e.gx, e.gy, e.theta});
        });
        run_stage(11, [&] {
            sp = sparse_vpx(edges, road.vpy, kGradientFloor, cfg.xi, W);
            rep.vpx_votes = static_cast<int64_t>(sp.votes.size());
            rep.vpx_skipped = sp.skipped;
            r.ext_lo = sp.ext_lo;
            r.ext_cols = sp.ext_cols;
            for (const auto& v : sp.votes) r.votes.push_back({v.u_e, v.v_e, v.col});
            acc = accumulate_dense_vpx(sp, road.horizon, H - 1, cfg.chi, cfg.rho_vote);
            r.acc = acc.m;
            upath = dp_extract_upath(acc, cfg.lambda_x, cfg.paper_sign);
            rep.upath_has_evidence = upath.has_evidence;
            rep.upath_energy = upath.energy;
            r.upath = upath.points;
            if (!upath.has_evidence) throw StageFail{11, LK_MSG_NO_EDGE_EVIDENCE, 0};
            RansacConfig rc;
            rc.tolerance = cfg.tr_x;
            rc.inlier_fraction = cfg.eps_x;
            rc.sample_size = 5;
            rc.max_iterations = 200;
            rc.rng_seed = cfg.rng_seed;
            gamma = ransac_gamma(upath, rc, Real(1));
            for (int k = 0; k < 5; ++k) rep.gamma[k] = gamma.profile.gamma[k];
            rep.gamma_kappa = gamma.profile.kappa;
            rep.gamma_v_normalizer = gamma.profile.v_normalizer;
            rep.gamma_iterations = gamma.iterations;
            rep.gamma_inlier_fraction = gamma.inlier_fraction;
            rep.gamma_degraded = gamma.degraded;
            rep.gamma_inlier_count = static_cast<int64_t>(gamma.inliers.size());
            r.gamma_inliers = gamma.inliers;
            vp.v_top = road.horizon;
            vp.v_max = H - 1;
            vp.vpx = vpx_profile(gamma.profile, H);
            vp.vpy = road.vpy.value;
            r.vpx = vp.vpx;
        });
        run_stage(12, [&] {
            m0 = build_m0(grad, edges, vp, cfg.nu, cfg.varsigma, cfg.sigma_g);
            m1 = build_m1(m0);
            r.m0 = m0.data;
            r.m1 = m1.data;
            const Real tr = std::isnan(cfg.tr_lpv) ? auto_lane_threshold(m1, vp.v_top, vp.v_max)
                                                   : cfg.tr_lpv;
            rep.tr_lpv_used = tr;
            energy = aggregate_energy(m1, vp, cfg.xi, cfg.lambda_g, cfg.threads);
            r.energy = energy.h;
            lanes = select_lanes(energy, tr, cfg.min_lane_sep, vp);
            rep.lane_count = static_cast<int64_t>(lanes.lanes.size());
            for (size_t i = 0; i < lanes.lanes.size(); ++i) {
                const Lane& l = lanes.lanes[i];
                if (i < LK_MAX_INLINE_LANES) {
                    rep.lane_bottom_col[i] = l.bottom_col;
                    rep.lane_energy[i] = l.energy;
                }
                r.lanes.push_back({l.bottom_col, static_cast<int32_t>(l.polyline.size()), l.energy});
                // polyline (v ascending, NaN rows dropped) back to the dense track layout
                std::vector<Real> track(vp.v_max - vp.v_top + 1,
                                        std::numeric_limits<Real>::quiet_NaN());
                for (const auto& [v, u] : l.polyline) track[v - vp.v_top] = u;
                r.polylines.insert(r.polylines.end(), track.begin(), track.end());
            }
        });
    } catch (const StageFail& f) {
        rep.status = LK_ERR_FRAME;
        rep.failed_stage = f.stage;
        rep.msg = f.msg;
        rep.err_row = f.row;
    } catch (const Error& e) {
        rep.status = LK_ERR_FRAME;
        rep.failed_stage = stage;
        rep.msg = msg_of(e.what());
    }
}

}  // namespace

#define LK_PREFIX(name) lkref_##name
#include "result_capi.inc"

extern "C" {

// lanekit::gen_scene (synth.hpp:103-200) + the 8-bit quantisation of
// write_png_gray (image_io.hpp:184-193). Returns 0, or 1 with msg filled.
int lkref_gen_scene(const lk_scene_params* p, uint8_t* left, uint8_t* right, uint8_t* disp,
                    int32_t* horizon, char* msg, int msglen) {
    SceneParams sp;
    sp.width = p->width;
    sp.height = p->height;
    for (int k = 0; k < 3; ++k) sp.beta[k] = p->beta[k];
    for (int k = 0; k < 5; ++k) sp.gamma[k] = p->gamma[k];
    sp.d_max = p->d_max;
    sp.lane_bottoms.assign(p->lane_bottoms, p->lane_bottoms + p->n_lanes);
    sp.lane_width = p->lane_width;
    sp.lane_brightness = p->lane_brightness;
    sp.road_base = p->road_base;
    sp.sky_level = p->sky_level;
    sp.texture_amplitude = p->texture_amplitude;
    sp.noise_sigma = p->noise_sigma;
    sp.rng_seed = p->rng_seed;
    try {
        const SyntheticScene sc = gen_scene(sp);
        auto q = [](Real x) {
            const long v = std::lround(x * 255.0);
            return static_cast<uint8_t>(std::clamp(v, 0L, 255L));
        };
        for (size_t i = 0; i < sc.left.data.size(); ++i) {
            if (left) left[i] = q(sc.left.data[i]);
            if (right) right[i] = q(sc.right.data[i]);
            if (disp) disp[i] = static_cast<uint8_t>(sc.true_disparity.data[i]);
        }
        if (horizon) *horizon = sc.horizon;
        return 0;
    } catch (const Error& e) {
        if (msg && msglen > 0) {
            std::strncpy(msg, e.what(), msglen - 1);
            msg[msglen - 1] = 0;
        }
        return 1;
    }
}

// Stages 1-4 exactly as run_pipeline composes them (pipeline.hpp:161-182):
// precompute_stats on both images, match_srp for the left and the right
// reference, lrc_check. Same outputs as orc_stereo.
int lkref_stereo(const uint8_t* left, const uint8_t* right, int W, int H, int rho, int d_max,
                 int tau, int tr_lrc, double sigma_floor, double* mu_l, double* sig_l,
                 uint8_t* disp_l, uint8_t* disp_r, uint8_t* disparity) {
    try {
        GrayImage L(W, H, 0), R(W, H, 0);
        for (size_t i = 0; i < L.data.size(); ++i) {
            L.data[i] = left[i] / 255.0;  // image_io.hpp:147
            R.data[i] = right[i] / 255.0;
        }
        StereoConfig sc;
        sc.rho = rho;
        sc.d_min = 0;
        sc.d_max = d_max;
        sc.tau = tau;
        sc.tr_lrc = tr_lrc;
        sc.sigma_floor = sigma_floor;
        sc.threads = 1;
        const BlockStats ls = precompute_stats(L, rho);
        const BlockStats rs = precompute_stats(R, rho);
        const DisparityMap dl = match_srp(L, R, ls, rs, RefView::left, sc);
        const DisparityMap dr = match_srp(R, L, rs, ls, RefView::right, sc);
        const DisparityMap out = lrc_check(dl, dr, tr_lrc);
        for (size_t i = 0; i < L.data.size(); ++i) {
            if (mu_l) mu_l[i] = ls.mu.data[i];
            if (sig_l) sig_l[i] = ls.sigma.data[i];
            if (disp_l) disp_l[i] = static_cast<uint8_t>(dl.data[i]);
            if (disp_r) disp_r[i] = static_cast<uint8_t>(dr.data[i]);
            if (disparity) disparity[i] = static_cast<uint8_t>(out.data[i]);
        }
        return 0;
    } catch (const Error&) {
        return 1;
    }
}

// run_pipeline on stereo pairs (stages 1-4 then 5-12, pipeline.hpp:118-270),
// frame-parallel on `threads` host threads: the CPU baseline of the stereo bench.
int lkref_run_stereo_batch(const uint8_t* left, const uint8_t* right, int n, int W, int H,
                           const lk_config* cfg, int threads, lk_frame_report* reps) {
    if (threads < 1) threads = 1;
    const size_t frame = static_cast<size_t>(W) * H;
    std::vector<std::thread> pool;
    std::atomic<int> next{0};
    auto worker = [&] {
        orc::Result r;
        std::vector<uint8_t> disp(frame);
        for (int i = next++; i < n; i = next++) {
            lkref_stereo(left + frame * i, right + frame * i, W, H, cfg->rho, cfg->d_max, cfg->tau,
                         cfg->tr_lrc, cfg->sigma_floor, nullptr, nullptr, nullptr, nullptr,
                         disp.data());
            compute_frame(left + frame * i, disp.data(), W, H, *cfg, r);
            if (reps) reps[i] = r.rep;
        }
    };
    for (int t = 0; t < threads; ++t) pool.emplace_back(worker);
    for (auto& t : pool) t.join();
    int failed = 0;
    if (reps)
        for (int i = 0; i < n; ++i) failed += reps[i].status != 0;
    return failed;
}

}  // extern "C"
