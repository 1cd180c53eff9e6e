// oracle_capi.cpp — TEST INFRASTRUCTURE ONLY. C entry points of the CPU
// restatement (liblk_oracle.so) for the pytest parity suite (ctypes).
#include <atomic>
#include <vector>

#include "lk_oracle.hpp"

static void compute_frame(const uint8_t* g, const uint8_t* d, int W, int H, const lk_config& c,
                          orc::Result& r) {
    orc::run_frame(g, d, W, H, c, r);
}

#define LK_PREFIX(name) orc_##name
#include "result_capi.inc"

namespace {
std::vector<orc::Pt> to_pts(const int32_t* p, int n) {
    std::vector<orc::Pt> v(n);
    for (int i = 0; i < n; ++i) v[i] = {p[2 * i], p[2 * i + 1]};
    return v;
}
}  // namespace

extern "C" {

double orc_dp_min_path(int stages, int states, const double* data, const int32_t* offs,
                       int n_off, const double* pen, int32_t* path_out) {
    std::vector<int> path;
    const double e = orc::dp_min_path(stages, states, data, offs, n_off, pen, path);
    for (int i = 0; i < stages; ++i) path_out[i] = path[i];
    return e;
}

int orc_fit_parabola(const int32_t* pts, int n, double* out) {
    return orc::fit_parabola(to_pts(pts, n), out) ? 0 : 1;
}

int orc_fit_quartic(const int32_t* pts, int n, double kappa, double vnorm, double* out,
                    double* s) {
    return orc::fit_quartic(to_pts(pts, n), kappa, vnorm, out, s) ? 0 : 1;
}

// Returns 0 or the lk_msg of the RANSAC failure. inl_out needs room for n pairs.
int orc_ransac(int kind, const int32_t* pts, int n, double tol, double eps, int max_iter,
               uint64_t seed, double* model, double* s, int32_t* iters, double* frac,
               int32_t* degraded, int32_t* inl_out, int32_t* n_inl) {
    try {
        orc::RansacOut o = orc::ransac(kind, to_pts(pts, n), tol, eps, max_iter, seed);
        for (int i = 0; i < 5; ++i) model[i] = o.model[i];
        *s = o.s;
        *iters = o.iterations;
        *frac = o.fraction;
        *degraded = o.degraded;
        *n_inl = static_cast<int32_t>(o.inliers.size());
        for (size_t i = 0; i < o.inliers.size(); ++i) {
            inl_out[2 * i] = o.inliers[i].first;
            inl_out[2 * i + 1] = o.inliers[i].second;
        }
        return 0;
    } catch (const orc::Fail& f) {
        return f.msg;
    }
}

double orc_piecewise_weight(double te, double tv, double sg) {
    return orc::piecewise_weight(te, tv, sg);
}

void orc_lane_track(double u, const double* vpx, const double* vpy, int v_top, int v_max,
                    double* track) {
    orc::lane_track(u, vpx, vpy, v_top, v_max, track);
}

double orc_auto_lane_threshold(const double* m1, int W, int H, int v_top, int v_max) {
    return orc::auto_lane_threshold(m1, W, H, v_top, v_max);
}

}  // extern "C"
