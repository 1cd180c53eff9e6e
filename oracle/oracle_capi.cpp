// oracle_capi.cpp — TEST INFRASTRUCTURE ONLY. C entry points of the CPU
// restatement (liblk_oracle.so) for the pytest parity suite (ctypes).
#include <algorithm>
#include <atomic>
#include <climits>
#include <cmath>
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

// ---- more unit-level restatements for the known-answer tests
namespace {

// road_profile.hpp:161-176
int horizon_row(const double* b, int rows, int* in_range) {
    double root;
    *in_range = 0;
    if (b[2] == 0) {
        if (b[1] <= 0) return 0;
        root = -b[0] / b[1];
    } else {
        const double disc = b[1] * b[1] - 4 * b[2] * b[0];
        if (disc <= 0) return 0;
        root = (-b[1] + std::sqrt(disc)) / (2 * b[2]);
    }
    const long long r = std::llround(root);
    if (r < 0 || r >= rows) return 0;
    *in_range = 1;
    return static_cast<int>(r);
}

}  // namespace

extern "C" {

int orc_horizon_row(const double* beta, int rows, int32_t* in_range) {
    int ir = 0;
    const int r = horizon_row(beta, rows, &ir);
    *in_range = ir;
    return r;
}

// road_profile.hpp:184-199
void orc_vpy_profile(const double* b, int rows, double* value, uint8_t* singular) {
    for (int v = 0; v < rows; ++v) {
        const double vv = static_cast<double>(v);
        const double fp = b[1] + 2 * b[2] * vv;
        if (std::abs(fp) < 1e-12) {
            singular[v] = 1;
            value[v] = vv;
            continue;
        }
        singular[v] = 0;
        value[v] = vv - (b[0] + b[1] * vv + b[2] * vv * vv) / fp;
    }
}

// vanish.hpp:24-30
int orc_extended_col_lo(double xi, int width) {
    return -static_cast<int>(std::llround(xi * width));
}
int orc_extended_col_count(double xi, int width) {
    return static_cast<int>(std::llround((2 * xi + 1) * width));
}

// vanish.hpp:49-70 for explicit edges (u, v, gx, gy); returns the vote count,
// cols_out[i] = vote column or INT32_MIN for a skipped edge.
int orc_sparse_vpx(const int32_t* uv, const double* g, int n, const double* vpy,
                   const uint8_t* singular, int rows, double xi, int width, int32_t* cols_out) {
    const int lo = orc_extended_col_lo(xi, width);
    const int hi = lo + orc_extended_col_count(xi, width) - 1;
    int votes = 0;
    for (int i = 0; i < n; ++i) {
        const int u = uv[2 * i], v = uv[2 * i + 1];
        const double gx = g[2 * i], gy = g[2 * i + 1];
        if (v < 0 || v >= rows || singular[v] || std::abs(gx) < 1e-3) {
            cols_out[i] = INT32_MIN;
            continue;
        }
        const double col = u + (v - vpy[v]) * (gy / gx);
        const long long c = std::llround(col);
        cols_out[i] = static_cast<int>(std::clamp(c, static_cast<long long>(lo),
                                                  static_cast<long long>(hi)));
        ++votes;
    }
    return votes;
}

// vanish.hpp:113-148 (sliding band) for explicit votes (col, row); acc is
// [(v_max - v_top + 1)][ext_cols].
void orc_accumulate(const int32_t* col_row, int n, int ext_lo, int ext_cols, int v_top,
                    int v_max, int chi, double rho_vote, double* acc) {
    const int nrows = v_max - v_top + 1;
    std::vector<std::vector<int>> by_row(nrows);
    for (int i = 0; i < n; ++i) {
        const int c = col_row[2 * i], r = col_row[2 * i + 1];
        if (r < v_top || r > v_max) continue;
        by_row[r - v_top].push_back(c - ext_lo);
    }
    std::vector<int32_t> cnt(ext_cols, 0);
    int top_cur = v_max + 1, bot_cur = v_max;
    for (int v = v_max; v >= v_top; --v) {
        int bt, bb;
        if (v > v_max - chi - 1) {
            bt = v;
            bb = v_max;
        } else if (v >= v_top + chi) {
            bt = v - chi;
            bb = v + chi;
        } else {
            bt = v_top;
            bb = v + chi;
        }
        for (int r = bt; r < top_cur; ++r)
            for (int c : by_row[r - v_top]) ++cnt[c];
        top_cur = bt;
        for (int r = bb + 1; r <= bot_cur; ++r)
            for (int c : by_row[r - v_top]) --cnt[c];
        bot_cur = bb;
        double* row = acc + static_cast<size_t>(v - v_top) * ext_cols;
        for (int c = 0; c < ext_cols; ++c) row[c] = -rho_vote * cnt[c];
    }
}

// lanes.hpp:106-129 on an explicit m1 map and V_p profile.
void orc_aggregate_energy(const double* m1, int W, int H, const double* vpx, const double* vpy,
                          int v_top, int v_max, double xi, double lambda_g, double* out) {
    const int lo = orc_extended_col_lo(xi, W), cols = orc_extended_col_count(xi, W);
    std::vector<double> track(v_max - v_top + 1);
    for (int ci = 0; ci < cols; ++ci) {
        orc::lane_track(static_cast<double>(lo + ci), vpx, vpy, v_top, v_max, track.data());
        double e = 0;
        for (int v = v_max; v >= v_top; --v) {
            double contrib = 0;
            const double tu = track[v - v_top];
            if (!std::isnan(tu)) {
                const long long r = std::llround(tu);
                if (r >= 0 && r < W && v >= 0 && v < H)
                    contrib = m1[static_cast<size_t>(v) * W + static_cast<int>(r)];
            }
            e = contrib + lambda_g * e;
        }
        out[ci] = e;
    }
}

// lanes.hpp:144-178 minus the polylines: kept histogram indices, strongest first.
int orc_select_lanes(const double* h, int n, double tr, int min_sep, int32_t* kept_out) {
    std::vector<int> cand;
    for (int i = 1; i + 1 < n; ++i)
        if (h[i] < h[i - 1] && h[i] < h[i + 1] && h[i] < tr) cand.push_back(i);
    std::sort(cand.begin(), cand.end(), [&](int a, int b) {
        if (h[a] != h[b]) return h[a] < h[b];
        return a < b;
    });
    int nk = 0;
    for (int i : cand) {
        bool close = false;
        for (int k = 0; k < nk; ++k)
            if (std::abs(i - kept_out[k]) < min_sep) {
                close = true;
                break;
            }
        if (!close) kept_out[nk++] = i;
    }
    return nk;
}

}  // extern "C"
