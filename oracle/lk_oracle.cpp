// lk_oracle.cpp — TEST INFRASTRUCTURE ONLY: CPU restatement of lanekit
// stages 5-12 (see lk_oracle.hpp for the contract). Citations are
// file:line into /root/reference/proj/include/lanekit/.
#include "lk_oracle.hpp"

#include <algorithm>
#include <cfloat>
#include <cmath>
#include <cstring>
#include <limits>
#include <random>

namespace orc {

namespace {

constexpr Real kNaN = std::numeric_limits<Real>::quiet_NaN();

// common.hpp:28-35 — fold an index back into [0, n) (edge-inclusive mirror).
int mirror(int i, int n) {
    if (n <= 1) return 0;
    while (i < 0 || i >= n) {
        if (i < 0) i = -i - 1;
        if (i >= n) i = 2 * n - 1 - i;
    }
    return i;
}

// ------------------------------------------------------------------ LDLT
// Eigen 3.4 ldlt_inplace<Lower>::unblocked + LDLT::_solve_impl restated
// (SURVEY.md Appendix B). Eigen is absent here; this defines the bits the
// GPU reproduces. Dot products are sequential from index 0.
struct Ldlt {
    int n = 0;
    Real a[25];  // row-major, lower triangle used
    int t[5];
};

void ldlt_factor(Ldlt& f) {
    const int n = f.n;
    Real* A = f.a;
    Real temp[5];
    for (int k = 0; k < n; ++k) {
        int p = k;
        Real big = std::fabs(A[k * n + k]);
        for (int i = k + 1; i < n; ++i) {
            const Real c = std::fabs(A[i * n + i]);
            if (c > big) {
                big = c;
                p = i;
            }
        }
        f.t[k] = p;
        if (p != k) {
            for (int j = 0; j < k; ++j) std::swap(A[k * n + j], A[p * n + j]);
            for (int i = p + 1; i < n; ++i) std::swap(A[i * n + k], A[i * n + p]);
            std::swap(A[k * n + k], A[p * n + p]);
            for (int i = k + 1; i < p; ++i) std::swap(A[i * n + k], A[p * n + i]);
        }
        if (k > 0) {
            for (int j = 0; j < k; ++j) temp[j] = A[j * n + j] * A[k * n + j];
            Real dot = A[k * n] * temp[0];
            for (int j = 1; j < k; ++j) dot = dot + A[k * n + j] * temp[j];
            A[k * n + k] = A[k * n + k] - dot;
            for (int i = k + 1; i < n; ++i) {
                Real s = A[i * n] * temp[0];
                for (int j = 1; j < k; ++j) s = s + A[i * n + j] * temp[j];
                A[i * n + k] = A[i * n + k] - s;
            }
        }
        const Real akk = A[k * n + k];
        const bool valid = std::fabs(akk) > 0;
        if (k == 0 && !valid) {
            for (int j = 0; j < n; ++j) f.t[j] = j;
            break;
        }
        if (valid)
            for (int i = k + 1; i < n; ++i) A[i * n + k] = A[i * n + k] / akk;
    }
}

void ldlt_solve(const Ldlt& f, const Real* b, Real* x) {
    const int n = f.n;
    const Real* A = f.a;
    for (int i = 0; i < n; ++i) x[i] = b[i];
    for (int k = 0; k < n; ++k) std::swap(x[k], x[f.t[k]]);
    for (int i = 0; i < n; ++i)
        for (int s = i + 1; s < n; ++s) x[s] = x[s] - x[i] * A[s * n + i];
    for (int i = 0; i < n; ++i) {
        const Real d = A[i * n + i];
        if (std::fabs(d) > DBL_MIN)
            x[i] = x[i] / d;
        else
            x[i] = 0;
    }
    for (int i = n - 2; i >= 0; --i) {
        Real s = A[(i + 1) * n + i] * x[i + 1];
        for (int j = i + 2; j < n; ++j) s = s + A[j * n + i] * x[j];
        x[i] = x[i] - s;
    }
    for (int k = n - 1; k >= 0; --k) std::swap(x[k], x[f.t[k]]);
}

int distinct_rows(const std::vector<Pt>& pts) {
    std::vector<int> rows;
    rows.reserve(pts.size());
    for (const Pt& p : pts) rows.push_back(p.second);
    std::sort(rows.begin(), rows.end());
    return static_cast<int>(std::unique(rows.begin(), rows.end()) - rows.begin());
}

Real beta_res2(const Real* m, const Pt& p) {  // road_profile.hpp:124-128
    const Real v = static_cast<Real>(p.second);
    const Real r = static_cast<Real>(p.first) - (m[0] + m[1] * v + m[2] * v * v);
    return r * r;
}

Real quartic_eval(const Real* g, Real v) {  // vanish.hpp:191-193 (Horner)
    return g[0] + v * (g[1] + v * (g[2] + v * (g[3] + v * g[4])));
}

Real gamma_res2(const Real* m, const Pt& p) {  // vanish.hpp:258-261
    const Real r = static_cast<Real>(p.first) - quartic_eval(m, static_cast<Real>(p.second));
    return r * r;
}

Real road_f(const Real* b, Real v) { return b[0] + b[1] * v + b[2] * v * v; }  // :145-147
Real road_fprime(const Real* b, Real v) { return b[1] + 2 * b[2] * v; }       // :149-151

}  // namespace

// ------------------------------------------------------------------ DP
// dp.hpp:29-73. data row-major [stages][states]; pen[oi] = penalty(offsets[oi]).
Real dp_min_path(int stages, int states, const Real* data, const int* offsets, int n_off,
                 const Real* pen, std::vector<int>& path) {
    constexpr Real kInf = std::numeric_limits<Real>::infinity();
    std::vector<Real> prev(states), cur(states);
    std::vector<int8_t> choice(static_cast<size_t>(stages) * states, 0);
    for (int s = 0; s < states; ++s) prev[s] = data[s];
    for (int st = 1; st < stages; ++st) {
        const Real* row = data + static_cast<size_t>(st) * states;
        for (int s = 0; s < states; ++s) {
            Real best = kInf;
            int best_off = 0;
            for (int oi = 0; oi < n_off; ++oi) {
                const int ps = s + offsets[oi];
                if (ps < 0 || ps >= states) continue;
                const Real e = prev[ps] + pen[oi];
                if (e < best) {
                    best = e;
                    best_off = offsets[oi];
                }
            }
            cur[s] = best + row[s];
            choice[static_cast<size_t>(st) * states + s] = static_cast<int8_t>(best_off);
        }
        prev.swap(cur);
    }
    int term = 0;
    for (int s = 1; s < states; ++s)
        if (prev[s] < prev[term]) term = s;
    path.assign(stages, 0);
    path[stages - 1] = term;
    for (int st = stages - 1; st > 0; --st)
        path[st - 1] = path[st] + choice[static_cast<size_t>(st) * states + path[st]];
    return prev[term];
}

// ------------------------------------------------------------------ fits
// road_profile.hpp:86-111 — parabola through (d, v) via 3x3 normal equations.
bool fit_parabola(const std::vector<Pt>& pts, Real out[3]) {
    if (distinct_rows(pts) < 3) return false;
    Real s = 1;
    for (const Pt& p : pts) s = std::max(s, std::abs(static_cast<Real>(p.second)));
    Ldlt f;
    f.n = 3;
    std::fill(f.a, f.a + 9, 0.0);
    Real b[3] = {0, 0, 0};
    for (const Pt& p : pts) {
        const Real t = static_cast<Real>(p.second) / s;
        const Real phi[3] = {1.0, t, t * t};
        for (int i = 0; i < 3; ++i)
            for (int j = 0; j < 3; ++j) f.a[i * 3 + j] = f.a[i * 3 + j] + phi[i] * phi[j];
        const Real d = static_cast<Real>(p.first);
        for (int i = 0; i < 3; ++i) b[i] = b[i] + d * phi[i];
    }
    ldlt_factor(f);
    Real x[3];
    ldlt_solve(f, b, x);
    out[0] = x[0];
    out[1] = x[1] / s;
    out[2] = x[2] / (s * s);
    return true;
}

// vanish.hpp:201-243 — quartic u = g(v), kappa-scaled normal equations plus
// one refinement pass. Eigen rewrites kappa*(phi*phi^T) as (kappa*phi)*phi^T.
bool fit_quartic(const std::vector<Pt>& pts, Real kappa, Real v_normalizer, Real out[5],
                 Real* s_out) {
    if (distinct_rows(pts) < 5) return false;
    if (kappa <= 0) return false;
    Real s = v_normalizer;
    if (s <= 0) {
        s = 1;
        for (const Pt& p : pts) s = std::max(s, std::abs(static_cast<Real>(p.second)));
    }
    Ldlt f;
    f.n = 5;
    Real a[25];
    std::fill(a, a + 25, 0.0);
    Real b[5] = {0, 0, 0, 0, 0};
    for (const Pt& p : pts) {
        const Real t = static_cast<Real>(p.second) / s;
        const Real phi[5] = {1.0, t, t * t, t * t * t, t * t * t * t};
        for (int i = 0; i < 5; ++i) {
            const Real ki = kappa * phi[i];
            for (int j = 0; j < 5; ++j) a[i * 5 + j] = a[i * 5 + j] + ki * phi[j];
        }
        const Real ku = kappa * static_cast<Real>(p.first);
        for (int i = 0; i < 5; ++i) b[i] = b[i] + ku * phi[i];
    }
    std::copy(a, a + 25, f.a);
    ldlt_factor(f);
    Real x[5], r[5], dx[5];
    ldlt_solve(f, b, x);
    for (int i = 0; i < 5; ++i) {
        Real ax = a[i * 5] * x[0];
        for (int j = 1; j < 5; ++j) ax = ax + a[i * 5 + j] * x[j];
        r[i] = b[i] - ax;
    }
    ldlt_solve(f, r, dx);
    for (int i = 0; i < 5; ++i) x[i] = x[i] + dx[i];
    Real sk = 1;
    for (int k = 0; k < 5; ++k) {
        out[k] = x[k] / sk;
        sk *= s;
    }
    if (s_out) *s_out = s;
    return true;
}

// ------------------------------------------------------------------ RANSAC
// ransac.hpp:36-119 — trimming RANSAC; kind 3 = ransac_beta
// (road_profile.hpp:121-137), kind 5 = ransac_gamma with kappa 1 (vanish.hpp:253-270).
RansacOut ransac(int kind, const std::vector<Pt>& points, Real tol, Real eps, int max_iter,
                 uint64_t seed) {
    const int k = kind;
    if (static_cast<int>(points.size()) < k) throw Fail{0, LK_MSG_RANSAC_FEW_POINTS, 0};
    auto fit = [&](const std::vector<Pt>& s, Real* m, Real* sn) -> bool {
        if (kind == 3) return fit_parabola(s, m);
        return fit_quartic(s, 1.0, 0.0, m, sn);
    };
    auto res2 = [&](const Real* m, const Pt& p) -> Real {
        return kind == 3 ? beta_res2(m, p) : gamma_res2(m, p);
    };

    std::mt19937_64 rng(seed);
    std::vector<Pt> m = points, sample(k), inl;
    std::vector<int> idx;
    RansacOut out;
    Real best_fraction = -1;
    Real best_model[5] = {0, 0, 0, 0, 0}, best_s = 0;
    bool have_model = false;

    for (int iter = 0; iter < max_iter; ++iter) {
        out.iterations = iter + 1;
        if (static_cast<int>(m.size()) < k) break;
        idx.resize(m.size());
        for (size_t i = 0; i < idx.size(); ++i) idx[i] = static_cast<int>(i);
        for (int i = 0; i < k; ++i) {
            const size_t j = i + static_cast<size_t>(rng() % (idx.size() - i));
            std::swap(idx[i], idx[j]);
            sample[i] = m[idx[i]];
        }
        Real model[5] = {0, 0, 0, 0, 0}, ms = 0;
        if (!fit(sample, model, &ms)) continue;  // degenerate sample, iteration consumed
        inl.clear();
        for (const Pt& p : m)
            if (res2(model, p) < tol) inl.push_back(p);
        const Real fraction = static_cast<Real>(inl.size()) / static_cast<Real>(m.size());
        if (fraction > best_fraction) {
            best_fraction = fraction;
            std::copy(model, model + 5, best_model);
            best_s = ms;
            have_model = true;
        }
        if (fraction >= best_fraction && fraction > Real(0.5) && static_cast<int>(inl.size()) >= k)
            m = inl;
        if (best_fraction >= eps) break;
    }
    if (!have_model) throw Fail{0, LK_MSG_RANSAC_NO_FIT, 0};

    inl.clear();
    for (const Pt& p : m)
        if (res2(best_model, p) < tol) inl.push_back(p);
    std::copy(best_model, best_model + 5, out.model);
    out.s = best_s;
    for (int round = 0; round < 3 && static_cast<int>(inl.size()) >= k; ++round) {
        Real refit[5] = {0, 0, 0, 0, 0}, rs = 0;
        if (!fit(inl, refit, &rs)) break;
        std::copy(refit, refit + 5, out.model);
        out.s = rs;
        std::vector<Pt> next;
        for (const Pt& p : points)
            if (res2(refit, p) < tol) next.push_back(p);
        const bool settled = next == inl;
        inl = std::move(next);
        if (settled) break;
    }
    out.inliers = inl.empty() ? m : inl;
    out.fraction = best_fraction;
    out.degraded = best_fraction < eps;
    return out;
}

// ------------------------------------------------------------------ lanes
// lanes.hpp:20-25
Real piecewise_weight(Real theta_e, Real theta_vp, Real sigma_g) {
    Real d = std::fmod(std::abs(theta_e - theta_vp), kPi);
    if (d > kPi / 2) d = kPi - d;
    if (d > kPi / 6) return 0;
    return std::exp(-(d / (sigma_g * sigma_g)) * (36 / kPi));
}

// lanes.hpp:83-96 — track[i] holds row v_top + i.
void lane_track(Real u_bottom, const Real* vpx, const Real* vpy, int v_top, int v_max,
                Real* track) {
    const int n = v_max - v_top + 1;
    for (int i = 0; i < n; ++i) track[i] = kNaN;
    track[n - 1] = u_bottom;
    for (int v = v_max - 1; v >= v_top; --v) {
        const Real u_next = track[v + 1 - v_top];
        const Real py = vpy[v + 1];
        const Real denom = static_cast<Real>(v + 1) - py;
        if (std::abs(denom) < 0.5) break;
        track[v - v_top] = (vpx[v + 1] + v * u_next - py * u_next) / denom;
    }
}

// lanes.hpp:182-193
Real auto_lane_threshold(const Real* m1, int W, int H, int v_top, int v_max) {
    std::vector<Real> mags;
    for (int v = std::max(0, v_top); v <= std::min(H - 1, v_max); ++v)
        for (int u = 0; u < W; ++u) mags.push_back(std::abs(m1[static_cast<size_t>(v) * W + u]));
    if (mags.empty()) return 0;
    const size_t k = static_cast<size_t>(std::floor(0.99 * (mags.size() - 1)));
    std::nth_element(mags.begin(), mags.begin() + k, mags.end());
    return -0.15 * static_cast<Real>(v_max - v_top + 1) * mags[k];
}

// ------------------------------------------------------------------ pipeline
// pipeline.hpp:184-270 with the disparity injected (stages 5-12).
void run_frame(const uint8_t* grey, const uint8_t* dispu8, int W, int H, const lk_config& cfg,
               Result& r) {
    r = Result{};
    lk_frame_report& rep = r.rep;
    rep.width = W;
    rep.height = H;
    rep.rng_seed = cfg.rng_seed;
    r.W = W;
    r.H = H;
    int stage = 1;
    try {
        if (W <= 0 || H <= 0) throw Fail{1, LK_MSG_EMPTY_INPUT, 0};
        const size_t N = static_cast<size_t>(W) * H;
        std::vector<int> disp(N);
        for (size_t i = 0; i < N; ++i) disp[i] = dispu8[i];
        long valid = 0;
        for (size_t i = 0; i < N; ++i) valid += disp[i] != 0;
        rep.valid_disparities = valid;

        // ---- stage 5: build_vdisparity (road_profile.hpp:32-45)
        stage = 5;
        const int dmax = cfg.d_max, D1 = dmax + 1;
        r.D1 = D1;
        r.vdisp.assign(static_cast<size_t>(H) * D1, 0);
        for (int v = 0; v < H; ++v)
            for (int u = 0; u < W; ++u) {
                const int d = disp[static_cast<size_t>(v) * W + u];
                if (d >= 1 && d <= dmax) ++r.vdisp[static_cast<size_t>(v) * D1 + d];
            }

        // ---- stage 6: dp_extract_vpath (road_profile.hpp:54-78)
        stage = 6;
        {
            const int stages = D1;
            std::vector<Real> data(static_cast<size_t>(stages) * H);
            for (int st = 0; st < stages; ++st)
                for (int v = 0; v < H; ++v)
                    data[static_cast<size_t>(st) * H + v] =
                        -static_cast<Real>(r.vdisp[static_cast<size_t>(v) * D1 + (dmax - st)]);
            const int offs[7] = {0, 1, 2, 3, 4, 5, 6};
            Real pen[7];
            for (int i = 0; i < 7; ++i)
                pen[i] = cfg.paper_sign ? -cfg.lambda_y * offs[i] : cfg.lambda_y * offs[i];
            std::vector<int> path;
            rep.vpath_energy = dp_min_path(stages, H, data.data(), offs, 7, pen, path);
            for (int i = 0; i < stages; ++i) r.vpath.emplace_back(dmax - i, path[i]);
            bool ev = false;
            for (int32_t c : r.vdisp)
                if (c > 0) {
                    ev = true;
                    break;
                }
            rep.vpath_has_evidence = ev;
            if (!ev) throw Fail{6, LK_MSG_NO_ROAD_EVIDENCE, 0};
        }

        // ---- stage 7: ransac_beta + make_road_profile (pipeline.hpp:193-208)
        stage = 7;
        Real beta[3];
        {
            RansacOut o = ransac(3, r.vpath, cfg.tr_y, cfg.eps_y, 200, cfg.rng_seed);
            std::copy(o.model, o.model + 3, beta);
            r.beta_inliers = o.inliers;
            std::copy(beta, beta + 3, rep.beta);
            rep.beta_iterations = o.iterations;
            rep.beta_inlier_fraction = o.fraction;
            rep.beta_degraded = o.degraded;
            rep.beta_inlier_count = static_cast<int64_t>(o.inliers.size());
        }
        // horizon_row (road_profile.hpp:161-176)
        int horizon = 0;
        bool in_range = true;
        {
            Real root = 0;
            bool ok = true;
            if (beta[2] == 0) {
                if (beta[1] <= 0)
                    ok = false;
                else
                    root = -beta[0] / beta[1];
            } else {
                const Real disc = beta[1] * beta[1] - 4 * beta[2] * beta[0];
                if (disc <= 0)
                    ok = false;
                else
                    root = (-beta[1] + std::sqrt(disc)) / (2 * beta[2]);
            }
            if (ok) {
                const long long rr = std::llround(root);
                if (rr < 0 || rr >= H)
                    ok = false;
                else
                    horizon = static_cast<int>(rr);
            }
            if (!ok) {
                horizon = 0;
                in_range = false;
            }
        }
        // vpy_profile (road_profile.hpp:184-199)
        r.vpy.assign(H, 0);
        r.vpy_singular.assign(H, 0);
        for (int v = 0; v < H; ++v) {
            const Real fp = road_fprime(beta, static_cast<Real>(v));
            if (std::abs(fp) < 1e-12) {
                r.vpy_singular[v] = 1;
                r.vpy[v] = static_cast<Real>(v);
                continue;
            }
            r.vpy[v] = static_cast<Real>(v) - road_f(beta, static_cast<Real>(v)) / fp;
        }
        rep.horizon = horizon;
        rep.horizon_in_range = in_range;
        for (int v = horizon; v < H; ++v)  // make_road_profile (road_profile.hpp:223-225)
            if (r.vpy_singular[v]) throw Fail{7, LK_MSG_SINGULAR_VPY, v};

        // ---- stage 8: road_mask (preprocess.hpp:14-26)
        stage = 8;
        r.mask.assign(N, 0);
        long mask_px = 0;
        for (int v = horizon; v < H; ++v) {
            const Real fv = road_f(beta, static_cast<Real>(v));
            for (int u = 0; u < W; ++u) {
                const int d = disp[static_cast<size_t>(v) * W + u];
                if (d != 0 && std::abs(static_cast<Real>(d) - fv) <= cfg.varpi) {
                    r.mask[static_cast<size_t>(v) * W + u] = 1;
                    ++mask_px;
                }
            }
        }
        rep.road_mask_pixels = mask_px;

        // ---- stage 9: bilateral_filter (preprocess.hpp:30-59). exp(a)*exp(b)
        // with a depending only on the tap and b only on the 8-bit pair, so
        // both factors are tabulated with the same libm calls: bit-identical.
        stage = 9;
        {
            const int rho = (cfg.bf_window - 1) / 2;
            const int win = 2 * rho + 1;
            const Real inv_s2 = 1.0 / (cfg.sigma_s * cfg.sigma_s);
            const Real inv_r2 = 1.0 / (cfg.sigma_r * cfg.sigma_r);
            std::vector<Real> ws(static_cast<size_t>(win) * win);
            for (int dj = -rho; dj <= rho; ++dj)
                for (int di = -rho; di <= rho; ++di) {
                    const Real ds = static_cast<Real>(di) * di + static_cast<Real>(dj) * dj;
                    ws[static_cast<size_t>(dj + rho) * win + (di + rho)] = std::exp(-ds * inv_s2);
                }
            std::vector<Real> val(256);
            for (int k = 0; k < 256; ++k) val[k] = k / 255.0;
            std::vector<Real> wr(256 * 256);
            for (int kc = 0; kc < 256; ++kc)
                for (int kv = 0; kv < 256; ++kv) {
                    const Real dr = val[kv] - val[kc];
                    wr[kc * 256 + kv] = std::exp(-dr * dr * inv_r2);
                }
            r.smoothed.assign(N, 0);
            std::vector<int> cols(win);
            for (int v = 0; v < H; ++v)
                for (int u = 0; u < W; ++u) {
                    const int kc = grey[static_cast<size_t>(v) * W + u];
                    const Real* wrow = &wr[kc * 256];
                    Real num = 0, den = 0;
                    for (int i = 0; i < win; ++i) cols[i] = mirror(u - rho + i, W);
                    for (int j = 0; j < win; ++j) {
                        const uint8_t* grow = grey + static_cast<size_t>(mirror(v - rho + j, H)) * W;
                        const Real* wsr = &ws[static_cast<size_t>(j) * win];
                        for (int i = 0; i < win; ++i) {
                            const int kv = grow[cols[i]];
                            const Real w = wsr[i] * wrow[kv];
                            num += w * val[kv];
                            den += w;
                        }
                    }
                    r.smoothed[static_cast<size_t>(v) * W + u] = num / den;
                }
        }

        // ---- stage 10: sobel_gradients + edge_map (preprocess.hpp:67-113)
        stage = 10;
        if (W < 3 || H < 3) throw Fail{10, LK_MSG_SOBEL_TOO_SMALL, 0};
        r.gx.assign(N, 0);
        r.gy.assign(N, 0);
        r.mag.assign(N, 0);
        r.theta.assign(N, 0);
        {
            const Real* img = r.smoothed.data();
            auto px = [&](int u, int v) {
                return img[static_cast<size_t>(mirror(v, H)) * W + mirror(u, W)];
            };
            for (int v = 0; v < H; ++v)
                for (int u = 0; u < W; ++u) {
                    const Real gx = (px(u + 1, v - 1) - px(u - 1, v - 1)) +
                                    2 * (px(u + 1, v) - px(u - 1, v)) +
                                    (px(u + 1, v + 1) - px(u - 1, v + 1));
                    const Real gy = (px(u - 1, v + 1) - px(u - 1, v - 1)) +
                                    2 * (px(u, v + 1) - px(u, v - 1)) +
                                    (px(u + 1, v + 1) - px(u + 1, v - 1));
                    const size_t i = static_cast<size_t>(v) * W + u;
                    r.gx[i] = gx;
                    r.gy[i] = gy;
                    r.mag[i] = std::sqrt(gx * gx + gy * gy);
                    Real th = std::atan2(gy, gx);
                    if (th <= -kPi) th = kPi;
                    r.theta[i] = th;
                }
            const Real thr = cfg.sobel_threshold / Real(255);
            for (int v = 0; v < H; ++v)
                for (int u = 0; u < W; ++u) {
                    const size_t i = static_cast<size_t>(v) * W + u;
                    if (!r.mask[i]) continue;
                    if (r.mag[i] < thr) continue;
                    r.edges.push_back({u, v, r.gx[i], r.gy[i], r.theta[i]});
                }
            rep.edge_pixels = static_cast<int64_t>(r.edges.size());
        }

        // ---- stage 11: V_px (pipeline.hpp:230-258)
        stage = 11;
        const int ext_lo = -static_cast<int>(std::llround(cfg.xi * W));      // vanish.hpp:24-26
        const int ext_cols = static_cast<int>(std::llround((2 * cfg.xi + 1) * W));  // :28-30
        r.ext_lo = ext_lo;
        r.ext_cols = ext_cols;
        const int v_top = horizon, v_max = H - 1;
        {
            // sparse_vpx (vanish.hpp:49-70)
            const int ext_hi = ext_lo + ext_cols - 1;
            long skipped = 0;
            for (const lk_edge& e : r.edges) {
                if (e.v < 0 || e.v >= H || r.vpy_singular[e.v] || std::abs(e.gx) < 1e-3) {
                    ++skipped;
                    continue;
                }
                const Real col = e.u + (e.v - r.vpy[e.v]) * (e.gy / e.gx);
                const long long c = std::llround(col);
                const int cc = static_cast<int>(std::clamp(c, static_cast<long long>(ext_lo),
                                                           static_cast<long long>(ext_hi)));
                r.votes.push_back({e.u, e.v, cc});
            }
            rep.vpx_votes = static_cast<int64_t>(r.votes.size());
            rep.vpx_skipped = skipped;

            // accumulate_dense_vpx (vanish.hpp:113-148): sliding band
            const int nrows = v_max - v_top + 1;
            r.acc.assign(static_cast<size_t>(nrows) * ext_cols, 0);
            std::vector<std::vector<int>> by_row(nrows);
            for (const lk_vote& vt : r.votes) {
                if (vt.v_e < v_top || vt.v_e > v_max) continue;
                by_row[vt.v_e - v_top].push_back(vt.col - ext_lo);
            }
            std::vector<int32_t> cnt(ext_cols, 0);
            int top_cur = v_max + 1, bot_cur = v_max;
            const int chi = cfg.chi;
            for (int v = v_max; v >= v_top; --v) {
                int bt, bb;  // vote_band (vanish.hpp:101-105)
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
                for (int rr = bt; rr < top_cur; ++rr)
                    for (int c : by_row[rr - v_top]) ++cnt[c];
                top_cur = bt;
                for (int rr = bb + 1; rr <= bot_cur; ++rr)
                    for (int c : by_row[rr - v_top]) --cnt[c];
                bot_cur = bb;
                Real* row = &r.acc[static_cast<size_t>(v - v_top) * ext_cols];
                for (int c = 0; c < ext_cols; ++c) row[c] = -cfg.rho_vote * cnt[c];
            }

            // dp_extract_upath (vanish.hpp:156-182)
            const int stages = nrows;
            std::vector<Real> data(static_cast<size_t>(stages) * ext_cols);
            for (int st = 0; st < stages; ++st)
                std::copy(&r.acc[static_cast<size_t>(v_max - v_top - st) * ext_cols],
                          &r.acc[static_cast<size_t>(v_max - v_top - st) * ext_cols] + ext_cols,
                          &data[static_cast<size_t>(st) * ext_cols]);
            const int offs[11] = {0, -1, 1, -2, 2, -3, 3, -4, 4, -5, 5};
            Real pen[11];
            for (int i = 0; i < 11; ++i)
                pen[i] = cfg.paper_sign ? cfg.lambda_x * offs[i] : cfg.lambda_x * std::abs(offs[i]);
            std::vector<int> path;
            rep.upath_energy = dp_min_path(stages, ext_cols, data.data(), offs, 11, pen, path);
            for (int i = 0; i < stages; ++i) r.upath.emplace_back(ext_lo + path[i], v_max - i);
            bool ev = false;
            for (Real x : r.acc)
                if (x != 0) {
                    ev = true;
                    break;
                }
            rep.upath_has_evidence = ev;
            if (!ev) throw Fail{11, LK_MSG_NO_EDGE_EVIDENCE, 0};

            RansacOut o = ransac(5, r.upath, cfg.tr_x, cfg.eps_x, 200, cfg.rng_seed);
            std::copy(o.model, o.model + 5, rep.gamma);
            rep.gamma_kappa = 1;
            rep.gamma_v_normalizer = o.s;
            rep.gamma_iterations = o.iterations;
            rep.gamma_inlier_fraction = o.fraction;
            rep.gamma_degraded = o.degraded;
            rep.gamma_inlier_count = static_cast<int64_t>(o.inliers.size());
            r.gamma_inliers = o.inliers;
            r.vpx.assign(H, 0);  // vpx_profile (vanish.hpp:276-281)
            for (int v = 0; v < H; ++v) r.vpx[v] = quartic_eval(o.model, static_cast<Real>(v));
        }

        // ---- stage 12: lanes (pipeline.hpp:260-270)
        stage = 12;
        {
            // build_m0 (lanes.hpp:30-61)
            std::vector<Real> wg(N, 0.0);
            for (const lk_edge& e : r.edges) {
                if (!(e.v >= v_top && e.v <= v_max)) continue;
                const Real dx = r.vpx[e.v] - e.u;
                const Real dy = r.vpy[e.v] - e.v;
                if (std::abs(dx) < 1e-12 && std::abs(dy) < 1e-12) continue;
                const Real theta_ray = std::atan2(dy, dx);
                const Real theta_tangent = e.theta + kPi / 2;
                wg[static_cast<size_t>(e.v) * W + e.u] =
                    e.gx * piecewise_weight(theta_tangent, theta_ray, cfg.sigma_g);
            }
            r.m0.assign(N, 0);
            for (int v = 0; v < H; ++v)
                for (int u = 0; u < W; ++u) {
                    Real s = 0;
                    for (int y = -cfg.varsigma; y <= cfg.varsigma; ++y) {
                        const int vv = v + y;
                        if (vv < 0 || vv >= H) continue;
                        for (int x = -cfg.nu; x <= cfg.nu; ++x) {
                            const int uu = u + x;
                            if (uu < 0 || uu >= W) continue;
                            s += wg[static_cast<size_t>(vv) * W + uu];
                        }
                    }
                    r.m0[static_cast<size_t>(v) * W + u] = s;
                }
            // build_m1 (lanes.hpp:67-76)
            r.m1.assign(N, 0);
            const Real* m0 = r.m0.data();
            auto M = [&](int u, int v) { return m0[static_cast<size_t>(v) * W + u]; };
            for (int v = 1; v < H - 1; ++v)
                for (int u = 1; u < W - 1; ++u)
                    r.m1[static_cast<size_t>(v) * W + u] =
                        (M(u + 1, v - 1) - M(u - 1, v - 1)) + 2 * (M(u + 1, v) - M(u - 1, v)) +
                        (M(u + 1, v + 1) - M(u - 1, v + 1));
            const Real tr = std::isnan(cfg.tr_lpv)
                                ? auto_lane_threshold(r.m1.data(), W, H, v_top, v_max)
                                : cfg.tr_lpv;
            rep.tr_lpv_used = tr;

            // aggregate_energy (lanes.hpp:106-129)
            const int nrows = v_max - v_top + 1;
            std::vector<Real> track(nrows);
            r.energy.assign(ext_cols, 0);
            for (int ci = 0; ci < ext_cols; ++ci) {
                lane_track(static_cast<Real>(ext_lo + ci), r.vpx.data(), r.vpy.data(), v_top,
                           v_max, track.data());
                Real e = 0;
                for (int v = v_max; v >= v_top; --v) {
                    Real contrib = 0;
                    const Real tu = track[v - v_top];
                    if (!std::isnan(tu)) {
                        const long long rr = std::llround(tu);
                        if (rr >= 0 && rr < W && v >= 0 && v < H)
                            contrib = r.m1[static_cast<size_t>(v) * W + static_cast<int>(rr)];
                    }
                    e = contrib + cfg.lambda_g * e;
                }
                r.energy[ci] = e;
            }

            // select_lanes (lanes.hpp:144-178)
            const std::vector<Real>& h = r.energy;
            const int n = ext_cols;
            std::vector<int> cand;
            for (int i = 1; i + 1 < n; ++i)
                if (h[i] < h[i - 1] && h[i] < h[i + 1] && h[i] < tr) cand.push_back(i);
            std::sort(cand.begin(), cand.end(), [&](int a, int b) {
                if (h[a] != h[b]) return h[a] < h[b];
                return a < b;
            });
            std::vector<int> kept;
            for (int i : cand) {
                bool close = false;
                for (int k : kept)
                    if (std::abs(i - k) < cfg.min_lane_sep) {
                        close = true;
                        break;
                    }
                if (close) continue;
                kept.push_back(i);
                lk_lane lane{};
                lane.bottom_col = ext_lo + i;
                lane.energy = h[i];
                lane_track(static_cast<Real>(lane.bottom_col), r.vpx.data(), r.vpy.data(), v_top,
                           v_max, track.data());
                int np = 0;
                for (int v = v_top; v <= v_max; ++v) np += !std::isnan(track[v - v_top]);
                lane.n_points = np;
                r.polylines.insert(r.polylines.end(), track.begin(), track.end());
                r.lanes.push_back(lane);
            }
            rep.lane_count = static_cast<int64_t>(r.lanes.size());
            for (size_t i = 0; i < r.lanes.size() && i < LK_MAX_INLINE_LANES; ++i) {
                rep.lane_bottom_col[i] = r.lanes[i].bottom_col;
                rep.lane_energy[i] = r.lanes[i].energy;
            }
        }
    } catch (const Fail& f) {
        rep.status = LK_ERR_FRAME;
        rep.failed_stage = f.stage ? f.stage : stage;
        rep.msg = f.msg;
        rep.err_row = f.row;
    }
}

}  // namespace orc
