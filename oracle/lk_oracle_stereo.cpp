// lk_oracle_stereo.cpp — TEST INFRASTRUCTURE ONLY. CPU restatement of stages
// 1-4 of run_pipeline (pipeline.hpp:161-182): block statistics from integral
// images, search-range-propagated NCC matching for both reference views, and
// the left-right consistency check. Pinned against the compiled reference
// (lkref_stereo, oracle/ref_wrapper.cpp) bit for bit by tests/test_stereo.py.
// Never linked into the product; only tests/, smoke() and bench.py's
// reference leg load it.
#include <algorithm>
#include <climits>
#include <cmath>
#include <cstdint>
#include <cstdlib>
#include <utility>
#include <vector>

namespace {

struct Map {
    int W = 0, H = 0;
    std::vector<double> a;
    double at(int u, int v) const { return a[(size_t)v * W + u]; }
};

// build_integral (integral.hpp:22-35): in(u, v) = in(u, v-1) + in(u-1, v)
// - in(u-1, v-1) + x(u, v), left to right, reads at -1 give 0.
Map integral(const Map& x) {
    Map s{x.W, x.H, std::vector<double>(x.a.size())};
    auto at = [&](int u, int v) { return (u < 0 || v < 0) ? 0.0 : s.a[(size_t)v * s.W + u]; };
    for (int v = 0; v < x.H; ++v)
        for (int u = 0; u < x.W; ++u)
            s.a[(size_t)v * s.W + u] = at(u, v - 1) + at(u - 1, v) - at(u - 1, v - 1) + x.at(u, v);
    return s;
}

// block_sum (integral.hpp:39-47)
double block_sum(const Map& in, int u, int v, int rho) {
    auto at = [&](int x, int y) { return (x < 0 || y < 0) ? 0.0 : in.at(x, y); };
    return at(u + rho, v + rho) + at(u - rho - 1, v - rho - 1) - at(u - rho - 1, v + rho) -
           at(u + rho, v - rho - 1);
}

// precompute_stats (stereo.hpp:39-60): mu / sigma, 0 where the block leaves the image
void stats(const Map& img, int rho, Map& mu, Map& sigma) {
    Map sq = img;
    for (double& x : sq.a) x = x * x;
    const Map in = integral(img), in2 = integral(sq);
    mu = Map{img.W, img.H, std::vector<double>(img.a.size(), 0.0)};
    sigma = mu;
    const double n = double(2 * rho + 1) * double(2 * rho + 1);
    for (int v = rho; v < img.H - rho; ++v)
        for (int u = rho; u < img.W - rho; ++u) {
            const double m = block_sum(in, u, v, rho) / n;
            const double var = block_sum(in2, u, v, rho) / n - m * m;
            mu.a[(size_t)v * img.W + u] = m;
            sigma.a[(size_t)v * img.W + u] = std::sqrt(std::max(0.0, var));
        }
}

// ncc_cost (stereo.hpp:67-84): left block at ul, right block at ur
double ncc(const Map& L, const Map& R, const Map& muL, const Map& sgL, const Map& muR,
           const Map& sgR, int ul, int ur, int v, int rho) {
    double dot = 0;
    for (int y = -rho; y <= rho; ++y)
        for (int x = 0; x <= 2 * rho; ++x) dot += L.at(ul - rho + x, v + y) * R.at(ur - rho + x, v + y);
    const double n = double(2 * rho + 1) * double(2 * rho + 1);
    return (dot - n * muL.at(ul, v) * muR.at(ur, v)) / (n * sgL.at(ul, v) * sgR.at(ur, v));
}

// match_srp (stereo.hpp:114-196). view 0: left reference (other column u - d),
// view 1: right reference (u + d). Candidates: SearchRanges (:89-112).
std::vector<int> srp(const Map& L, const Map& R, const Map& muL, const Map& sgL, const Map& muR,
                     const Map& sgR, int view, int rho, int d_min, int d_max, int tau,
                     double floor_) {
    const int W = L.W, H = L.H;
    std::vector<int> disp((size_t)W * H, 0);
    const Map& refsg = view ? sgR : sgL;
    const Map& othsg = view ? sgL : sgR;
    const int v_bottom = H - 1 - rho;
    for (int v = v_bottom; v >= rho; --v) {
        for (int u = rho; u < W - rho; ++u) {
            if (refsg.at(u, v) < floor_) {
                disp[(size_t)v * W + u] = 0;
                continue;
            }
            std::vector<std::pair<int, int>> iv;
            auto add = [&](int lo, int hi) {
                lo = std::max(lo, d_min);
                hi = std::min(hi, d_max);
                if (lo <= hi) iv.push_back({lo, hi});
            };
            if (v == v_bottom) {
                add(d_min, d_max);
            } else {
                for (int k = u - 1; k <= u + 1; ++k) {
                    if (k < 0 || k >= W) continue;
                    const int l = disp[(size_t)(v + 1) * W + k];
                    add(l - tau, l + tau);
                }
                if (iv.empty()) add(d_min, d_max);
            }
            std::sort(iv.begin(), iv.end());
            double best = 0;
            int best_d = -1;
            int next = INT_MIN;
            for (const auto& p : iv) {
                for (int d = std::max(p.first, next); d <= p.second; ++d) {
                    const int uo = view ? u + d : u - d;
                    if (uo < rho || uo >= W - rho) continue;
                    if (othsg.at(uo, v) < floor_) continue;
                    const double c = view ? ncc(L, R, muL, sgL, muR, sgR, uo, u, v, rho)
                                          : ncc(L, R, muL, sgL, muR, sgR, u, uo, v, rho);
                    if (best_d < 0 || c > best) {
                        best = c;
                        best_d = d;
                    }
                }
                next = std::max(next, p.second + 1);
            }
            disp[(size_t)v * W + u] = best_d < 0 ? 0 : best_d;
        }
    }
    return disp;
}

}  // namespace

extern "C" {

// Stages 1-4 on one u8 stereo pair (k means k/255.0). Outputs (any may be
// NULL): stats_left mu / sigma (f64 [H][W]), the two SRP maps and the LRC
// result (u8 [H][W]).
int orc_stereo(const uint8_t* left, const uint8_t* right, int W, int H, int rho, int d_max,
               int tau, int tr_lrc, double sigma_floor, double* mu_l, double* sig_l,
               uint8_t* disp_l, uint8_t* disp_r, uint8_t* disparity) {
    if (W <= 2 * rho || H <= 2 * rho) return 1;
    Map L{W, H, std::vector<double>((size_t)W * H)}, R = L;
    for (size_t i = 0; i < L.a.size(); ++i) {
        L.a[i] = left[i] / 255.0;  // image_io.hpp:147
        R.a[i] = right[i] / 255.0;
    }
    Map muL, sgL, muR, sgR;
    stats(L, rho, muL, sgL);
    stats(R, rho, muR, sgR);
    const std::vector<int> dl = srp(L, R, muL, sgL, muR, sgR, 0, rho, 0, d_max, tau, sigma_floor);
    const std::vector<int> dr = srp(L, R, muL, sgL, muR, sgR, 1, rho, 0, d_max, tau, sigma_floor);
    for (int v = 0; v < H; ++v)  // lrc_check (stereo.hpp:263-276)
        for (int u = 0; u < W; ++u) {
            const size_t i = (size_t)v * W + u;
            const int d = dl[i], ur = u - d;
            int o = 0;
            if (ur >= 0 && ur < W && std::abs(d - dr[(size_t)v * W + ur]) <= tr_lrc) o = d;
            if (disparity) disparity[i] = (uint8_t)o;
            if (disp_l) disp_l[i] = (uint8_t)dl[i];
            if (disp_r) disp_r[i] = (uint8_t)dr[i];
            if (mu_l) mu_l[i] = muL.a[i];
            if (sig_l) sig_l[i] = sgL.a[i];
        }
    return 0;
}

}  // extern "C"
