// synth.cpp — synthetic stereo scene generator (host, test-kit input).
//
// Restates lanekit::gen_scene (synth.hpp:103-200) with its hash value noise
// (synth.hpp:20-58) and the 8-bit quantisation of write_png_gray
// (image_io.hpp:184-193), so frames fed to the GPU carry exactly the bytes
// the reference's own tooling would write. Extensions for the stress config
// (not in the reference): fronto-parallel obstacle boxes with constant
// disparity and their own texture, and a pitch change above which the road
// profile continues as a straight line with a slope jump.
// Compiled with -O3 -ffp-contract=off, like the reference's Release build.
#include <algorithm>
#include <atomic>
#include <cmath>
#include <string>
#include <thread>
#include <vector>

#include "../../include/lanekit_b200.h"

namespace {

constexpr double kPi = 3.14159265358979323846;

uint64_t hash64(uint64_t x) {  // synth.hpp:20-25 (splitmix64 finaliser)
    x += 0x9e3779b97f4a7c15ULL;
    x = (x ^ (x >> 30)) * 0xbf58476d1ce4e5b9ULL;
    x = (x ^ (x >> 27)) * 0x94d049bb133111ebULL;
    return x ^ (x >> 31);
}

double hash_unit(uint64_t seed, uint64_t salt, int64_t x, int64_t y) {  // synth.hpp:28-33
    uint64_t h = hash64(seed ^ (salt * 0xd6e8feb86659fd93ULL));
    h = hash64(h ^ static_cast<uint64_t>(x));
    h = hash64(h ^ static_cast<uint64_t>(y));
    return static_cast<double>(h >> 11) * 0x1.0p-53;
}

double value_noise(uint64_t seed, uint64_t salt, double x, double y, double cx,
                   double cy) {  // synth.hpp:37-51
    const double gx = x / cx, gy = y / cy;
    const double fx = std::floor(gx), fy = std::floor(gy);
    const int64_t x0 = static_cast<int64_t>(fx), y0 = static_cast<int64_t>(fy);
    double tx = gx - fx, ty = gy - fy;
    tx = tx * tx * (3 - 2 * tx);
    ty = ty * ty * (3 - 2 * ty);
    auto corner = [&](int64_t a, int64_t b) { return 2 * hash_unit(seed, salt, a, b) - 1; };
    const double c00 = corner(x0, y0), c10 = corner(x0 + 1, y0);
    const double c01 = corner(x0, y0 + 1), c11 = corner(x0 + 1, y0 + 1);
    const double top = c00 + tx * (c10 - c00);
    const double bot = c01 + tx * (c11 - c01);
    return top + ty * (bot - top);
}

double hash_gauss(uint64_t seed, uint64_t salt, int64_t x, int64_t y) {  // synth.hpp:54-58
    const double u1 = hash_unit(seed, salt, x, y);
    const double u2 = hash_unit(seed, salt + 0x71ULL, x, y);
    return std::sqrt(-2 * std::log(1 - u1)) * std::cos(2 * kPi * u2);
}

double road_f(const double* b, double v) { return b[0] + b[1] * v + b[2] * v * v; }
double road_fp(const double* b, double v) { return b[1] + 2 * b[2] * v; }

bool horizon_row(const double* b, int rows, int* out) {  // road_profile.hpp:161-176
    double root;
    if (b[2] == 0) {
        if (b[1] <= 0) return false;
        root = -b[0] / b[1];
    } else {
        const double disc = b[1] * b[1] - 4 * b[2] * b[0];
        if (disc <= 0) return false;
        root = (-b[1] + std::sqrt(disc)) / (2 * b[2]);
    }
    const long long r = std::llround(root);
    if (r < 0 || r >= rows) return false;
    *out = static_cast<int>(r);
    return true;
}

// lanes.hpp:83-96 — track[i] is row v_top + i, NaN once truncated.
void lane_track(double u_bottom, const std::vector<double>& vpx, const std::vector<double>& vpy,
                int v_top, int v_max, std::vector<double>& track) {
    const int n = v_max - v_top + 1;
    track.assign(n, std::numeric_limits<double>::quiet_NaN());
    track[n - 1] = u_bottom;
    for (int v = v_max - 1; v >= v_top; --v) {
        const double u_next = track[v + 1 - v_top];
        const double py = vpy[v + 1];
        const double denom = static_cast<double>(v + 1) - py;
        if (std::abs(denom) < 0.5) break;
        track[v - v_top] = (vpx[v + 1] + v * u_next - py * u_next) / denom;
    }
}

uint8_t quantise(double x) {  // image_io.hpp:186-188
    const long q = std::lround(x * 255.0);
    return static_cast<uint8_t>(std::clamp(q, 0L, 255L));
}

thread_local std::string g_msg;

lk_status synth_one(const lk_scene_params& p, uint8_t* gl, uint8_t* gr, uint8_t* dm,
                    int32_t* horizon_out) {
    const int W = p.width, H = p.height;
    if (W < 16 || H < 16) return g_msg = "scene: image too small", LK_ERR_INVALID_ARGUMENT;
    if (p.d_max < 1) return g_msg = "scene: d_max must be positive", LK_ERR_INVALID_ARGUMENT;
    if (p.n_lanes < 0 || p.n_lanes > 8 || p.n_obstacles < 0 || p.n_obstacles > 4)
        return g_msg = "scene: bad lane / obstacle count", LK_ERR_INVALID_ARGUMENT;
    int h = 0;
    if (!horizon_row(p.beta, H, &h))
        return g_msg = "scene: beta has no horizon inside the image", LK_ERR_INVALID_ARGUMENT;
    const int v_max = H - 1;
    if (road_fp(p.beta, h) <= 0 || road_fp(p.beta, v_max) <= 0)
        return g_msg = "scene: beta must be increasing over the road rows", LK_ERR_INVALID_ARGUMENT;

    // Road disparity per row. Extension: above pitch_row the profile is the
    // tangent line at pitch_row with its slope scaled by (1 + pitch_jump).
    const bool pitch = p.pitch_row >= 0 && p.pitch_row < H;
    int road_top = h;
    double line_f0 = 0, line_slope = 0;
    if (pitch) {
        if (p.pitch_row < h || !(1 + p.pitch_jump > 0))
            return g_msg = "scene: pitch row above the horizon or slope flip", LK_ERR_INVALID_ARGUMENT;
        line_f0 = road_f(p.beta, p.pitch_row);
        line_slope = road_fp(p.beta, p.pitch_row) * (1 + p.pitch_jump);
        const double root = p.pitch_row - line_f0 / line_slope;
        road_top = static_cast<int>(std::clamp(std::llround(root), 0LL, (long long)p.pitch_row));
    }
    auto profile = [&](int v) {
        if (pitch && v < p.pitch_row) return line_f0 + line_slope * (v - p.pitch_row);
        return road_f(p.beta, static_cast<double>(v));
    };
    std::vector<int> shift(H, 0);
    for (int v = road_top; v < H; ++v) {
        const long long d = std::llround(profile(v));
        if (d < 0 || d > p.d_max)
            return g_msg = "scene: beta leaves [0, d_max] on road rows", LK_ERR_INVALID_ARGUMENT;
        shift[v] = static_cast<int>(d);
    }
    // true vanishing-point profile of the base road (synth.hpp:126-134)
    std::vector<double> vpx(H), vpy(H);
    for (int v = 0; v < H; ++v) {
        const double t = static_cast<double>(v);
        const double fp = road_fp(p.beta, t);
        vpy[v] = std::abs(fp) < 1e-12 ? t : t - road_f(p.beta, t) / fp;  // road_profile.hpp:184-199
        vpx[v] = p.gamma[0] + t * (p.gamma[1] + t * (p.gamma[2] + t * (p.gamma[3] + t * p.gamma[4])));
    }
    int max_shift = shift[v_max];
    for (int k = 0; k < p.n_obstacles; ++k) max_shift = std::max(max_shift, p.obstacle_disp[k]);
    const int wide = W + max_shift;
    std::vector<double> field(static_cast<size_t>(wide) * H);
    for (int v = 0; v < H; ++v)  // synth.hpp:137-155
        for (int u = 0; u < wide; ++u) {
            double& x = field[static_cast<size_t>(v) * wide + u];
            if (v < road_top) {
                x = p.sky_level;
                continue;
            }
            const double n = 0.55 * value_noise(p.rng_seed, 11, u, v, 2.0, 16.0) +
                             0.35 * value_noise(p.rng_seed, 13, u, v, 5.0, 40.0) +
                             0.1 * (2 * hash_unit(p.rng_seed, 17, u, v) - 1);
            x = p.road_base + p.texture_amplitude * n;
        }
    std::vector<double> lb_t, rb_t;
    for (int li = 0; li < p.n_lanes; ++li) {  // synth.hpp:159-182
        const double bottom = p.lane_bottoms[li];
        lane_track(bottom - p.lane_width / 2, vpx, vpy, h, v_max, lb_t);
        lane_track(bottom + p.lane_width / 2, vpx, vpy, h, v_max, rb_t);
        for (int v = v_max; v >= h; --v) {
            const int i = v - h;
            const double lb = lb_t[i], rb = rb_t[i];
            if (std::isnan(lb) || std::isnan(rb) || rb - lb < 0.5) break;
            const int u0 = std::max(0, static_cast<int>(std::floor(lb - 1)));
            const int u1 = std::min(wide - 1, static_cast<int>(std::ceil(rb + 1)));
            for (int u = u0; u <= u1; ++u) {
                const double cov =
                    std::clamp(std::min(rb, u + 0.5) - std::max(lb, u - 0.5), 0.0, 1.0);
                if (cov <= 0) continue;
                double& x = field[static_cast<size_t>(v) * wide + u];
                x = x + cov * (p.lane_brightness - x);
            }
        }
    }
    std::vector<int> dmap(static_cast<size_t>(W) * H);
    for (int v = 0; v < H; ++v)  // synth.hpp:184-198
        for (int u = 0; u < W; ++u) {
            double l = field[static_cast<size_t>(v) * wide + u];
            double r = field[static_cast<size_t>(v) * wide + u + shift[v]];
            if (p.noise_sigma > 0) {
                l += p.noise_sigma * hash_gauss(p.rng_seed, 21, u, v);
                r += p.noise_sigma * hash_gauss(p.rng_seed, 23, u, v);
            }
            const size_t i = static_cast<size_t>(v) * W + u;
            if (gl) gl[i] = quantise(std::clamp(l, 0.0, 1.0));
            if (gr) gr[i] = quantise(std::clamp(r, 0.0, 1.0));
            dmap[i] = shift[v];
        }
    // Extension: obstacles (later boxes occlude earlier ones).
    for (int k = 0; k < p.n_obstacles; ++k) {
        const int* b = p.obstacle_box[k];
        const int dob = p.obstacle_disp[k];
        for (int v = std::max(0, b[1]); v <= std::min(H - 1, b[3]); ++v)
            for (int u = std::max(0, b[0]); u <= std::min(W - 1, b[2]); ++u) {
                const size_t i = static_cast<size_t>(v) * W + u;
                const double tex = 0.5 + 0.25 * value_noise(p.rng_seed, 31 + k, u, v, 3.0, 3.0);
                double l = tex;
                if (p.noise_sigma > 0) l += p.noise_sigma * hash_gauss(p.rng_seed, 21, u, v);
                if (gl) gl[i] = quantise(std::clamp(l, 0.0, 1.0));
                dmap[i] = dob;
                const int ur = u - dob;  // the right view sees the box shifted left
                if (gr && ur >= 0) gr[static_cast<size_t>(v) * W + ur] = quantise(std::clamp(tex, 0.0, 1.0));
            }
    }
    if (dm)
        for (size_t i = 0; i < dmap.size(); ++i) dm[i] = static_cast<uint8_t>(std::clamp(dmap[i], 0, 255));
    if (horizon_out) *horizon_out = road_top;
    return LK_OK;
}

}  // namespace

extern "C" {

void lk_scene_default(lk_scene_params* p) {  // synth.hpp:62-80
    *p = lk_scene_params{};
    p->width = 640;
    p->height = 360;
    p->beta[0] = -15.0;
    p->beta[1] = 0.15;
    p->beta[2] = 0.0001;
    p->gamma[0] = 320.0;
    p->d_max = 192;
    p->n_lanes = 3;
    p->lane_bottoms[0] = 160.0;
    p->lane_bottoms[1] = 320.0;
    p->lane_bottoms[2] = 480.0;
    p->lane_width = 6.0;
    p->lane_brightness = 0.85;
    p->road_base = 0.35;
    p->sky_level = 0.75;
    p->texture_amplitude = 0.15;
    p->noise_sigma = 0.0;
    p->rng_seed = 1;
    p->pitch_row = -1;
}

const char* lk_synth_last_error(void) { return g_msg.c_str(); }

lk_status lk_synth_scene(const lk_scene_params* p, uint8_t* gl, uint8_t* gr, uint8_t* dm,
                         int32_t* horizon) {
    if (!p) return LK_ERR_INVALID_ARGUMENT;
    return synth_one(*p, gl, gr, dm, horizon);
}

lk_status lk_synth_stereo_batch(const lk_scene_params* params, int n, uint8_t* left,
                                uint8_t* right, uint8_t* disp, int threads) {
    if (!params || n < 0) return LK_ERR_INVALID_ARGUMENT;
    if (threads < 1) threads = 1;
    std::atomic<int> next{0};
    std::atomic<int> bad{0};
    std::vector<std::thread> pool;
    for (int t = 0; t < threads; ++t)
        pool.emplace_back([&] {
            for (int i = next++; i < n; i = next++) {
                const size_t off = static_cast<size_t>(i) * params[0].width * params[0].height;
                if (params[i].width != params[0].width || params[i].height != params[0].height ||
                    synth_one(params[i], left ? left + off : nullptr, right ? right + off : nullptr,
                              disp ? disp + off : nullptr, nullptr) != LK_OK)
                    bad = 1;
            }
        });
    for (auto& t : pool) t.join();
    return bad ? LK_ERR_INVALID_ARGUMENT : LK_OK;
}

lk_status lk_synth_batch(const lk_scene_params* params, int n, uint8_t* grey, uint8_t* disp,
                         int threads) {
    return lk_synth_stereo_batch(params, n, grey, nullptr, disp, threads);
}

}  // extern "C"
