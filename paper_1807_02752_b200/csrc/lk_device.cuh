// lk_device.cuh — device-side layout and exact-arithmetic helpers shared by
// the stage kernels. Every translation unit is compiled with --fmad=false so
// each double + and * rounds exactly like the reference's SSE2 build
// (no -march, no FMA contraction: reference proj/CMakeLists.txt:8-10).
#pragma once

#include <cstdint>

#include "../../include/lanekit_b200.h"

namespace lkg {

constexpr double kPi = 3.14159265358979323846;  // common.hpp:11
constexpr int kSkipCol = INT32_MIN;              // edge without a vote (vanish.hpp:59-62)

// Per-frame scratch scalars that are not part of the public report.
struct FrameAux {
    unsigned long long hist_total;  // pixels counted by the v-disparity (evidence)
    unsigned long long mask_px;
    unsigned long long edge_px;
    unsigned long long votes;
    unsigned long long skipped;
    unsigned int p99_cands;         // candidates in the p99 exponent bucket
    unsigned int p99_bucket;
    unsigned int p99_bucket2;      // next 12 bits inside the exponent bucket
    unsigned int p99_done;         // the percentile is exactly +0 (rank among the zeros)
    unsigned int p99_level2;       // bucket too large: narrowed by a second histogram
    unsigned int fneed;             // need-list length of the FP32 bilateral (k_prescreen)
    unsigned long long p99_zeros;  // |m1| values that are exactly zero
    unsigned long long p99_rank;    // rank of the percentile inside the bucket
    double tr;                      // tr_lpv used
    int lanes;                      // kept lanes
    unsigned int uncertain_gates;   // w_g gates within kGateEps of pi/6 (k_wg)
    unsigned long long max_wg;      // max |w_g| (IEEE bits of a non-negative double)
};

// Everything a kernel needs, passed by value. Pointers index frame-major
// buffers sized for the context's max_batch.
struct Dev {
    // geometry
    int W, H, D1, d_max, ext_lo, ext_cols, rho, win, words_per_row;
    int lane_cap;
    int hooks;
    size_t px;  // W*H
    // config (config.hpp:16-46)
    double lambda_y, tr_y, eps_y, varpi, rho_vote, lambda_x, tr_x, eps_x, sigma_g, lambda_g,
        tr_lpv;
    int chi, nu, varsigma, min_lane_sep, paper_sign, max_iter;
    double upen[11];  // u-path transition penalty per offset index (vanish.hpp:163-166)
    int upk[11];      // exact-int path keys: (int)upen * 16 + index
    unsigned int p99_l2_min;  // bucket size above which the p99 uses a 2nd histogram level
    double sobel_s_star;  // smallest s with !(sqrt(s) < threshold): exact sqrt-free test
    float sobel_s_star_lo;  // largest float <= sobel_s_star (FP32 candidate screen)
    // inputs
    const uint8_t* grey;    // left grey (stereo) or the only grey
    const uint8_t* disp;
    // stereo front end, stages 1-4 (LK_FLAG_STEREO; stereo.hpp)
    int stereo;
    int srho, tau, tr_lrc;  // block radius, search propagation bound, LRC tolerance
    double sigma_floor;
    const uint8_t* right;   // [B][H][W] right grey
    double* sat;            // [B][4][H][W] integral images: left, left^2, right, right^2
    double* mu_l;           // [B][H][W] block statistics (0 on the border)
    double* sig_l;
    double* mu_r;
    double* sig_r;
    uint8_t* disp_l;        // [B][H][W] SRP disparity, left / right reference
    uint8_t* disp_r;
    uint8_t* disp_out;      // the LRC result = the disparity input of stages 5-12
    // tables built on the host with the reference's libm
    const double* ws;       // [win*win] exp(-ds*inv_s2)
    const double* wr;       // [256][256] exp(-dr*dr*inv_r2)
    unsigned long long wr_tex;  // texture object over wr (int2 texels)
    const double* val;      // [256] k/255.0
    const uint64_t* rng;    // mt19937_64(seed) outputs 0..max_iter*5-1
    // outputs / intermediates
    lk_frame_report* rep;
    FrameAux* aux;
    int8_t* vchoice;        // [B][D1][H]
    int32_t* vpath;         // [B][D1][2]
    int32_t* beta_inl;      // [B][D1][2]
    double* vpy;            // [B][H]
    uint8_t* vsing;         // [B][H]
    double* fv;             // [B][H]
    double* vpx;            // [B][H]
    double* smoothed;       // [B][H][W] (fast path: exact only around edge candidates)
    float* smoothed_f;      // [B][H][W] certified approximation (fast path)
    uint32_t* need;         // [B][need_cap] pixels (v << 16 | u) whose exact smoothed value the
                            // fast path needs (3x3 neighbourhoods of Sobel candidates)
    uint32_t* need_cnt;     // [B]
    uint32_t* ctile;        // [B][n_stile] Sobel tiles holding candidates
    uint32_t* ctile_cnt;    // [B]
    int need_cap, n_stile;
    const float2* need_tab; // [511] (R(delta), R(delta) * delta), delta = i - 255 (k_bilateral_need)
    uint32_t* pbits;        // [B][H][words_per_row] pre-screen survivors ("possibly an edge")
    uint32_t* fneed;        // [B][px] pixels (v << 16 | u) whose s~ the Sobel screen needs
    uint32_t* ebits;        // [B][H][words_per_row]
    int n_seg;              // edge-list segments per row (ceil(W / SB_TW))
    int32_t* seg_cnt;       // [B][H][n_seg]
    int32_t* seg_off;       // [B][H][n_seg]
    int32_t* row_off;       // [B][H+1]
    int32_t* e_uv;          // [B][px]  u | v << 16
    double* e_gx;           // [B][px]
    double* e_gy;
    double* e_th;
    double* e_wg;
    int32_t* e_col;         // [B][px]  vote column or kSkipCol
    int8_t* uchoice;        // [B][H][ext_cols]
    int32_t* upath;         // [B][H][2]
    int32_t* gamma_inl;     // [B][H][2]
    double* m1;             // [B][H][W] (only tiles flagged in m1_nz are written)
    uint8_t* m1_nz;         // [B][m_nty][m_ntx] m0/m1 tile has a non-zero
    int m_tile_shift, m_ntx, m_nty;  // m0/m1 tile: (1 << m_tile_shift) rows x M_TW cols
    int vote_cap;           // k_vanish: vote columns staged in shared memory
    unsigned int* p99hist;  // [B][2048]
    unsigned int* p99hist2; // [B][4096]
    unsigned long long* p99cand;  // [B][px]
    double* energy;         // [B][ext_cols]
    int2* mrange;           // [B][H] road-mask disparity interval per row (empty above the horizon)
    int32_t* track_np;      // [B][ext_cols] finite points of each column's lane_track
    uint8_t* e_touch;       // [B][ext_cols] the column's track read a cell within reach of a w_g != 0
    uint8_t* wg_nz;         // [B][m_nty][m_ntx] m0/m1 tiles with a non-zero w_g in reach
    lk_lane* lanes;         // [B][lane_cap]
    double* polylines;      // [B][lane_cap][H] (hooks)
    // hooks (LK_FLAG_HOOKS)
    uint8_t* mask;
    double* gx;
    double* gy;
    double* mag;
    double* theta;
    double* acc;            // [B][H][ext_cols] rows from horizon
    double* m0;
};

// std::llround as glibc/x86-64 behaves: round half away from zero; NaN and
// |x| >= 2^63 give LLONG_MIN (cvttsd2si "integer indefinite").
__device__ __forceinline__ long long llround_ref(double x) {
    if (!(fabs(x) < 9223372036854775808.0)) return (long long)0x8000000000000000ULL;
    return llround(x);
}

// common.hpp:28-35
__device__ __forceinline__ int mirror(int i, int n) {
    if (n <= 1) return 0;
    while (i < 0 || i >= n) {
        if (i < 0) i = -i - 1;
        if (i >= n) i = 2 * n - 1 - i;
    }
    return i;
}

// road_mask's test |double(d) - f(v)| <= varpi (preprocess.hpp:14-25) over the
// integers d in [1, 255] holds on an interval [lo, hi] (fl(d - f) is monotone
// in d) inside [f - varpi - 1, f + varpi + 1] (the double subtraction errs by
// < 1e-13): found by evaluating the reference's expression; lo > hi = empty.
__device__ __forceinline__ int2 mask_interval(double fr, double varpi) {
    auto test = [&](int x) { return fabs((double)x - fr) <= varpi; };
    const double a = fr - varpi - 1.0, b = fr + varpi + 1.0;
    const int l0 = a >= 1.0 ? (a <= 255.0 ? (int)ceil(a) : 256) : 1;  // NaN -> 1
    const int h0 = b <= 255.0 ? (b >= 1.0 ? (int)floor(b) : 0) : 255;  // NaN -> 255
    int lo = 256, hi = 0;
    for (int x = l0; x <= h0; ++x)
        if (test(x)) {
            lo = x;
            break;
        }
    for (int x = h0; x >= lo; --x)
        if (test(x)) {
            hi = x;
            break;
        }
    return make_int2(lo, hi);
}

__device__ __forceinline__ bool frame_failed(const Dev& d, int f) {
    return d.rep[f].status != 0;
}

__device__ __forceinline__ void fail_frame(const Dev& d, int f, int stage, int msg, int row = 0) {
    lk_frame_report& r = d.rep[f];
    r.status = LK_ERR_FRAME;
    r.failed_stage = stage;
    r.msg = msg;
    r.err_row = row;
}

// Rounds up to 8-byte alignment by pointer arithmetic (not an integer
// round-trip), so the compiler keeps the shared-memory address space and
// emits LDS/STS rather than generic LD/ST.
__device__ __forceinline__ double* align8(void* p) {
    char* c = (char*)p;
    return (double*)(c + ((8 - ((uintptr_t)c & 7)) & 7));
}

// a / b, correctly rounded, given y = RN(1 / b): q0 = RN(a y), r = a - q0 b
// (exact, FMA), q = RN(q0 + r y) (Markstein's theorem; checked against IEEE
// division on 3e10 cases by tools/markstein_check.cu). Zero, non-finite or
// extreme operands fall back to the IEEE division, so the result is always
// bit-identical to a / b. Lets several quotients share one reciprocal.
__device__ __forceinline__ double div_rn(double a, double b, double y) {
    const double aa = fabs(a), ab = fabs(b);
    if (aa >= 0x1p-500 && aa <= 0x1p500 && ab >= 0x1p-500 && ab <= 0x1p500) {
        const double q0 = __dmul_rn(a, y);
        return __fma_rn(__fma_rn(-q0, b, a), y, q0);
    }
    return a / b;
}

// Ordered double -> u64 key (total order equal to '<' for non-NaN values).
__device__ __forceinline__ unsigned long long order_key(double x) {
    unsigned long long b = (unsigned long long)__double_as_longlong(x);
    return (b & 0x8000000000000000ULL) ? ~b : (b | 0x8000000000000000ULL);
}

}  // namespace lkg
