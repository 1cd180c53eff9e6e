// lk_fastpath.cu — certified fast front end (stages 9-10) for throughput runs.
//
// The exact bilateral (k_bilateral_tile) is bound by random 8-byte gathers
// into the exact weight table. But the only consumers of the smoothed image
// downstream of stage 10 are the EDGE pixels (gx, gy, theta, votes, w_g all
// come from the edge list, preprocess.hpp:103-113), and the only integer
// decision taken on non-edge pixels is "not an edge". So:
//
//  1. k_bilateral_fast computes every pixel approximately: weights
//     2^(c_t + c2*dr^2) with MUFU ex2 and FP32 row-partial sums. A rigorous
//     bound |s~ - s| <= kEpsSmooth holds against the exact double result
//     (derivation in DESIGN.md §3; the worst error measured on 10^8 pixels is
//     recorded in profiles/).
//  2. k_sobel_refine evaluates Sobel on s~ and propagates the bound to
//     s = gx^2 + gy^2. A masked pixel whose s can still reach the threshold is
//     a candidate. Every pixel in a candidate's 3x3 neighbourhood gets its
//     EXACT bilateral (the LUT arithmetic of k_bilateral_tile), and the
//     candidate's edge decision and gradients use those exact values.
//
// The edge set, every edge's gx/gy, and everything downstream are therefore
// bit-identical to the exact path; only the (unexported) smoothed values of
// pixels far from any edge are approximate. Hooks mode always runs the exact
// path, so the SMOOTHED/GX/GY/MAG/THETA maps it exports are exact.
#include <cuda_runtime.h>

#include "lk_kernels.h"

namespace lkg {

constexpr double kEpsSmooth = 2.5e-5;  // bound on |s~ - s| (absolute, values in [0, 1])

__device__ __forceinline__ float ex2_approx(float x) {
    float y;
    asm("ex2.approx.ftz.f32 %0, %1;" : "=f"(y) : "f"(x));
    return y;
}

// ---- 1. approximate bilateral: tile BT_W x BT_H, BT_R outputs per thread
//
// Taps (2q, 2q+1) of a window row are processed as one packed f32x2 lane pair
// (FADD2 / FMUL2 / FFMA2), which halves the FP32 issue slots and leaves the
// range factor as the limiter. Tap pairs in the mask TB take it from a
// 511-entry shared-memory table instead of MUFU ex2, so the XU and the LSU
// pipes share the work. The table index comes from the float difference
// itself: dr*1020*RC is within 3e-3 of the integer 4 RC (k_q - k_p), so one FFMA with
// 1.5*2^23 rounds it into the low mantissa bits (no integer keys staged).
// w = S_t * R[dr] rounds three times in FP32 (~2e-7 relative), inside the
// ex2.approx error the bound in DESIGN.md already budgets.
//
// all = 0 (the pipeline): s~ is consumed only by the Sobel of road-mask pixels
// (k_sobel_refine), i.e. within one pixel of a masked pixel (mirroring at the
// border stays within that pixel). Tiles whose one-pixel ring holds no masked
// pixel are skipped; the test is the exact mask of k_sobel_refine
// (road_mask, preprocess.hpp:14-25). all = 1 computes every tile (lk_fast_path_error).
//
// The table is replicated RC times, entry-major (word i * RC + copy), and lane
// L reads copy L % RC: lanes with different entries then collide in a bank
// at most 32 / RC ways (RC = 16: 2-way) instead of up to 16-way.
template <int RHO, int TB>
__global__ void __launch_bounds__(256, 3) k_bilateral_fast(Dev d, FastBfParam p, int all) {
    constexpr int WIN = 2 * RHO + 1, TWh = BT_W + 2 * RHO, THh = BT_H + 2 * RHO;
    constexpr int NPX = TWh * THh;
    constexpr int RC = BF_TABLE_COPIES;
    static_assert(WIN == 11, "packed tap pairs assume an 11-wide window");
    __shared__ float s_v[NPX], s_vf[256], s_R[TB ? 512 * RC : 1];
    __shared__ int s_row[THh], s_col[TWh];
    const int f = blockIdx.z;
    if (frame_failed(d, f)) return;
    const int u0 = blockIdx.x * BT_W, v0 = blockIdx.y * BT_H;
    if (!all) {
        const int horizon = (int)d.rep[f].horizon;
        if (v0 + BT_H < horizon) return;  // ring rows all above the horizon
        const uint8_t* dp = d.disp + (size_t)f * d.px;
        const double* fv = d.fv + (size_t)f * d.H;
        int any = 0;
        for (int i = threadIdx.x; i < (BT_H + 2) * (BT_W + 2) && !any; i += blockDim.x) {
            const int r = i / (BT_W + 2), c = i - r * (BT_W + 2);
            const int v = v0 - 1 + r, u = u0 - 1 + c;
            if (v >= horizon && v >= 0 && v < d.H && u >= 0 && u < d.W) {
                const int dv = dp[(size_t)v * d.W + u];
                any = dv != 0 && fabs((double)dv - fv[v]) <= d.varpi;
            }
        }
        if (!__syncthreads_or(any)) return;
    }
    const uint8_t* g = d.grey + (size_t)f * d.px;
    s_vf[threadIdx.x] = __ldg(d.fast_tab + threadIdx.x);
    if (TB) {
        const float r0 = __ldg(d.fast_tab + 256 + threadIdx.x);
        const float r1 = __ldg(d.fast_tab + 512 + threadIdx.x);
#pragma unroll
        for (int k = 0; k < RC; ++k) {
            s_R[threadIdx.x * RC + k] = r0;
            s_R[(threadIdx.x + 256) * RC + k] = r1;
        }
    }
    if (threadIdx.x < THh) s_row[threadIdx.x] = mirror(v0 + (int)threadIdx.x - RHO, d.H) * d.W;
    if (threadIdx.x < TWh) s_col[threadIdx.x] = mirror(u0 + (int)threadIdx.x - RHO, d.W);
    __syncthreads();
    for (int i = threadIdx.x; i < NPX; i += blockDim.x) {
        const int ty = i / TWh, tx = i - ty * TWh;
        s_v[i] = s_vf[g[(size_t)s_row[ty] + s_col[tx]]];
    }
    __syncthreads();
    const int tx = threadIdx.x % BT_W, ty = threadIdx.x / BT_W;
    const int r0 = ty * BT_R;
    float va[BT_R], num[BT_R], den[BT_R];
    float2 nva[BT_R];
#pragma unroll
    for (int r = 0; r < BT_R; ++r) {
        va[r] = s_v[(r0 + r + RHO) * TWh + tx + RHO];
        nva[r] = make_float2(-va[r], -va[r]);
        num[r] = den[r] = 0.f;
    }
    const float2 c2 = make_float2(p.c2, p.c2);
    constexpr float kMagic = 12582912.0f;  // 1.5 * 2^23: float + kMagic rounds to an integer
    // t = dr*S + kMagic + S, S = 4 * 255 * RC: its bit pattern is
    // __float_as_int(kMagic) + the BYTE offset 4 * RC * (k_q - k_p + 255) of the
    // entry, so the LDS needs one add of the thread's base (its copy) only
    constexpr float kS = 1020.f * RC;
    const float2 kscale = make_float2(kS, kS), mg = make_float2(kMagic + kS, kMagic + kS);
    const char* Rb = reinterpret_cast<const char*>(s_R) + 4 * (threadIdx.x % RC) -
                     __float_as_int(kMagic);
#pragma unroll
    for (int jj = 0; jj < BT_R + 2 * RHO; ++jj) {
        const int prow = (r0 + jj) * TWh + tx;
        float2 vp[5];
#pragma unroll
        for (int q = 0; q < 5; ++q) vp[q] = make_float2(s_v[prow + 2 * q], s_v[prow + 2 * q + 1]);
        const float vl = s_v[prow + 10];
#pragma unroll
        for (int r = 0; r < BT_R; ++r) {
            const int dj = jj - r;
            if (dj < 0 || dj >= WIN) continue;
            // row partial sums keep the FP32 error small (two interleaved chains)
            float2 rn = make_float2(0.f, 0.f), rd = make_float2(0.f, 0.f);
#pragma unroll
            for (int q = 0; q < 5; ++q) {
                const float2 dr = __fadd2_rn(vp[q], nva[r]);
                float2 w;
                if ((TB >> q) & 1) {
                    const float2 t = __ffma2_rn(dr, kscale, mg);
                    w = __fmul2_rn(p.sp[dj][q],
                                   make_float2(*reinterpret_cast<const float*>(Rb + __float_as_int(t.x)),
                                               *reinterpret_cast<const float*>(Rb + __float_as_int(t.y))));
                } else {
                    const float2 x = __ffma2_rn(c2, __fmul2_rn(dr, dr), p.cp[dj][q]);
                    w = make_float2(ex2_approx(x.x), ex2_approx(x.y));
                }
                rn = __ffma2_rn(w, vp[q], rn);
                rd = __fadd2_rn(w, rd);
            }
            const float dr = vl - va[r];
            const float w = ex2_approx(fmaf(p.c2, dr * dr, p.c[dj * WIN + 10]));
            num[r] += fmaf(w, vl, rn.x + rn.y);
            den[r] += (rd.x + rd.y) + w;
        }
    }
    const int u = u0 + tx;
#pragma unroll
    for (int r = 0; r < BT_R; ++r) {
        const int v = v0 + r0 + r;
        if (u < d.W && v < d.H)
            d.smoothed_f[(size_t)f * d.px + (size_t)v * d.W + u] = __fdiv_rn(num[r], den[r]);
    }
}

// Exact bilateral at in-image pixel (u, v) from the staged mirrored grey tile
// (origin gx0, gy0): the arithmetic of k_bilateral_tile / preprocess.hpp:38-56,
// same j-major / i-minor accumulation. The weight-table gathers of row j+1
// are issued before row j is accumulated (two-row software pipeline), so the
// L1/L2 latency overlaps the dependent add chain; k/255 comes from smem.
template <int RHO>
__device__ __forceinline__ double exact_bilateral(const Dev& d, const WsParam& ws,
                                                  const uint8_t* s_g, const double* s_val,
                                                  int gw, int gx0, int gy0, int u, int v) {
    constexpr int WIN = 2 * RHO + 1;
    const uint8_t* c = s_g + (v - gy0) * gw + (u - gx0);
    const double* wrow = d.wr + (int)c[0] * 256;
    double num = 0.0, den = 0.0;
    double wr_cur[WIN];
    {
        const uint8_t* row = c - RHO * gw - RHO;
#pragma unroll
        for (int i = 0; i < WIN; ++i) wr_cur[i] = __ldg(wrow + row[i]);
    }
#pragma unroll 1
    for (int j = 0; j < WIN; ++j) {
        double wr_nxt[WIN];
        if (j + 1 < WIN) {
            const uint8_t* row = c + (j + 1 - RHO) * gw - RHO;
#pragma unroll
            for (int i = 0; i < WIN; ++i) wr_nxt[i] = __ldg(wrow + row[i]);
        }
        const uint8_t* row = c + (j - RHO) * gw - RHO;
#pragma unroll
        for (int i = 0; i < WIN; ++i) {
            const double w = ws.w[j * WIN + i] * wr_cur[i];
            num += w * s_val[row[i]];
            den += w;
        }
#pragma unroll
        for (int i = 0; i < WIN; ++i) wr_cur[i] = wr_nxt[i];
    }
    return num / den;
}

// ---- 2. Sobel on s~ with the propagated bound, exact refinement, edge bits
//
// Tile SB_TW x SB_TH, 256 threads; thread t owns pixels (row (t>>7) + 2k,
// col t & 127), k < 4, so each warp covers 32 consecutive pixels of a row
// and its ballot is a candidate / edge word directly.
//
// Candidate screening runs in FP32 on s~ (values in [0, 1]). Its rounding
// error is folded into the certified bound: each FP32 Sobel component is
// within 11 * 2^-24 < 1e-6 of the exact-arithmetic Sobel of s~, which is
// within 8 * kEpsSmooth of the Sobel of the exact smoothed image; the
// reference's FP64 evaluation of that Sobel adds < 1e-15. With D = 8 eps +
// 1e-6, |s - s_f| <= D(2|gx_f| + D) + D(2|gy_f| + D) + 3 * 2^-24 * s_f, where
// s_f = fl32(gx_f^2 + gy_f^2). ds below over-covers this (x1.001, +4e-7 s_f,
// +1e-9) and the test uses s*_lo = the largest float <= s*, so every pixel
// with s >= s* is a candidate.
template <int RHO>
__global__ void __launch_bounds__(256, 3) k_sobel_refine(Dev d, WsParam ws) {
    constexpr int FW = SB_TW + 2, FH = SB_TH + 2;               // tile + 1-px ring
    constexpr int GW = SB_TW + 2 + 2 * RHO, GH = SB_TH + 2 + 2 * RHO;  // grey for the ring
    constexpr int NWORD = (FW + 31) / 32;                       // ring row bitmap words
    constexpr int TWORD = SB_TW / 32;                           // tile row bitmap words
    constexpr int NF = (FH * FW + 255) / 256, NG = (GH * GW + 255) / 256;
    static_assert(SB_TW == 128 && SB_TH == 8, "pixel ownership assumes a 128 x 8 tile");
    __shared__ float s_f[FH * FW];
    __shared__ uint8_t s_g[GH * GW];
    __shared__ double s_ex[FH * FW];
    __shared__ double s_val[256];
    __shared__ short s_need[FH * FW];
    __shared__ unsigned s_cw[SB_TH][TWORD];
    __shared__ int s_nneed, s_seg[SB_TH], s_tot[2];
    const int f = blockIdx.z;
    if (frame_failed(d, f)) return;
    if (d.W < 3 || d.H < 3) {  // preprocess.hpp:68-69
        if (blockIdx.x == 0 && blockIdx.y == 0 && threadIdx.x == 0)
            fail_frame(d, f, 10, LK_MSG_SOBEL_TOO_SMALL);
        return;
    }
    const int W = d.W, H = d.H, tid = threadIdx.x, lane = tid & 31;
    const int u0 = blockIdx.x * SB_TW, v0 = blockIdx.y * SB_TH;
    const int horizon = (int)d.rep[f].horizon;
    if (v0 + SB_TH <= horizon) {  // the mask is empty above the horizon
        if (tid < SB_TH && v0 + tid < H)
            d.seg_cnt[((size_t)f * H + v0 + tid) * d.n_seg + blockIdx.x] = 0;
        return;
    }
    const float* sf = d.smoothed_f + (size_t)f * d.px;
    const uint8_t* grey = d.grey + (size_t)f * d.px;
    const int pc = tid & (SB_TW - 1), pr0 = tid >> 7;  // owned pixels: (pr0 + 2k, pc)
    // independent loads first: disparity and profile of the owned pixels, s~ tile
    int dv[4];
    double fvv[4];
#pragma unroll
    for (int k = 0; k < 4; ++k) {
        const int v = v0 + pr0 + 2 * k, u = u0 + pc;
        const bool in = v < H && u < W;
        dv[k] = in ? d.disp[(size_t)f * d.px + (size_t)v * W + u] : 0;
        fvv[k] = in ? d.fv[(size_t)f * H + v] : 0.0;
    }
    {
        float t[NF];
#pragma unroll
        for (int q = 0; q < NF; ++q) {
            const int i = tid + q * 256;
            t[q] = 0.f;
            if (i < FH * FW) {
                const int r = i / FW, c = i - r * FW;
                t[q] = sf[(size_t)mirror(v0 - 1 + r, H) * W + mirror(u0 - 1 + c, W)];
            }
        }
#pragma unroll
        for (int q = 0; q < NF; ++q)
            if (tid + q * 256 < FH * FW) s_f[tid + q * 256] = t[q];
    }
    if (tid < SB_TH) s_seg[tid] = 0;
    if (tid < 2) s_tot[tid] = 0;
    if (tid == 0) s_nneed = 0;
    __syncthreads();
    const float D = (float)(8.0 * kEpsSmooth + 1e-6);
    int n_mask = 0, any_cand = 0;
    unsigned cand_bits = 0;  // bit k: owned pixel k is a candidate
#pragma unroll
    for (int k = 0; k < 4; ++k) {
        const int r = pr0 + 2 * k, v = v0 + r, u = u0 + pc;
        const bool m = v < H && u < W && v >= horizon && dv[k] != 0 &&
                       fabs((double)dv[k] - fvv[k]) <= d.varpi;  // road_mask, preprocess.hpp:14-25
        n_mask += m;
        bool cand = false;
        if (m) {
            const float* a = s_f + r * FW + pc;  // row v-1, col u-1
            const float* b = a + FW;
            const float* cc = b + FW;
            const float gx = ((a[2] - a[0]) + 2.f * (b[2] - b[0])) + (cc[2] - cc[0]);
            const float gy = ((cc[0] - a[0]) + 2.f * (cc[1] - a[1])) + (cc[2] - a[2]);
            const float s = gx * gx + gy * gy;
            const float ds = 1.001f * (D * (2.f * fabsf(gx) + D) + D * (2.f * fabsf(gy) + D)) +
                             4e-7f * s + 1e-9f;
            cand = s + ds >= d.sobel_s_star_lo;
        }
        cand_bits |= (unsigned)cand << k;
        const unsigned bal = __ballot_sync(0xffffffffu, cand);
        if (lane == 0) s_cw[r][pc >> 5] = bal;
        any_cand |= cand;
    }
    if (!__syncthreads_or(any_cand)) {  // no edge can exist in this tile (most tiles)
        for (int o = 16; o; o >>= 1) n_mask += __shfl_xor_sync(0xffffffffu, n_mask, o);
        if (lane == 0 && n_mask) atomicAdd(&d.aux[f].mask_px, (unsigned long long)n_mask);
        if (tid < SB_TH && v0 + tid < H)
            d.seg_cnt[((size_t)f * H + v0 + tid) * d.n_seg + blockIdx.x] = 0;
        return;
    }
    {  // grey for the exact bilateral of the ring (loads first), k/255 table
        uint8_t t[NG];
#pragma unroll
        for (int q = 0; q < NG; ++q) {
            const int i = tid + q * 256;
            t[q] = 0;
            if (i < GH * GW) {
                const int r = i / GW, c = i - r * GW;
                t[q] = grey[(size_t)mirror(v0 - 1 - RHO + r, H) * W + mirror(u0 - 1 - RHO + c, W)];
            }
        }
        s_val[tid] = __ldg(d.val + tid);
#pragma unroll
        for (int q = 0; q < NG; ++q)
            if (tid + q * 256 < GH * GW) s_g[tid + q * 256] = t[q];
    }
    // pixels of tile + ring inside a candidate's 3x3 need the exact value:
    // ring bit C of ring row R <-> tile (R - 1, C - 1); need = 3x3 dilation
    if (tid < FH * NWORD) {
        const int R = tid / NWORD, w = tid - R * NWORD;
        auto tw = [&](int k) -> unsigned {  // OR of tile rows R-2..R, word k
            unsigned x = 0;
            if (k >= 0 && k < TWORD)
#pragma unroll
                for (int y = R - 2; y <= R; ++y)
                    if (y >= 0 && y < SB_TH) x |= s_cw[y][k];
            return x;
        };
        const unsigned t0 = tw(w), t1 = tw(w - 1);
        // (T | T << 1 | T << 2) restricted to ring bits 32w .. 32w + 31
        unsigned need = t0 | __funnelshift_l(t1, t0, 1) | __funnelshift_l(t1, t0, 2);
        if (w == NWORD - 1) need &= (FW % 32) ? (1u << (FW % 32)) - 1u : 0xffffffffu;
        if (need) {
            int o = atomicAdd(&s_nneed, __popc(need));
            while (need) {
                const int bit = __ffs(need) - 1;
                need &= need - 1;
                s_need[o++] = (short)(R * FW + 32 * w + bit);
            }
        }
    }
    __syncthreads();
    const int gx0 = u0 - 1 - RHO, gy0 = v0 - 1 - RHO;
    for (int k = tid; k < s_nneed; k += blockDim.x) {
        const int i = s_need[k];
        const int r = i / FW, c = i - r * FW;
        // ring positions outside the image hold their mirror pixel (preprocess.hpp:71-72)
        const int v = mirror(v0 - 1 + r, H), u = mirror(u0 - 1 + c, W);
        const double e = exact_bilateral<RHO>(d, ws, s_g, s_val, GW, gx0, gy0, u, v);
        s_ex[i] = e;
        d.smoothed[(size_t)f * d.px + (size_t)v * W + u] = e;  // read back by k_edge_emit
    }
    __syncthreads();
    int n_edge = 0;
#pragma unroll
    for (int k = 0; k < 4; ++k) {
        const int r = pr0 + 2 * k, v = v0 + r;
        bool edge = false;
        if ((cand_bits >> k) & 1) {  // candidate => masked and in the image
            const double* a = s_ex + r * FW + pc;  // row v-1, col u-1
            const double* b = a + FW;
            const double* cc = b + FW;
            const double gx = (a[2] - a[0]) + 2 * (b[2] - b[0]) + (cc[2] - cc[0]);
            const double gy = (cc[0] - a[0]) + 2 * (cc[1] - a[1]) + (cc[2] - a[2]);
            edge = gx * gx + gy * gy >= d.sobel_s_star;
            n_edge += edge;
        }
        const unsigned bal = __ballot_sync(0xffffffffu, edge);
        if (lane == 0 && v < H) {
            const int word = (u0 + pc) >> 5;
            if (word < d.words_per_row) d.ebits[((size_t)f * H + v) * d.words_per_row + word] = bal;
            if (bal) atomicAdd(&s_seg[r], __popc(bal));
        }
    }
    for (int o = 16; o; o >>= 1) {
        n_edge += __shfl_xor_sync(0xffffffffu, n_edge, o);
        n_mask += __shfl_xor_sync(0xffffffffu, n_mask, o);
    }
    if (lane == 0) {
        if (n_edge) atomicAdd(&s_tot[0], n_edge);
        if (n_mask) atomicAdd(&s_tot[1], n_mask);
    }
    __syncthreads();
    if (threadIdx.x < SB_TH && v0 + threadIdx.x < H)
        d.seg_cnt[((size_t)f * H + v0 + threadIdx.x) * d.n_seg + blockIdx.x] = s_seg[threadIdx.x];
    if (threadIdx.x == 0) {
        if (s_tot[0]) atomicAdd(&d.aux[f].edge_px, (unsigned long long)s_tot[0]);
        if (s_tot[1]) atomicAdd(&d.aux[f].mask_px, (unsigned long long)s_tot[1]);
    }
}

void launch_fast_bilateral(const Dev& d, const LaunchPlan& lp, int n, cudaStream_t s, int all) {
    const dim3 g((d.W + BT_W - 1) / BT_W, (d.H + BT_H - 1) / BT_H, n);
    switch (lp.fast_table) {
#define LK_BF(M) \
    case M: k_bilateral_fast<5, M><<<g, 256, 0, s>>>(d, lp.fbf, all); break;
        LK_BF(0) LK_BF(2) LK_BF(10) LK_BF(14) LK_BF(21) LK_BF(27) LK_BF(31)
#undef LK_BF
        default: k_bilateral_fast<5, 10><<<g, 256, 0, s>>>(d, lp.fbf, all); break;
    }
}

void launch_sobel_refine(const Dev& d, const LaunchPlan& lp, int n, cudaStream_t s) {
    const dim3 g((d.W + SB_TW - 1) / SB_TW, (d.H + SB_TH - 1) / SB_TH, n);
    k_sobel_refine<5><<<g, 256, 0, s>>>(d, lp.ws);
}

// Largest |s~ - s| of a batch (verification of kEpsSmooth): both maps full.
__global__ void k_fast_error(const float* a, const double* b, size_t n, double* out) {
    double m = 0;
    for (size_t i = (size_t)blockIdx.x * blockDim.x + threadIdx.x; i < n;
         i += (size_t)gridDim.x * blockDim.x)
        m = fmax(m, fabs((double)a[i] - b[i]));
    for (int o = 16; o; o >>= 1) m = fmax(m, __shfl_xor_sync(0xffffffffu, m, o));
    if ((threadIdx.x & 31) == 0)
        atomicMax((unsigned long long*)out, (unsigned long long)__double_as_longlong(m));
}

cudaError_t fast_error(const Dev& d, int n, cudaStream_t s, double* out_dev) {
    k_fast_error<<<296, 256, 0, s>>>(d.smoothed_f, d.smoothed, (size_t)n * d.px, out_dev);
    return cudaGetLastError();
}

}  // namespace lkg
