// lk_fastpath.cu — certified fast front end (stages 9-10) for throughput runs.
//
// The exact bilateral (k_bilateral_tile) is bound by random 8-byte gathers
// into the exact weight table. But the only consumers of the smoothed image
// downstream of stage 10 are the EDGE pixels (gx, gy, theta, votes, w_g all
// come from the edge list, preprocess.hpp:103-113), and the only integer
// decision taken on non-edge pixels is "not an edge". So:
//
//  0. k_prescreen certifies, from integer box sums of the raw grey bytes,
//     which road-mask pixels cannot be edges (most of them): only the
//     survivors and their 3x3 neighbourhoods go on.
//  1. k_bilateral_need computes the neighbourhood ("need") pixels
//     approximately in FP32 from an exact-index shared range table. A
//     rigorous bound |s~ - s| <= kEpsSmooth holds against the exact double
//     result (derivation in DESIGN.md §3; the worst error measured is checked
//     by tests/test_gpu_fastpath.py).
//  2. k_sobel_screen evaluates Sobel on s~ at the survivors and propagates the
//     bound to s = gx^2 + gy^2. A survivor whose s can still reach the
//     threshold is a candidate; its 3x3 neighbourhood goes to the frame's
//     exact need list.
//  3. k_refine_exact gives every exact need pixel its EXACT bilateral (the LUT
//     arithmetic of k_bilateral_tile), and k_sobel_decide takes each
//     candidate's edge decision from those exact values.
//
// The edge set, every edge's gx/gy, and everything downstream are therefore
// bit-identical to the exact path; only the (unexported) smoothed values of
// pixels far from any edge are approximate. Hooks mode always runs the exact
// path, so the SMOOTHED/GX/GY/MAG/THETA maps it exports are exact.
#include <cuda_runtime.h>

#include <algorithm>
#include <climits>

#include "lk_kernels.h"

namespace lkg {

constexpr double kEpsSmooth = 2.5e-5;  // bound on |s~ - s| (absolute, values in [0, 1])


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
// Three kernels, so that the exact FP64 refinement (a 121-tap dependent
// chain per pixel, ~1.6 % of the pixels) runs at full occupancy instead of
// leaving most of a tile's threads waiting at a barrier:
//   k_sobel_screen  (tile 128 x SB_TH): FP32 Sobel of s~ with the certified bound
//                   below; candidate bits -> ebits, need pixels (the 3x3
//                   neighbourhoods of candidates) -> the frame's need list,
//                   candidate tiles -> the frame's tile list;
//   k_refine_exact  one thread per need pixel: the exact LUT bilateral
//                   (preprocess.hpp:38-56) -> smoothed;
//   k_sobel_decide  per candidate tile: the exact Sobel of the candidates ->
//                   edge bits, segment counts, edge count.
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
//
// Thread t of a tile owns pixels (row (t>>7) * SB_TH / 2 + k, col t & 127), k < SB_TH / 2, so
// each warp covers 32 consecutive pixels of a row and its ballot is a
// candidate / edge word directly.
__global__ void __launch_bounds__(128) k_sobel_screen(Dev d) {
    constexpr int FW = SB_TW + 2, FH = SB_TH + 2;  // tile + 1-px ring
    constexpr int NWORD = (FW + 31) / 32;          // ring row bitmap words
    constexpr int TWORD = SB_TW / 32;              // tile row bitmap words
    static_assert(SB_TW == 128 && SB_TH * TWORD <= 128, "one thread per survivor word");
    __shared__ unsigned s_cw[SB_TH][TWORD];
    __shared__ unsigned s_need[FH][NWORD];
    __shared__ int s_nneed, s_base;
    const int f = blockIdx.z;
    if (frame_failed(d, f)) return;
    if (d.W < 3 || d.H < 3) {  // preprocess.hpp:68-69
        if (blockIdx.x == 0 && blockIdx.y == 0 && threadIdx.x == 0)
            fail_frame(d, f, 10, LK_MSG_SOBEL_TOO_SMALL);
        return;
    }
    const int W = d.W, H = d.H, tid = threadIdx.x;
    const int u0 = blockIdx.x * SB_TW, v0 = blockIdx.y * SB_TH;
    const int horizon = (int)d.rep[f].horizon;
    if (v0 + SB_TH <= horizon) {  // the mask is empty above the horizon
        if (tid < SB_TH && v0 + tid < H)
            d.seg_cnt[((size_t)f * H + v0 + tid) * d.n_seg + blockIdx.x] = 0;
        return;
    }
    const float* sf = d.smoothed_f + (size_t)f * d.px;
    // only pre-screen survivors (masked pixels that can still be edges) are
    // screened, one thread per survivor: the tile's 64 survivor words are
    // prefix-summed, and survivor i (in row-major order) is the n-th set bit
    // of its word (__fns). Each reads the s~ of its 3x3 neighbourhood (need
    // pixels of k_bilateral_need, mirrored at the border, preprocess.hpp:71-72).
    __shared__ unsigned s_pw[SB_TH * TWORD], s_pre[SB_TH * TWORD + 1];
    static_assert(SB_TH * TWORD == 64, "two warps scan the survivor words");
    const float D = (float)(8.0 * kEpsSmooth + 1e-6);
    if (tid < SB_TH * TWORD) {
        const int r = tid / TWORD, w = (u0 >> 5) + tid % TWORD;
        const unsigned x = v0 + r < H && w < d.words_per_row
                               ? d.pbits[((size_t)f * H + v0 + r) * d.words_per_row + w] : 0u;
        s_pw[tid] = x;
        s_cw[r][tid % TWORD] = 0;
        // inclusive prefix of the popcounts over the 64 words (two warps)
        unsigned c = __popc(x);
        for (int o = 1; o < 32; o <<= 1) {
            const unsigned y = __shfl_up_sync(0xffffffffu, c, o);
            if ((tid & 31) >= o) c += y;
        }
        s_pre[tid + 1] = c;  // warp-local for now
    }
    if (tid == 0) s_pre[0] = 0;
    __syncthreads();
    if (tid >= 32 && tid < 64) s_pre[tid + 1] += s_pre[32];  // second warp's offset
    __syncthreads();
    const unsigned total = s_pre[SB_TH * TWORD];
    if (total == 0) {  // no survivor: no edge in this tile
        if (tid < SB_TH && v0 + tid < H)
            d.seg_cnt[((size_t)f * H + v0 + tid) * d.n_seg + blockIdx.x] = 0;
        return;
    }
    bool anyc = false;
    for (unsigned i = tid; i < total; i += blockDim.x) {
        int lo = 0, hi = SB_TH * TWORD;  // word: s_pre[lo] <= i < s_pre[lo + 1]
        while (hi - lo > 1) {
            const int mid = (lo + hi) >> 1;
            if (s_pre[mid] <= i) lo = mid; else hi = mid;
        }
        const int bit = (int)__fns(s_pw[lo], 0, (int)(i - s_pre[lo]) + 1);
        const int r = lo / TWORD, v = v0 + r, u = u0 + 32 * (lo % TWORD) + bit;
        const float* ra = sf + (size_t)mirror(v - 1, H) * W;
        const float* rb = sf + (size_t)v * W;
        const float* rc = sf + (size_t)mirror(v + 1, H) * W;
        const int ul = mirror(u - 1, W), ur = mirror(u + 1, W);
        const float a0 = ra[ul], a1 = ra[u], a2 = ra[ur];
        const float b0 = rb[ul], b2 = rb[ur];
        const float c0 = rc[ul], c1 = rc[u], c2 = rc[ur];
        const float gx = ((a2 - a0) + 2.f * (b2 - b0)) + (c2 - c0);
        const float gy = ((c0 - a0) + 2.f * (c1 - a1)) + (c2 - a2);
        const float sg = gx * gx + gy * gy;
        const float ds = 1.001f * (D * (2.f * fabsf(gx) + D) + D * (2.f * fabsf(gy) + D)) +
                         4e-7f * sg + 1e-9f;
        if (sg + ds >= d.sobel_s_star_lo) {
            atomicOr(&s_cw[r][lo % TWORD], 1u << bit);
            anyc = true;
        }
    }
    const unsigned cw = anyc ? 1u : 0u;
    if (tid == 0) s_nneed = 0;
    if (!__syncthreads_or(cw != 0)) {  // no edge can exist in this tile (most tiles)
        if (tid < SB_TH && v0 + tid < H)
            d.seg_cnt[((size_t)f * H + v0 + tid) * d.n_seg + blockIdx.x] = 0;
        return;
    }
    // candidate words -> ebits (k_sobel_decide keeps the edges among them)
    if (tid < SB_TH * TWORD) {
        const int r = tid / TWORD, w = tid - r * TWORD, word = (u0 >> 5) + w;
        if (v0 + r < H && word < d.words_per_row)
            d.ebits[((size_t)f * H + v0 + r) * d.words_per_row + word] = s_cw[r][w];
    }
    // pixels of tile + ring inside a candidate's 3x3 need the exact value:
    // ring bit C of ring row R <-> tile (R - 1, C - 1); need = 3x3 dilation
    unsigned need = 0;
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
        need = t0 | __funnelshift_l(t1, t0, 1) | __funnelshift_l(t1, t0, 2);
        if (w == NWORD - 1) need &= (FW % 32) ? (1u << (FW % 32)) - 1u : 0xffffffffu;
        s_need[R][w] = need;
        if (need) atomicAdd(&s_nneed, __popc(need));
    }
    __syncthreads();
    if (tid == 0) {
        s_base = (int)atomicAdd(&d.need_cnt[f], (unsigned)s_nneed);
        const unsigned ct = atomicAdd(&d.ctile_cnt[f], 1u);
        d.ctile[(size_t)f * d.n_stile + ct] = blockIdx.y * gridDim.x + blockIdx.x;
    }
    __syncthreads();
    if (tid < FH * NWORD && need) {
        const int R = tid / NWORD, w = tid - R * NWORD;
        int o = s_base;  // this word's slot: the need bits of the words before it
        for (int j = 0; j < R * NWORD + w; ++j) o += __popc(s_need[j / NWORD][j % NWORD]);
        uint32_t* out = d.need + (size_t)f * d.need_cap;
        // ring positions outside the image hold their mirror pixel (preprocess.hpp:71-72)
        const int v = mirror(v0 - 1 + R, H);
        while (need) {
            const int bit = __ffs(need) - 1;
            need &= need - 1;
            const int u = mirror(u0 - 1 + 32 * w + bit, W);
            out[o++] = ((uint32_t)v << 16) | (uint32_t)u;
        }
    }
}

// Exact bilateral of one need pixel (u, v) straight from global memory: the
// arithmetic of k_bilateral_tile / preprocess.hpp:38-56, j-major / i-minor,
// the grey bytes and weight-table gathers of row j+1 issued before row j's
// dependent add chain. One thread per pixel keeps every SM full of chains.
// k/255.0 is computed exactly (grey_value); an interior window row is read as four
// 32-bit words (the input buffers carry 16 bytes of padding).
template <int RHO>
__device__ __forceinline__ void refine_row(const uint8_t* g, size_t rowoff, const int (&col)[2 * RHO + 1],
                                           bool inner, int u, uint8_t (&k)[2 * RHO + 1]) {
    constexpr int WIN = 2 * RHO + 1;
    static_assert(WIN <= 13, "four words cover the row");
    if (inner) {
        const uintptr_t a = reinterpret_cast<uintptr_t>(g + rowoff + u - RHO);
        const uint32_t* w = reinterpret_cast<const uint32_t*>(a & ~(uintptr_t)3);
        const unsigned sh = 8u * (unsigned)(a & 3);
        uint32_t x[4];
#pragma unroll
        for (int i = 0; i < 4; ++i) x[i] = __ldg(w + i);
        uint32_t y[4];
#pragma unroll
        for (int i = 0; i < 3; ++i) y[i] = __funnelshift_r(x[i], x[i + 1], sh);
        y[3] = x[3] >> sh;
#pragma unroll
        for (int i = 0; i < WIN; ++i) k[i] = (uint8_t)(y[i >> 2] >> (8 * (i & 3)));
    } else {
#pragma unroll
        for (int i = 0; i < WIN; ++i) k[i] = __ldg(g + rowoff + col[i]);
    }
}

// k / 255.0 correctly rounded without a table: q0 = RN(k y), y = RN(1/255),
// then one Markstein step q = RN(q0 + RN(k - q0 255) y) (both FMAs). Exact for
// all 256 k (checked exhaustively; 24 of the plain products q0 are off by one
// ulp). The FP64 pipe is ~14 % busy in this kernel while a shared-memory table
// of doubles cost ~1.5 bank-conflict wavefronts per lookup on the LSU pipe,
// which the weight-table gathers already keep ~77 % busy.
__device__ __forceinline__ double grey_value(uint8_t k) {
    constexpr double y = 1.0 / 255.0;
    const double x = (double)k;
    const double q0 = __dmul_rn(x, y);
    return __fma_rn(__fma_rn(-q0, 255.0, x), y, q0);
}

template <int RHO>
__global__ void __launch_bounds__(256) k_refine_exact(Dev d, WsParam ws) {
    constexpr int WIN = 2 * RHO + 1;
    const int f = blockIdx.y;
    if (frame_failed(d, f)) return;
    const unsigned cnt = d.need_cnt[f];
    if (blockIdx.x * blockDim.x >= cnt) return;
    const uint32_t* list = d.need + (size_t)f * d.need_cap;
    const uint8_t* g = d.grey + (size_t)f * d.px;
    const int W = d.W, H = d.H;
    for (unsigned i = blockIdx.x * blockDim.x + threadIdx.x; i < cnt; i += gridDim.x * blockDim.x) {
        const uint32_t e = list[i];
        const int v = (int)(e >> 16), u = (int)(e & 0xffffu);
        const bool inner = u >= RHO && v >= RHO && u + RHO < W && v + RHO < H;
        int col[WIN];
#pragma unroll
        for (int k = 0; k < WIN; ++k) col[k] = inner ? u - RHO + k : mirror(u - RHO + k, W);
        auto rowoff = [&](int j) {
            return (size_t)(inner ? v - RHO + j : mirror(v - RHO + j, H)) * W;
        };
        const double* wrow = d.wr + (int)g[(size_t)v * W + u] * 256;
        double num = 0.0, den = 0.0;
        uint8_t k_cur[WIN];
        double wr_cur[WIN];
        refine_row<RHO>(g, rowoff(0), col, inner, u, k_cur);
#pragma unroll
        for (int k = 0; k < WIN; ++k) wr_cur[k] = __ldg(wrow + k_cur[k]);
#pragma unroll 1
        for (int j = 0; j < WIN; ++j) {
            uint8_t k_nxt[WIN];
            double wr_nxt[WIN];
            if (j + 1 < WIN) {
                refine_row<RHO>(g, rowoff(j + 1), col, inner, u, k_nxt);
#pragma unroll
                for (int k = 0; k < WIN; ++k) wr_nxt[k] = __ldg(wrow + k_nxt[k]);
            }
#pragma unroll
            for (int k = 0; k < WIN; ++k) {
                const double w = ws.w[j * WIN + k] * wr_cur[k];
                num += w * grey_value(k_cur[k]);
                den += w;
            }
#pragma unroll
            for (int k = 0; k < WIN; ++k) {
                k_cur[k] = k_nxt[k];
                wr_cur[k] = wr_nxt[k];
            }
        }
        d.smoothed[(size_t)f * d.px + (size_t)v * W + u] = num / den;
    }
}

// ---- 0. certified pre-screen (k_prescreen) and the need-list bilateral
//
// Which masked pixels can possibly be edges, decided from integer box sums
// of the raw grey bytes, before any bilateral arithmetic. With
// delta_q = v_q - v_p, beta the normalised spatial weights of p's window,
// r_q = exp(-kappa delta_q^2) the range factors (kappa = 1/sigma_r^2) and
// e_q = 1 - r_q in [0, min(1, kappa delta_q^2)]:
//   s(p) - g(p) = (ebar * m1 - sum beta e delta) / (1 - ebar),
// g the beta-weighted mean, m1 = g - v_p, ebar = sum beta e <= kappa m2,
// m2 = sum beta delta^2, |e delta| <= fmax delta^2 (fmax = sup (1 - exp(-kappa
// x^2)) / x). The spatial weights lie in [w_min, 1] (w_min = 0.99944 at the
// default sigma_s = 300), so beta-moments are bounded by box moments: m2 <=
// m2b / w_min, |m1| <= |m1b| + ew sqrt(m2b), |g - b| <= ew sqrt(m2b), ew =
// 1/w_min - 1, with b the 11x11 box mean (mirrored window) and m1b, m2b the
// box moments of delta. Hence |s - b| <= E with
//   E = (kappa A2 A1 + fmax A2) / (1 - kappa A2) + ew sqrt(m2b),
//   A2 = m2b / w_min, A1 = |m1b| + ew sqrt(m2b)      (E = inf if kappa A2 >= 0.95).
// The box sums S1 = sum k, S2 = sum k^2 (k the u8 grey) are integers below
// 2^24, exact in FP32, and so are M1 = S1 - 121 k_p and M2 = S2 - 2 k_p S1 +
// 121 k_p^2 (m1b = M1 / (121*255), m2b = M2 / (121*255^2)). E is evaluated in
// FP32 (relative error < 1e-5 including the 1 - kappa A2 >= 0.05 division)
// and inflated by 1.0001, + 1e-9 for the reference's own double rounding.
// The exact Sobel of s then satisfies |gx - gx_b| <= Ex = sum |c_k| E(p + k)
// (gx_b = Sobel(S1) / (121*255), an exact integer Sobel), and a masked pixel
// is a *survivor* unless (|gx_b| + Ex)^2 + (|gy_b| + Ey)^2 (x 1.00001) < s*_lo:
// a non-survivor has s_g < s*, so it is provably not an edge. On the KITTI
// batch ~6 % of the masked pixels survive; only the 3x3 neighbourhoods of the
// survivors (~9 %) need s~ (the FP32 bilateral below), instead of every tile
// near the road.
//
// CTA = one frame, walking down its rows from the horizon. Lane l of warp w
// owns the quad q = 30 w - 1 + l (image columns 4q .. 4q + 3, evaluated at
// their mirror columns outside the image); lanes 1-30 are the warp's output
// quads, lanes 0 and 31 the neighbours its Sobels read, so warps never wait
// for each other inside a row. Per input row a lane loads the 14 window bytes
// of its quad as five words, forms H1 = sum k and H2 = sum k^2 of the first
// column's 11 bytes with dp4a and slides them across the quad; the vertical
// running sums S1, S2 (exact int) subtract the row that left the window (a
// shared ring of packed H1 | H2 << 12 of the last 16 input rows). E rows are
// kept in registers (rows r - 1, r, r + 1), the neighbour columns come by
// shuffle, and the Sobel test of P row r runs as soon as E row r + 1 exists.
// Survivor nibbles go to a shared row bitmap (one match/reduce OR per word
// group); every PQ_RB rows the need rows (3x3 dilation, one row behind) are
// appended to the frame's list and the survivor words written to pbits.
constexpr int PQ_RB = 16;  // rows per need block
constexpr int PQ_RING = 11;  // H ring: the 11 input rows of the current window
constexpr int PQ_SR = 20;  // survivor bitmap ring rows (>= PQ_RB + 3)
constexpr uint32_t kOnes = 0x01010101u;
#ifndef PQ_PFD_N
#define PQ_PFD_N 2
#endif
constexpr int PQ_PFD = PQ_PFD_N;  // rows staged ahead (cp.async): grey row e + 5 and disparity row e - 1
// bytes of one staged row: the 16-byte chunks covering W bytes at any alignment
__host__ __device__ __forceinline__ int pq_row_bytes(int W) { return ((W + 30) >> 4 << 4) + 16; }

__device__ __forceinline__ void pq_cp16(void* smem, const void* gmem) {
    asm volatile("cp.async.cg.shared.global [%0], [%1], 16;\n" ::"r"((uint32_t)__cvta_generic_to_shared(smem)),
                 "l"(gmem)
                 : "memory");
}
__device__ __forceinline__ void pq_cp8(void* smem, const void* gmem) {
    asm volatile("cp.async.ca.shared.global [%0], [%1], 8;\n" ::"r"((uint32_t)__cvta_generic_to_shared(smem)),
                 "l"(gmem)
                 : "memory");
}
__device__ __forceinline__ void pq_commit() { asm volatile("cp.async.commit_group;\n" ::: "memory"); }
template <int N>
__device__ __forceinline__ void pq_wait() { asm volatile("cp.async.wait_group %0;\n" ::"n"(N) : "memory"); }

__device__ __forceinline__ uint32_t pq_byte(uint32_t w, int i) { return (w >> (8 * i)) & 0xffu; }

// the 14 window bytes 4q - 5 .. 4q + 8 of a (mirrored) row as t0..t3 (bytes 0-13)
__device__ __forceinline__ void pq_bytes(const uint8_t* row, int q, int W, bool fast, uint32_t& t0,
                                         uint32_t& t1, uint32_t& t2, uint32_t& t3) {
    if (fast) {
        const uintptr_t a = reinterpret_cast<uintptr_t>(row + 4 * q - 5);
        const uint32_t* w = reinterpret_cast<const uint32_t*>(a & ~(uintptr_t)3);
        const unsigned sh = 8u * (unsigned)(a & 3);
        const uint32_t w0 = __ldg(w), w1 = __ldg(w + 1), w2 = __ldg(w + 2), w3 = __ldg(w + 3),
                       w4 = __ldg(w + 4);
        t0 = __funnelshift_r(w0, w1, sh);
        t1 = __funnelshift_r(w1, w2, sh);
        t2 = __funnelshift_r(w2, w3, sh);
        t3 = __funnelshift_r(w3, w4, sh);
    } else {
        uint32_t b[14];
#pragma unroll
        for (int i = 0; i < 14; ++i) {  // one reflection suffices: overhang < 160 <= W
            const int x = 4 * q - 5 + i;
            b[i] = __ldg(row + (W >= 160 ? (x < 0 ? -x - 1 : x >= W ? 2 * W - 1 - x : x) : mirror(x, W)));
        }
        t0 = b[0] | b[1] << 8 | b[2] << 16 | b[3] << 24;
        t1 = b[4] | b[5] << 8 | b[6] << 16 | b[7] << 24;
        t2 = b[8] | b[9] << 8 | b[10] << 16 | b[11] << 24;
        t3 = b[12] | b[13] << 8;
    }
}

__global__ void __launch_bounds__(768) k_prescreen(Dev d, PrescreenParam p) {
    extern __shared__ __align__(16) uint32_t pq_sm[];
    const int f = blockIdx.x, seg = blockIdx.y, nseg = gridDim.y;
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    const int nt = blockDim.x, W = d.W, H = d.H, wpr = d.words_per_row;
    uint4* ring = reinterpret_cast<uint4*>(pq_sm);                 // [PQ_RING][nt]
    uint32_t* sbits = pq_sm + PQ_RING * 4 * nt;                     // [PQ_SR][wpr + 1]
    const int sbw = wpr + 1;
    // staged rows (16-byte aligned): grey [PQ_PFD + 1][RB], disparity [PQ_PFD + 1][RB], mask intervals
    const int RB = pq_row_bytes(W);
    uint8_t* rowG = reinterpret_cast<uint8_t*>(sbits + ((PQ_SR * sbw + 3) & ~3));
    uint8_t* rowD = rowG + (PQ_PFD + 1) * RB;
    int2* rowM = reinterpret_cast<int2*>(rowD + (PQ_PFD + 1) * RB);
    if (tid == 0 && seg == 0) {  // the Sobel screen appends to these
        d.need_cnt[f] = 0;
        d.ctile_cnt[f] = 0;
    }
    if (frame_failed(d, f)) return;
    const int horizon = (int)d.rep[f].horizon;
    const int P0 = max(horizon, 0);
    // survivor words of the rows a Sobel tile reads but the walk does not reach
    if (seg == 0)
        for (int i = tid; i < wpr * (P0 - (P0 & ~(SB_TH - 1))); i += nt) {
            const int r = (P0 & ~(SB_TH - 1)) + i / wpr;
            if (r < H) d.pbits[((size_t)f * H + r) * wpr + i % wpr] = 0;
        }
    if (P0 >= H) return;
    // this segment's rows [pa, pb) of P0 .. H - 1: it emits their need rows
    // (segment 0 also row P0 - 1) and survivor words, and tests P rows
    // [t_lo, t_hi] (one more on each side for the dilation)
    const int L = (H - P0 + nseg - 1) / nseg;
    const int pa = P0 + seg * L, pb = min(pa + L, H);
    if (pa >= pb) return;
    const int t_lo = max(pa - 1, P0), t_hi = min(pb, H - 1);
    const int n_lo = seg == 0 ? max(P0 - 1, 0) : pa;
    for (int i = tid; i < PQ_SR * sbw; i += nt) sbits[i] = 0;
    const int q = 30 * warp - 1 + lane;
    const int qlast = (W - 1) >> 2;
    const bool outq = lane >= 1 && lane <= 30 && q <= qlast;  // an output quad
    const bool fast = 4 * q - 5 >= 0 && 4 * q + 11 < W;       // window words inside the row
    const bool bigH = H >= 16;
    const uint8_t* g = d.grey + (size_t)f * d.px;
    const uint8_t* dp = d.disp + (size_t)f * d.px;
    int S1[4] = {0, 0, 0, 0}, S2[4] = {0, 0, 0, 0};  // box sums of k, k^2 (exact) per column
    uint32_t cen[6] = {0, 0, 0, 0, 0, 0};  // centre bytes (columns 4q..4q+3) of input rows, newest first
    // H1, H2 of the quad's 4 columns for input row rin (mirrored), packed H1 | H2 << 12
    auto hsums = [&](uint32_t t0, uint32_t t1, uint32_t t2, uint32_t t3, uint4& hp) {
        const uint32_t t2m = t2 & 0x00ffffffu;
        int h1 = (int)__dp4a(t0, kOnes, __dp4a(t1, kOnes, __dp4a(t2m, kOnes, 0u)));
        int h2 = (int)__dp4a(t0, t0, __dp4a(t1, t1, __dp4a(t2m, t2m, 0u)));
        const int o0 = pq_byte(t0, 0), o1 = pq_byte(t0, 1), o2 = pq_byte(t0, 2);
        const int n0 = pq_byte(t2, 3), n1 = pq_byte(t3, 0), n2 = pq_byte(t3, 1);
        hp.x = (uint32_t)h1 | (uint32_t)h2 << 12;
        h1 += n0 - o0;
        h2 += n0 * n0 - o0 * o0;
        hp.y = (uint32_t)h1 | (uint32_t)h2 << 12;
        h1 += n1 - o1;
        h2 += n1 * n1 - o1 * o1;
        hp.z = (uint32_t)h1 | (uint32_t)h2 << 12;
        h1 += n2 - o2;
        h2 += n2 * n2 - o2 * o2;
        hp.w = (uint32_t)h1 | (uint32_t)h2 << 12;
#pragma unroll
        for (int i = 5; i > 0; --i) cen[i] = cen[i - 1];
        cen[0] = __funnelshift_r(t1, t2, 8);  // bytes 5 .. 8 = columns 4q .. 4q + 3
    };
    auto hrow = [&](int rin, uint4& hp) {
        const int rr = bigH ? (rin < 0 ? -rin - 1 : rin >= H ? 2 * H - 1 - rin : rin) : mirror(rin, H);
        uint32_t t0, t1, t2, t3;
        pq_bytes(g + (size_t)rr * W, q, W, fast, t0, t1, t2, t3);
        hsums(t0, t1, t2, t3, hp);
    };
    // the same from a staged grey row (bytes [0, W) of row rr at offset (src & 15))
    auto hrow_staged = [&](int rr, int slot, uint4& hp) {
        const uint8_t* sb = rowG + slot * RB + ((reinterpret_cast<uintptr_t>(g + (size_t)rr * W)) & 15);
        uint32_t t0, t1, t2, t3;
        if (fast) {
            const uintptr_t a = reinterpret_cast<uintptr_t>(sb + 4 * q - 5);
            const uint32_t* w = reinterpret_cast<const uint32_t*>(a & ~(uintptr_t)3);
            const unsigned sh = 8u * (unsigned)(a & 3);
            const uint32_t w0 = w[0], w1 = w[1], w2 = w[2], w3 = w[3], w4 = w[4];
            t0 = __funnelshift_r(w0, w1, sh);
            t1 = __funnelshift_r(w1, w2, sh);
            t2 = __funnelshift_r(w2, w3, sh);
            t3 = __funnelshift_r(w3, w4, sh);
        } else {
            uint32_t b[14];
#pragma unroll
            for (int i = 0; i < 14; ++i) {  // W >= 160 here: one reflection suffices
                const int x = 4 * q - 5 + i;
                b[i] = sb[x < 0 ? -x - 1 : x >= W ? 2 * W - 1 - x : x];
            }
            t0 = b[0] | b[1] << 8 | b[2] << 16 | b[3] << 24;
            t1 = b[4] | b[5] << 8 | b[6] << 16 | b[7] << 24;
            t2 = b[8] | b[9] << 8 | b[10] << 16 | b[11] << 24;
            t3 = b[12] | b[13] << 8;
        }
        hsums(t0, t1, t2, t3, hp);
    };
    auto addrow = [&](const uint4& hp, int sg) {
        const uint32_t h[4] = {hp.x, hp.y, hp.z, hp.w};
#pragma unroll
        for (int j = 0; j < 4; ++j) {
            S1[j] += sg * (int)(h[j] & 0xfffu);
            S2[j] += sg * (int)(h[j] >> 12);
        }
    };
    // E of column j (centre byte of 5 rows ago) is
    //   ((kappa A2 A1 + fmax A2)(1 + 2 kappa A2) + ew sq) * 1.0001 + 1e-9,
    //   A2 = m2 / w_min, A1 = m1 + ew sq, sq = 10 m2 + 0.025 >= sqrt(m2) (AM-GM at 0.05),
    // infinite when kappa A2 >= 1/2 (1 / (1 - km) <= 1 + 2 km needs km <= 1/2)
    const int e0 = max(t_lo - 1, 0);  // first E row
    const int e_last = t_hi + 1;      // == H: the last step mirrors E row H
    for (int i = -5; i <= 5; ++i) {
        uint4 hp;
        hrow(e0 + i, hp);
        addrow(hp, 1);
        ring[(i + 5) * nt + tid] = hp;  // slot k <-> input row e0 - 5 + k (mod PQ_RING)
    }
    // E rows of the quad, (S1, E) per column, plus the left neighbour's column 3
    // (l) and the right neighbour's column 0 (r); three rotate without copies
    struct RowE {
        float2 v[4], l, r;
    };
    // E of columns j0, j0 + 1 as one packed f32x2 evaluation (evalE's formula)
    auto evalE2 = [&](int j0) {
        const int k0 = (int)pq_byte(cen[5], j0), k1 = (int)pq_byte(cen[5], j0 + 1);
        const float2 m1 = __fmul2_rn(make_float2((float)abs(S1[j0] - 121 * k0), (float)abs(S1[j0 + 1] - 121 * k1)),
                                     make_float2(p.c1, p.c1));
        const float2 m2 = __fmul2_rn(make_float2((float)(S2[j0] - 2 * k0 * S1[j0] + 121 * k0 * k0),
                                                 (float)(S2[j0 + 1] - 2 * k1 * S1[j0 + 1] + 121 * k1 * k1)),
                                     make_float2(p.c2, p.c2));
        const float2 A2 = __fmul2_rn(m2, make_float2(p.inv_wmin, p.inv_wmin));
        const float2 km = __fmul2_rn(A2, make_float2(p.kappa, p.kappa));
        const float2 sq = __ffma2_rn(m2, make_float2(10.f, 10.f), make_float2(0.025f, 0.025f));
        const float2 ew = make_float2(p.ew, p.ew);
        const float2 A1 = __ffma2_rn(ew, sq, m1);
        const float2 e = __fmul2_rn(__ffma2_rn(km, A1, __fmul2_rn(make_float2(p.fmax, p.fmax), A2)),
                                    __ffma2_rn(make_float2(2.f, 2.f), km, make_float2(1.f, 1.f)));
        const float2 r = __ffma2_rn(__ffma2_rn(ew, sq, e), make_float2(1.0001f, 1.0001f),
                                    make_float2(1e-9f, 1e-9f));
        return make_float2(km.x >= 0.5f ? 1e30f : r.x, km.y >= 0.5f ? 1e30f : r.y);
    };
    auto make_row = [&](RowE& C) {
        const float2 e01 = evalE2(0), e23 = evalE2(2);
        C.v[0] = make_float2((float)S1[0], e01.x);
        C.v[1] = make_float2((float)S1[1], e01.y);
        C.v[2] = make_float2((float)S1[2], e23.x);
        C.v[3] = make_float2((float)S1[3], e23.y);
        C.l = make_float2(__shfl_up_sync(0xffffffffu, C.v[3].x, 1), __shfl_up_sync(0xffffffffu, C.v[3].y, 1));
        C.r = make_float2(__shfl_down_sync(0xffffffffu, C.v[0].x, 1), __shfl_down_sync(0xffffffffu, C.v[0].y, 1));
    };
    int nmask = 0;
    // P row r from E rows A = E(r - 1), B = E(r), C = E(r + 1): exact integer
    // Sobel of S1 and |c|-weighted Sobel of E as packed (S1, E) pairs
    const float2 np = make_float2(-1.f, 1.f), two = make_float2(2.f, 2.f);
    auto test_row = [&](int r, const RowE& A, const RowE& B, const RowE& C, int slot) {
        // mask inputs of the quad: disparity bytes 4q .. 4q + 3 and the row interval
        uint32_t dw = 0;
        int2 mr = make_int2(256, 0);
        if (outq) {
            const uint8_t* dr;
            if (slot >= 0) {  // staged
                mr = rowM[slot];
                dr = rowD + slot * RB + ((reinterpret_cast<uintptr_t>(dp + (size_t)r * W)) & 15) + 4 * q;
            } else {
                mr = d.mrange[(size_t)f * H + r];
                dr = dp + (size_t)r * W + 4 * q;
            }
            if (4 * q + 4 <= W) {
                const uintptr_t a = reinterpret_cast<uintptr_t>(dr);
                const uint32_t* wp = reinterpret_cast<const uint32_t*>(a & ~(uintptr_t)3);
                dw = __funnelshift_r(wp[0], wp[1], 8u * (unsigned)(a & 3));
            } else {
                for (int j = 0; j < 4 && 4 * q + j < W; ++j) dw |= (uint32_t)dr[j] << (8 * j);
            }
        }
        // every pixel of the quad is evaluated (no divergence); the road mask
        // and the image edge gate the survivor bits
        uint32_t nib = 0, mnib = 0;
#pragma unroll
        for (int j = 0; j < 4; ++j) {
            const int dv = (int)pq_byte(dw, j);
            const bool m = outq && 4 * q + j < W && dv >= mr.x && dv <= mr.y;
            const float2 a0 = j ? A.v[j - 1] : A.l, a1 = A.v[j], a2 = j < 3 ? A.v[j + 1] : A.r;
            const float2 b0 = j ? B.v[j - 1] : B.l, b2 = j < 3 ? B.v[j + 1] : B.r;
            const float2 c0 = j ? C.v[j - 1] : C.l, c1 = C.v[j], c2 = j < 3 ? C.v[j + 1] : C.r;
            // (gx, ex): x = right - left, y = right + left; rows weighted 1, 2, 1
            const float2 hx = __fadd2_rn(__ffma2_rn(__ffma2_rn(b0, np, b2), two, __ffma2_rn(a0, np, a2)),
                                         __ffma2_rn(c0, np, c2));
            // (gy, ey): x = bottom - top, y = bottom + top; columns weighted 1, 2, 1
            const float2 hy = __fadd2_rn(__ffma2_rn(__ffma2_rn(a1, np, c1), two, __ffma2_rn(a0, np, c0)),
                                         __ffma2_rn(a2, np, c2));
            const float tx = fmaf(fabsf(hx.x), p.c1, hx.y), ty = fmaf(fabsf(hy.x), p.c1, hy.y);
            mnib |= (uint32_t)m << j;
            nib |= (uint32_t)(m && fmaf(tx, tx, ty * ty) * 1.00001f >= p.s_star_lo) << j;
        }
        if (r >= pa && r < pb) nmask += __popc(mnib);
        // OR the nibbles of each 32-column word into the shared row bitmap
        const int wd = outq ? (4 * q) >> 5 : -1;
        const unsigned grp = __match_any_sync(0xffffffffu, wd);
        const uint32_t word = __reduce_or_sync(grp, nib << ((4 * q) & 31));
        if (wd >= 0 && lane == __ffs(grp) - 1 && word) atomicOr(&sbits[(r % PQ_SR) * sbw + wd], word);
    };
    // need rows rb .. re - 1 from the survivor rows around them (ring), then pbits
    auto need_rows = [&](int rb, int re) {
        __syncthreads();
        const int ntask = (re - rb) * wpr;
        for (int base0 = 0; base0 < ntask; base0 += nt) {
            const int ti = base0 + tid;
            uint32_t nw = 0;
            int r = 0, w = 0;
            if (ti < ntask) {
                r = rb + ti / wpr;
                w = ti % wpr;
                auto orw = [&](int ww) -> uint32_t {
                    if (ww < 0 || ww >= wpr) return 0u;
                    uint32_t x = r >= t_lo ? sbits[(r % PQ_SR) * sbw + ww] : 0u;
                    if (r - 1 >= t_lo) x |= sbits[((r - 1) % PQ_SR) * sbw + ww];
                    if (r + 1 <= t_hi) x |= sbits[((r + 1) % PQ_SR) * sbw + ww];
                    return x;
                };
                const uint32_t X = orw(w);
                nw = X | (X << 1 | orw(w - 1) >> 31) | (X >> 1 | orw(w + 1) << 31);
                const int ub = 32 * w;
                if (W - ub < 32) nw &= (1u << (W - ub)) - 1u;
                if (r >= pa) d.pbits[((size_t)f * H + r) * wpr + w] = sbits[(r % PQ_SR) * sbw + w];
            }
            const int cnt = __popc(nw);
            int pre = cnt;
            for (int o = 1; o < 32; o <<= 1) {
                const int x = __shfl_up_sync(0xffffffffu, pre, o);
                if (lane >= o) pre += x;
            }
            const int tot = __shfl_sync(0xffffffffu, pre, 31);
            unsigned bo = 0;
            if (lane == 0 && tot) bo = atomicAdd(&d.aux[f].fneed, (unsigned)tot);
            bo = __shfl_sync(0xffffffffu, bo, 0) + (unsigned)(pre - cnt);
            uint32_t* out = d.fneed + (size_t)f * d.px;
            while (nw) {
                const int bb = __ffs(nw) - 1;
                nw &= nw - 1;
                out[bo++] = ((uint32_t)r << 16) | (uint32_t)(32 * w + bb);
            }
        }
        __syncthreads();
        // survivor rows older than re - 2 are no longer read: clear them for reuse
        for (int i = tid; i < (re - rb) * sbw; i += nt) {
            const int r = rb - 1 + i / sbw;
            if (r >= t_lo && r < re - 1) sbits[(r % PQ_SR) * sbw + i % sbw] = 0;
        }
        __syncthreads();
    };
    int need_from = n_lo;  // next need row to emit
    int slot = 0;          // ring slot of input row e - 6 (e the next E row); e + 5 reuses it
    // one row step: E row e into N (its storage held E(e - 3)), then P row e - 1
    // with M = E(e - 2) (O = E(e - 1)); at e == H, N = E(H - 1) (the mirror of row H)
    // staging (bigH): group j = step e0 + 1 + j holds grey row e0 + 6 + j (mirrored), disparity
    // row e0 + j and its mask interval, in slot j % (PQ_PFD + 1); PQ_PFD groups in flight
    const bool staged = bigH && W >= 160;
    auto stage_rows = [&](int j) {
        const int slot = j % (PQ_PFD + 1);
        const int rin = e0 + 6 + j, rd = e0 + j;
        const int rr = rin < 0 ? -rin - 1 : rin >= H ? 2 * H - 1 - rin : rin;
        const uintptr_t ag = reinterpret_cast<uintptr_t>(g + (size_t)rr * W);
        const int ng = rin <= min(e_last, H - 1) + 5 ? (int)(((ag & 15) + W + 15) >> 4) : 0;  // consumed by steps e < H
        const bool dok = rd >= t_lo && rd <= t_hi;
        const uintptr_t ad = reinterpret_cast<uintptr_t>(dp + (size_t)(dok ? rd : 0) * W);
        const int nd = dok ? (int)(((ad & 15) + W + 15) >> 4) : 0;
        for (int i = tid; i < ng + nd; i += nt) {
            if (i < ng)
                pq_cp16(rowG + slot * RB + 16 * i, reinterpret_cast<const void*>((ag & ~(uintptr_t)15) + 16 * i));
            else
                pq_cp16(rowD + slot * RB + 16 * (i - ng),
                        reinterpret_cast<const void*>((ad & ~(uintptr_t)15) + 16 * (i - ng)));
        }
        if (dok && tid == nt - 1) pq_cp8(rowM + slot, d.mrange + (size_t)f * H + rd);
        pq_commit();
    };
    auto step = [&](int e, RowE& M, RowE& O, RowE& N) {
        const int j = e - e0 - 1, ss = j % (PQ_PFD + 1);  // staging slot of this step
        if (staged) {
            pq_wait<PQ_PFD - 1>();  // group j has landed
            __syncthreads();        // ... for every thread; slot of group j - 1 is free
            stage_rows(j + PQ_PFD);
        }
        if (e < H) {
            uint4 hp;
            if (staged) {
                const int rin = e + 5;
                hrow_staged(rin >= H ? 2 * H - 1 - rin : rin, ss, hp);
            } else {
                hrow(e + 5, hp);
            }
            addrow(ring[slot * nt + tid], -1);
            addrow(hp, 1);
            ring[slot * nt + tid] = hp;  // (PQ_RING = 11: row e + 5 takes row e - 6's slot)
            slot = slot + 1 == PQ_RING ? 0 : slot + 1;
            make_row(N);
        } else {
            N = O;
        }
        const int r = e - 1;
        if (r >= t_lo) test_row(r, r == 0 ? O : M, O, N, staged ? ss : -1);  // mirror(-1) = 0
        // rows up to r are tested: need rows up to r - 1 are final
        if ((r - need_from + 1 >= PQ_RB && r >= t_lo) || r == t_hi) {
            const int re = r == t_hi ? pb : r;
            if (re > need_from) need_rows(need_from, re);
            need_from = re;
        }
    };
    RowE X, Y, Z;
    make_row(Z);  // E row e0
    Y = Z;        // (rolls into the A slot of the first test, which only happens for r >= P0)
    __syncthreads();  // sbits cleared
    if (staged)
        for (int j = 0; j < PQ_PFD; ++j) stage_rows(j);
    for (int e = e0 + 1; e <= e_last; e += 3) {
        step(e, Y, Z, X);
        if (e + 1 <= e_last) step(e + 1, Z, X, Y);
        if (e + 2 <= e_last) step(e + 2, X, Y, Z);
    }
    for (int o = 16; o; o >>= 1) nmask += __shfl_xor_sync(0xffffffffu, nmask, o);
    if (lane == 0 && nmask) atomicAdd(&d.aux[f].mask_px, (unsigned long long)nmask);
}

size_t prescreen_smem(int W, int nt) {
    const size_t sb = ((size_t)PQ_SR * ((W + 31) / 32 + 1) + 3) & ~(size_t)3;
    return (size_t)PQ_RING * nt * 16 + sb * 4 + (size_t)2 * (PQ_PFD + 1) * pq_row_bytes(W) +
           (size_t)(PQ_PFD + 1) * 8;
}

// Row segments per frame: 2 for batches that fill the GPU; small batches
// (the drop-in's one frame at a time) split each frame's walk further, so the
// latency of a batch is a few short walks instead of one long one (each
// segment re-reads its 11-row window head, ~12 rows of extra work).
int prescreen_segments(int H, int n) {
    if (H < 128) return 1;
    if (n >= 16) return 2;
    const int s = 32 / (n < 1 ? 1 : n);
    const int cap = H / 24;  // segments of at least 24 rows
    return s < 2 ? 2 : s > cap ? (cap < 2 ? 2 : cap) : s;
}

int prescreen_threads(int W) {
    const int qlast = (W - 1) >> 2;
    return 32 * ((qlast + 1 + 29) / 30);
}

// FP32 bilateral of the need pixels (k_prescreen's list), one thread per
// pixel, the frames' lists flattened over a persistent grid. Each tap
// reads (R(delta), R(delta) * delta) from a shared table (delta = k_q - k_p,
// 16 lane copies entry-major: a half-warp's 8-byte loads hit 32 distinct
// banks) and adds S_t * R to den and S_t * R * delta to num (two FMAs, S_t
// an immediate constant-bank operand); s~ = (k_p + num / den) / 255. The sums
// of a pixel run in j-major / i-minor order. Error: the weights are exact to
// 3 ulp, each FMA chain of 121 terms adds <= 121 ulp of sum |S R delta| <=
// 255 den (num) or of den, so |num/den - q| <= ~246 * 255 * 2^-24 and
// |s~ - s| <= ~248 * 2^-24 < 1.5e-5 < kEpsSmooth.
// all = 1: every pixel of every frame (lk_fast_path_error).
__global__ void __launch_bounds__(256) k_bilateral_need(Dev d, NeedBfParam p, int n, int all) {
    extern __shared__ float2 s_T[];  // [511][16]
    const int tid = threadIdx.x, lane = tid & 31;
    for (int i = tid; i < 511 * 16; i += 256) s_T[i] = d.need_tab[i >> 4];
    __syncthreads();
    const unsigned T = gridDim.x * blockDim.x, t = blockIdx.x * blockDim.x + tid;
    const unsigned tb = (unsigned)__cvta_generic_to_shared(s_T) + 8u * (lane & 15);
    const int W = d.W, H = d.H;
    // the frames' lists flattened: prefix sums of their lengths, NC frames at a time
    constexpr int NC = 64;
    __shared__ unsigned s_pre[NC + 1];
    for (int f0 = 0; f0 < n; f0 += NC) {
        const int nc = min(NC, n - f0);
        __syncthreads();  // the previous chunk's prefix array is no longer read
        if (tid < 32) {   // one warp scans the chunk's counts
            unsigned carry = 0;
            for (int c0 = 0; c0 < nc; c0 += 32) {
                const int f = f0 + c0 + lane;
                unsigned x = 0;
                if (c0 + lane < nc)
                    x = frame_failed(d, f) ? 0u : all ? (unsigned)d.px : d.aux[f].fneed;
                for (int o = 1; o < 32; o <<= 1) {
                    const unsigned y = __shfl_up_sync(0xffffffffu, x, o);
                    if (lane >= o) x += y;
                }
                if (c0 + lane < nc) s_pre[c0 + lane + 1] = carry + x;
                carry += __shfl_sync(0xffffffffu, x, 31);
            }
            if (lane == 0) s_pre[0] = 0;
        }
        __syncthreads();
        const unsigned total = s_pre[nc];
        for (unsigned gi = t; gi < total; gi += T) {
            int lo = 0, hi = nc;  // frame: s_pre[lo] <= gi < s_pre[lo + 1]
            while (hi - lo > 1) {
                const int mid = (lo + hi) >> 1;
                if (s_pre[mid] <= gi) lo = mid; else hi = mid;
            }
            const int f = f0 + lo;
            const unsigned i = gi - s_pre[lo];
            const uint8_t* g = d.grey + (size_t)f * d.px;
            const uint32_t* list = d.fneed + (size_t)f * d.px;
            int u, v;
            if (all) {
                v = (int)(i / (unsigned)W);
                u = (int)i - v * W;
            } else {
                const uint32_t e = list[i];
                v = (int)(e >> 16);
                u = (int)(e & 0xffffu);
            }
            const int kp = g[(size_t)v * W + u];
            const unsigned C = tb + 128u * (unsigned)(255 - kp);
            const bool inner = u >= 5 && v >= 5 && u + 5 < W && v + 5 < H;
            int col[11];
#pragma unroll
            for (int k = 0; k < 11; ++k) col[k] = inner ? u - 5 + k : mirror(u - 5 + k, W);
            float num = 0.f, den = 0.f;
            uint8_t kc[11];
            refine_row<5>(g, (size_t)(inner ? v - 5 : mirror(v - 5, H)) * W, col, inner, u, kc);
#pragma unroll
            for (int j = 0; j < 11; ++j) {
                uint8_t kn[11];
                if (j < 10)
                    refine_row<5>(g, (size_t)(inner ? v - 4 + j : mirror(v - 4 + j, H)) * W, col,
                                  inner, u, kn);
#pragma unroll
                for (int k = 0; k < 11; ++k) {
                    float2 rt;
                    asm("ld.shared.v2.f32 {%0, %1}, [%2];"
                        : "=f"(rt.x), "=f"(rt.y)
                        : "r"(C + 128u * kc[k]));
                    den = fmaf(p.S[j * 11 + k], rt.x, den);
                    num = fmaf(p.S[j * 11 + k], rt.y, num);
                }
                if (j < 10)
#pragma unroll
                    for (int k = 0; k < 11; ++k) kc[k] = kn[k];
            }
            d.smoothed_f[(size_t)f * d.px + (size_t)v * W + u] =
                ((float)kp + __fdiv_rn(num, den)) * (1.f / 255.f);
        }
    }
}

// Exact Sobel (preprocess.hpp:76-81) of the candidates of each candidate
// tile, on the exact smoothed values k_refine_exact wrote for their 3x3
// neighbourhoods: edge bits replace the candidate bits, then the segment and
// edge counts the scan and the report need.
__global__ void __launch_bounds__(128) k_sobel_decide(Dev d) {
    __shared__ int s_seg[SB_TH], s_tot;
    const int f = blockIdx.y;
    if (frame_failed(d, f)) return;
    const unsigned cnt = d.ctile_cnt[f];
    const int W = d.W, H = d.H, tid = threadIdx.x, lane = tid & 31;
    // thread t: column t & 127 of rows (t >> 7) + rstep * k (128 threads: every row)
    const int pc = tid & (SB_TW - 1), pr0 = tid >> 7, rstep = blockDim.x >> 7;
    const double* sm = d.smoothed + (size_t)f * d.px;
    const int nbx = (W + SB_TW - 1) / SB_TW;
    for (unsigned t = blockIdx.x; t < cnt; t += gridDim.x) {
        const int tile = (int)d.ctile[(size_t)f * d.n_stile + t];
        const int by = tile / nbx, bx = tile - by * nbx;
        const int u0 = bx * SB_TW, v0 = by * SB_TH;
        __syncthreads();  // the previous tile's counters have been written out
        if (tid < SB_TH) s_seg[tid] = 0;
        if (tid == 0) s_tot = 0;
        __syncthreads();
        int n_edge = 0;
        for (int r = pr0; r < SB_TH; r += rstep) {
            const int v = v0 + r, u = u0 + pc;
            const bool in = v < H && u < W;
            const int word = u >> 5;
            const unsigned cw = in ? d.ebits[((size_t)f * H + v) * d.words_per_row + word] : 0u;
            bool edge = false;
            if ((cw >> (u & 31)) & 1) {  // candidate => masked and in the image
                // its 3x3 neighbourhood (mirrored at the border, preprocess.hpp:71-72)
                // holds exact values: k_refine_exact computed every need pixel
                const double* ra = sm + (size_t)mirror(v - 1, H) * W;
                const double* rb = sm + (size_t)v * W;
                const double* rc = sm + (size_t)mirror(v + 1, H) * W;
                const int ul = mirror(u - 1, W), ur = mirror(u + 1, W);
                const double a0 = ra[ul], a1 = ra[u], a2 = ra[ur];
                const double b0 = rb[ul], b2 = rb[ur];
                const double c0 = rc[ul], c1 = rc[u], c2 = rc[ur];
                const double gx = (a2 - a0) + 2 * (b2 - b0) + (c2 - c0);
                const double gy = (c0 - a0) + 2 * (c1 - a1) + (c2 - a2);
                edge = gx * gx + gy * gy >= d.sobel_s_star;
                n_edge += edge;
            }
            const unsigned bal = __ballot_sync(0xffffffffu, edge);
            __syncwarp();
            if (lane == 0 && v < H && word < d.words_per_row) {
                d.ebits[((size_t)f * H + v) * d.words_per_row + word] = bal;
                if (bal) atomicAdd(&s_seg[r], __popc(bal));
            }
        }
        for (int o = 16; o; o >>= 1) n_edge += __shfl_xor_sync(0xffffffffu, n_edge, o);
        if (lane == 0 && n_edge) atomicAdd(&s_tot, n_edge);
        __syncthreads();
        if (tid < SB_TH && v0 + tid < H)
            d.seg_cnt[((size_t)f * H + v0 + tid) * d.n_seg + bx] = s_seg[tid];
        if (tid == 0 && s_tot) atomicAdd(&d.aux[f].edge_px, (unsigned long long)s_tot);
    }
}

constexpr size_t kNeedTabSmem = 511 * 16 * sizeof(float2);

cudaError_t configure_fastpath(int W) {
    cudaError_t e = cudaFuncSetAttribute(k_bilateral_need, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                         kNeedTabSmem);
    if (e == cudaSuccess)
        e = cudaFuncSetAttribute(k_prescreen, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                 prescreen_smem(W, prescreen_threads(W)));
    return e;
}

int need_bilateral_ctas(int sm_count) {
    int per_sm = 0;
    if (cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, k_bilateral_need, 256, kNeedTabSmem) !=
            cudaSuccess || per_sm < 1)
        per_sm = 1;
    return sm_count * per_sm;
}

// Stage 9 of the throughput path: the certified pre-screen, then the FP32
// bilateral of its need pixels (all = 1: every pixel, for lk_fast_path_error).
void launch_fast_bilateral(const Dev& d, const LaunchPlan& lp, int n, cudaStream_t s, int all) {
    if (!all)
        k_prescreen<<<dim3(n, prescreen_segments(d.H, n)), prescreen_threads(d.W),
                      prescreen_smem(d.W, prescreen_threads(d.W)), s>>>(d, lp.ps);
    k_bilateral_need<<<lp.need_ctas, 256, kNeedTabSmem, s>>>(d, lp.nbf, n, all);
}

void launch_sobel_refine(const Dev& d, const LaunchPlan& lp, int n, cudaStream_t s) {
    const dim3 g((d.W + SB_TW - 1) / SB_TW, (d.H + SB_TH - 1) / SB_TH, n);
    k_sobel_screen<<<g, 128, 0, s>>>(d);
    k_refine_exact<5><<<dim3(lp.refine_ctas, n), 256, 0, s>>>(d, lp.ws);
    k_sobel_decide<<<dim3(lp.decide_ctas, n), 128, 0, s>>>(d);
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
