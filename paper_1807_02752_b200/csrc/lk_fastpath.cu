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
// itself: dr*1020 is within 1e-4 of the integer 4(k_q - k_p), so one FFMA with
// 1.5*2^23 rounds it into the low mantissa bits (no integer keys staged).
// w = S_t * R[dr] rounds three times in FP32 (~2e-7 relative), inside the
// ex2.approx error the bound in DESIGN.md already budgets.
//
// all = 0 (the pipeline): s~ is consumed only by the Sobel of road-mask pixels
// (k_sobel_refine), i.e. within one pixel of a masked pixel (mirroring at the
// border stays within that pixel). Tiles whose one-pixel ring holds no masked
// pixel are skipped; the test is the exact mask of k_sobel_refine
// (road_mask, preprocess.hpp:14-25). all = 1 computes every tile (lk_fast_path_error).
template <int RHO, int TB>
__global__ void __launch_bounds__(256, 3) k_bilateral_fast(Dev d, FastBfParam p, int all) {
    constexpr int WIN = 2 * RHO + 1, TWh = BT_W + 2 * RHO, THh = BT_H + 2 * RHO;
    constexpr int NPX = TWh * THh;
    static_assert(WIN == 11, "packed tap pairs assume an 11-wide window");
    __shared__ float s_v[NPX], s_vf[256], s_R[512];
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
        s_R[threadIdx.x] = __ldg(d.fast_tab + 256 + threadIdx.x);
        s_R[threadIdx.x + 256] = __ldg(d.fast_tab + 512 + threadIdx.x);
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
    // t = dr*1020 + kMagic + 1020: its bit pattern is __float_as_int(kMagic) + the
    // BYTE offset 4*(k_q - k_p + 255) of the table entry, so the LDS needs no
    // address arithmetic beyond one add of a uniform base
    const float2 k1020 = make_float2(1020.f, 1020.f), mg = make_float2(kMagic + 1020.f, kMagic + 1020.f);
    const char* Rb = reinterpret_cast<const char*>(s_R) - __float_as_int(kMagic);
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
                    const float2 t = __ffma2_rn(dr, k1020, mg);
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
// (origin gx0, gy0): the arithmetic of k_bilateral_tile / preprocess.hpp:38-56.
template <int RHO>
__device__ __forceinline__ double exact_bilateral(const Dev& d, const WsParam& ws,
                                                  const uint8_t* s_g, int gw, int gx0, int gy0,
                                                  int u, int v) {
    constexpr int WIN = 2 * RHO + 1;
    const uint8_t* c = s_g + (v - gy0) * gw + (u - gx0);
    const double* wrow = d.wr + (int)c[0] * 256;
    double num = 0.0, den = 0.0;
#pragma unroll 1
    for (int j = 0; j < WIN; ++j) {
        const uint8_t* row = c + (j - RHO) * gw - RHO;
#pragma unroll
        for (int i = 0; i < WIN; ++i) {
            const int kv = row[i];
            const double w = ws.w[j * WIN + i] * __ldg(wrow + kv);
            num += w * __ldg(d.val + kv);
            den += w;
        }
    }
    return num / den;
}

// ---- 2. Sobel on s~ with the propagated bound, exact refinement, edge bits
template <int RHO>
__global__ void __launch_bounds__(256) k_sobel_refine(Dev d, WsParam ws) {
    constexpr int FW = SB_TW + 4, FH = SB_TH + 4;              // s~ tile, 2-px halo
    constexpr int NW = SB_TW + 2, NH = SB_TH + 2;              // tile + 1-px ring
    constexpr int GW = SB_TW + 2 + 2 * RHO, GH = SB_TH + 2 + 2 * RHO;  // grey for the ring
    __shared__ float s_f[FH * FW];
    __shared__ uint8_t s_g[GH * GW];
    __shared__ uint8_t s_cand[SB_TH * SB_TW];
    __shared__ double s_ex[NH * NW];
    __shared__ short s_need[NH * NW];
    __shared__ int s_nneed, s_seg[SB_TH], s_tot[2];
    const int f = blockIdx.z;
    if (frame_failed(d, f)) return;
    if (d.W < 3 || d.H < 3) {  // preprocess.hpp:68-69
        if (blockIdx.x == 0 && blockIdx.y == 0 && threadIdx.x == 0)
            fail_frame(d, f, 10, LK_MSG_SOBEL_TOO_SMALL);
        return;
    }
    const int W = d.W, H = d.H;
    const int u0 = blockIdx.x * SB_TW, v0 = blockIdx.y * SB_TH;
    const int horizon = (int)d.rep[f].horizon;
    if (v0 + SB_TH <= horizon) {  // the mask is empty above the horizon
        if (threadIdx.x < SB_TH && v0 + threadIdx.x < H)
            d.seg_cnt[((size_t)f * H + v0 + threadIdx.x) * d.n_seg + blockIdx.x] = 0;
        return;
    }
    const float* sf = d.smoothed_f + (size_t)f * d.px;
    const uint8_t* grey = d.grey + (size_t)f * d.px;
    // mirrored row offsets / columns of the grey halo (the s~ halo is its inner part)
    __shared__ int s_rowg[GH], s_colg[GW];
    for (int i = threadIdx.x; i < GH; i += blockDim.x) s_rowg[i] = mirror(v0 - 1 - RHO + i, H) * W;
    for (int i = threadIdx.x; i < GW; i += blockDim.x) s_colg[i] = mirror(u0 - 1 - RHO + i, W);
    __syncthreads();
    for (int i = threadIdx.x; i < FH * FW; i += blockDim.x) {
        const int r = i / FW, c = i - r * FW;  // s~ row v0-2+r = grey row index r + RHO - 1
        s_f[i] = sf[(size_t)s_rowg[r + RHO - 1] + s_colg[c + RHO - 1]];
    }
    if (threadIdx.x < SB_TH) s_seg[threadIdx.x] = 0;
    if (threadIdx.x < 2) s_tot[threadIdx.x] = 0;
    if (threadIdx.x == 0) s_nneed = 0;
    __syncthreads();
    const double dg = 8.0 * kEpsSmooth;  // |gx~ - gx|, |gy~ - gy| bound (sum of |Sobel taps| = 8)
    int n_mask = 0, any_cand = 0;
    for (int i = threadIdx.x; i < SB_TH * SB_TW; i += blockDim.x) {
        const int r = i / SB_TW, c = i - r * SB_TW;
        const int v = v0 + r, u = u0 + c;
        uint8_t cand = 0;
        if (v < H && u < W) {
            const int dv = d.disp[(size_t)f * d.px + (size_t)v * W + u];
            const bool m = v >= horizon && dv != 0 &&
                           fabs((double)dv - d.fv[(size_t)f * H + v]) <= d.varpi;
            n_mask += m;
            if (m) {
                const float* a = s_f + (r + 1) * FW + (c + 1);  // row v-1, col u-1
                const float* b = a + FW;
                const float* cc = b + FW;
                const double gx = ((double)a[2] - a[0]) + 2 * ((double)b[2] - b[0]) +
                                  ((double)cc[2] - cc[0]);
                const double gy = ((double)cc[0] - a[0]) + 2 * ((double)cc[1] - a[1]) +
                                  ((double)cc[2] - a[2]);
                const double s = gx * gx + gy * gy;
                const double ds = dg * (2 * fabs(gx) + dg) + dg * (2 * fabs(gy) + dg) + 1e-14;
                cand = s + ds >= d.sobel_s_star;
            }
        }
        s_cand[i] = cand;
        any_cand |= cand;
    }
    if (!__syncthreads_or(any_cand)) {  // no edge can exist in this tile (most tiles)
        for (int o = 16; o; o >>= 1) n_mask += __shfl_xor_sync(0xffffffffu, n_mask, o);
        if ((threadIdx.x & 31) == 0 && n_mask)
            atomicAdd(&d.aux[f].mask_px, (unsigned long long)n_mask);
        if (threadIdx.x < SB_TH && v0 + threadIdx.x < H)
            d.seg_cnt[((size_t)f * H + v0 + threadIdx.x) * d.n_seg + blockIdx.x] = 0;
        return;
    }
    for (int i = threadIdx.x; i < GH * GW; i += blockDim.x) {
        const int r = i / GW, c = i - r * GW;
        s_g[i] = grey[(size_t)s_rowg[r] + s_colg[c]];
    }
    // pixels of tile + ring inside a candidate's 3x3 need the exact bilateral
    for (int i = threadIdx.x; i < NH * NW; i += blockDim.x) {
        const int r = i / NW, c = i - r * NW;  // ring coords: tile pixel (r-1, c-1)
        bool need = false;
        for (int y = r - 2; y <= r && !need; ++y)
            for (int x = c - 2; x <= c; ++x)
                if (y >= 0 && y < SB_TH && x >= 0 && x < SB_TW && s_cand[y * SB_TW + x]) {
                    need = true;
                    break;
                }
        if (need) s_need[atomicAdd(&s_nneed, 1)] = (short)i;
    }
    __syncthreads();
    const int gx0 = u0 - 1 - RHO, gy0 = v0 - 1 - RHO;
    for (int k = threadIdx.x; k < s_nneed; k += blockDim.x) {
        const int i = s_need[k];
        const int r = i / NW, c = i - r * NW;
        // ring positions outside the image hold their mirror pixel (preprocess.hpp:71-72)
        const int v = mirror(v0 - 1 + r, H), u = mirror(u0 - 1 + c, W);
        const double e = exact_bilateral<RHO>(d, ws, s_g, GW, gx0, gy0, u, v);
        s_ex[i] = e;
        d.smoothed[(size_t)f * d.px + (size_t)v * W + u] = e;  // read back by k_edge_emit
    }
    __syncthreads();
    const int lane = threadIdx.x & 31;
    int n_edge = 0;
#pragma unroll
    for (int k = 0; k < SB_TW * SB_TH / 256; ++k) {
        const int i = threadIdx.x + k * 256;
        const int r = i / SB_TW, c = i % SB_TW;
        const int v = v0 + r;
        bool edge = false;
        if (s_cand[i]) {  // candidate => masked and in the image
            const double* a = s_ex + r * NW + c;  // row v-1, col u-1
            const double* b = a + NW;
            const double* cc = b + NW;
            const double gx = (a[2] - a[0]) + 2 * (b[2] - b[0]) + (cc[2] - cc[0]);
            const double gy = (cc[0] - a[0]) + 2 * (cc[1] - a[1]) + (cc[2] - a[2]);
            edge = gx * gx + gy * gy >= d.sobel_s_star;
            n_edge += edge;
        }
        const unsigned bal = __ballot_sync(0xffffffffu, edge);
        if (lane == 0 && v < H) {
            const int word = (u0 + c) >> 5;
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
