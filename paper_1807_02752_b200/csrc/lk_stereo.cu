// lk_stereo.cu — stages 1-4 of run_pipeline (pipeline.hpp:161-182): block
// statistics, search-range-propagated NCC matching for both reference views,
// and the left-right consistency check. Everything the reference computes in
// double is replayed operation for operation (--fmad=false), so every
// disparity is bit-identical to stereo.hpp.
#include <cuda_runtime.h>

#include <climits>

#include "lk_kernels.h"

namespace lkg {

// ---- stage 1a: summed-area tables (integral.hpp:22-35)
//
// in(u, v) = ((in(u, v-1) + in(u-1, v)) - in(u-1, v-1)) + x(u, v), with reads
// outside the image as 0. One warp per table (left, left^2, right, right^2 of
// one frame). Lane l owns row 32g + l of row group g and runs one column
// behind lane l-1: at step t it computes column u = t - l, and the two
// values it needs from the row above (columns u and u-1) are lane l-1's
// results of steps t-1 and t-2, fetched by shuffle. Lane 0 reads them from
// the previous group's last row. The recurrence and its rounding are the
// reference's, element for element.
__global__ void __launch_bounds__(128) k_integral(Dev d) {
    extern __shared__ double sh_int[];  // [4 warps][W] last row of the previous group
    __shared__ double s_val[256];
    const int f = blockIdx.x;
    for (int i = threadIdx.x; i < 256; i += blockDim.x) s_val[i] = d.val[i];
    __syncthreads();
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const int W = d.W, H = d.H;
    const bool sq = warp & 1;  // stats of x^2 (stereo.hpp:45)
    const uint8_t* img = (warp >= 2 ? d.right : d.grey) + (size_t)f * d.px;
    double* out = d.sat + ((size_t)f * 4 + warp) * d.px;
    double* last = sh_int + (size_t)warp * W;  // row 32g - 1, kept on chip for lane 0
    for (int g = 0; g * 32 < H; ++g) {
        __syncwarp();  // lane 31's writes of the previous group are visible to lane 0
        const int v = g * 32 + lane;
        const bool row_ok = v < H;
        const uint8_t* irow = img + (size_t)(row_ok ? v : 0) * W;
        double mine1 = 0.0, mine2 = 0.0;  // my results of the last two steps
        int k_next = (row_ok && lane == 0) ? irow[0] : 0;  // pixel of the next step
        // lane 0: last[u] prefetched one step ahead; last[u-1] is the previous step's
        double above_u = (v > 0 && lane == 0) ? last[0] : 0.0, above_prev = 0.0;
        for (int t = 0; t < W + 31; ++t) {
            const int u = t - lane;
            const bool act = row_ok && u >= 0 && u < W;
            const int k = k_next;
            if (row_ok && u + 1 >= 0 && u + 1 < W) k_next = irow[u + 1];  // prefetch
            double up = __shfl_up_sync(0xffffffffu, mine1, 1);    // in(u, v-1)
            double diag = __shfl_up_sync(0xffffffffu, mine2, 1);  // in(u-1, v-1)
            if (lane == 0) {  // the row above comes from the previous group (u = t >= 0)
                diag = above_prev;                                  // last[u-1] (0 at u = 0)
                up = (v > 0 && u < W) ? above_u : 0.0;              // last[u]
                above_prev = up;
                above_u = (v > 0 && u + 1 < W) ? last[u + 1] : 0.0;
            }
            double val = 0.0;
            if (act) {
                double x = s_val[k];
                if (sq) x = x * x;
                val = ((up + mine1) - diag) + x;  // mine1 = in(u-1, v)
                out[(size_t)v * W + u] = val;
            }
            mine2 = mine1;
            mine1 = val;
            // lane 31 hands its row to the next group's lane 0 (read after __syncwarp)
            if (lane == 31 && act) last[u] = val;
        }
    }
}

// block_sum (integral.hpp:39-47): ((r1 + r2) - r3) - r4; reads at -1 are 0
__device__ __forceinline__ double block_sum(const double* in, int W, int u, int v, int rho) {
    auto at = [&](int x, int y) { return (x < 0 || y < 0) ? 0.0 : in[(size_t)y * W + x]; };
    const double r1 = at(u + rho, v + rho);
    const double r2 = at(u - rho - 1, v - rho - 1);
    const double r3 = at(u - rho - 1, v + rho);
    const double r4 = at(u + rho, v - rho - 1);
    return ((r1 + r2) - r3) - r4;
}

// ---- stage 1b: per-pixel block mean / deviation (precompute_stats, stereo.hpp:39-60)
__global__ void __launch_bounds__(256) k_block_stats(Dev d) {
    const int f = blockIdx.z, v = blockIdx.y;
    const int u = blockIdx.x * blockDim.x + threadIdx.x;
    const int W = d.W, H = d.H, rho = d.srho;
    if (u >= W) return;
    const size_t i = (size_t)f * d.px + (size_t)v * W + u;
    const double n = (double)(2 * rho + 1) * (double)(2 * rho + 1);
    const bool inner = v >= rho && v < H - rho && u >= rho && u < W - rho;
#pragma unroll
    for (int side = 0; side < 2; ++side) {
        double mu = 0.0, sigma = 0.0;  // border blocks stay unmatchable
        if (inner) {
            const double* in = d.sat + ((size_t)f * 4 + 2 * side) * d.px;
            mu = block_sum(in, W, u, v, rho) / n;
            const double var = block_sum(in + d.px, W, u, v, rho) / n - mu * mu;
            sigma = sqrt((0.0 < var) ? var : 0.0);  // std::max(Real(0), var)
        }
        (side ? d.mu_r : d.mu_l)[i] = mu;
        (side ? d.sig_r : d.sig_l)[i] = sigma;
    }
}

// ---- stages 2/3: match_srp (stereo.hpp:157-196) for one (frame, view)
//
// Rows run bottom to top inside one CTA (each row's search ranges come from
// the row below). The 2*rho+1 rows of the OTHER image that the current row's
// blocks touch live in shared memory as doubles (a ring indexed by row mod
// 2*rho+1); the reference block of a pixel is loaded once into registers and
// every candidate's 49-term dot product accumulates y-major / x-minor in the
// reference's order. Cost: (dot - n*mu_l*mu_r) / (n*sl*sr) with the LEFT
// block's statistics first (ncc_cost, stereo.hpp:67-84); the best is the
// highest cost, smallest d on ties (ascending candidates, strict '>').
template <int RHO>
__global__ void __launch_bounds__(256) k_srp(Dev d) {
    constexpr int B = 2 * RHO + 1;
    extern __shared__ double sh_srp[];
    const int f = blockIdx.x, view = blockIdx.y;  // 0: left reference, 1: right
    const int W = d.W, H = d.H;
    double* ring = sh_srp;                              // [B][W]
    uint8_t* drow = (uint8_t*)(ring + (size_t)B * W);   // [2][W] disparity of rows v+1, v
    const size_t fo = (size_t)f * d.px;
    const uint8_t* ref = (view ? d.right : d.grey) + fo;
    const uint8_t* oth = (view ? d.grey : d.right) + fo;
    const double* ref_sig = (view ? d.sig_r : d.sig_l) + fo;
    const double* oth_sig = (view ? d.sig_l : d.sig_r) + fo;
    const double* mu_l = d.mu_l + fo;
    const double* mu_r = d.mu_r + fo;
    const double* sg_l = d.sig_l + fo;
    const double* sg_r = d.sig_r + fo;
    uint8_t* out = (view ? d.disp_r : d.disp_l) + fo;
    const double* val = d.val;
    const double n = (double)B * (double)B;
    const double floor_ = d.sigma_floor;
    const int d_min = 0, d_max = d.d_max, tau = d.tau;
    const int v_bottom = H - 1 - RHO;
    // rows never matched stay 0 (DisparityMap disp(w, h, 0))
    for (size_t i = threadIdx.x; i < (size_t)W * RHO; i += blockDim.x) {
        out[i] = 0;
        out[(size_t)(H - RHO) * W + i] = 0;
    }
    auto load_row = [&](int y) {  // other-image row y into its ring slot
        double* dst = ring + (size_t)(y % B) * W;
        const uint8_t* src = oth + (size_t)y * W;
        for (int u = threadIdx.x; u < W; u += blockDim.x) dst[u] = __ldg(val + src[u]);
    };
    for (int y = v_bottom - RHO; y <= v_bottom + RHO; ++y) load_row(y);
    for (int v = v_bottom; v >= RHO; --v) {
        if (v < v_bottom) load_row(v - RHO);
        __syncthreads();
        uint8_t* cur = drow + (size_t)(v & 1) * W;
        const uint8_t* below = drow + (size_t)((v + 1) & 1) * W;
        for (int u = threadIdx.x; u < W; u += blockDim.x) {
            int res = 0;
            if (u >= RHO && u < W - RHO && !(ref_sig[(size_t)v * W + u] < floor_)) {
                // search ranges (SearchRanges, stereo.hpp:89-112): up to three
                // clamped intervals, iterated ascending without repeats
                int lo[3], hi[3], cnt = 0;
                auto add = [&](int a, int b) {
                    a = max(a, d_min);
                    b = min(b, d_max);
                    if (a > b) return;
                    lo[cnt] = a;
                    hi[cnt] = b;
                    ++cnt;
                };
                if (v == v_bottom) {
                    add(d_min, d_max);
                } else {
                    for (int k = u - 1; k <= u + 1; ++k) {
                        if (k < 0 || k >= W) continue;
                        const int l = below[k];
                        add(l - tau, l + tau);
                    }
                    if (cnt == 0) add(d_min, d_max);  // every interval clamped away
                }
                // std::sort of (lo, hi) pairs
                for (int a = 1; a < cnt; ++a)
                    for (int b = a; b > 0 && (lo[b] < lo[b - 1] ||
                                              (lo[b] == lo[b - 1] && hi[b] < hi[b - 1]));
                         --b) {
                        const int tl = lo[b], th = hi[b];
                        lo[b] = lo[b - 1];
                        hi[b] = hi[b - 1];
                        lo[b - 1] = tl;
                        hi[b - 1] = th;
                    }
                double rb[B][B];  // the reference block
#pragma unroll
                for (int y = 0; y < B; ++y)
#pragma unroll
                    for (int x = 0; x < B; ++x)
                        rb[y][x] = __ldg(val + ref[(size_t)(v + y - RHO) * W + u - RHO + x]);
                double best_cost = 0.0;
                int best_d = -1;
                int next = INT_MIN;
                for (int iv = 0; iv < cnt; ++iv) {
                    for (int dd = max(lo[iv], next); dd <= hi[iv]; ++dd) {
                        const int uo = view ? u + dd : u - dd;
                        if (uo < RHO || uo >= W - RHO) continue;
                        if (oth_sig[(size_t)v * W + uo] < floor_) continue;
                        double dot = 0.0;
#pragma unroll
                        for (int y = 0; y < B; ++y) {
                            const double* o = ring + (size_t)((v + y - RHO) % B) * W + uo - RHO;
#pragma unroll
                            for (int x = 0; x < B; ++x) dot += rb[y][x] * o[x];
                        }
                        const int ul = view ? uo : u, ur = view ? u : uo;
                        const size_t il = (size_t)v * W + ul, ir = (size_t)v * W + ur;
                        const double c = (dot - n * mu_l[il] * mu_r[ir]) / (n * sg_l[il] * sg_r[ir]);
                        if (best_d < 0 || c > best_cost) {
                            best_cost = c;
                            best_d = dd;
                        }
                    }
                    next = max(next, hi[iv] + 1);
                }
                res = best_d < 0 ? 0 : best_d;
            }
            cur[u] = (uint8_t)res;
            out[(size_t)v * W + u] = (uint8_t)res;
        }
        __syncthreads();
    }
}

// ---- stage 4: lrc_check (stereo.hpp:263-276), written as the stage-5 input
__global__ void __launch_bounds__(256) k_lrc(Dev d) {
    const size_t n = d.px;
    const int f = blockIdx.y;
    const size_t fo = (size_t)f * n;
    for (size_t i = (size_t)blockIdx.x * blockDim.x + threadIdx.x; i < n;
         i += (size_t)gridDim.x * blockDim.x) {
        const int v = (int)(i / (size_t)d.W), u = (int)(i - (size_t)v * d.W);
        const int dl = d.disp_l[fo + i];
        const int ur = u - dl;
        int o = 0;
        if (ur >= 0 && ur < d.W && abs(dl - (int)d.disp_r[fo + (size_t)v * d.W + ur]) <= d.tr_lrc)
            o = dl;
        d.disp_out[fo + i] = (uint8_t)o;
    }
}

size_t stereo_smem(const Dev& d) { return (size_t)(2 * d.srho + 1) * d.W * 8 + 2 * (size_t)d.W; }

cudaError_t configure_stereo(const Dev& d) {
    cudaError_t e = cudaFuncSetAttribute(k_integral, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                         (int)((size_t)4 * d.W * 8));
    for (auto fn : {k_srp<1>, k_srp<2>, k_srp<3>, k_srp<4>, k_srp<5>})
        if (e == cudaSuccess)
            e = cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                     (int)stereo_smem(d));
    return e;
}

int stereo_launches() { return 4; }

cudaError_t launch_stereo(const Dev& d, int n, cudaStream_t s, cudaEvent_t* ev) {
    cudaStreamCaptureStatus cap = cudaStreamCaptureStatusNone;
    cudaStreamIsCapturing(s, &cap);
    auto mark = [&](int k) {
        if (!ev) return;
        if (cap == cudaStreamCaptureStatusActive)
            cudaEventRecordWithFlags(ev[k], s, cudaEventRecordExternal);
        else
            cudaEventRecord(ev[k], s);
    };
    mark(0);
    k_integral<<<n, 128, (size_t)4 * d.W * 8, s>>>(d);
    k_block_stats<<<dim3((d.W + 255) / 256, d.H, n), 256, 0, s>>>(d);
    mark(1);
    const dim3 g(n, 2);  // both reference views concurrently
    switch (d.srho) {  // the block radius fixes the register block
        case 1: k_srp<1><<<g, 256, stereo_smem(d), s>>>(d); break;
        case 2: k_srp<2><<<g, 256, stereo_smem(d), s>>>(d); break;
        case 4: k_srp<4><<<g, 256, stereo_smem(d), s>>>(d); break;
        case 5: k_srp<5><<<g, 256, stereo_smem(d), s>>>(d); break;
        default: k_srp<3><<<g, 256, stereo_smem(d), s>>>(d); break;
    }
    mark(2);
    mark(3);
    k_lrc<<<dim3(64, n), 256, 0, s>>>(d);
    mark(4);
    return cudaGetLastError();
}

}  // namespace lkg
