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
constexpr int IR = 64;  // k_integral output ring: columns per row kept on chip
__global__ void __launch_bounds__(128) k_integral(Dev d) {
    extern __shared__ double sh_int[];  // [4 warps][W] last row of the previous group, then rings
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
    // the group's results go through a [32 rows][IR columns] ring and leave in
    // row segments of 32 columns (one coalesced 256-byte store per row)
    // instead of 32 one-lane-per-row stores per step
    double* ring = sh_int + (size_t)4 * W + (size_t)warp * 32 * IR;
    auto flush = [&](int g, int c0) {  // columns c0 .. c0 + 31 (complete) of rows 32g ..
        __syncwarp();
        const int u = c0 + lane;
        if (u < W)
            for (int r = 0; r < 32; ++r) {
                const int vr = g * 32 + r;
                if (vr < H) out[(size_t)vr * W + u] = ring[r * IR + (u & (IR - 1))];
            }
        __syncwarp();
    };
    for (int g = 0; g * 32 < H; ++g) {
        __syncwarp();  // lane 31's writes of the previous group are visible to lane 0
        const int v = g * 32 + lane;
        const bool row_ok = v < H;
        const uint8_t* irow = img + (size_t)(row_ok ? v : 0) * W;
        double mine1 = 0.0, mine2 = 0.0;  // my results of the last two steps
        // lane 0: last[u] prefetched one step ahead; last[u-1] is the previous step's
        double above_u = (v > 0 && lane == 0) ? last[0] : 0.0, above_prev = 0.0;
        // input bytes in blocks of PB steps, loaded one block ahead (L2 latency)
        constexpr int PB = 8;
        auto load_block = [&](int t0, int (&kb)[PB]) {
#pragma unroll
            for (int j = 0; j < PB; ++j) {
                const int u = t0 + j - lane;
                kb[j] = (row_ok && u >= 0 && u < W) ? irow[u] : 0;
            }
        };
        int kb_cur[PB], kb_nxt[PB];
        load_block(0, kb_cur);
        for (int t0 = 0; t0 < W + 31; t0 += PB) {
            load_block(t0 + PB, kb_nxt);
#pragma unroll
            for (int j = 0; j < PB; ++j) {
                const int t = t0 + j;
                const int u = t - lane;
                double up = __shfl_up_sync(0xffffffffu, mine1, 1);    // in(u, v-1)
                double diag = __shfl_up_sync(0xffffffffu, mine2, 1);  // in(u-1, v-1)
                if (lane == 0) {  // the row above comes from the previous group (u = t >= 0)
                    diag = above_prev;                                  // last[u-1] (0 at u = 0)
                    up = (v > 0 && u < W) ? above_u : 0.0;              // last[u]
                    above_prev = up;
                    above_u = (v > 0 && u + 1 < W) ? last[u + 1] : 0.0;
                }
                double val = 0.0;
                const bool act = row_ok && u >= 0 && u < W;
                if (act) {
                    double x = s_val[kb_cur[j]];
                    if (sq) x = x * x;
                    val = ((up + mine1) - diag) + x;  // mine1 = in(u-1, v)
                    ring[lane * IR + (u & (IR - 1))] = val;
                }
                mine2 = mine1;
                mine1 = val;
                // lane 31 hands its row to the next group's lane 0 (read after __syncwarp)
                if (lane == 31 && act) last[u] = val;
                // column c is complete at step c + 31: columns [t - 62, t - 30) leave
                // before lane 0 reuses their slots (step t - 62 + IR)
                if (t >= 62 && ((t - 62) & 31) == 0) flush(g, t - 62);
            }
#pragma unroll
            for (int j = 0; j < PB; ++j) kb_cur[j] = kb_nxt[j];
        }
        // the blocks the steps did not reach (every column is complete now)
        const int tl = ((W + 31 + PB - 1) / PB) * PB - 1;  // the last step run
        for (int c0 = tl >= 62 ? ((tl - 62) / 32 + 1) * 32 : 0; c0 < W; c0 += 32) flush(g, c0);
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
// the row below). Shared memory holds the 2*rho+1 grey rows of BOTH images
// that the current row's blocks touch (u8 rings indexed by row mod 2*rho+1)
// and the row's block statistics.
//
// Certified integer correlation. The reference's dot product is a sequential
// FP64 sum of 49 rounded products of rounded k/255 values; the exact integer
// K = sum k_l * k_r (DP4A on packed bytes) gives dot ~ x = K / 65025 with
// |dot_ref - x| <= 49 * 3u + 48 * 49u + 2u < 2700u (u = 2^-53, every term
// <= 1; x carries two roundings). A = n mu_l mu_r and B = n sl sr are
// evaluated exactly as the reference does, and c~ = (x - A) * fl(1/B) is
// within a few u|c| of fl(fl(x - A) / B), so
//   |c_ref - c~| <= (2700u + 2u |x - A|) / B + 6u (|c~| + 1) =: E
// (covered with slack below). The candidate with the best c~ (smallest d on
// ties) is certified when every other candidate's c~ + E lies below its
// c~ - E: those cannot reach the reference's best cost, not even tie it.
// Otherwise every candidate is re-evaluated with the reference's FP64 dot in
// its exact order and compared with its exact rule (ascending d, '>').
template <int RHO>
__device__ __forceinline__ double exact_dot(const uint8_t* rr, const uint8_t* ro, int W, int v,
                                            int ucol_ref, int ucol_oth, bool ref_is_left,
                                            const double* val) {
    constexpr int B = 2 * RHO + 1, RB = B + 1;
    double dot = 0.0;
    for (int y = 0; y < B; ++y) {
        const int slot = ((v + y - RHO) % RB) * W;
        for (int x = 0; x < B; ++x) {
            const double a = __ldg(val + rr[slot + ucol_ref - RHO + x]);
            const double b = __ldg(val + ro[slot + ucol_oth - RHO + x]);
            dot += ref_is_left ? a * b : b * a;  // pl[x] * pr[x] (stereo.hpp:77-81)
        }
    }
    return dot;
}

__device__ __forceinline__ void cp_async8(void* smem, const void* gmem) {
    const unsigned sa = (unsigned)__cvta_generic_to_shared(smem);
    asm volatile("cp.async.ca.shared.global [%0], [%1], 8;\n" ::"r"(sa), "l"(gmem));
}
__device__ __forceinline__ void cp_async_wait_all() {
    asm volatile("cp.async.commit_group;\ncp.async.wait_group 0;\n" ::: "memory");
}

// 4 bytes of a u8 row starting at byte offset o (any alignment), little endian
__device__ __forceinline__ unsigned bytes4(const uint8_t* row, int o) {
    const unsigned* w = reinterpret_cast<const unsigned*>(row + (o & ~3));
    return __funnelshift_r(w[0], w[1], (o & 3) * 8);
}

template <int RHO>
__global__ void __launch_bounds__(256) k_srp(Dev d) {
    constexpr int B = 2 * RHO + 1;
    constexpr int RB = B + 1;        // ring slots: the block rows + the prefetched row
    constexpr int NW = (B + 3) / 4;  // packed words per block row
    static_assert(B <= 12, "block rows are packed into at most 3 words");
    extern __shared__ double sh_srp[];
    const int f = blockIdx.x, view = blockIdx.y;  // 0: left reference, 1: right
    const int W = d.W, H = d.H;
    const int WP = (W + 16 + 3) & ~3;         // padded u8 row pitch (word reads past the end)
    double* sbuf = sh_srp;                    // [2][4][W] statistics of rows v (and v-1, prefetched)
    uint8_t* rr = (uint8_t*)(sbuf + (size_t)8 * W);  // [RB][WP] reference-image rows
    uint8_t* ro = rr + (size_t)RB * WP;       // [RB][WP] other-image rows
    uint8_t* drow = ro + (size_t)RB * WP;     // [2][W] disparity of rows v+1, v
    const size_t fo = (size_t)f * d.px;
    const uint8_t* ref = (view ? d.right : d.grey) + fo;
    const uint8_t* oth = (view ? d.grey : d.right) + fo;
    uint8_t* out = (view ? d.disp_r : d.disp_l) + fo;
    const double* val = d.val;
    const double n = (double)B * (double)B;
    const double floor_ = d.sigma_floor;
    const int d_min = 0, d_max = d.d_max, tau = d.tau;
    const int v_bottom = H - 1 - RHO;
    constexpr double kU = 1.1102230246251565e-16;  // 2^-53
    for (size_t i = threadIdx.x; i < (size_t)W * RHO; i += blockDim.x) {
        out[i] = 0;  // rows never matched stay 0 (DisparityMap disp(w, h, 0))
        out[(size_t)(H - RHO) * W + i] = 0;
    }
    for (int i = threadIdx.x; i < 2 * RB * WP; i += blockDim.x) rr[i] = 0;  // pads read as 0
    __syncthreads();
    auto load_rows = [&](int y) {  // grey row y of both images into its ring slot
        uint8_t* a = rr + (size_t)(y % RB) * WP;
        uint8_t* b = ro + (size_t)(y % RB) * WP;
        const uint8_t* sa = ref + (size_t)y * W;
        const uint8_t* sb = oth + (size_t)y * W;
        for (int u = threadIdx.x; u < W; u += blockDim.x) {
            a[u] = sa[u];
            b[u] = sb[u];
        }
    };
    auto fetch_stats = [&](int v) {  // row v's four statistics, asynchronously
        double* dst = sbuf + (size_t)(v & 1) * 4 * W;
        const size_t i0 = fo + (size_t)v * W;
        for (int u = threadIdx.x; u < W; u += blockDim.x) {
            cp_async8(dst + u, d.mu_l + i0 + u);
            cp_async8(dst + W + u, d.mu_r + i0 + u);
            cp_async8(dst + 2 * W + u, d.sig_l + i0 + u);
            cp_async8(dst + 3 * W + u, d.sig_r + i0 + u);
        }
    };
    for (int y = v_bottom - RHO; y <= v_bottom + RHO; ++y) load_rows(y);
    fetch_stats(v_bottom);
    cp_async_wait_all();
    __syncthreads();
    constexpr int PF = 8;  // prefetched grey bytes per thread
    const bool reg_pf = W <= PF * (int)blockDim.x;  // wider rows load at the end of the row
    for (int v = v_bottom; v >= RHO; --v) {
        // prefetch row v-1's statistics (async) and grey row v-1-RHO (registers)
        const bool more = v - 1 >= RHO;
        uint8_t pa[PF], pb[PF];
        if (more) fetch_stats(v - 1);
        if (more && reg_pf) {
            const uint8_t* sa = ref + (size_t)(v - 1 - RHO) * W;
            const uint8_t* sb = oth + (size_t)(v - 1 - RHO) * W;
#pragma unroll
            for (int k = 0; k < PF; ++k) {
                const int u = threadIdx.x + k * blockDim.x;
                pa[k] = u < W ? sa[u] : 0;
                pb[k] = u < W ? sb[u] : 0;
            }
        }
        const double* s_mul = sbuf + (size_t)(v & 1) * 4 * W;
        const double* s_mur = s_mul + W;
        const double* s_sgl = s_mur + W;
        const double* s_sgr = s_sgl + W;
        const double* ref_sg = view ? s_sgr : s_sgl;
        const double* oth_sg = view ? s_sgl : s_sgr;
        uint8_t* cur = drow + (size_t)(v & 1) * W;
        const uint8_t* below = drow + (size_t)((v + 1) & 1) * W;
        for (int u = threadIdx.x; u < W; u += blockDim.x) {
            int res = 0;
            if (u >= RHO && u < W - RHO && !(ref_sg[u] < floor_)) {
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
                for (int a = 1; a < cnt; ++a)  // std::sort of (lo, hi) pairs
                    for (int b = a; b > 0 && (lo[b] < lo[b - 1] ||
                                              (lo[b] == lo[b - 1] && hi[b] < hi[b - 1]));
                         --b) {
                        const int tl = lo[b], th = hi[b];
                        lo[b] = lo[b - 1];
                        hi[b] = hi[b - 1];
                        lo[b - 1] = tl;
                        hi[b - 1] = th;
                    }
                // the reference block, packed (bytes past the block are zero)
                unsigned rw[B][NW];
#pragma unroll
                for (int y = 0; y < B; ++y) {
                    const uint8_t* row = rr + (size_t)((v + y - RHO) % RB) * WP;
#pragma unroll
                    for (int k = 0; k < NW; ++k) {
                        unsigned w = bytes4(row, u - RHO + 4 * k);
                        const int keep = B - 4 * k;  // bytes of this word inside the block
                        if (keep < 4) w &= (1u << (8 * keep)) - 1u;
                        rw[y][k] = w;
                    }
                }
                // approximate costs: the best (smallest d on ties) and M, the
                // largest c~ + E over every other candidate (including bests it
                // displaced). Certified iff M < best_c - best_e.
                double best_c = 0.0, best_e = 0.0, M = -1e300;
                int best_d = -1;
                int next = INT_MIN;
                const double mu_ref = view ? s_mur[u] : s_mul[u];
                const double sg_ref = view ? s_sgr[u] : s_sgl[u];
                for (int iv = 0; iv < cnt; ++iv) {
                    for (int dd = max(lo[iv], next); dd <= hi[iv]; ++dd) {
                        const int uo = view ? u + dd : u - dd;
                        if (uo < RHO || uo >= W - RHO) continue;
                        if (oth_sg[uo] < floor_) continue;
                        unsigned K = 0;
#pragma unroll
                        for (int y = 0; y < B; ++y) {
                            const uint8_t* row = ro + (size_t)((v + y - RHO) % RB) * WP;
                            const int o = uo - RHO;
                            const unsigned* w = reinterpret_cast<const unsigned*>(row + (o & ~3));
                            const int sh = (o & 3) * 8;
                            unsigned wd[NW + 1];
#pragma unroll
                            for (int k = 0; k <= NW; ++k) wd[k] = w[k];
#pragma unroll
                            for (int k = 0; k < NW; ++k)
                                K = __dp4a(rw[y][k], __funnelshift_r(wd[k], wd[k + 1], sh), K);
                        }
                        // A and B in the reference's order: n * (left stats) * (right stats)
                        const double mu_o = view ? s_mul[uo] : s_mur[uo];
                        const double sg_o = view ? s_sgl[uo] : s_sgr[uo];
                        const double A = view ? n * mu_o * mu_ref : n * mu_ref * mu_o;
                        const double Bn = view ? n * sg_o * sg_ref : n * sg_ref * sg_o;
                        const double ib = 1.0 / Bn;
                        const double x = (double)K * (1.0 / 65025.0);
                        const double num = x - A;
                        const double c = num * ib;  // within 4u|c| of fl(fl(x - A) / B)
                        const double e = 1.01 * ((2700.0 * kU + 2.0 * kU * fabs(num)) * ib +
                                                 6.0 * kU * (fabs(c) + 1.0)) + 1e-300;
                        if (best_d < 0 || c > best_c) {
                            if (best_d >= 0) M = fmax(M, best_c + best_e);
                            best_c = c;
                            best_e = e;
                            best_d = dd;
                        } else {
                            M = fmax(M, c + e);
                        }
                    }
                    next = max(next, hi[iv] + 1);
                }
                if (best_d >= 0 && !(M < best_c - best_e)) {
                    // ambiguous (rare): the reference's loop verbatim (stereo.hpp:124-144)
                    double bc = 0.0;
                    int bd = -1;
                    next = INT_MIN;
                    for (int iv = 0; iv < cnt; ++iv) {
                        for (int dd = max(lo[iv], next); dd <= hi[iv]; ++dd) {
                            const int uo = view ? u + dd : u - dd;
                            if (uo < RHO || uo >= W - RHO) continue;
                            if (oth_sg[uo] < floor_) continue;
                            const double dot = exact_dot<RHO>(rr, ro, WP, v, u, uo, view == 0, val);
                            const int ul = view ? uo : u, ur = view ? u : uo;
                            const double c = (dot - n * s_mul[ul] * s_mur[ur]) /
                                             (n * s_sgl[ul] * s_sgr[ur]);
                            if (bd < 0 || c > bc) {
                                bc = c;
                                bd = dd;
                            }
                        }
                        next = max(next, hi[iv] + 1);
                    }
                    best_d = bd;
                }
                res = best_d < 0 ? 0 : best_d;
            }
            cur[u] = (uint8_t)res;
            out[(size_t)v * W + u] = (uint8_t)res;
        }
        if (more && !reg_pf) load_rows(v - 1 - RHO);
        if (more && reg_pf) {
            uint8_t* a = rr + (size_t)((v - 1 - RHO) % RB) * WP;
            uint8_t* b = ro + (size_t)((v - 1 - RHO) % RB) * WP;
#pragma unroll
            for (int k = 0; k < PF; ++k) {
                const int u = threadIdx.x + k * blockDim.x;
                if (u < W) {
                    a[u] = pa[k];
                    b[u] = pb[k];
                }
            }
        }
        cp_async_wait_all();
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

size_t integral_smem(const Dev& d) { return (size_t)4 * d.W * 8 + (size_t)4 * 32 * IR * 8; }

size_t stereo_smem(const Dev& d) {
    const size_t wp = (size_t)((d.W + 16 + 3) & ~3);
    return (size_t)8 * d.W * 8 + 2 * (size_t)(2 * d.srho + 2) * wp + 2 * (size_t)d.W;
}

cudaError_t configure_stereo(const Dev& d) {
    cudaError_t e = cudaFuncSetAttribute(k_integral, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                         (int)integral_smem(d));
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
    k_integral<<<n, 128, integral_smem(d), s>>>(d);
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
