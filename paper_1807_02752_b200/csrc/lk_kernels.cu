// lk_kernels.cu — sm_100a kernels for lanekit stages 5-12.
//
// Built with --fmad=false: every double + - * / rounds exactly as the
// reference's SSE2 build does, so FP-derived integer decisions (mask, edges,
// votes, DP paths, RANSAC sets, lane columns) are reproduced bit for bit.
// Transcendentals: the bilateral's exp factors come from host-built glibc
// tables (exact); atan2 (Sobel theta, w_g ray) and exp (w_g) use CUDA's
// libdevice (<= 2 ulp from glibc, covered by the parity tolerance).
#include <cuda_runtime.h>

#include "lk_fit.cuh"
#include "lk_kernels.h"

namespace lkg {

// =====================================================================
// K1  build_vdisparity (road_profile.hpp:32-45) + valid-disparity count.
// grid (ceil(H/R), n), 256 threads = 8 warps; warp w takes rows w, w+8, ...
// of the CTA's R rows, so a row's histogram key is warp-uniform. The rows'
// bytes arrive in shared memory by one TMA bulk copy (cp.async.bulk, mbarrier
// transaction count). A row whose bytes all equal its first (road rows, the
// sky) is one warp-level aggregate: a single shared atomic of W. Other rows go
// 16-byte chunk by chunk: a uniform chunk extends the lane's (d, count) run, a
// mixed one is merged per byte, and the lanes' runs are added with one shared
// atomic per distinct d (all lanes equal: one add of the warp sum; else
// __match_any_sync groups and their leaders). Only the transposed histogram
// [D1][H] is written (the v-path DP's layout; the VDISPARITY hook transposes
// it back on the host).
// =====================================================================

constexpr int K1_UNROLL = 3;  // 3 x 32 x 16 B covers a 1242-px row in one round

// Byte b (0..15) of a 16-byte chunk, without a local-memory array.
__device__ __forceinline__ int chunk_byte(const uint4& q, int b) {
    const int k = b >> 2;
    const uint32_t w = k == 0 ? q.x : k == 1 ? q.y : k == 2 ? q.z : q.w;
    return (w >> (8 * (b & 3))) & 0xff;
}

// Bytes [lo, hi) of a row chunk, per byte (road_profile.hpp:42): valid and
// counted totals, runs of equal d merged into per-lane shared atomics; the
// last run is returned in (key, cnt) for the warp-aggregated add. Out of line:
// it is rare and keeps the hot loop small.
struct VdRun {
    int key, cnt, valid, counted;
};

__device__ __noinline__ VdRun vd_row_chunk(uint4 q, int lo, int hi, int d_max, int32_t* hrow) {
    VdRun o{-1, 0, 0, 0};
    for (int b = lo; b < hi; ++b) {
        const int dv = chunk_byte(q, b);
        o.valid += dv != 0;
        const int k = (dv >= 1 && dv <= d_max) ? dv : -1;
        if (k != o.key) {
            if (o.cnt) atomicAdd(&hrow[o.key], o.cnt);
            o.key = k;
            o.cnt = 0;
        }
        o.cnt += k >= 0;
        o.counted += k >= 0;
    }
    return o;
}

// Warp-aggregated shared atomic of (key, cnt) per lane; cnt == 0 = nothing.
// Called by whole warps.
__device__ __forceinline__ void vd_warp_add(int32_t* hrow, int key, int cnt) {
    const unsigned full = 0xffffffffu;
    key = cnt ? key : -1;
    const int k0 = __shfl_sync(full, key, 0);
    if (__all_sync(full, key == k0)) {
        const int sum = __reduce_add_sync(full, cnt);
        if (k0 >= 0 && (threadIdx.x & 31) == 0) atomicAdd(&hrow[k0], sum);
        return;
    }
    const unsigned grp = __match_any_sync(full, key);
    const int sum = __reduce_add_sync(grp, cnt);
    if (key >= 0 && (threadIdx.x & 31) == __ffs(grp) - 1) atomicAdd(&hrow[key], sum);
}

// One full 16-byte chunk's contribution: a uniform chunk extends the lane's
// run (key, cnt); a mixed one goes through vd_row_chunk. A lane's run is
// flushed with a per-lane atomic only when its key changes.
__device__ __forceinline__ void vd_chunk(const uint4& q, int d_max, int32_t* hrow, int& key,
                                         int& cnt, unsigned& valid, unsigned& counted) {
    const uint32_t b0 = (q.x & 0xffu) * 0x01010101u;
    const int dv = q.x & 0xff;
    if (((q.x ^ b0) | (q.y ^ b0) | (q.z ^ b0) | (q.w ^ b0)) == 0) {
        valid += dv ? 16 : 0;
        if (dv >= 1 && dv <= d_max) {  // road_profile.hpp:42
            counted += 16;
            if (dv != key) {
                if (cnt) atomicAdd(&hrow[key], cnt);
                key = dv;
                cnt = 0;
            }
            cnt += 16;
        }
    } else {
        const VdRun o = vd_row_chunk(q, 0, 16, d_max, hrow);
        valid += o.valid;
        counted += o.counted;
        if (o.cnt) {
            if (o.key != key) {
                if (cnt) atomicAdd(&hrow[key], cnt);
                key = o.key;
                cnt = 0;
            }
            cnt += o.cnt;
        }
    }
}

// ---- one-shot TMA bulk staging (cp.async.bulk + mbarrier transaction count)
__device__ __forceinline__ uint32_t smem_u32(const void* p) {
    return (uint32_t)__cvta_generic_to_shared(p);
}

__device__ __forceinline__ void mbar_init(uint64_t* bar, unsigned count) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(count)
                 : "memory");
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
}

// Arms the barrier with the byte count, then one bulk copy global -> shared
// (addresses and size multiples of 16) that completes the transaction.
__device__ __forceinline__ void bulk_load(void* dst, const void* src, unsigned bytes,
                                          uint64_t* bar) {
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(bar)),
                 "r"(bytes)
                 : "memory");
    asm volatile(
        "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::
            "r"(smem_u32(dst)),
        "l"(src), "r"(bytes), "r"(smem_u32(bar))
        : "memory");
}

// Several bulk copies on one barrier: arm it once with their total bytes
// (mbar_expect), then issue each copy (bulk_copy; 16-byte aligned, size a
// multiple of 16).
__device__ __forceinline__ void mbar_expect(uint64_t* bar, unsigned bytes) {
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(bar)),
                 "r"(bytes)
                 : "memory");
}

__device__ __forceinline__ void bulk_copy(void* dst, const void* src, unsigned bytes, uint64_t* bar) {
    asm volatile(
        "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::
            "r"(smem_u32(dst)),
        "l"(src), "r"(bytes), "r"(smem_u32(bar))
        : "memory");
}

__device__ __forceinline__ void mbar_wait(uint64_t* bar, unsigned parity) {
    asm volatile(
        "{\n .reg .pred p;\n"
        "WAIT_%=:\n mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n"
        " @!p bra WAIT_%=;\n}" ::"r"(smem_u32(bar)),
        "r"(parity)
        : "memory");
}

// Row r of the CTA = head bytes [rp, a) + full 16-byte chunks [a, e) + tail
// bytes [e, rp + W), all in shared memory. One warp round covers the row's first
// 32*K1_UNROLL chunks plus one head/tail byte per lane (lanes 0-15 head,
// 16-31 tail).
__device__ __forceinline__ void vd_row_geometry(const uint8_t* rp, int W, int& head, int& nfull) {
    head = (int)((16 - (reinterpret_cast<uintptr_t>(rp) & 15)) & 15);
    if (head > W) head = W;
    nfull = (W - head) >> 4;
}

// K1 CTA = (block of R rows, frame). Thread 0 stages the rows' bytes (the
// 16-byte aligned span around them) into shared memory with one bulk copy
// while the others zero the histogram; the warps then count rows from shared
// memory (warp w: rows w, w+8, ...). dynamic smem: barrier, hist [R][D1], span.
__global__ void __launch_bounds__(256) k_vdisparity(Dev d, int32_t* vhistT, int R) {
    extern __shared__ __align__(128) unsigned char k1s[];
    uint64_t* bar = reinterpret_cast<uint64_t*>(k1s);
    int32_t* sh_hist = reinterpret_cast<int32_t*>(k1s + 16);
    const int D1 = d.D1, W = d.W, d_max = d.d_max;
    uint8_t* span = k1s + 16 + (((size_t)R * D1 * 4 + 15) & ~(size_t)15);
    const int f = blockIdx.y;
    const int v0 = blockIdx.x * R;
    const int rows = min(R, d.H - v0);
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    const uint8_t* start = d.disp + (size_t)f * d.px + (size_t)v0 * W;
    const uintptr_t a = reinterpret_cast<uintptr_t>(start) & ~(uintptr_t)15;
    const uintptr_t e = (reinterpret_cast<uintptr_t>(start) + (size_t)rows * W + 15) & ~(uintptr_t)15;
    if (threadIdx.x == 0) {  // (the inputs carry 16 bytes of padding past the last frame)
        mbar_init(bar, 1);
        bulk_load(span, reinterpret_cast<const void*>(a), (unsigned)(e - a), bar);
    }
    for (int i = threadIdx.x; i < R * D1; i += blockDim.x) sh_hist[i] = 0;
    unsigned valid = 0, counted = 0;
    const uint8_t* sbase = span + (reinterpret_cast<uintptr_t>(start) - a);
    constexpr int RC = 32 * K1_UNROLL;  // chunks per warp round
    __syncthreads();  // barrier initialised, histogram zeroed
    mbar_wait(bar, 0);
    for (int r = warp; r < rows; r += 8) {
        const uint8_t* rp = sbase + (size_t)r * W;
        int head, nfull;
        vd_row_geometry(rp, W, head, nfull);
        const uint4* a0 = reinterpret_cast<const uint4*>(rp + head);
        const int tail = W - head - 16 * nfull;  // < 16
        const int hb = lane < head ? (int)rp[lane]
                     : (lane >= 16 && lane - 16 < tail) ? (int)rp[head + 16 * nfull + (lane - 16)]
                                                        : -1;
        uint4 q[K1_UNROLL];
#pragma unroll
        for (int j = 0; j < K1_UNROLL; ++j) {
            const int c = lane + 32 * j;
            q[j] = c < nfull ? a0[c] : make_uint4(0, 0, 0, 0);
        }
        int32_t* hrow = sh_hist + r * D1;
        // whole-row test: every byte of the row equal to its first byte
        const int ref = rp[0];
        const uint32_t b4 = (uint32_t)ref * 0x01010101u;
        uint32_t diff = hb >= 0 ? (uint32_t)(hb ^ ref) : 0u;
#pragma unroll
        for (int j = 0; j < K1_UNROLL; ++j)
            if (lane + 32 * j < nfull)
                diff |= (q[j].x ^ b4) | (q[j].y ^ b4) | (q[j].z ^ b4) | (q[j].w ^ b4);
        if (nfull <= RC && __all_sync(0xffffffffu, diff == 0)) {
            if (lane == 0) {  // the warp's whole-row aggregate: one shared atomic
                valid += ref ? W : 0;
                if (ref >= 1 && ref <= d_max) {  // road_profile.hpp:42
                    atomicAdd(&hrow[ref], W);
                    counted += W;
                }
            }
            continue;
        }
        // mixed row: per chunk (uniform chunks merged into lane runs, mixed
        // chunks per byte), then one warp-aggregated add of the lane runs
        int key = -1, cnt = 0;
        for (int c0 = 0; c0 < nfull; c0 += RC) {
            if (c0) {
#pragma unroll
                for (int j = 0; j < K1_UNROLL; ++j) {
                    const int c = c0 + lane + 32 * j;
                    q[j] = c < nfull ? a0[c] : make_uint4(0, 0, 0, 0);
                }
            }
#pragma unroll
            for (int j = 0; j < K1_UNROLL; ++j)
                if (c0 + lane + 32 * j < nfull)
                    vd_chunk(q[j], d_max, hrow, key, cnt, valid, counted);
        }
        vd_warp_add(hrow, key, cnt);
        int bk = -1, bc = 0;  // head / tail bytes, one per lane
        if (hb >= 0) {
            valid += hb != 0;
            if (hb >= 1 && hb <= d_max) {
                bk = hb;
                bc = 1;
                ++counted;
            }
        }
        vd_warp_add(hrow, bk, bc);
    }
    for (int o = 16; o; o >>= 1) {
        valid += __shfl_xor_sync(0xffffffffu, valid, o);
        counted += __shfl_xor_sync(0xffffffffu, counted, o);
    }
    if (lane == 0) {
        if (valid) atomicAdd((unsigned long long*)&d.rep[f].valid_disparities,
                             (unsigned long long)valid);
        if (counted) atomicAdd(&d.aux[f].hist_total, (unsigned long long)counted);
    }
    __syncthreads();
    // transposed store [D1][H]: warp per column, lane = row (R <= 32: runs of R ints)
    int32_t* outT = vhistT + (size_t)f * D1 * d.H + v0;
    for (int c = warp; c < D1; c += 8)
        if (lane < rows) outT[(size_t)c * d.H + lane] = sh_hist[lane * D1 + c];
    if (blockIdx.x == 0 && threadIdx.x == 0) {
        lk_frame_report& rep = d.rep[f];
        rep.width = d.W;
        rep.height = d.H;
    }
}

// Rows per K1 CTA: as many as keep the CTA's shared memory (histogram rows +
// staged bytes) within ~56 KB (4 CTAs per SM), at most one per lane.
int vdisparity_rows(int W, int D1) {
    const int r = (56 * 1024 - 160) / (W + 4 * D1 + 1);
    return r < 1 ? 1 : r > K1_ROWS ? K1_ROWS : r;
}

size_t vdisparity_smem(int W, int D1) {
    const int R = vdisparity_rows(W, D1);
    return 16 + (((size_t)R * D1 * 4 + 15) & ~(size_t)15) + (size_t)R * W + 32;
}

// Block-wide (value, index) argmin, first index among equal minima (the
// terminal scan of dp.hpp:60-62). Returns the index to every thread.
__device__ int block_argmin(double val, int idx, double* sv, int* si) {
    for (int o = 16; o; o >>= 1) {
        const double ov = __shfl_xor_sync(0xffffffffu, val, o);
        const int oi = __shfl_xor_sync(0xffffffffu, idx, o);
        if (ov < val || (ov == val && oi < idx)) {
            val = ov;
            idx = oi;
        }
    }
    const int w = threadIdx.x >> 5, nw = blockDim.x >> 5;
    __syncthreads();
    if ((threadIdx.x & 31) == 0) {
        sv[w] = val;
        si[w] = idx;
    }
    __syncthreads();
    if (threadIdx.x < 32) {
        val = threadIdx.x < nw ? sv[threadIdx.x] : __longlong_as_double(0x7ff0000000000000LL);
        idx = threadIdx.x < nw ? si[threadIdx.x] : 0x7fffffff;
        for (int o = 16; o; o >>= 1) {
            const double ov = __shfl_xor_sync(0xffffffffu, val, o);
            const int oi = __shfl_xor_sync(0xffffffffu, idx, o);
            if (ov < val || (ov == val && oi < idx)) {
                val = ov;
                idx = oi;
            }
        }
        if (threadIdx.x == 0) si[0] = idx;
    }
    __syncthreads();
    const int r = si[0];
    __syncthreads();
    return r;
}

// =====================================================================
// K2a  dp_extract_vpath (road_profile.hpp:54-78) on dp_min_path (dp.hpp:29-73).
// One CTA per frame; states = rows in parallel, stages = disparities in
// sequence. Offsets {0..6} are scanned in list order with strict '<', energy
// order (prev + pen) + data. Choices live in shared memory when they fit.
// =====================================================================
__global__ void __launch_bounds__(512) k_vpath(Dev d, const int32_t* vhistT, int choice_in_smem) {
    extern __shared__ double sh[];
    const int f = blockIdx.x;
    if (frame_failed(d, f)) return;
    const int H = d.H, D1 = d.D1;
    double* prev = sh;
    double* cur = sh + H;
    __shared__ double sv[32];
    __shared__ int si[32];
    int8_t* choice = choice_in_smem ? (int8_t*)(sh + 2 * H) : d.vchoice + (size_t)f * D1 * H;
    const int32_t* hT = vhistT + (size_t)f * D1 * H;
    double pen[7];
    for (int o = 0; o < 7; ++o) pen[o] = d.paper_sign ? -d.lambda_y * o : d.lambda_y * o;
    // stage 0 <-> d = d_max
    for (int s = threadIdx.x; s < H; s += blockDim.x)
        prev[s] = -(double)hT[(size_t)d.d_max * H + s];
    __syncthreads();
    // the next stage's histogram column is loaded while this stage runs, so
    // the 64 sequential stages do not each wait on a global load
    constexpr int VP_MAXS = 4;  // states per thread held in registers (H <= 2048)
    const bool regs = H <= VP_MAXS * (int)blockDim.x;
    int cnext[VP_MAXS];
    auto load_col = [&](int st) {
        const int32_t* col = hT + (size_t)(d.d_max - st) * H;
#pragma unroll
        for (int k = 0; k < VP_MAXS; ++k) {
            const int s = threadIdx.x + k * blockDim.x;
            cnext[k] = s < H ? col[s] : 0;
        }
    };
    if (regs && D1 > 1) load_col(1);
    // integral lambda_y (default 30): the energies are integers, exact in
    // double, so the DP runs on int keys 8 E + o whose minimum is the smallest
    // energy and, among ties, the first offset in scan order (strict '<',
    // dp.hpp:43-51); rows past H hold sentinels instead of a bound test
    const bool use_int = regs && d.lambda_y == floor(d.lambda_y) && d.lambda_y <= 1e4 &&
                         (double)d.W * (double)D1 + 7e4 * (double)D1 < 1e8;
    if (use_int) {
        int* pi = reinterpret_cast<int*>(prev);
        int* ci = reinterpret_cast<int*>(cur);
        int ik[7];
#pragma unroll
        for (int o = 0; o < 7; ++o) ik[o] = (int)pen[o] * 8 + o;
        __syncthreads();  // prev's doubles read above
        for (int s = threadIdx.x; s < H + 7; s += blockDim.x) {
            pi[s] = s < H ? -hT[(size_t)d.d_max * H + s] * 8 : (1 << 30);
            if (s >= H) ci[s] = 1 << 30;
        }
        __syncthreads();
        for (int st = 1; st < D1; ++st) {
            int ccur[VP_MAXS];
#pragma unroll
            for (int k = 0; k < VP_MAXS; ++k) ccur[k] = cnext[k];
            if (st + 1 < D1) load_col(st + 1);
            int8_t* chr = choice + (size_t)st * H;
#pragma unroll
            for (int k = 0; k < VP_MAXS; ++k) {
                const int s = threadIdx.x + k * blockDim.x;
                if (s >= H) break;
                int best = pi[s] + ik[0];
#pragma unroll
                for (int o = 1; o < 7; ++o) best = min(best, pi[s + o] + ik[o]);
                ci[s] = (best & ~7) - ccur[k] * 8;
                chr[s] = (int8_t)(best & 7);
            }
            __syncthreads();
            int* t = pi;
            pi = ci;
            ci = t;
        }
        int mvi = 0x7fffffff, mi = 0x7fffffff;
        for (int s = threadIdx.x; s < H; s += blockDim.x)
            if (pi[s] < mvi) {  // (pi >> 3 ordered like pi: the low bits hold no offset at the end)
                mvi = pi[s];
                mi = s;
            }
        const int term = block_argmin((double)(mvi >> 3), mi, sv, si);
        if (threadIdx.x == 0) {
            int32_t* pts = d.vpath + (size_t)f * D1 * 2;
            int p = term;
            pts[(D1 - 1) * 2] = d.d_max - (D1 - 1);
            pts[(D1 - 1) * 2 + 1] = p;
            for (int st = D1 - 1; st > 0; --st) {
                p += choice[(size_t)st * H + p];
                pts[(st - 1) * 2] = d.d_max - (st - 1);
                pts[(st - 1) * 2 + 1] = p;
            }
            lk_frame_report& rep = d.rep[f];
            rep.vpath_energy = (double)(pi[term] >> 3);
            const bool ev = d.aux[f].hist_total > 0;
            rep.vpath_has_evidence = ev;
            if (!ev) fail_frame(d, f, 6, LK_MSG_NO_ROAD_EVIDENCE);  // pipeline.hpp:189-190
        }
        return;
    }
    for (int st = 1; st < D1; ++st) {
        const int32_t* col = hT + (size_t)(d.d_max - st) * H;
        int ccur[VP_MAXS];
#pragma unroll
        for (int k = 0; k < VP_MAXS; ++k) ccur[k] = cnext[k];
        if (regs && st + 1 < D1) load_col(st + 1);
#pragma unroll
        for (int k = 0; k < VP_MAXS; ++k) {
            const int s = threadIdx.x + k * blockDim.x;
            if (!regs || s >= H) break;
            double best = __longlong_as_double(0x7ff0000000000000LL);
            int bo = 0;
#pragma unroll
            for (int o = 0; o < 7; ++o) {
                const int ps = s + o;
                if (ps >= H) continue;
                const double e = prev[ps] + pen[o];
                if (e < best) {
                    best = e;
                    bo = o;
                }
            }
            cur[s] = best + -(double)ccur[k];
            choice[(size_t)st * H + s] = (int8_t)bo;
        }
        if (!regs)
            for (int s = threadIdx.x; s < H; s += blockDim.x) {
                double best = __longlong_as_double(0x7ff0000000000000LL);
                int bo = 0;
#pragma unroll
                for (int o = 0; o < 7; ++o) {
                    const int ps = s + o;
                    if (ps >= H) continue;
                    const double e = prev[ps] + pen[o];
                    if (e < best) {
                        best = e;
                        bo = o;
                    }
                }
                cur[s] = best + -(double)col[s];
                choice[(size_t)st * H + s] = (int8_t)bo;
            }
        __syncthreads();
        double* t = prev;
        prev = cur;
        cur = t;
    }
    double mv = __longlong_as_double(0x7ff0000000000000LL);
    int mi = 0x7fffffff;
    for (int s = threadIdx.x; s < H; s += blockDim.x)
        if (prev[s] < mv) {
            mv = prev[s];
            mi = s;
        }
    const int term = block_argmin(mv, mi, sv, si);
    if (threadIdx.x == 0) {
        int32_t* pts = d.vpath + (size_t)f * D1 * 2;
        int p = term;
        pts[(D1 - 1) * 2] = d.d_max - (D1 - 1);
        pts[(D1 - 1) * 2 + 1] = p;
        for (int st = D1 - 1; st > 0; --st) {
            p += choice[(size_t)st * H + p];
            pts[(st - 1) * 2] = d.d_max - (st - 1);
            pts[(st - 1) * 2 + 1] = p;
        }
        lk_frame_report& rep = d.rep[f];
        rep.vpath_energy = prev[term];
        const bool ev = d.aux[f].hist_total > 0;
        rep.vpath_has_evidence = ev;
        if (!ev) fail_frame(d, f, 6, LK_MSG_NO_ROAD_EVIDENCE);  // pipeline.hpp:189-190
    }
}

// =====================================================================
// K2b  ransac_beta (road_profile.hpp:121-137) + make_road_profile
// (road_profile.hpp:145-227): horizon, V_py, singular rows, f(v) per row.
// One CTA (128 threads) per frame; warp 0 runs the RANSAC.
// =====================================================================
__global__ void __launch_bounds__(128) k_road_fit(Dev d) {
    extern __shared__ int sh_i[];
    const int f = blockIdx.x;
    if (frame_failed(d, f)) return;
    const int n = d.D1, H = d.H;
    constexpr int NW = 4;  // 128 threads
    int* px = sh_i;
    int* pv = px + n;
    int* bufs[NW + 2];
    for (int b = 0; b < NW + 2; ++b) bufs[b] = pv + n + b * n;
    double* tbuf = align8(pv + n + (NW + 2) * n);
    __shared__ RansacState st;
    __shared__ int s_bad_row;
    const int32_t* pts = d.vpath + (size_t)f * n * 2;
    for (int i = threadIdx.x; i < n; i += blockDim.x) {
        px[i] = pts[2 * i];
        pv[i] = pts[2 * i + 1];
    }
    if (threadIdx.x == 0) s_bad_row = 0x7fffffff;
    __syncthreads();
    block_ransac<3, NW>(px, pv, n, d.tr_y, d.eps_y, d.max_iter, d.rng, bufs, tbuf, st);
    lk_frame_report& rep = d.rep[f];
    if (st.msg) {  // ransac_trim threw: the report keeps its defaults (pipeline.hpp:199-207)
        if (threadIdx.x == 0) fail_frame(d, f, 7, st.msg);
        return;
    }
    const double b0 = st.model[0], b1 = st.model[1], b2 = st.model[2];
    // horizon_row (road_profile.hpp:161-176)
    int horizon = 0;
    bool in_range = true;
    {
        double root = 0;
        bool ok = true;
        if (b2 == 0) {
            if (b1 <= 0)
                ok = false;
            else
                root = -b0 / b1;
        } else {
            const double disc = b1 * b1 - 4 * b2 * b0;
            if (disc <= 0)
                ok = false;
            else
                root = (-b1 + sqrt(disc)) / (2 * b2);
        }
        if (ok) {
            const long long r = llround_ref(root);
            if (r < 0 || r >= H)
                ok = false;
            else
                horizon = (int)r;
        }
        if (!ok) {
            horizon = 0;
            in_range = false;
        }
    }
    // vpy_profile (road_profile.hpp:184-199) and road_f per row
    int bad = 0x7fffffff;
    for (int v = threadIdx.x; v < H; v += blockDim.x) {
        const double vv = (double)v;
        const double fp = b1 + 2 * b2 * vv;
        const double fvv = b0 + b1 * vv + b2 * vv * vv;
        uint8_t sing = 0;
        double vpy;
        if (fabs(fp) < 1e-12) {
            sing = 1;
            vpy = vv;
            if (v >= horizon) bad = min(bad, v);
        } else {
            vpy = vv - fvv / fp;
        }
        d.vpy[(size_t)f * H + v] = vpy;
        d.vsing[(size_t)f * H + v] = sing;
        d.fv[(size_t)f * H + v] = fvv;
        d.mrange[(size_t)f * H + v] = v >= horizon ? mask_interval(fvv, d.varpi) : make_int2(256, 0);
    }
    if (bad != 0x7fffffff) atomicMin(&s_bad_row, bad);
    for (int i = threadIdx.x; i < st.n_inl; i += blockDim.x) {
        const int id = st.inl[i];
        d.beta_inl[((size_t)f * n + i) * 2] = px[id];
        d.beta_inl[((size_t)f * n + i) * 2 + 1] = pv[id];
    }
    __syncthreads();
    if (threadIdx.x == 0) {
        rep.beta[0] = b0;
        rep.beta[1] = b1;
        rep.beta[2] = b2;
        rep.beta_iterations = st.iterations;
        rep.beta_inlier_fraction = st.fraction;
        rep.beta_degraded = st.degraded;
        rep.beta_inlier_count = st.n_inl;
        rep.horizon = horizon;
        rep.horizon_in_range = in_range;
        if (s_bad_row != 0x7fffffff)  // road_profile.hpp:223-225
            fail_frame(d, f, 7, LK_MSG_SINGULAR_VPY, s_bad_row);
    }
}

// =====================================================================
// K3a  bilateral_filter (preprocess.hpp:30-59), 8-bit input.
// w = exp(-ds*inv_s2) * exp(-dr*dr*inv_r2): the first factor depends only on
// the tap (ws table), the second only on the (centre, neighbour) byte pair
// (wr table), both tabulated on the host with the reference's libm, so the
// product and the j-major / i-minor sums are bit-identical. Tile 32x8 with a
// mirrored halo staged in shared memory.
// =====================================================================

template <int RHO>
__global__ void __launch_bounds__(256) k_bilateral(Dev d) {
    extern __shared__ double sh_bf[];
    const int rho = RHO >= 0 ? RHO : d.rho;
    const int win = 2 * rho + 1;
    const int f = blockIdx.z;
    if (frame_failed(d, f)) return;
    const int TWh = BF_TW + 2 * rho, THh = BF_TH + 2 * rho;
    double* s_val = sh_bf;               // [256]
    double* s_ws = s_val + 256;          // [win*win]
    uint8_t* s_px = (uint8_t*)(s_ws + win * win);  // [THh][TWh]
    const int u0 = blockIdx.x * BF_TW, v0 = blockIdx.y * BF_TH;
    const uint8_t* g = d.grey + (size_t)f * d.px;
    for (int i = threadIdx.x; i < 256; i += blockDim.x) s_val[i] = d.val[i];
    for (int i = threadIdx.x; i < win * win; i += blockDim.x) s_ws[i] = d.ws[i];
    for (int i = threadIdx.x; i < TWh * THh; i += blockDim.x) {
        const int ty = i / TWh, tx = i - ty * TWh;
        const int gu = mirror(u0 + tx - rho, d.W), gv = mirror(v0 + ty - rho, d.H);
        s_px[i] = g[(size_t)gv * d.W + gu];
    }
    __syncthreads();
    const int tx = threadIdx.x % BF_TW, ty = threadIdx.x / BF_TW;
    const int u = u0 + tx, v = v0 + ty;
    if (u >= d.W || v >= d.H) return;
    const int kc = s_px[(ty + rho) * TWh + tx + rho];
    const double* __restrict__ wrow = d.wr + kc * 256;
    double num = 0.0, den = 0.0;
    if (RHO >= 0) {
#pragma unroll
        for (int j = 0; j < 2 * RHO + 1; ++j) {
            const uint8_t* prow = s_px + (ty + j) * TWh + tx;
#pragma unroll
            for (int i = 0; i < 2 * RHO + 1; ++i) {
                const int kv = prow[i];
                const double w = s_ws[j * (2 * RHO + 1) + i] * __ldg(wrow + kv);
                num += w * s_val[kv];
                den += w;
            }
        }
    } else {
        for (int j = 0; j < win; ++j) {
            const uint8_t* prow = s_px + (ty + j) * TWh + tx;
            for (int i = 0; i < win; ++i) {
                const int kv = prow[i];
                const double w = s_ws[j * win + i] * __ldg(wrow + kv);
                num += w * s_val[kv];
                den += w;
            }
        }
    }
    d.smoothed[(size_t)f * d.px + (size_t)v * d.W + u] = num / den;
}

// ---------------------------------------------------------------------
// K3a' tiled bilateral for the default 11x11 window (RHO = 5).
// The exact wr LUT is 512 KB. A tile of BT_W x BT_H outputs (plus its 5-px
// mirrored halo) only touches the values V present in that region, and
// wr[a][b] == wr[b][a] exactly (a-b == -(b-a) in IEEE arithmetic), so the CTA
// compacts V (typically 40-130 values) and stages the exact symmetric
// sub-table, |V|(|V|+1)/2 doubles, in shared memory: every tap's weight is one
// LDS.64 instead of an L1/L2 gather (tiles with |V| > BT_TRI_N fall back to
// __ldg on the full table). The 121 spatial factors ws are a by-value kernel
// parameter, so they reach the DMULs as constant-bank operands. Each thread
// produces BT_R vertically adjacent outputs: a window row is loaded once
// (conflict-free, consecutive lanes) and folded into every output whose
// window contains it, still in the reference's j-major / i-minor order.
// ---------------------------------------------------------------------
// Table-lookup mode of the tiled bilateral (a profiling experiment kept as a
// switch): 0 = exact sub-table in shared memory (LSU pipe); 1 = the full
// table via __ldg; 2 = the full table via tex1Dfetch (TEX pipe); 3 = hybrid,
// even taps from shared memory, odd taps through the texture path.
template <int RHO, int MODE>
__device__ __forceinline__ void bilateral_rows(const Dev& d, const WsParam& ws,
                                               const double* s_sub, const int* s_map,
                                               const double* s_v, const uint32_t* s_kt,
                                               const uint8_t* s_g, int f, int u0, int v0) {
    constexpr int WIN = 2 * RHO + 1, TWh = BT_W + 2 * RHO;
    const int tx = threadIdx.x % BT_W, ty = threadIdx.x / BT_W;
    const int r0 = ty * BT_R;
    int ca[BT_R], ta[BT_R], craw[BT_R];
#pragma unroll
    for (int r = 0; r < BT_R; ++r) {
        const int kc = s_g[(r0 + r + RHO) * TWh + tx + RHO];
        craw[r] = kc * 256;
        ca[r] = (MODE == 0 || MODE == 3) ? s_map[kc] : 0;
        ta[r] = (ca[r] * (ca[r] + 1)) >> 1;
    }
    double num[BT_R], den[BT_R];
#pragma unroll
    for (int r = 0; r < BT_R; ++r) num[r] = den[r] = 0.0;
#pragma unroll
    for (int jj = 0; jj < BT_R + 2 * RHO; ++jj) {
        const int prow = (r0 + jj) * TWh + tx;
        uint32_t kt[WIN];
        double vv[WIN];
#pragma unroll
        for (int i = 0; i < WIN; ++i) {
            kt[i] = s_kt[prow + i];
            vv[i] = s_v[prow + i];
        }
#pragma unroll
        for (int r = 0; r < BT_R; ++r) {
            const int dj = jj - r;
            if (dj < 0 || dj >= WIN) continue;
#pragma unroll
            for (int i = 0; i < WIN; ++i) {
                const int b = (int)(kt[i] & 0xffu);            // local index
                const int raw = (int)((kt[i] >> 8) & 0xffu);   // 8-bit value
                double wrv;
                if (MODE == 0 || (MODE == 3 && (i & 1) == 0)) {
                    const int tb = (int)(kt[i] >> 16);
                    wrv = s_sub[b <= ca[r] ? ta[r] + b : tb + ca[r]];
                } else if (MODE == 1) {
                    wrv = __ldg(d.wr + craw[r] + raw);
                } else {
                    const int2 t = tex1Dfetch<int2>((cudaTextureObject_t)d.wr_tex, craw[r] + raw);
                    wrv = __hiloint2double(t.y, t.x);
                }
                const double w = ws.w[dj * WIN + i] * wrv;
                num[r] += w * vv[i];
                den[r] += w;
            }
        }
    }
    const int u = u0 + tx;
#pragma unroll
    for (int r = 0; r < BT_R; ++r) {
        const int v = v0 + r0 + r;
        if (u < d.W && v < d.H) d.smoothed[(size_t)f * d.px + (size_t)v * d.W + u] = num[r] / den[r];
    }
}

template <int RHO, int MODE>
__global__ void __launch_bounds__(256, 2) k_bilateral_tile(Dev d, WsParam ws) {
    constexpr int TWh = BT_W + 2 * RHO, THh = BT_H + 2 * RHO;
    constexpr int NPX = TWh * THh;
    extern __shared__ double sm_bt[];
    double* s_v = sm_bt;                         // [NPX] neighbour values k/255.0
    uint32_t* s_kt = (uint32_t*)(s_v + NPX);     // [NPX] local | value << 8 | tri(local) << 16
    int* s_map = (int*)(s_kt + NPX);             // [256] value -> local index
    int* s_inv = s_map + 256;                    // [256] local index -> value
    uint8_t* s_g = (uint8_t*)(s_inv + 256);      // [NPX] raw 8-bit grey
    uint8_t* s_fv = s_g + NPX;                   // [256] value present
    double* s_sub = align8(s_fv + 256);          // [TRI] symmetric exact sub-table (MODE 0/3)
    __shared__ int s_warp[8];
    __shared__ int s_n;
    const int f = blockIdx.z;
    if (frame_failed(d, f)) return;
    const int u0 = blockIdx.x * BT_W, v0 = blockIdx.y * BT_H;
    const uint8_t* g = d.grey + (size_t)f * d.px;
    for (int i = threadIdx.x; i < 256; i += blockDim.x) s_fv[i] = 0;
    __syncthreads();
    for (int i = threadIdx.x; i < NPX; i += blockDim.x) {
        const int ty = i / TWh, tx = i - ty * TWh;
        const int gu = mirror(u0 + tx - RHO, d.W), gv = mirror(v0 + ty - RHO, d.H);
        const int k = g[(size_t)gv * d.W + gu];
        s_g[i] = (uint8_t)k;
        s_v[i] = d.val[k];
        s_fv[k] = 1;  // benign race: every writer stores 1
    }
    __syncthreads();
    if (MODE == 1 || MODE == 2) {
        for (int i = threadIdx.x; i < NPX; i += blockDim.x) s_kt[i] = (uint32_t)s_g[i] << 8;
        __syncthreads();
        bilateral_rows<RHO, MODE>(d, ws, s_sub, s_map, s_v, s_kt, s_g, f, u0, v0);
        return;
    }
    {  // exclusive scan of the presence vector -> value <-> local index
        const int t = threadIdx.x, lane = t & 31, w = t >> 5;
        const int fv = s_fv[t];
        int iv = fv;
        for (int o = 1; o < 32; o <<= 1) {
            const int b = __shfl_up_sync(0xffffffffu, iv, o);
            if (lane >= o) iv += b;
        }
        if (lane == 31) s_warp[w] = iv;
        __syncthreads();
        int ov = 0;
        for (int k = 0; k < w; ++k) ov += s_warp[k];
        iv += ov - fv;
        s_map[t] = iv;
        if (fv) s_inv[iv] = t;
        if (t == 255) s_n = iv + fv;
    }
    __syncthreads();
    const int nv = s_n;
    if (nv <= BT_TRI_N) {
        const int ntri = nv * (nv + 1) / 2;
        for (int e = threadIdx.x; e < ntri; e += blockDim.x) {
            // e = b(b+1)/2 + a, a <= b
            int b = (int)((sqrt(8.0 * e + 1.0) - 1.0) * 0.5);
            while (b * (b + 1) / 2 > e) --b;
            while ((b + 1) * (b + 2) / 2 <= e) ++b;
            const int a = e - b * (b + 1) / 2;
            s_sub[e] = __ldg(d.wr + s_inv[a] * 256 + s_inv[b]);
        }
        for (int i = threadIdx.x; i < NPX; i += blockDim.x) {
            const uint32_t raw = s_g[i], b = (uint32_t)s_map[raw];
            s_kt[i] = b | (raw << 8) | (((b * (b + 1)) >> 1) << 16);
        }
        __syncthreads();
        bilateral_rows<RHO, MODE>(d, ws, s_sub, s_map, s_v, s_kt, s_g, f, u0, v0);
    } else {  // more than BT_TRI_N values in this tile: full table through L1
        for (int i = threadIdx.x; i < NPX; i += blockDim.x) s_kt[i] = (uint32_t)s_g[i] << 8;
        __syncthreads();
        bilateral_rows<RHO, 1>(d, ws, s_sub, s_map, s_v, s_kt, s_g, f, u0, v0);
    }
}

// Sobel taps on the smoothed image with mirrored borders (preprocess.hpp:71-81).
__device__ __forceinline__ void sobel_at(const double* img, int W, int H, int u, int v,
                                         double& gx, double& gy) {
    const int um = mirror(u - 1, W), up = mirror(u + 1, W), uc = mirror(u, W);
    const double* rm = img + (size_t)mirror(v - 1, H) * W;
    const double* rc = img + (size_t)mirror(v, H) * W;
    const double* rp = img + (size_t)mirror(v + 1, H) * W;
    gx = (rm[up] - rm[um]) + 2 * (rc[up] - rc[um]) + (rp[up] - rp[um]);
    gy = (rp[um] - rm[um]) + 2 * (rp[uc] - rm[uc]) + (rp[up] - rm[up]);
}

// =====================================================================
// K3b  road_mask (preprocess.hpp:14-26) + sobel_gradients (:67-90) +
// edge_map test (:103-113). Tile SB_TW x SB_TH with the mirrored 1-px halo
// of the smoothed image staged in shared memory: the tile's SB_TH + 2 row
// interiors (SB_TW doubles, 1 KB each) arrive by TMA bulk copies on one
// mbarrier while the threads load the two mirrored halo columns; tiles at the
// right border (or an odd width: rows not 16-byte aligned) stage element-wise.
// The magnitude test !(sqrt(s) < t) is evaluated exactly as s >= s* (s* from
// the host). Writes the edge bitmap and, per (row, SB_TW-column segment), the
// edge count.
// =====================================================================
__global__ void __launch_bounds__(256) k_sobel_edges(Dev d) {
    constexpr int SW = SB_TW + 2;   // staged columns u0 - 1 .. u0 + SB_TW
    constexpr int SWP = SB_TW + 4;  // row pitch: column u0 - 1 + c at index 1 + c (interior 16-B aligned)
    __shared__ __align__(16) double s_img[(SB_TH + 2) * SWP];
    __shared__ uint64_t s_bar;
    __shared__ int s_seg[SB_TH];
    __shared__ int s_tot[2];
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
    if (!d.hooks && v0 + SB_TH <= horizon) {  // the mask is empty above the horizon
        if (threadIdx.x < SB_TH && v0 + threadIdx.x < H)
            d.seg_cnt[((size_t)f * H + v0 + threadIdx.x) * d.n_seg + blockIdx.x] = 0;
        return;
    }
    const double* img = d.smoothed + (size_t)f * d.px;
    __shared__ int s_col[SW];
    __shared__ int s_row[SB_TH + 2];
    for (int i = threadIdx.x; i < SW; i += blockDim.x) s_col[i] = mirror(u0 - 1 + i, W);
    if (threadIdx.x < SB_TH + 2) s_row[threadIdx.x] = mirror(v0 - 1 + threadIdx.x, H) * W;
    __syncthreads();
    const bool tma = u0 + SB_TW <= W && (W & 1) == 0 && (reinterpret_cast<uintptr_t>(img) & 15) == 0;
    if (tma) {
        if (threadIdx.x == 0) {
            mbar_init(&s_bar, 1);
            mbar_expect(&s_bar, (SB_TH + 2) * SB_TW * 8);
            for (int r = 0; r < SB_TH + 2; ++r)
                bulk_copy(s_img + r * SWP + 2, img + (size_t)s_row[r] + u0, SB_TW * 8, &s_bar);
        }
        if (threadIdx.x < 2 * (SB_TH + 2)) {  // the mirrored halo columns
            const int r = threadIdx.x >> 1, c = (threadIdx.x & 1) ? SW - 1 : 0;
            s_img[r * SWP + 1 + c] = img[(size_t)s_row[r] + s_col[c]];
        }
    } else {  // all loads in flight before the stores
        constexpr int NE = ((SB_TH + 2) * SW + 255) / 256;
        double t[NE];
#pragma unroll
        for (int k = 0; k < NE; ++k) {
            const int i = threadIdx.x + k * 256;
            if (i < (SB_TH + 2) * SW) t[k] = img[(size_t)s_row[i / SW] + s_col[i % SW]];
        }
#pragma unroll
        for (int k = 0; k < NE; ++k) {
            const int i = threadIdx.x + k * 256;
            if (i < (SB_TH + 2) * SW) s_img[(i / SW) * SWP + 1 + i % SW] = t[k];
        }
    }
    if (threadIdx.x < SB_TH) s_seg[threadIdx.x] = 0;
    if (threadIdx.x < 2) s_tot[threadIdx.x] = 0;
    __syncthreads();
    if (tma) mbar_wait(&s_bar, 0);
    const int lane = threadIdx.x & 31;
    int n_edge = 0, n_mask = 0;
#pragma unroll
    for (int k = 0; k < SB_TW * SB_TH / 256; ++k) {
        const int i = threadIdx.x + k * 256;
        const int r = i / SB_TW, c = i % SB_TW;
        const int v = v0 + r, u = u0 + c;
        bool edge = false;
        if (v < H && u < W) {
            const double* a = s_img + r * SWP + 1 + c;  // row v-1, col u-1
            const double* b = a + SWP;                   // row v
            const double* cc = b + SWP;                  // row v+1
            const double gx = (a[2] - a[0]) + 2 * (b[2] - b[0]) + (cc[2] - cc[0]);
            const double gy = (cc[0] - a[0]) + 2 * (cc[1] - a[1]) + (cc[2] - a[2]);
            const double s = gx * gx + gy * gy;
            const int dv = d.disp[(size_t)f * d.px + (size_t)v * W + u];
            const bool m = v >= horizon && dv != 0 &&
                           fabs((double)dv - d.fv[(size_t)f * H + v]) <= d.varpi;
            n_mask += m;
            edge = m && s >= d.sobel_s_star;
            n_edge += edge;
            if (d.hooks) {
                const size_t gi = (size_t)f * d.px + (size_t)v * W + u;
                d.mask[gi] = m;
                d.gx[gi] = gx;
                d.gy[gi] = gy;
                d.mag[gi] = sqrt(s);
                double th = atan2(gy, gx);
                if (th <= -kPi) th = kPi;
                d.theta[gi] = th;
            }
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

// Exclusive scan of the per-segment edge counts in row-major order: every
// (row, segment) gets the index of its first edge in the frame's edge list;
// row_off[v] is the first edge of row v (row_off[H] = edge count).
__global__ void __launch_bounds__(1024) k_edge_scan(Dev d) {
    const int f = blockIdx.x;
    if (frame_failed(d, f)) return;
    __shared__ int s_w[32];
    const int total = d.H * d.n_seg;
    const int per = (total + blockDim.x - 1) / blockDim.x;
    const int start = threadIdx.x * per;
    const int32_t* cnt = d.seg_cnt + (size_t)f * total;
    int32_t* off = d.seg_off + (size_t)f * total;
    int sum = 0;
    for (int i = start; i < min(start + per, total); ++i) sum += cnt[i];
    const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
    int inc = sum;
    for (int o = 1; o < 32; o <<= 1) {
        const int t = __shfl_up_sync(0xffffffffu, inc, o);
        if (lane >= o) inc += t;
    }
    if (lane == 31) s_w[w] = inc;
    __syncthreads();
    if (w == 0) {
        int x = s_w[lane];
        for (int o = 1; o < 32; o <<= 1) {
            const int t = __shfl_up_sync(0xffffffffu, x, o);
            if (lane >= o) x += t;
        }
        s_w[lane] = x;
    }
    __syncthreads();
    int run = inc - sum + (w > 0 ? s_w[w - 1] : 0);
    for (int i = start; i < min(start + per, total); ++i) {
        off[i] = run;
        run += cnt[i];
    }
    __syncthreads();
    int32_t* roff = d.row_off + (size_t)f * (d.H + 1);
    for (int v = threadIdx.x; v < d.H; v += blockDim.x) roff[v] = off[(size_t)v * d.n_seg];
    if (threadIdx.x == blockDim.x - 1) roff[d.H] = run;
}

// =====================================================================
// K3c  edge list in row-major order (edge_map, preprocess.hpp:103-113) +
// sparse_vpx votes (vanish.hpp:49-70). One warp per (row, segment): the
// segment's bitmap words are walked in u order and each edge is written at
// its scanned position, so the list order equals the reference's.
// =====================================================================
// One warp emits the edges of one 128-px row segment (row v, segment sx).
__device__ __forceinline__ void emit_segment(const Dev& d, int f, int v, int sx, int lane) {
    const int W = d.W, H = d.H;
    const int seg = v * d.n_seg + sx;
    // every input of the segment requested at once (one memory latency)
    const int cnt = d.seg_cnt[(size_t)f * H * d.n_seg + seg];
    const int base = d.seg_off[(size_t)f * H * d.n_seg + seg];
    const uint32_t* bits = d.ebits + ((size_t)f * H + v) * d.words_per_row;
    uint32_t bw[SB_TW / 32];
#pragma unroll
    for (int w = 0; w < SB_TW / 32; ++w) {
        const int word = sx * (SB_TW / 32) + w;
        bw[w] = word < d.words_per_row ? bits[word] : 0u;
    }
    const double vpy = d.vpy[(size_t)f * H + v];
    const bool sing = d.vsing[(size_t)f * H + v] != 0;
    if (cnt == 0) return;  // empty segment
    const double* img = d.smoothed + (size_t)f * d.px;
    const int ext_hi = d.ext_lo + d.ext_cols - 1;
    int run = 0, n_vote = 0, n_skip = 0;
#pragma unroll
    for (int w = 0; w < SB_TW / 32; ++w) {
        const int word = sx * (SB_TW / 32) + w;
        const uint32_t b = bw[w];
        if ((b >> lane) & 1u) {
            const int u = word * 32 + lane;
            const size_t e = (size_t)f * d.px + base + run + __popc(b & ((1u << lane) - 1u));
            double gx, gy;
            sobel_at(img, W, H, u, v, gx, gy);
            d.e_uv[e] = u | (v << 16);  // theta (atan2) is k_wg's, over all edges in parallel
            d.e_gx[e] = gx;
            d.e_gy[e] = gy;
            int col = kSkipCol;
            if (!(sing || fabs(gx) < 1e-3)) {  // kGradientFloor, vanish.hpp:20, 59
                const double c = (double)u + ((double)v - vpy) * (gy / gx);
                long long cc = llround_ref(c);
                cc = cc < d.ext_lo ? d.ext_lo : (cc > ext_hi ? ext_hi : cc);
                col = (int)cc;
                ++n_vote;
            } else {
                ++n_skip;
            }
            d.e_col[e] = col;
        }
        run += __popc(b);
    }
    for (int o = 16; o; o >>= 1) {
        n_vote += __shfl_xor_sync(0xffffffffu, n_vote, o);
        n_skip += __shfl_xor_sync(0xffffffffu, n_skip, o);
    }
    if (lane == 0) {
        if (n_vote) atomicAdd(&d.aux[f].votes, (unsigned long long)n_vote);
        if (n_skip) atomicAdd(&d.aux[f].skipped, (unsigned long long)n_skip);
    }
}

// Exact path: a warp per segment over the whole frame.
__global__ void __launch_bounds__(256) k_edge_emit(Dev d) {
    const int f = blockIdx.y;
    if (frame_failed(d, f)) return;
    const int seg = blockIdx.x * 8 + (threadIdx.x >> 5);
    if (seg >= d.H * d.n_seg) return;
    emit_segment(d, f, seg / d.n_seg, seg % d.n_seg, threadIdx.x & 31);
}

// Fast path: edges exist only in the Sobel screen's candidate tiles (one
// 128-px segment column x SB_TH rows each), so only those are visited.
__global__ void __launch_bounds__(256) k_edge_emit_tiles(Dev d) {
    const int f = blockIdx.y;
    if (frame_failed(d, f)) return;
    const unsigned cnt = d.ctile_cnt[f];
    const int warp = threadIdx.x >> 5, nw = blockDim.x >> 5;
    for (unsigned t = blockIdx.x; t < cnt; t += gridDim.x) {
        const int tile = (int)d.ctile[(size_t)f * d.n_stile + t];
        const int by = tile / d.n_seg, bx = tile - by * d.n_seg;
        for (int r = warp; r < SB_TH; r += nw) {  // a warp per 128-px row segment
            const int v = by * SB_TH + r;
            if (v < d.H) emit_segment(d, f, v, bx, threadIdx.x & 31);
        }
    }
}

// lanes.hpp:20-25
// Gate margin of the certificate (lk_frame_report.uncertain): the two atan2
// (libdevice, <= 2 ulp; glibc <= 1 ulp) move te - tv, hence dd, by < 1e-14.
constexpr double kGateEps = 1e-12;

__device__ __forceinline__ double piecewise_weight(double te, double tv, double sg,
                                                   bool* uncertain = nullptr) {
    double dd = fmod(fabs(te - tv), kPi);
    if (dd > kPi / 2) dd = kPi - dd;
    if (uncertain) *uncertain = fabs(dd - kPi / 6) <= kGateEps;
    if (dd > kPi / 6) return 0.0;
    return exp(-(dd / (sg * sg)) * (36 / kPi));
}

// =====================================================================
// K4a accumulate_dense_vpx (vanish.hpp:113-148) + dp_extract_upath
// (:156-182). One CTA per frame.
// The banded accumulator is never materialised: per-column band counts slide
// with the DP stage (exact integer +-1 updates from the per-row vote lists),
// and each DP stage reads -rho_vote * count directly.
// =====================================================================

// One DP stage over the thread's SP consecutive states, operands from a
// register window prev[s0-5 .. s0+SP+4]. INT: exact packed keys
// (energy << 4 | offset index), whose minimum is the smallest energy and,
// among ties, the earliest offset in list order — the strict-'<' scan of
// dp.hpp:43-51. Otherwise doubles with the reference's scan verbatim.
// Offset of list entry oi in {0, -1, 1, -2, 2, ...} (dp.hpp:43-51 scan order).
__device__ __forceinline__ int upath_off(int oi) { return (oi & 1) ? -((oi + 1) >> 1) : (oi >> 1); }

// One DP stage over the thread's SP consecutive states, operands from a
// register window prev[s0-5 .. s0+SP+4] (the rows carry 5 sentinel entries
// on each side, so no bounds tests). INT: exact packed keys
// (energy << 4 | offset index), whose minimum is the smallest energy and,
// among ties, the earliest offset in list order — the strict-'<' scan of
// dp.hpp:43-51; energies are stored x16, so keys are prev16 + d.upk[oi] with
// upk = pen * 16 + oi from the host (constant-bank operands), reduced with
// 3-input mins. Otherwise
// doubles with the reference's scan verbatim. ch[s] receives the winning
// offset INDEX (the backtrack maps it to the offset).
template <int SP, bool INT>
__device__ __forceinline__ void upath_stage(const Dev& d, const void* prevv, void* curv,
                                            const int* cnt, int8_t* ch, int C, double nrv,
                                            int nrv_i) {
    const int s0 = threadIdx.x * SP;
    if (s0 >= C) return;
    if (INT) {
        const int* prev = (const int*)prevv;
        int* cur = (int*)curv;
        int w16[SP + 10];
#pragma unroll
        for (int k = 0; k < SP + 10; ++k) w16[k] = prev[s0 - 5 + k];  // stored x16 already
#pragma unroll
        for (int j = 0; j < SP; ++j) {
            const int s = s0 + j;
            if (s >= C) break;
            int key[11];
#pragma unroll
            for (int oi = 0; oi < 11; ++oi) key[oi] = w16[j + 5 + upath_off(oi)] + d.upk[oi];
            const int m0 = __vimin3_s32(key[0], key[1], key[2]);
            const int m1 = __vimin3_s32(key[3], key[4], key[5]);
            const int m2 = __vimin3_s32(key[6], key[7], key[8]);
            const int best = __vimin3_s32(__vimin3_s32(m0, m1, m2), key[9], key[10]);
            cur[s] = (best & ~15) + nrv_i * cnt[s];  // x16: prev*16 + pen*16 + 16 nrv cnt
            ch[s] = (int8_t)(best & 15);
        }
    } else {
        const double* prev = (const double*)prevv;
        double* cur = (double*)curv;
        double wv[SP + 10];
#pragma unroll
        for (int k = 0; k < SP + 10; ++k) wv[k] = prev[s0 - 5 + k];
#pragma unroll
        for (int j = 0; j < SP; ++j) {
            const int s = s0 + j;
            if (s >= C) break;
            double best = __longlong_as_double(0x7ff0000000000000LL);
            int boi = 0;
#pragma unroll
            for (int oi = 0; oi < 11; ++oi) {
                const double e = wv[j + 5 + upath_off(oi)] + d.upen[oi];
                if (e < best) {
                    best = e;
                    boi = oi;
                }
            }
            cur[s] = best + nrv * cnt[s];
            ch[s] = (int8_t)boi;
        }
    }
}

template <int SP, int NT>
__global__ void __launch_bounds__(NT, NT <= 512 ? 2 : 1) k_vanish(Dev d) {
    extern __shared__ double sh4[];
    const int f = blockIdx.x;
    if (frame_failed(d, f)) return;
    const int H = d.H, C = d.ext_cols;
    lk_frame_report& rep = d.rep[f];
    const int v_top = (int)rep.horizon, v_max = H - 1;
    const int nrows = v_max - v_top + 1;
    double* prev = sh4 + 8;  // DP rows with 8 pad slots on each side
    double* cur = prev + C + 16;
    int* const cnt0 = (int*)(cur + C + 8);  // band counts, double-buffered
    int* const cnt1 = cnt0 + C;
    int* px = cnt1 + C;
    int* pv = px + H;
    int8_t* win = (int8_t*)(pv + H);  // [BT_CHUNK][2*BT_SPAN+1]
    int* s_roff = (int*)(win + BT_CHUNK * (2 * BT_SPAN + 1) + 4 - (BT_CHUNK * (2 * BT_SPAN + 1)) % 4);
    uint16_t* s_vcol = (uint16_t*)(s_roff + H + 1);  // [d.vote_cap] vote column - ext_lo
    __shared__ double sv[32];
    __shared__ int si[32];
    __shared__ int s_votes;
#ifdef LK_VANISH_PROF
    const long long t0 = clock64();
    long long t_band = 0, t_dp = 0;
#endif
    const int32_t* groff = d.row_off + (size_t)f * (H + 1);
    const int32_t* ecol = d.e_col + (size_t)f * d.px;
    int8_t* choice = d.uchoice + (size_t)f * H * C;
    // per-row vote lists staged once (the band updates of every stage read them)
    const int e_first = groff[v_top], n_edges_in = groff[H] - e_first;
    const bool staged = n_edges_in <= d.vote_cap;
    for (int r = threadIdx.x; r <= H; r += blockDim.x) s_roff[r] = groff[r];
    if (staged)
        for (int e = threadIdx.x; e < n_edges_in; e += blockDim.x) {
            const int c = ecol[e_first + e];
            s_vcol[e] = c == kSkipCol ? (uint16_t)0xffff : (uint16_t)(c - d.ext_lo);
        }
    const int* roff = s_roff;
    for (int c = threadIdx.x; c < 2 * C; c += blockDim.x) cnt0[c] = 0;
    if (threadIdx.x == 0) s_votes = 0;
    __syncthreads();
    // vote_band (vanish.hpp:101-105) of stage stg: rows [bt, bb]
    auto band = [&](int stg, int& bt, int& bb) {
        const int v = v_max - stg;
        if (v > v_max - d.chi - 1) {
            bt = v;
            bb = v_max;
        } else if (v >= v_top + d.chi) {
            bt = v - d.chi;
            bb = v + d.chi;
        } else {
            bt = v_top;
            bb = v + d.chi;
        }
    };
    // moves counts cn from band [t0, b0] to band [t1, b1] (both slide upwards):
    // rows [t1, t0) enter, rows (b1, b0] leave; exact integer +-1 updates
    auto slide = [&](int* cn, int t0, int b0, int t1, int b1) {
        if (t1 < t0)
            for (int e = roff[t1] + threadIdx.x; e < roff[t0]; e += blockDim.x) {
                const int c = staged ? (int)s_vcol[e - e_first]
                                     : (ecol[e] == kSkipCol ? 0xffff : ecol[e] - d.ext_lo);
                if (c != 0xffff) atomicAdd(&cn[c], 1);
            }
        if (b1 < b0)
            for (int e = roff[b1 + 1] + threadIdx.x; e < roff[b0 + 1]; e += blockDim.x) {
                const int c = staged ? (int)s_vcol[e - e_first]
                                     : (ecol[e] == kSkipCol ? 0xffff : ecol[e] - d.ext_lo);
                if (c != 0xffff) atomicSub(&cn[c], 1);
            }
    };
    const double nrv = -d.rho_vote;
    // exact int32 path: integral lambda_x / rho_vote and |energies| < 2^25
    const double lx = d.lambda_x, rv = d.rho_vote;
    const bool use_int = SP > 0 && lx == floor(lx) && rv == floor(rv) && lx < 1e6 && rv < 1e6 &&
                         (double)nrows * (rv * (double)d.aux[f].votes + 5.0 * lx) < 33554432.0;
    // int path: energies are stored x16 (< 2^29), so a stage's keys need no multiply
    const int nrv_i = use_int ? -16 * (int)rv : 0;
    if (threadIdx.x < 10) {  // sentinels: states outside [0, C) never win
        const int k = threadIdx.x < 5 ? (int)threadIdx.x - 5 : C + (int)threadIdx.x - 5;
        if (use_int) {
            ((int*)prev)[k] = 1 << 30;
            ((int*)cur)[k] = 1 << 30;
        } else {
            prev[k] = __longlong_as_double(0x7ff0000000000000LL);
            cur[k] = __longlong_as_double(0x7ff0000000000000LL);
        }
    }
    int my_votes = 0;  // every row of [v_top, v_max] enters the band exactly once
    for (int e = groff[v_top] + threadIdx.x; e < groff[H]; e += blockDim.x)
        my_votes += (staged ? s_vcol[e - e_first] != 0xffff : ecol[e] != kSkipCol);
    // Invariant at stage stg: cnt{stg & 1} holds band(stg) (read by the DP),
    // the other buffer holds band(stg - 1) and is slid to band(stg + 1) during
    // the same phase, so one barrier per stage covers both.
    int tm1 = v_max + 1, bm1 = v_max, t0b, b0b;  // band(stg - 1) (empty before 0), band(stg)
    band(0, t0b, b0b);
    slide(cnt0, tm1, bm1, t0b, b0b);
    __syncthreads();
#ifdef LK_VANISH_PROF
    const long long t1 = clock64();
#endif
    if (SP > 0 && use_int && !d.hooks) {
        // The product loop (int keys, no hooks), with the per-stage work cut
        // to the DP itself: the offsets' key constants in registers, the
        // thread's window / counts / choice row as running pointers, stage 0
        // peeled, no per-state bound test for threads whose states are all
        // inside [0, C). Same operations per state as upath_stage<SP, true>.
        constexpr int S = SP > 0 ? SP : 1;
        int* pv = (int*)prev;
        int* cu = (int*)cur;
        const int s0 = threadIdx.x * S;
        const bool act = s0 < C, full = s0 + S <= C;
        // the band slide goes to a warp without states when there is one (the
        // DP warps then issue only their DP), else to warp 0
        const int slide_warp = ((NT / 32 - 1) * 32) * S >= C ? NT / 32 - 1 : 0;
        int uk[11];
#pragma unroll
        for (int oi = 0; oi < 11; ++oi) uk[oi] = d.upk[oi];
        for (int c = threadIdx.x; c < C; c += blockDim.x) pv[c] = nrv_i * cnt0[c];  // stage 0
        if (nrows > 1) {  // cnt1: band(-1) (empty) -> band(1)
            int t1b, b1b;
            band(1, t1b, b1b);
            slide(cnt1, tm1, bm1, t1b, b1b);
            tm1 = t0b;
            bm1 = b0b;
            t0b = t1b;
            b0b = b1b;
        }
        __syncthreads();
        int8_t* ch = choice + C + s0;  // stage 1's choice row
        for (int stg = 1; stg < nrows; ++stg) {
            const int* cn = ((stg & 1) ? cnt1 : cnt0) + s0;
            if (act) {
                int w16[S + 10];
                const int* pw = pv + s0 - 5;  // 5 sentinels on each side of the rows
#pragma unroll
                for (int k = 0; k < S + 10; ++k) w16[k] = pw[k];
#pragma unroll
                for (int j = 0; j < S; ++j) {
                    if (!full && s0 + j >= C) break;
                    int key[11];
#pragma unroll
                    for (int oi = 0; oi < 11; ++oi) key[oi] = w16[j + 5 + upath_off(oi)] + uk[oi];
                    const int m0 = __vimin3_s32(key[0], key[1], key[2]);
                    const int m1 = __vimin3_s32(key[3], key[4], key[5]);
                    const int m2 = __vimin3_s32(key[6], key[7], key[8]);
                    const int best = __vimin3_s32(__vimin3_s32(m0, m1, m2), key[9], key[10]);
                    cu[s0 + j] = (best & ~15) + nrv_i * cn[j];
                    ch[j] = (int8_t)(best & 15);
                }
            }
            // warp 0 alone slides the other buffer, band(stg - 1) -> band(stg + 1)
            // (a row holds a few dozen votes: one or two lane strides), so the
            // other warps issue only their DP
            if (stg + 1 < nrows && (int)(threadIdx.x >> 5) == slide_warp) {
                int t1b, b1b;
                band(stg + 1, t1b, b1b);
                int* cb = (stg & 1) ? cnt0 : cnt1;
                auto wslide = [&](int e0, int e1, int dlt) {
                    for (int e = e0 + (int)(threadIdx.x & 31); e < e1; e += 32) {
                        const int c = staged ? (int)s_vcol[e - e_first]
                                             : (ecol[e] == kSkipCol ? 0xffff : ecol[e] - d.ext_lo);
                        if (c != 0xffff) atomicAdd(&cb[c], dlt);
                    }
                };
                if (t1b < tm1) wslide(roff[t1b], roff[tm1], 1);             // rows entering
                if (b1b < bm1) wslide(roff[b1b + 1], roff[bm1 + 1], -1);    // rows leaving
                tm1 = t0b;
                bm1 = b0b;
                t0b = t1b;
                b0b = b1b;
            }
            __syncthreads();
            int* t = pv;
            pv = cu;
            cu = t;
            ch += C;
        }
        prev = (double*)pv;  // the last stage's energies (read below)
    } else
    for (int stg = 0; stg < nrows; ++stg) {
#ifdef LK_VANISH_PROF
        const long long tb = clock64();
#endif
        const int v = v_max - stg;
        const int* cnt = (stg & 1) ? cnt1 : cnt0;
        if (d.hooks) {
            double* arow = d.acc + ((size_t)f * H + (v - v_top)) * C;
            for (int c = threadIdx.x; c < C; c += blockDim.x) arow[c] = nrv * cnt[c];
        }
        if (stg == 0) {
            if (use_int)
                for (int c = threadIdx.x; c < C; c += blockDim.x) ((int*)prev)[c] = nrv_i * cnt[c];
            else
                for (int c = threadIdx.x; c < C; c += blockDim.x) prev[c] = nrv * cnt[c];
        } else if (SP > 0) {
            int8_t* ch = choice + (size_t)stg * C;
            if (use_int)
                upath_stage<(SP > 0 ? SP : 1), true>(d, prev, cur, cnt, ch, C, nrv, nrv_i);
            else
                upath_stage<(SP > 0 ? SP : 1), false>(d, prev, cur, cnt, ch, C, nrv, nrv_i);
        } else {
            int8_t* ch = choice + (size_t)stg * C;
            for (int s = threadIdx.x; s < C; s += blockDim.x) {
                double best = __longlong_as_double(0x7ff0000000000000LL);
                int boi = 0;
#pragma unroll
                for (int o = 0; o < 11; ++o) {
                    const int ps = s + upath_off(o);
                    if (ps < 0 || ps >= C) continue;
                    const double e = prev[ps] + d.upen[o];
                    if (e < best) {
                        best = e;
                        boi = o;
                    }
                }
                cur[s] = best + nrv * cnt[s];
                ch[s] = (int8_t)boi;
            }
        }
        if (stg + 1 < nrows) {  // other buffer: band(stg - 1) -> band(stg + 1)
            int t1b, b1b;
            band(stg + 1, t1b, b1b);
            slide((stg & 1) ? cnt0 : cnt1, tm1, bm1, t1b, b1b);
            tm1 = t0b;
            bm1 = b0b;
            t0b = t1b;
            b0b = b1b;
        }
        __syncthreads();
#ifdef LK_VANISH_PROF
        t_dp += clock64() - tb;
#endif
        if (stg > 0) {
            double* t = prev;
            prev = cur;
            cur = t;
        }
    }
    for (int o = 16; o; o >>= 1) my_votes += __shfl_xor_sync(0xffffffffu, my_votes, o);
    if ((threadIdx.x & 31) == 0 && my_votes) atomicAdd(&s_votes, my_votes);
    double mv = __longlong_as_double(0x7ff0000000000000LL);
    int mi = 0x7fffffff;
    for (int s = threadIdx.x; s < C; s += blockDim.x) {
        const double e = use_int ? (double)(((const int*)prev)[s] >> 4) : prev[s];
        if (e < mv) {
            mv = e;
            mi = s;
        }
    }
#ifdef LK_VANISH_PROF
    const long long t2 = clock64();
#endif
    const int term = block_argmin(mv, mi, sv, si);
    const double energy = use_int ? (double)(((const int*)prev)[term] >> 4) : prev[term];
    // backtrack (dp.hpp:67-71) in windows of BT_CHUNK stages staged in smem
    int p = term;
    if (threadIdx.x == 0) {
        px[nrows - 1] = d.ext_lo + p;
        pv[nrows - 1] = v_max - (nrows - 1);
    }
    const int span = 2 * BT_SPAN + 1;
    for (int hi = nrows - 1; hi > 0; hi -= BT_CHUNK) {
        const int lo = max(1, hi - BT_CHUNK + 1);  // stages lo..hi are read
        const int c0 = p - BT_SPAN;
        __syncthreads();
        {  // U independent loads in flight per thread before the stores
            constexpr int U = 8;
            const int total = (hi - lo + 1) * span;
            for (int i0 = threadIdx.x; i0 < total; i0 += U * blockDim.x) {
                int8_t w[U];
#pragma unroll
                for (int u = 0; u < U; ++u) {
                    const int i = i0 + u * blockDim.x;
                    const int r = i / span, c = c0 + (i - r * span);
                    w[u] = (i < total && c >= 0 && c < C) ? choice[(size_t)(lo + r) * C + c] : 0;
                }
#pragma unroll
                for (int u = 0; u < U; ++u)
                    if (i0 + u * blockDim.x < total) win[i0 + u * blockDim.x] = w[u];
            }
        }
        __syncthreads();
        if (threadIdx.x == 0) {
            for (int stg = hi; stg >= lo; --stg) {
                p += upath_off(win[(stg - lo) * span + (p - c0)]);
                px[stg - 1] = d.ext_lo + p;
                pv[stg - 1] = v_max - (stg - 1);
            }
            si[0] = p;
        }
        __syncthreads();
        p = si[0];
    }
    __syncthreads();
    int32_t* up = d.upath + (size_t)f * H * 2;
    for (int i = threadIdx.x; i < nrows; i += blockDim.x) {
        up[2 * i] = px[i];
        up[2 * i + 1] = pv[i];
    }
    if (threadIdx.x == 0) {
        rep.upath_energy = energy;
#ifdef LK_VANISH_PROF
        rep.gamma_kappa = (double)(t1 - t0);
        rep.gamma_v_normalizer = (double)t_band;
        rep.gamma_inlier_fraction = (double)t_dp;
        rep.gamma[0] = (double)(t2 - t1);
        rep.gamma[1] = (double)(clock64() - t2);
#endif
        rep.upath_has_evidence = s_votes > 0;
        if (s_votes == 0) fail_frame(d, f, 11, LK_MSG_NO_EDGE_EVIDENCE);  // pipeline.hpp:238-239
    }
}


// =====================================================================
// K4b  ransac_gamma (vanish.hpp:253-270) on the u-path points, vpx_profile
// (:276-281), then the w_g edge weights of build_m0 (lanes.hpp:35-44).
// One CTA per frame; warp 0 runs the RANSAC.
// =====================================================================
__global__ void __launch_bounds__(32 * GAMMA_NW, 2) k_gamma_fit(Dev d) {
    extern __shared__ int sh_g[];
    const int f = blockIdx.x;
    if (frame_failed(d, f)) return;
    const int H = d.H;
    lk_frame_report& rep = d.rep[f];
    const int v_top = (int)rep.horizon, v_max = H - 1;
    const int nrows = v_max - v_top + 1;
    constexpr int NW = GAMMA_NW;  // speculative RANSAC iterations per round, one warp each
    int* px = sh_g;
    int* pv = px + H;
    int* bufs[NW + 2];
    for (int b = 0; b < NW + 2; ++b) bufs[b] = pv + H + b * H;
    double* tbuf = align8(pv + H + (NW + 2) * H);
    // the draws of every iteration staged on chip (a round's first load is
    // then a shared-memory read, not an L2 round trip)
    uint64_t* s_rng = reinterpret_cast<uint64_t*>(tbuf + 6 * H);
    for (int i = threadIdx.x; i < d.max_iter * 5; i += blockDim.x) s_rng[i] = d.rng[i];
    __shared__ RansacState st;
    const int32_t* up = d.upath + (size_t)f * H * 2;
    for (int i = threadIdx.x; i < nrows; i += blockDim.x) {
        px[i] = up[2 * i];
        pv[i] = up[2 * i + 1];
    }
    uint8_t* wnz = d.wg_nz + (size_t)f * d.m_nty * d.m_ntx;  // marked after w_g below
    for (int i = threadIdx.x; i < d.m_nty * d.m_ntx; i += blockDim.x) wnz[i] = 0;
    __syncthreads();
#ifdef LK_GAMMA_PROF
    const long long t0 = clock64();
#endif
    block_ransac<5, NW>(px, pv, nrows, d.tr_x, d.eps_x, d.max_iter, s_rng, bufs, tbuf, st);
#ifdef LK_GAMMA_PROF
    const long long t1 = clock64();
#endif
    if (st.msg) {  // ransac_trim threw: the report keeps its defaults (pipeline.hpp:245-251)
        if (threadIdx.x == 0) fail_frame(d, f, 11, st.msg);
        return;
    }
    const double g0 = st.model[0], g1 = st.model[1], g2 = st.model[2], g3 = st.model[3],
                 g4 = st.model[4];
    double* vpx = d.vpx + (size_t)f * H;
    for (int v = threadIdx.x; v < H; v += blockDim.x) {
        const double vv = (double)v;
        vpx[v] = g0 + vv * (g1 + vv * (g2 + vv * (g3 + vv * g4)));
    }
    for (int i = threadIdx.x; i < st.n_inl; i += blockDim.x) {
        const int id = st.inl[i];
        d.gamma_inl[((size_t)f * H + i) * 2] = px[id];
        d.gamma_inl[((size_t)f * H + i) * 2 + 1] = pv[id];
    }
    if (threadIdx.x == 0) {
#ifndef LK_VANISH_PROF
        for (int k = 0; k < 5; ++k) rep.gamma[k] = st.model[k];
        rep.gamma_kappa = 1.0;
        rep.gamma_v_normalizer = st.s;
#endif
        rep.gamma_iterations = st.iterations;
#ifndef LK_VANISH_PROF
        rep.gamma_inlier_fraction = st.fraction;
#endif
        rep.gamma_degraded = st.degraded;
        rep.gamma_inlier_count = st.n_inl;
    }
    __syncthreads();
    // w_g per edge: k_wg (all frames' edges in parallel)
#ifdef LK_GAMMA_PROF
    __syncthreads();
    if (threadIdx.x == 0) {
        rep.gamma_kappa = (double)(st.t_loop - t0);
        rep.gamma_v_normalizer = (double)(t1 - st.t_loop);
        rep.gamma_inlier_fraction = (double)(clock64() - t1);
        rep.beta[0] = (double)st.t_fit;
        rep.beta[1] = (double)st.t_cls;
        rep.beta[2] = (double)st.t_commit;
        rep.vpath_energy = (double)st.rounds;
    }
#endif
}

// Per edge: theta = atan2(gy, gx) (sobel_gradients, preprocess.hpp:85-87; it
// feeds only w_g and the EDGES hook) and w_g (build_m0's weight,
// lanes.hpp:35-44) after k_gamma_fit has written V_px. Grid (X, frames),
// threads stride over the frame's edges. Also
// marks the m0/m1 tiles whose w_g window (k_m0_m1: rows v0-1-vs .. v0+th+vs,
// cols u0-1-nu .. u0+M_TW+nu) holds a non-zero w_g (k_gamma_fit zeroed them).
__global__ void __launch_bounds__(256) k_wg(Dev d) {
    const int f = blockIdx.y;
    const lk_frame_report& rep = d.rep[f];
    // edges exist once stage 10 has passed; a stage-11 failure still exports them
    if (rep.status != 0 && rep.failed_stage <= 10) return;
    const bool fit = rep.status == 0;
    const int H = d.H, v_top = (int)d.rep[f].horizon, v_max = H - 1;
    const double* vpx = d.vpx + (size_t)f * H;
    const double* vpy = d.vpy + (size_t)f * H;
    uint8_t* wnz = d.wg_nz + (size_t)f * d.m_nty * d.m_ntx;
    const int n_edges = d.row_off[(size_t)f * (H + 1) + H];
    const size_t eb = (size_t)f * d.px;
    unsigned n_unc = 0;
    double wmax = 0.0;
    for (int e = blockIdx.x * blockDim.x + threadIdx.x; e < n_edges; e += gridDim.x * blockDim.x) {
        const int uv = d.e_uv[eb + e];
        const int u = uv & 0xffff, v = uv >> 16;
        const double gx = d.e_gx[eb + e];
        double th = atan2(d.e_gy[eb + e], gx);  // sobel_gradients' theta (preprocess.hpp:85-87)
        if (th <= -kPi) th = kPi;
        d.e_th[eb + e] = th;
        if (!fit) continue;
        double wg = 0.0;
        if (v >= v_top && v <= v_max) {
            const double dx = vpx[v] - (double)u;
            const double dy = vpy[v] - (double)v;
            if (!(fabs(dx) < 1e-12 && fabs(dy) < 1e-12)) {
                const double theta_ray = atan2(dy, dx);
                const double theta_tangent = th + kPi / 2;
                bool unc;
                wg = gx * piecewise_weight(theta_tangent, theta_ray, d.sigma_g, &unc);
                n_unc += unc;
            }
        }
        wmax = fmax(wmax, fabs(wg));
        d.e_wg[eb + e] = wg;
        if (wg != 0.0) {
            const int th = 1 << d.m_tile_shift;
            const int ax = u - M_TW - d.nu, ay = v - th - d.varsigma;  // first tiles: ceil(a / size)
            const int tx0 = ax > 0 ? (ax + M_TW - 1) / M_TW : 0, tx1 = min(d.m_ntx - 1, (u + 1 + d.nu) / M_TW);
            const int ty0 = ay > 0 ? (ay + th - 1) / th : 0, ty1 = min(d.m_nty - 1, (v + 1 + d.varsigma) / th);
            for (int ty = ty0; ty <= ty1; ++ty)
                for (int tx = tx0; tx <= tx1; ++tx) wnz[ty * d.m_ntx + tx] = 1;
        }
    }
    // certificate inputs (k_select): uncertain gates and the largest |w_g|
    for (int o = 16; o; o >>= 1) {
        n_unc += __shfl_xor_sync(0xffffffffu, n_unc, o);
        wmax = fmax(wmax, __shfl_xor_sync(0xffffffffu, wmax, o));
    }
    if ((threadIdx.x & 31) == 0) {
        if (n_unc) atomicAdd(&d.aux[f].uncertain_gates, n_unc);
        if (wmax > 0.0) atomicMax(&d.aux[f].max_wg, (unsigned long long)__double_as_longlong(wmax));
    }
}

// =====================================================================
// K5a  build_m0 (lanes.hpp:46-60) + build_m1 (:67-76) + the exponent
// histogram of |m1| over the road rows for the auto threshold (:182-193).
// Tile M_TW x M_TH; w_g scattered from the row-ordered edge list into a
// zeroed shared tile; the box sum keeps the y-major / x-minor order (adding
// the zeros the reference adds is exact, so the order is all that matters).
// =====================================================================

__global__ void __launch_bounds__(256) k_m0_m1(Dev d, int tile_h, int want_hist) {
    extern __shared__ double sh5[];
    __shared__ unsigned s_live;
    const int f = blockIdx.y;
    if (d.rep[f].status != 0) return;
    if (d.W < 3 || d.H < 3) {  // lanes.hpp:68 (stage 10 already rejects this)
        if (blockIdx.x == 0 && threadIdx.x == 0) fail_frame(d, f, 12, LK_MSG_M1_TOO_SMALL);
        return;
    }
    const int v_top = (int)d.rep[f].horizon;
    // The CTA's tiles t = blockIdx.x + k gridDim.x (k < 32; 8 at launch): their k_wg flags
    // are loaded at once (one latency), so the many all-zero tiles cost a bit
    // test each instead of a CTA; their zero counts go out in one atomic.
    const int ntile = d.m_nty * d.m_ntx;
    if (threadIdx.x < 32) {
        const int t = blockIdx.x + threadIdx.x * gridDim.x;
        const unsigned b = __ballot_sync(0xffffffffu, t < ntile && d.wg_nz[(size_t)f * ntile + t]);
        if (threadIdx.x == 0) s_live = b;
    }
    __syncthreads();
    const unsigned live_mask = s_live;
    unsigned long long zcount = 0;  // thread 0: road-row pixels of the all-zero tiles
    for (int kt = 0, t = blockIdx.x; t < ntile; ++kt, t += gridDim.x) {
    const int nonzero = (live_mask >> kt) & 1;
    const int tx = t % d.m_ntx, ty = t / d.m_ntx;
    const int W = d.W, H = d.H, nu = d.nu, vs = d.varsigma;
    const int u0 = tx * M_TW, v0 = ty * tile_h;
    const int v_max = H - 1;
    // w_g is zero above v_top, so m0 vanishes on rows < v_top - vs and m1 on
    // rows < v_top - vs - 1: without hooks those rows are skipped (zero).
    const int first_row = d.hooks ? 0 : max(0, v_top - vs - 1);
    if (v0 + tile_h <= first_row) continue;
    if (d.hooks && v0 + tile_h <= v_top - vs - 1) {
        for (int i = threadIdx.x; i < tile_h * M_TW; i += blockDim.x) {
            const int v = v0 + i / M_TW, u = u0 + i % M_TW;
            if (v >= H || u >= W) continue;
            const size_t gi = (size_t)f * d.px + (size_t)v * W + u;
            d.m1[gi] = 0.0;
            d.m0[gi] = 0.0;
        }
        continue;
    }
    // wg region rows [v0-1-vs, v0+tile_h+vs], cols [u0-1-nu, u0+M_TW+nu]
    const int gr0 = v0 - 1 - vs, gc0 = u0 - 1 - nu;
    const int GH = tile_h + 2 + 2 * vs, GW = M_TW + 2 + 2 * nu;
    // m0 region rows [v0-1, v0+tile_h], cols [u0-1, u0+M_TW]
    const int MH = tile_h + 2, MW = M_TW + 2;
    double* gw = sh5;
    double* m0 = gw + GH * GW;
    unsigned int* hist = (unsigned int*)(m0 + MH * MW);
    const int32_t* roff = d.row_off + (size_t)f * (H + 1);
    const size_t eb = (size_t)f * d.px;
    const int r_lo = max(max(gr0, 0), v_top), r_hi = min(gr0 + GH - 1, v_max);
    // A tile without a non-zero w_g in reach has m0 = m1 = +0 everywhere: it
    // is flagged instead of written (readers of m1 consult the flag), so such
    // tiles (most of them) skip the staging entirely.
    if (nonzero) {
        if ((GH * GW & 1) == 0)
            for (int i = threadIdx.x; i < GH * GW / 2; i += blockDim.x)
                reinterpret_cast<double2*>(gw)[i] = make_double2(0.0, 0.0);
        else
            for (int i = threadIdx.x; i < GH * GW; i += blockDim.x) gw[i] = 0.0;
        if (want_hist)
            for (int i = threadIdx.x; i < 2048; i += blockDim.x) hist[i] = 0;
        __syncthreads();
        for (int e = roff[r_lo] + threadIdx.x; e < roff[r_hi + 1]; e += blockDim.x) {
            const int uv = d.e_uv[eb + e];
            const int u = uv & 0xffff, v = uv >> 16;
            if (u >= gc0 && u < gc0 + GW) gw[(v - gr0) * GW + (u - gc0)] = d.e_wg[eb + e];
        }
        __syncthreads();
    }
    const int t_lo = max(0, v_top), t_hi = min(H - 1, v_max);
    if (threadIdx.x == 0) d.m1_nz[(size_t)f * ntile + t] = (uint8_t)nonzero;
    if (!nonzero) {
        if (d.hooks)
            for (int i = threadIdx.x; i < tile_h * M_TW; i += blockDim.x) {
                const int v = v0 + i / M_TW, u = u0 + i % M_TW;
                if (v >= H || u >= W) continue;
                const size_t gi = (size_t)f * d.px + (size_t)v * W + u;
                d.m1[gi] = 0.0;
                d.m0[gi] = 0.0;
            }
        if (want_hist && threadIdx.x == 0) {
            const int rows = max(0, min(v0 + tile_h - 1, t_hi) - max(v0, t_lo) + 1);
            zcount += (unsigned long long)rows * min(M_TW, W - u0);
        }
        continue;
    }
    // box sum, y-major / x-minor (lanes.hpp:46-60). Positions outside the image
    // hold zeros in gw: adding +-0.0 to a running sum that starts at +0.0 never
    // changes it, so summing them instead of skipping is bit-identical.
    if (nu == 1 && (GW & 1) == 0) {
        // 3-wide window: a thread sums 2 consecutive outputs of a row, each
        // in its own y-major / x-minor order, from two 16-byte loads of the 4
        // columns they span. Consecutive lanes' loads are then contiguous (16 B
        // apart): with 4 outputs per thread they were 32 B apart and every
        // load took twice the shared-memory wavefronts (ncu: 25 M conflicts).
        // A thread also covers R consecutive rows: each staged row it loads
        // feeds every one of its R x Q outputs whose window holds it (rows
        // r .. r + 2 vs in increasing order, columns x-minor, as before), so
        // R outputs share their overlapping rows' loads.
        constexpr int Q = 2, R = 6;
        const int per_row = (MW + Q - 1) / Q;
        const int ngrp = (MH + R - 1) / R;
        for (int i = threadIdx.x; i < ngrp * per_row; i += blockDim.x) {
            const int rg = i / per_row, c = (i - rg * per_row) * Q;
            const int r0 = rg * R, rn = min(R, MH - r0);
            const double2* g0 = reinterpret_cast<const double2*>(gw + r0 * GW + c);  // 16-byte aligned
            double s[R][Q];
#pragma unroll
            for (int rr = 0; rr < R; ++rr) s[rr][0] = s[rr][1] = 0.0;
            for (int y = 0; y < rn + 2 * vs; ++y) {
                const double2 a = g0[0], b = g0[1];  // columns c .. c+3 of staged row r0 + y
                const double g[4] = {a.x, a.y, b.x, b.y};
#pragma unroll
                for (int rr = 0; rr < R; ++rr) {
                    const int dy = y - rr;  // the window row of output row r0 + rr
                    if (dy >= 0 && dy <= 2 * vs) {
#pragma unroll
                        for (int k = 0; k < Q; ++k) {
                            s[rr][k] += g[k];
                            s[rr][k] += g[k + 1];
                            s[rr][k] += g[k + 2];
                        }
                    }
                }
                g0 += GW / 2;
            }
#pragma unroll
            for (int rr = 0; rr < R; ++rr)
#pragma unroll
                for (int k = 0; k < Q; ++k)
                    if (rr < rn && c + k < MW) m0[(r0 + rr) * MW + c + k] = s[rr][k];
        }
    } else {
        for (int i = threadIdx.x; i < MH * MW; i += blockDim.x) {
            const int r = i / MW, c = i - r * MW;
            const double* g0 = gw + r * GW + c;  // row v-vs, col u-nu
            double s = 0.0;
            for (int y = 0; y <= 2 * vs; ++y)
                for (int x = 0; x <= 2 * nu; ++x) s += g0[y * GW + x];
            m0[i] = s;
        }
    }
    __syncthreads();
    const int lane = threadIdx.x & 31;
    for (int i = threadIdx.x; i < tile_h * M_TW; i += blockDim.x) {
        const int r = i / M_TW, c = i - r * M_TW;
        const int v = v0 + r, u = u0 + c;
        const bool live = v < H && u < W && v >= first_row;
        double m1 = 0.0;
        if (live && v >= 1 && v < H - 1 && u >= 1 && u < W - 1) {
            const double* a = m0 + r * MW + c;  // row v-1, col u-1
            const double* b = a + MW;            // row v
            const double* cc = b + MW;           // row v+1
            m1 = (a[2] - a[0]) + 2 * (b[2] - b[0]) + (cc[2] - cc[0]);
        }
        if (live) {
            const size_t gi = (size_t)f * d.px + (size_t)v * W + u;
            d.m1[gi] = m1;
            if (d.hooks) d.m0[gi] = m0[(r + 1) * MW + c + 1];
        }
        if (want_hist) {
            const bool in = live && v >= t_lo && v <= t_hi;
            const unsigned bin = (unsigned)((unsigned long long)__double_as_longlong(fabs(m1)) >> 52);
            const unsigned zb = __ballot_sync(__activemask(), in && bin == 0);
            const unsigned z0 = __ballot_sync(__activemask(), in && m1 == 0.0);
            if (lane == 0 && zb) atomicAdd(&hist[0], (unsigned)__popc(zb));
            if (lane == 0 && z0) atomicAdd(&d.aux[f].p99_zeros, (unsigned long long)__popc(z0));
            if (in && bin != 0) atomicAdd(&hist[bin], 1u);
        }
    }
    if (want_hist) {
        __syncthreads();
        unsigned int* gh = d.p99hist + (size_t)f * 2048;
        for (int i = threadIdx.x; i < 2048; i += blockDim.x)
            if (hist[i]) atomicAdd(&gh[i], hist[i]);
    }
    __syncthreads();  // the next tile restages gw / m0 / hist
    }
    if (want_hist && threadIdx.x == 0 && zcount) {
        atomicAdd(&d.p99hist[(size_t)f * 2048], (unsigned)zcount);
        atomicAdd(&d.aux[f].p99_zeros, zcount);
    }
}

// =====================================================================
// auto_lane_threshold (lanes.hpp:182-193): the k-th smallest |m1|,
// k = floor(0.99*(n-1)), selected EXACTLY on the IEEE bit patterns
// (non-negative doubles order like their bits). Level 1: exponent histogram
// (fused into K5a) -> bucket; level 2: histogram of the next 12 bits inside
// that bucket -> sub-bucket; the few values sharing those 24 leading bits are
// gathered and the remaining 40 bits resolved by MSB radix select.
// =====================================================================
__device__ __forceinline__ unsigned long long p99_n(const Dev& d, int f, int* t_lo) {
    const int v_top = (int)d.rep[f].horizon, v_max = d.H - 1;
    *t_lo = max(0, v_top);
    const int t_hi = min(d.H - 1, v_max);
    return (unsigned long long)(t_hi - *t_lo + 1) * d.W;
}

// Picks the bin holding rank `rank` among nb bins (blockDim = 256).
// One warp: the first index i of a[0..n) (n <= 256) whose running sum
// exceeds rank (n - 1 if none) and the sum of a[0..i), in every lane: the
// sequential scan `for (i < n - 1) { if (run + a[i] > rank) break; run += a[i]; }`
// as 8-entry lane sums, a warp prefix sum and one lane's scan of its 8.
template <class T>
__device__ __forceinline__ void warp_find(const T* a, int n, unsigned long long rank, int& idx,
                                          unsigned long long& before) {
    const int lane = threadIdx.x & 31;
    unsigned long long sum = 0;
#pragma unroll
    for (int j = 0; j < 8; ++j)
        if (8 * lane + j < n) sum += a[8 * lane + j];
    unsigned long long inc = sum;
    for (int o = 1; o < 32; o <<= 1) {
        const unsigned long long t = __shfl_up_sync(0xffffffffu, inc, o);
        if (lane >= o) inc += t;
    }
    const unsigned hit = __ballot_sync(0xffffffffu, inc > rank);
    const int L = hit ? __ffs(hit) - 1 : (n - 1) >> 3;
    int i = 0;
    unsigned long long run = 0;
    if (lane == L) {
        run = inc - sum;
        i = 8 * L;
        for (const int last = min(8 * L + 8, n) - 1; i < last; ++i) {
            if (run + a[i] > rank) break;
            run += a[i];
        }
    }
    idx = __shfl_sync(0xffffffffu, i, L);
    before = __shfl_sync(0xffffffffu, run, L);
}

__device__ void pick_bin(const unsigned int* h, int nb, unsigned long long rank, int* bin_out,
                         unsigned long long* rank_out) {
    __shared__ unsigned long long s_part[256];
    const int per = nb / 256;
    unsigned long long mine = 0;
    for (int b = 0; b < per; ++b) mine += h[threadIdx.x * per + b];
    s_part[threadIdx.x] = mine;
    __syncthreads();
    if (threadIdx.x < 32) {
        int t;
        unsigned long long run;
        warp_find(s_part, 256, rank, t, run);
        if (threadIdx.x != 0) return;
        int b = t * per;
        for (; b < (t + 1) * per - 1; ++b) {
            if (run + h[b] > rank) break;
            run += h[b];
        }
        *bin_out = b;
        *rank_out = rank - run;
    }
}

__global__ void __launch_bounds__(256) k_p99_bucket(Dev d) {
    const int f = blockIdx.x;
    if (frame_failed(d, f)) return;
    int t_lo;
    const unsigned long long n = p99_n(d, f, &t_lo);
    const unsigned long long k = (unsigned long long)floor(0.99 * (double)(n - 1));
    int b;
    unsigned long long r;
    pick_bin(d.p99hist + (size_t)f * 2048, 2048, k, &b, &r);
    if (threadIdx.x == 0) {
        d.aux[f].p99_bucket = b;
        d.aux[f].p99_rank = r;
        d.aux[f].p99_cands = 0;
        // +0 is the smallest |m1|: a rank among the zeros settles it (common when
        // fewer than 1% of the road pixels respond, e.g. 2560x1024 with lambda_g 1)
        const bool zero = b == 0 && r < d.aux[f].p99_zeros;
        d.aux[f].p99_done = zero;
        // a small bucket is gathered directly; a large one is narrowed first by
        // a second histogram level (12 more bits)
        d.aux[f].p99_level2 = d.p99hist[(size_t)f * 2048 + b] > d.p99_l2_min;
        d.aux[f].p99_bucket2 = 0;
        if (zero) {
            const int v_top = (int)d.rep[f].horizon, v_max = d.H - 1;
            const double tr = -0.15 * (double)(v_max - v_top + 1) * 0.0;
            d.aux[f].tr = tr;
            d.rep[f].tr_lpv_used = tr;
        }
    }
}

// |m1| bits of road-row pixel i (unwritten tiles are +0).
// Visits |m1| of the threshold rows [t_lo, H-1] tile by tile (M_TW x tile_h,
// the k_m0_m1 tiling): fn(bits, live) per pixel, 32-bit index arithmetic.
// Tiles k_m0_m1 flagged all-zero are only visited when zeros matter
// (want_zero: the selection key is the zero bucket).
template <class Fn>
__device__ __forceinline__ void for_m1_rows(const Dev& d, int f, int t_lo, bool want_zero, Fn fn) {
    const int th = 1 << d.m_tile_shift, ty0 = t_lo >> d.m_tile_shift;
    const int ntile = (d.m_nty - ty0) * d.m_ntx;
    const uint8_t* nz = d.m1_nz + ((size_t)f * d.m_nty + ty0) * d.m_ntx;
    const double* m1 = d.m1 + (size_t)f * d.px;
    for (int t = blockIdx.x; t < ntile; t += gridDim.x) {
        const bool live = nz[t] != 0;
        if (!live && !want_zero) continue;
        const int ty = ty0 + t / d.m_ntx, tx = t % d.m_ntx;
        for (int p = threadIdx.x; p < th * M_TW; p += blockDim.x) {
            const int v = ty * th + (p >> 7), u = tx * M_TW + (p & (M_TW - 1));
            if (v < t_lo || v >= d.H || u >= d.W) continue;
            fn(live ? (unsigned long long)__double_as_longlong(fabs(m1[(size_t)v * d.W + u])) : 0ULL, live);
        }
    }
}

__global__ void __launch_bounds__(256) k_p99_hist2(Dev d) {
    const int f = blockIdx.y;
    if (frame_failed(d, f) || d.aux[f].p99_done || !d.aux[f].p99_level2) return;
    __shared__ unsigned int h[4096];
    for (int i = threadIdx.x; i < 4096; i += blockDim.x) h[i] = 0;
    __syncthreads();
    int t_lo;
    const size_t n = p99_n(d, f, &t_lo);
    const unsigned bucket = d.aux[f].p99_bucket;
    (void)n;
    for_m1_rows(d, f, t_lo, bucket == 0, [&](unsigned long long b, bool) {
        if ((b >> 52) == bucket) atomicAdd(&h[(b >> 40) & 0xfff], 1u);
    });
    __syncthreads();
    unsigned int* gh = d.p99hist2 + (size_t)f * 4096;
    for (int i = threadIdx.x; i < 4096; i += blockDim.x)
        if (h[i]) atomicAdd(&gh[i], h[i]);
}

__global__ void __launch_bounds__(256) k_p99_bucket2(Dev d) {
    const int f = blockIdx.x;
    if (frame_failed(d, f) || d.aux[f].p99_done || !d.aux[f].p99_level2) return;
    int b;
    unsigned long long r;
    pick_bin(d.p99hist2 + (size_t)f * 4096, 4096, d.aux[f].p99_rank, &b, &r);
    if (threadIdx.x == 0) {
        d.aux[f].p99_bucket2 = b;
        d.aux[f].p99_rank = r;
    }
}

__global__ void __launch_bounds__(256) k_p99_collect(Dev d) {
    const int f = blockIdx.y;
    if (frame_failed(d, f) || d.aux[f].p99_done) return;
    int t_lo;
    const size_t n = p99_n(d, f, &t_lo);
    const bool l2 = d.aux[f].p99_level2;
    const int ksh = l2 ? 40 : 52;  // leading bits fixed by the histogram level(s)
    const unsigned long long key = l2 ? ((unsigned long long)d.aux[f].p99_bucket << 12) |
                                            d.aux[f].p99_bucket2
                                      : (unsigned long long)d.aux[f].p99_bucket;
    unsigned long long* out = d.p99cand + (size_t)f * d.px;
    (void)n;
    // a zero can only be a candidate of key 0
    for_m1_rows(d, f, t_lo, key == 0, [&](unsigned long long b, bool) {
        const bool hit = (b >> ksh) == key;
        const unsigned act = __activemask();
        const unsigned bal = __ballot_sync(act, hit);
        if (!bal) return;
        const int lane = threadIdx.x & 31;
        const int leader = __ffs(bal) - 1;
        unsigned base = 0;
        if (lane == leader) base = atomicAdd(&d.aux[f].p99_cands, (unsigned)__popc(bal));
        base = __shfl_sync(act, base, leader);
        if (hit) out[base + __popc(bal & ((1u << lane) - 1u))] = b;
    });
}

__global__ void __launch_bounds__(256) k_p99_select(Dev d) {
    const int f = blockIdx.x;
    if (frame_failed(d, f) || d.aux[f].p99_done) return;
    __shared__ unsigned int hist[256];
    __shared__ unsigned long long s_prefix, s_rank;
    const unsigned ncand = d.aux[f].p99_cands;
    const unsigned long long* c = d.p99cand + (size_t)f * d.px;
    const bool l2 = d.aux[f].p99_level2;
    int bits_left = l2 ? 40 : 52;  // bits below the histogram-fixed prefix
    unsigned long long prefix = ((unsigned long long)d.aux[f].p99_bucket << 52) |
                                ((unsigned long long)d.aux[f].p99_bucket2 << 40);
    unsigned long long mask = ~0ULL << bits_left;
    unsigned long long rank = d.aux[f].p99_rank;
    while (bits_left > 0) {
        const int w = min(8, bits_left), sh = bits_left - w;
        const unsigned dm = (1u << w) - 1u;
        for (int i = threadIdx.x; i < 256; i += blockDim.x) hist[i] = 0;
        __syncthreads();
        for (unsigned i = threadIdx.x; i < ncand; i += blockDim.x) {
            const unsigned long long x = c[i];
            if ((x & mask) == prefix) atomicAdd(&hist[(x >> sh) & dm], 1u);
        }
        __syncthreads();
        if (threadIdx.x < 32) {
            int dg;
            unsigned long long run;
            warp_find(hist, (int)dm + 1, rank, dg, run);
            if (threadIdx.x == 0) {
                s_prefix = prefix | ((unsigned long long)dg << sh);
                s_rank = rank - run;
            }
        }
        __syncthreads();
        prefix = s_prefix;
        rank = s_rank;
        mask |= (unsigned long long)dm << sh;
        bits_left = sh;
        __syncthreads();
    }
    if (threadIdx.x == 0) {
        const double p99 = __longlong_as_double((long long)prefix);
        const int v_top = (int)d.rep[f].horizon, v_max = d.H - 1;
        const double tr = -0.15 * (double)(v_max - v_top + 1) * p99;
        d.aux[f].tr = tr;
        d.rep[f].tr_lpv_used = tr;
    }
}

// =====================================================================
// K5c  aggregate_energy (lanes.hpp:106-129) with lane_track (:83-96) fused:
// one thread per extended bottom column, the track recursion and the decayed
// m1 sum run together from the bottom row upward.
// =====================================================================
// One lane_track step (lanes.hpp:91-94): u' = ((vpx + v u) - vpy u) / denom,
// the quotient as RN(a y) + one Markstein correction (= IEEE a / denom, see
// k_energy) unless an operand is zero, non-finite or extreme.
__device__ __forceinline__ double track_step(const double4 rw, int v, double u) {
    const double a = rw.x + (double)v * u - rw.y * u;
    const double aa = fabs(a);
    if (aa >= 0x1p-500 && aa <= 0x1p500 && fabs(rw.z) <= 0x1p500) {
        const double q0 = __dmul_rn(a, rw.w);
        return __fma_rn(__fma_rn(-q0, rw.z, a), rw.w, q0);
    }
    return a / rw.z;
}

// LG1: lambda_g == 1 (the default, config.hpp:38): c + 1.0 * e is c + e exactly
template <bool LG1>
__global__ void __launch_bounds__(128) k_energy(Dev d) {
    extern __shared__ double4 sh_e4[];  // per row v: (vpx[v+1], vpy[v+1], denom, 1/denom)
    __shared__ int s_dead;
    const int f = blockIdx.y;
    if (frame_failed(d, f)) return;
    const int W = d.W, H = d.H;
    const int v_top = (int)d.rep[f].horizon, v_max = H - 1;
    const double* vpx = d.vpx + (size_t)f * H;
    const double* vpy = d.vpy + (size_t)f * H;
    uint8_t* s_nz = (uint8_t*)(sh_e4 + H);  // the frame's m1 tile flags
    // Every column divides by the same denom at row v, so 1/denom is
    // computed once per row; each quotient is then q0 = RN(a y), r = a - q0 b
    // (exact, FMA), q = RN(q0 + r y), which is the correctly rounded a / b
    // (Markstein; checked against IEEE division on 3e10 cases by
    // tools/markstein_check.cu). Zero, non-finite or extreme operands take the
    // IEEE division. The track of EVERY column stops at the same row: the
    // first v (going up) with |denom| < 0.5 (lanes.hpp:91), found once here.
    if (threadIdx.x == 0) s_dead = -1;
    __syncthreads();
    for (int v = v_top + threadIdx.x; v < v_max; v += blockDim.x) {
        const double py = vpy[v + 1];
        const double den = (double)(v + 1) - py;
        sh_e4[v] = make_double4(vpx[v + 1], py, den, 1.0 / den);
        if (fabs(den) < 0.5) atomicMax(&s_dead, v);
    }
    for (int i = threadIdx.x; i < d.m_nty * d.m_ntx; i += blockDim.x)
        s_nz[i] = d.m1_nz[(size_t)f * d.m_nty * d.m_ntx + i];
    __syncthreads();
    const int ci = blockIdx.x * blockDim.x + threadIdx.x;
    if (ci >= d.ext_cols) return;
    const double* m1 = d.m1 + (size_t)f * d.px;
    const double lg = d.lambda_g;
    const double w_hi = (double)W - 0.5;
    const int v_alive = max(v_top, s_dead + 1);  // rows v_alive..v_max carry the track
    const double u_bottom = (double)(d.ext_lo + ci);
    double u = u_bottom;
    double e = 0.0;
    bool touched = false;  // read a cell within reach of a w_g != 0 (m1 tile flag)
    // Chunks of EC rows: the track recursion (lane_track, lanes.hpp:83-96)
    // yields EC gather indices, the EC m1 loads are then all in flight
    // together, and the decayed sum consumes them in row order.
    constexpr int EC = 8;
    for (int vc = v_max; vc >= v_alive; vc -= EC) {
        int idx[EC];
#pragma unroll
        for (int k = 0; k < EC; ++k) {
            const int v = vc - k;
            idx[k] = -1;
            if (v < v_alive) continue;
            if (v < v_max) u = track_step(sh_e4[v], v, u);
            // llround(u) in [0, W)  <=>  -0.5 < u < W - 0.5 (NaN fails); then
            // llround = trunc(RN(u + 0.5)): the sum is exact or rounds within
            // its unit interval for every such u except 0.5 - 2^-54, whose sum
            // rounds up to 1.0 (llround gives 0). One instruction fewer than
            // trunc + (frac >= 0.5) on this issue-bound loop.
            if (u > -0.5 && u < w_hi) {
                const int r = (int)(u + 0.5) - (u == 0x1.fffffffffffffp-2);
                if (s_nz[(v >> d.m_tile_shift) * d.m_ntx + (r >> 7)]) idx[k] = v * W + r;  // < 2^31
            }
        }
        double c[EC];
#pragma unroll
        for (int k = 0; k < EC; ++k) {
            c[k] = idx[k] >= 0 ? m1[idx[k]] : 0.0;
            touched |= idx[k] >= 0;
        }
#pragma unroll
        for (int k = 0; k < EC; ++k)
            if (vc - k >= v_alive) e = LG1 ? c[k] + e : c[k] + lg * e;
    }
    // rows after the track stops contribute +0.0 (kept: 0 + (-0.0) is +0.0)
    for (int v = v_alive - 1; v >= v_top; --v) e = 0.0 + lg * e;
    d.energy[(size_t)f * d.ext_cols + ci] = e;
    d.e_touch[(size_t)f * d.ext_cols + ci] = touched;
    // lane_track's finite points (lanes.hpp:83-96), for k_select: NaN is
    // absorbing in track_step (every operation propagates it), so a non-NaN
    // final u means every step was finite; otherwise (rare) recount.
    int np = 1 + max(0, v_max - v_alive);
    if (isnan(u)) {
        np = 1;
        double w = u_bottom;
        for (int v = v_max - 1; v >= v_alive; --v) {
            w = track_step(sh_e4[v], v, w);
            np += !isnan(w);
        }
    }
    d.track_np[(size_t)f * d.ext_cols + ci] = np;
}

// =====================================================================
// Certificate of the lane decisions (lk_frame_report.uncertain). The only
// arithmetic that differs from the reference's is libdevice's atan2 / exp in
// theta and w_g (<= 2 ulp; glibc <= 1 ulp); every later sum runs in the
// reference's order. With the gates certain (k_wg: none within kGateEps of
// pi/6), |w_g - w_g,ref| <= kWgRel |w_g| (the gate distance moves by < 1e-14,
// exp's argument by < 1e-14, exp by <= 3 ulp), so over the m0 box and the m1
// Sobel |m1 - m1,ref| <= 8 (2 nu + 1)(2 varsigma + 1) kWgRel max|w_g| =: e1,
// an energy (sum of lambda_g^k m1 over the track rows) moves by <= e1 S_lambda
// when its track reads a cell within reach of a w_g != 0 (the m1 tile flags,
// e_touch) and not at all otherwise, and the auto threshold (-0.15 rows p99 of
// |m1|) by <= 0.15 rows e1. A strict comparison is certain when its margin
// exceeds the two operands' bounds; the count is the minima tests that are not
// certain, plus order pairs of certain candidates within min_sep whose
// energies are within their bounds (the greedy suppression could flip).
// =====================================================================
constexpr double kWgRel = 1e-12;

__device__ void select_certificate(const Dev& d, int f, const double* h, double tr,
                                   unsigned int* cbits) {
    __shared__ unsigned int s_unc;
    const int n = d.ext_cols, H = d.H, v_top = (int)d.rep[f].horizon;
    const int rows = H - v_top;
    const double lg = d.lambda_g;
    const double wmax = __longlong_as_double((long long)d.aux[f].max_wg);
    const double e1 = 8.0 * (2 * d.nu + 1) * (2 * d.varsigma + 1) * kWgRel * wmax;
    const double sl = lg == 1.0 ? (double)rows : (pow(lg, (double)rows) - 1.0) / (lg - 1.0);
    const double eh = e1 * fabs(sl) * 1.01;
    const double etr = isnan(d.tr_lpv) ? 0.15 * rows * e1 * 1.01 : 0.0;
    const uint8_t* touch = d.e_touch + (size_t)f * n;
    if (threadIdx.x == 0) s_unc = 0;
    for (int w = threadIdx.x; w < (n + 31) >> 5; w += blockDim.x) cbits[w] = 0;
    __syncthreads();
    // 3-valued a < b: 1 certain true, 0 certain false, 2 uncertain
    auto lt3 = [](double a, double ea, double b, double eb) {
        const double dd = b - a, m = ea + eb;
        if (m == 0.0) return dd > 0.0 ? 1 : 0;
        return dd > m ? 1 : dd <= -m ? 0 : 2;
    };
    unsigned unc = 0;
    for (int i = threadIdx.x; i < n; i += blockDim.x) {
        if (i < 1 || i + 1 >= n) continue;
        const double ei = touch[i] ? eh : 0.0;
        const int a = lt3(h[i], ei, h[i - 1], touch[i - 1] ? eh : 0.0);
        const int b = lt3(h[i], ei, h[i + 1], touch[i + 1] ? eh : 0.0);
        const int c = lt3(h[i], ei, tr, etr);
        const bool fals = a == 0 || b == 0 || c == 0;
        if (!fals && (a == 2 || b == 2 || c == 2)) ++unc;
        if (!fals && a == 1 && b == 1 && c == 1) atomicOr(&cbits[i >> 5], 1u << (i & 31));
    }
    __syncthreads();
    const int sep = d.min_lane_sep;
    for (int i = threadIdx.x; i < n; i += blockDim.x) {
        if (!((cbits[i >> 5] >> (i & 31)) & 1) || !touch[i]) continue;
        // the certain candidates j within min_sep: set bits of the window's words
        const int lo = max(0, i - sep + 1), hi = min(n - 1, i + sep - 1);
        for (int w = lo >> 5; w <= (hi >> 5); ++w) {
            unsigned int bits = cbits[w];
            if (w == (lo >> 5)) bits &= ~0u << (lo & 31);
            if (w == (hi >> 5)) bits &= ~0u >> (31 - (hi & 31));
            while (bits) {
                const int j = 32 * w + __ffs(bits) - 1;
                bits &= bits - 1;
                if (j != i && fabs(h[i] - h[j]) <= eh + (touch[j] ? eh : 0.0))
                    unc += j > i || !touch[j];  // each touched pair once
            }
        }
    }
    for (int o = 16; o; o >>= 1) unc += __shfl_xor_sync(0xffffffffu, unc, o);
    if ((threadIdx.x & 31) == 0 && unc) atomicAdd(&s_unc, unc);
    __syncthreads();
    if (threadIdx.x == 0) d.rep[f].uncertain = (int64_t)(s_unc + d.aux[f].uncertain_gates);
    __syncthreads();
}

// =====================================================================
// K5d  select_lanes (lanes.hpp:144-178): strict interior minima under the
// threshold, sorted by (energy, column) with a shared-memory bitonic sort,
// greedy min_sep suppression, then each kept lane's track length.
// =====================================================================
__global__ void __launch_bounds__(256) k_select(Dev d, int sort_cap) {
    extern __shared__ unsigned long long sh_keys[];  // [sort_cap] keys, [sort_cap] cols
    const int f = blockIdx.x;
    if (frame_failed(d, f)) return;
    int* cols = (int*)(sh_keys + sort_cap);
    __shared__ int s_n, s_kept;
    const int n = d.ext_cols;
    const double* h = d.energy + (size_t)f * n;
    const double tr = isnan(d.tr_lpv) ? d.aux[f].tr : d.tr_lpv;
    if (threadIdx.x == 0) {
        s_n = 0;
        if (!isnan(d.tr_lpv)) d.rep[f].tr_lpv_used = tr;
    }
    __syncthreads();
    for (int i = threadIdx.x; i < n; i += blockDim.x) {
        if (i >= 1 && i + 1 < n && h[i] < h[i - 1] && h[i] < h[i + 1] && h[i] < tr) {
            const int slot = atomicAdd(&s_n, 1);
            if (slot < sort_cap) {
                sh_keys[slot] = order_key(h[i]);
                cols[slot] = i;
            }
        }
    }
    __syncthreads();
    select_certificate(d, f, h, tr, (unsigned int*)(cols + sort_cap) + ((n + 31) >> 5));
    const int m = min(s_n, sort_cap);
    int p2 = 1;
    while (p2 < m) p2 <<= 1;
    for (int i = m + threadIdx.x; i < p2; i += blockDim.x) {
        sh_keys[i] = ~0ULL;
        cols[i] = 0x7fffffff;
    }
    __syncthreads();
    for (int k = 2; k <= p2; k <<= 1)
        for (int j = k >> 1; j > 0; j >>= 1) {
            for (int i = threadIdx.x; i < p2; i += blockDim.x) {
                const int l = i ^ j;
                if (l > i) {
                    const bool up = (i & k) == 0;
                    const bool gt = sh_keys[i] > sh_keys[l] ||
                                    (sh_keys[i] == sh_keys[l] && cols[i] > cols[l]);
                    if (gt == up) {
                        const unsigned long long tk = sh_keys[i];
                        sh_keys[i] = sh_keys[l];
                        sh_keys[l] = tk;
                        const int tc = cols[i];
                        cols[i] = cols[l];
                        cols[l] = tc;
                    }
                }
            }
            __syncthreads();
        }
    lk_lane* lanes = d.lanes + (size_t)f * d.lane_cap;
    // greedy suppression (lanes.hpp:158-166) against a bitmap of kept columns:
    // "some kept k with |i - k| < min_sep" is a test of the bits in
    // [i - min_sep + 1, i + min_sep - 1], in the same candidate order
    unsigned int* kbits = (unsigned int*)(cols + sort_cap);
    const int nwords = (n + 31) >> 5;
    for (int i = threadIdx.x; i < nwords; i += blockDim.x) kbits[i] = 0;
    __syncthreads();
    if (threadIdx.x < 32) {
        // warp 0 walks the candidates in order; the first 128 kept columns sit
        // in registers (4 per lane), so "some kept k with |i - k| < min_sep"
        // is one ballot instead of a scan of the bitmap words (which still
        // records every kept column and takes over beyond 128)
        const int lane = threadIdx.x;
        constexpr int KR = 4;
        int kc[KR];
#pragma unroll
        for (int r = 0; r < KR; ++r) kc[r] = INT_MIN / 2;
        int kept = 0;
        const int sep = d.min_lane_sep;
        for (int q = 0; q < m; ++q) {
            const int i = cols[q];
            bool close = false;
            if (sep > 0) {
                bool near = false;
#pragma unroll
                for (int r = 0; r < KR; ++r) near |= abs(i - kc[r]) < sep;
                close = __any_sync(0xffffffffu, near);
                if (!close && kept > 32 * KR) {  // kept columns beyond the registers
                    const int lo = max(0, i - sep + 1), hi = min(n - 1, i + sep - 1);
                    for (int w = lo >> 5; w <= (hi >> 5) && !close; ++w) {
                        unsigned int bits = kbits[w];
                        if (w == (lo >> 5)) bits &= ~0u << (lo & 31);
                        if (w == (hi >> 5)) bits &= ~0u >> (31 - (hi & 31));
                        close = bits != 0;
                    }
                }
            }
            if (close) continue;
            if (lane == 0) kbits[i >> 5] |= 1u << (i & 31);
            if (kept < 32 * KR && lane == (kept & 31)) {
#pragma unroll
                for (int r = 0; r < KR; ++r)
                    if (r == (kept >> 5)) kc[r] = i;
            }
            if (lane == 0 && kept < d.lane_cap) {
                lanes[kept].bottom_col = d.ext_lo + i;
                lanes[kept].energy = h[i];
                lanes[kept].n_points = 0;
            }
            ++kept;
            __syncwarp();  // lane 0's bitmap word before the next candidate's scan
        }
        if (lane == 0) {
        s_kept = kept;
        lk_frame_report& rep = d.rep[f];
        rep.lane_count = kept;
        for (int k = 0; k < kept && k < LK_MAX_INLINE_LANES; ++k) {
            rep.lane_bottom_col[k] = lanes[k].bottom_col;
            rep.lane_energy[k] = lanes[k].energy;
        }
        }
    }
    __syncthreads();
    // polylines: lane_track per kept lane (lanes.hpp:161-166)
    const int H = d.H, v_top = (int)d.rep[f].horizon, v_max = H - 1, rows = v_max - v_top + 1;
    const double* vpx = d.vpx + (size_t)f * H;
    const double* vpy = d.vpy + (size_t)f * H;
    for (int k = threadIdx.x; k < min(s_kept, d.lane_cap); k += blockDim.x) {
        if (!d.hooks) {  // the same recursion already ran in k_energy for this column
            lanes[k].n_points = d.track_np[(size_t)f * n + (lanes[k].bottom_col - d.ext_lo)];
            continue;
        }
        double u = (double)lanes[k].bottom_col;
        double* poly = d.hooks ? d.polylines + ((size_t)f * d.lane_cap + k) * H : nullptr;
        int np = 1;
        if (poly) poly[rows - 1] = u;
        int v = v_max - 1;
        for (; v >= v_top; --v) {
            const double py = vpy[v + 1];
            const double denom = (double)(v + 1) - py;
            if (fabs(denom) < 0.5) break;
            u = (vpx[v + 1] + v * u - py * u) / denom;
            np += !isnan(u);
            if (poly) poly[v - v_top] = u;
        }
        if (poly)
            for (; v >= v_top; --v) poly[v - v_top] = __longlong_as_double(0x7ff8000000000000LL);
        lanes[k].n_points = np;
    }
}

// Copies the aux counters into the public report at the end of the batch.
__global__ void k_finish(Dev d, int n) {
    const int f = blockIdx.x * blockDim.x + threadIdx.x;
    if (f >= n) return;
    lk_frame_report& r = d.rep[f];
    const FrameAux& a = d.aux[f];
    r.road_mask_pixels = (int64_t)a.mask_px;
    r.edge_pixels = (int64_t)a.edge_px;
    r.vpx_votes = (int64_t)a.votes;
    r.vpx_skipped = (int64_t)a.skipped;
}

}  // namespace lkg

// ------------------------------------------------------------------ launchers
namespace lkg {

cudaError_t launch_pipeline(const Dev& d, const LaunchPlan& lp, int n, cudaStream_t s,
                            cudaEvent_t* stage_ev, bool mark_start) {
    cudaStreamCaptureStatus cap = cudaStreamCaptureStatusNone;
    cudaStreamIsCapturing(s, &cap);
    auto mark = [&](int stage) {  // event-record nodes when captured into the graph
        if (!stage_ev) return;
        if (cap == cudaStreamCaptureStatusActive)
            cudaEventRecordWithFlags(stage_ev[stage], s, cudaEventRecordExternal);
        else
            cudaEventRecord(stage_ev[stage], s);
    };
    if (mark_start) mark(0);
    {
        const int R = vdisparity_rows(d.W, d.D1);
        k_vdisparity<<<dim3((d.H + R - 1) / R, n), 256, vdisparity_smem(d.W, d.D1), s>>>(
            d, lp.vhistT, R);
    }
    mark(5);
    k_vpath<<<n, 512, lp.vpath_smem, s>>>(d, lp.vhistT, lp.vpath_choice_smem);
    mark(6);
    k_road_fit<<<n, 128, lp.road_smem, s>>>(d);
    mark(7);
    mark(8);  // road mask is fused into the Sobel pass (stage 10)
    const dim3 bg((d.W + BF_TW - 1) / BF_TW, (d.H + BF_TH - 1) / BF_TH, n);
    if (lp.fast_front) {
        launch_fast_bilateral(d, lp, n, s);
        mark(9);
        launch_sobel_refine(d, lp, n, s);
    } else if (d.rho == 5)
    {
        const dim3 g((d.W + BT_W - 1) / BT_W, (d.H + BT_H - 1) / BT_H, n);
        switch (lp.bt_mode) {
            case 1: k_bilateral_tile<5, 1><<<g, 256, lp.bt_smem, s>>>(d, lp.ws); break;
            case 2: k_bilateral_tile<5, 2><<<g, 256, lp.bt_smem, s>>>(d, lp.ws); break;
            case 3: k_bilateral_tile<5, 3><<<g, 256, lp.bt_smem, s>>>(d, lp.ws); break;
            default: k_bilateral_tile<5, 0><<<g, 256, lp.bt_smem, s>>>(d, lp.ws); break;
        }
    }
    else
        k_bilateral<-1><<<bg, 256, lp.bf_smem, s>>>(d);
    if (!lp.fast_front) {
        mark(9);
        k_sobel_edges<<<dim3((d.W + SB_TW - 1) / SB_TW, (d.H + SB_TH - 1) / SB_TH, n), 256, 0,
                        s>>>(d);
    }
    k_edge_scan<<<n, 1024, 0, s>>>(d);
    if (lp.fast_front)
        k_edge_emit_tiles<<<dim3(lp.decide_ctas, n), 128, 0, s>>>(d);
    else
        k_edge_emit<<<dim3((d.H * d.n_seg + 7) / 8, n), 256, 0, s>>>(d);
    mark(10);
    // u-path DP: NT threads x SP consecutive states each (SP = 0: strided fallback)
#define LK_VANISH(SP, NT) k_vanish<SP, NT><<<n, NT, lp.vanish_smem, s>>>(d)
    if (lp.upath_nt == 512) {
        switch (lp.upath_sp) {
            case 1: LK_VANISH(1, 512); break;
            case 2: LK_VANISH(2, 512); break;
            case 3: LK_VANISH(3, 512); break;
            case 4: LK_VANISH(4, 512); break;
            case 5: LK_VANISH(5, 512); break;
            case 6: LK_VANISH(6, 512); break;
            default: LK_VANISH(8, 512); break;
        }
    } else {
        switch (lp.upath_sp) {
            case 5: LK_VANISH(5, 1024); break;
            case 6: LK_VANISH(6, 1024); break;
            case 8: LK_VANISH(8, 1024); break;
            default: LK_VANISH(0, 1024); break;
        }
    }
#undef LK_VANISH
    k_gamma_fit<<<n, 32 * GAMMA_NW, lp.gamma_smem, s>>>(d);
    k_wg<<<dim3(8, n), 256, 0, s>>>(d);
    mark(11);
    const bool auto_tr = isnan(d.tr_lpv);
    // 8 tiles per CTA (measured 4 / 8 / 16 / 32: 278 / 277 / 268 / 280 us at
    // 1242x375, 284 / 267 / 278 / 343 us at 2560x1024)
    k_m0_m1<<<dim3((d.m_nty * d.m_ntx + 7) / 8, n), 256, lp.m_smem, s>>>(d, lp.m_tile_h, auto_tr ? 1 : 0);
    if (auto_tr) {
        k_p99_bucket<<<n, 256, 0, s>>>(d);
        k_p99_hist2<<<dim3(lp.collect_blocks, n), 256, 0, s>>>(d);
        k_p99_bucket2<<<n, 256, 0, s>>>(d);
        k_p99_collect<<<dim3(lp.collect_blocks, n), 256, 0, s>>>(d);
        k_p99_select<<<n, 256, 0, s>>>(d);
    }
    if (d.lambda_g == 1.0)
    k_energy<true><<<dim3((d.ext_cols + 127) / 128, n), 128,
               (size_t)d.H * sizeof(double4) + (size_t)d.m_nty * d.m_ntx, s>>>(d);
    else
    k_energy<false><<<dim3((d.ext_cols + 127) / 128, n), 128,
               (size_t)d.H * sizeof(double4) + (size_t)d.m_nty * d.m_ntx, s>>>(d);
    k_select<<<n, 256, lp.select_smem, s>>>(d, lp.sort_cap);
    k_finish<<<(n + 127) / 128, 128, 0, s>>>(d, n);
    mark(12);
    return cudaGetLastError();
}

// Road-row copy (lk_submit_batch): the first grey row stages 8-12 read per
// frame, max(0, horizon - 1 - rho) (the Sobel's row above, the filter radius;
// the mask is empty above the horizon, preprocess.hpp:18), or H for a frame
// that failed in stages 5-7 (it reads no grey).
__global__ void k_road_rows(Dev d, int n, int* rows) {
    const int f = blockIdx.x * blockDim.x + threadIdx.x;
    if (f >= n) return;
    rows[f] = frame_failed(d, f) ? d.H : min(max((int)d.rep[f].horizon - 1 - d.rho, 0), d.H);
}

// The front pass of a streamed batch: stages 5-7 into d's (scratch) buffers,
// then k_road_rows. The batch's own graph recomputes stages 5-7 identically.
cudaError_t launch_road_front(const Dev& d, const LaunchPlan& lp, int n, int* rows, cudaStream_t s) {
    const int R = vdisparity_rows(d.W, d.D1);
    k_vdisparity<<<dim3((d.H + R - 1) / R, n), 256, vdisparity_smem(d.W, d.D1), s>>>(d, lp.vhistT, R);
    k_vpath<<<n, 512, lp.vpath_smem, s>>>(d, lp.vhistT, lp.vpath_choice_smem);
    k_road_fit<<<n, 128, lp.road_smem, s>>>(d);
    k_road_rows<<<(n + 127) / 128, 128, 0, s>>>(d, n, rows);
    return cudaGetLastError();
}

void launch_exact_bilateral(const Dev& d, const LaunchPlan& lp, int n, cudaStream_t s) {
    const dim3 g((d.W + BT_W - 1) / BT_W, (d.H + BT_H - 1) / BT_H, n);
    k_bilateral_tile<5, 0><<<g, 256, lp.bt_smem, s>>>(d, lp.ws);
}

// Kernels per frame range: the exact path (k_bilateral_tile, k_sobel_edges) or
// the certified fast path (k_prescreen, k_bilateral_need, k_sobel_screen,
// k_refine_exact, k_sobel_decide: 3 more), 5 more with the auto threshold.
int launches_per_batch(const Dev& d, const LaunchPlan& lp) {
    return (isnan(d.tr_lpv) ? 19 : 14) + (lp.fast_front ? 3 : 0);
}

cudaError_t configure_kernels(const LaunchPlan& lp) {
    cudaError_t e;
    if ((e = cudaFuncSetAttribute(k_vdisparity, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                  lp.vdisp_smem)))
        return e;
    if ((e = cudaFuncSetAttribute(k_vpath, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                  lp.vpath_smem)))
        return e;
    if ((e = cudaFuncSetAttribute(k_road_fit, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                  lp.road_smem)))
        return e;
    for (auto fn : {k_bilateral_tile<5, 0>, k_bilateral_tile<5, 1>, k_bilateral_tile<5, 2>,
                    k_bilateral_tile<5, 3>})
        if ((e = cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize, lp.bt_smem)))
            return e;
    if ((e = cudaFuncSetAttribute(k_bilateral<-1>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                  lp.bf_smem)))
        return e;
    for (auto fn : {k_vanish<1, 512>, k_vanish<2, 512>, k_vanish<3, 512>, k_vanish<4, 512>,
                    k_vanish<5, 512>, k_vanish<6, 512>, k_vanish<8, 512>, k_vanish<5, 1024>,
                    k_vanish<6, 1024>, k_vanish<8, 1024>, k_vanish<0, 1024>})
        if ((e = cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                      lp.vanish_smem)))
            return e;
    if ((e = cudaFuncSetAttribute(k_gamma_fit, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                  lp.gamma_smem)))
        return e;
    if ((e = cudaFuncSetAttribute(k_m0_m1, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                  lp.m_smem)))
        return e;
    if ((e = cudaFuncSetAttribute(k_select, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                  lp.select_smem)))
        return e;
    return configure_fastpath(lp.fast_width);
}

}  // namespace lkg

// ------------------------------------------------------------------ FP64 probe
// Throughput of dependent-free DADD/DMUL streams (8 chains per thread) for the
// FP64 roofline denominator; ops counted as individual adds and multiplies.
namespace lkg {
__global__ void __launch_bounds__(256) k_fp64_probe(double* sink, int iters, double a, double b) {
    double x[8];
#pragma unroll
    for (int k = 0; k < 8; ++k) x[k] = threadIdx.x * 1e-3 + k;
    for (int i = 0; i < iters; ++i) {
#pragma unroll
        for (int k = 0; k < 8; ++k) x[k] = x[k] * a + b;  // 1 DMUL + 1 DADD (no contraction)
    }
    double s = 0;
#pragma unroll
    for (int k = 0; k < 8; ++k) s += x[k];
    if (s == 12345.678) sink[0] = s;
}

cudaError_t fp64_probe(int sms, double* ops_per_s) {
    double* sink;
    cudaError_t e = cudaMalloc(&sink, 8);
    if (e) return e;
    cudaEvent_t t0, t1;
    cudaEventCreate(&t0);
    cudaEventCreate(&t1);
    const int blocks = sms * 8, iters = 4096;
    k_fp64_probe<<<blocks, 256>>>(sink, 64, 0.999999, 1e-7);  // warm-up
    cudaEventRecord(t0);
    k_fp64_probe<<<blocks, 256>>>(sink, iters, 0.999999, 1e-7);
    cudaEventRecord(t1);
    e = cudaEventSynchronize(t1);
    float ms = 0;
    cudaEventElapsedTime(&ms, t0, t1);
    *ops_per_s = (double)blocks * 256 * iters * 8 * 2 / (ms * 1e-3);
    cudaEventDestroy(t0);
    cudaEventDestroy(t1);
    cudaFree(sink);
    return e ? e : cudaGetLastError();
}
}  // namespace lkg
