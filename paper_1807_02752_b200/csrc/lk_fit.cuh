// lk_fit.cuh — block-level trimming RANSAC with least-squares refits.
//
// Restates, on one CTA per frame:
//   detail::ransac_trim         ransac.hpp:36-119
//   fit_parabola_lsq            road_profile.hpp:86-111   (K = 3)
//   fit_quartic (kappa = 1)     vanish.hpp:201-243        (K = 5)
//   Eigen LDLT + solve
// The reference's sequential semantics are kept exactly:
//  * the sample sequence comes from a host-built table of mt19937_64(seed)
//    outputs (iteration `it` consumes outputs it*K .. it*K+K-1, ransac.hpp:54-64);
//  * SPECULATION: the NW warps of the CTA evaluate iterations it0..it0+NW-1
//    against the same candidate set m; thread 0 then commits them in order,
//    and the first iteration that trims m ends the round (later speculative
//    results used a stale m and are discarded) — identical to running the
//    iterations one by one;
//  * classification is lane-parallel with ORDER-PRESERVING ballot compaction;
//  * every normal-equation entry is summed sequentially in point order;
//  * the small LDLT solves run fully unrolled in registers (compile-time
//    indices; pivot swaps as predicated exchanges).
#pragma once

#include "lk_device.cuh"

namespace lkg {

constexpr int RS_MAX_WARPS = 16;

struct RansacState {  // lives in shared memory
    double model[5];
    double s;          // v normalizer of the model (quartic)
    double fraction;
    int iterations;
    int degraded;
    int msg;           // 0 ok, LK_MSG_RANSAC_*
    int n_inl;
    const int* inl;    // index list into the points (shared memory)
    // scratch
    double fit_model[5];
    double fit_s;
    double ab[32];     // normal-equation entries gathered for lane 0
    // speculative round
    double w_model[RS_MAX_WARPS][5];
    int w_ok[RS_MAX_WARPS];
    int w_cnt[RS_MAX_WARPS];
    int w_buf[RS_MAX_WARPS];  // buffer index holding warp w's compacted inliers
    int m_buf;                // buffer index holding m
    int msz;
    int it0;
    int done;
    int iterations_run;
    double best;
    int have;
    double best_model[5];
    double best_s;
    double w_s[RS_MAX_WARPS];
    double w_frac[RS_MAX_WARPS];  // inlier fraction of warp w's iteration (ransac.hpp:76)
#ifdef LK_GAMMA_PROF
    long long t_loop;
    long long t_fit, t_cls, t_commit;
    int rounds;
#endif
};

template <int K>
__device__ __forceinline__ double phi_k(int i, double t) {
    // (1, t, t*t, t*t*t, t*t*t*t) evaluated exactly as written
    // (road_profile.hpp:105, vanish.hpp:226)
    if (i == 0) return 1.0;
    if (i == 1) return t;
    if (i == 2) return t * t;
    if (i == 3) return t * t * t;
    return t * t * t * t;
}

template <int K>
__device__ __forceinline__ double res2(const double* m, int x, int v) {
    const double vv = (double)v;
    double r;
    if (K == 3) {  // road_profile.hpp:124-128
        r = (double)x - (m[0] + m[1] * vv + m[2] * vv * vv);
    } else {       // vanish.hpp:191-193, 258-261
        r = (double)x - (m[0] + vv * (m[1] + vv * (m[2] + vv * (m[3] + vv * m[4]))));
    }
    return r * r;
}

template <typename T>
__device__ __forceinline__ void xchg(T& a, T& b) {
    T t = a;
    a = b;
    b = t;
}

// x mod d for a 64-bit x and 0 < d < 2^16 (a RANSAC index range) exactly, in
// three 32-bit steps (16 bits of x at a time) instead of the 64-bit division
// routine: ((x_hi mod d) 2^16 + x[31:16]) mod d, then the same with x[15:0].
__device__ __forceinline__ unsigned mod64_small(unsigned long long x, unsigned d) {
    const unsigned hi = (unsigned)(x >> 32), lo = (unsigned)x;
    unsigned r = hi % d;
    r = ((r << 16) | (lo >> 16)) % d;
    return ((r << 16) | (lo & 0xffffu)) % d;
}

// ---- LDLT (Appendix B) in registers, row-major N x N, lower triangle used.
template <int N>
__device__ __forceinline__ void ldlt_factor(double (&A)[N][N], int (&t)[N]) {
    double temp[N];
#pragma unroll
    for (int k = 0; k < N; ++k) {
        int p = k;
        double big = fabs(A[k][k]);
#pragma unroll
        for (int i = k + 1; i < N; ++i) {
            const double c = fabs(A[i][i]);
            if (c > big) {
                big = c;
                p = i;
            }
        }
        t[k] = p;
#pragma unroll
        for (int q = k + 1; q < N; ++q) {
            if (p == q) {
#pragma unroll
                for (int j = 0; j < k; ++j) xchg(A[k][j], A[q][j]);
#pragma unroll
                for (int i = q + 1; i < N; ++i) xchg(A[i][k], A[i][q]);
                xchg(A[k][k], A[q][q]);
#pragma unroll
                for (int i = k + 1; i < q; ++i) xchg(A[i][k], A[q][i]);
            }
        }
        if (k > 0) {
#pragma unroll
            for (int j = 0; j < k; ++j) temp[j] = A[j][j] * A[k][j];
            double dot = A[k][0] * temp[0];
#pragma unroll
            for (int j = 1; j < k; ++j) dot = dot + A[k][j] * temp[j];
            A[k][k] = A[k][k] - dot;
#pragma unroll
            for (int i = k + 1; i < N; ++i) {
                double s = A[i][0] * temp[0];
#pragma unroll
                for (int j = 1; j < k; ++j) s = s + A[i][j] * temp[j];
                A[i][k] = A[i][k] - s;
            }
        }
        const double akk = A[k][k];
        const bool valid = fabs(akk) > 0.0;
        if (k == 0 && !valid) {  // whole diagonal zero: identity transpositions, stop
#pragma unroll
            for (int j = 0; j < N; ++j) t[j] = j;
            return;
        }
        if (valid) {
#pragma unroll
            for (int i = k + 1; i < N; ++i) A[i][k] = A[i][k] / akk;
        }
    }
}

template <int N>
__device__ __forceinline__ void apply_transposition(double (&x)[N], int k, int tk) {
#pragma unroll
    for (int q = 0; q < N; ++q)
        if (q > k && tk == q) xchg(x[k], x[q]);
}

template <int N>
__device__ __forceinline__ void ldlt_solve(const double (&A)[N][N], const int (&t)[N],
                                           const double (&b)[N], double (&x)[N]) {
#pragma unroll
    for (int i = 0; i < N; ++i) x[i] = b[i];
#pragma unroll
    for (int k = 0; k < N; ++k) apply_transposition<N>(x, k, t[k]);
#pragma unroll
    for (int i = 0; i < N; ++i)
#pragma unroll
        for (int s = i + 1; s < N; ++s) x[s] = x[s] - x[i] * A[s][i];
#pragma unroll
    for (int i = 0; i < N; ++i) {
        const double dd = A[i][i];
        if (fabs(dd) > 2.2250738585072014e-308)  // DBL_MIN
            x[i] = x[i] / dd;
        else
            x[i] = 0.0;
    }
#pragma unroll
    for (int i = N - 2; i >= 0; --i) {
        double s = A[i + 1][i] * x[i + 1];
#pragma unroll
        for (int j = i + 2; j < N; ++j) s = s + A[j][i] * x[j];
        x[i] = x[i] - s;
    }
#pragma unroll
    for (int k = N - 1; k >= 0; --k) apply_transposition<N>(x, k, t[k]);
}

// Normal equations (A, b) -> model, exactly as fit_parabola_lsq / fit_quartic
// finish: solve, one refinement pass for the quartic, rescale by s^k.
template <int K>
__device__ __forceinline__ void solve_model(const double (&A)[K][K], const double (&b)[K], double s,
                                            double* model) {
    double L[K][K], x[K];
    int t[K];
#pragma unroll
    for (int i = 0; i < K; ++i)
#pragma unroll
        for (int j = 0; j < K; ++j) L[i][j] = A[i][j];
    ldlt_factor<K>(L, t);
    ldlt_solve<K>(L, t, b, x);
    if (K == 5) {  // x += solve(b - a*x)  (vanish.hpp:230-232)
        double r[K], dx[K];
#pragma unroll
        for (int i = 0; i < K; ++i) {
            double ax = A[i][0] * x[0];
#pragma unroll
            for (int j = 1; j < K; ++j) ax = ax + A[i][j] * x[j];
            r[i] = b[i] - ax;
        }
        ldlt_solve<K>(L, t, r, dx);
#pragma unroll
        for (int i = 0; i < K; ++i) x[i] = x[i] + dx[i];
        double sk = 1.0;
#pragma unroll
        for (int k = 0; k < K; ++k) {
            model[k] = x[k] / sk;
            sk *= s;
        }
    } else {
        model[0] = x[0];
        model[1] = x[1] / s;
        model[2] = x[2] / (s * s);
    }
}

// One-lane fit of the K sample points (x[i], v[i]) in sample order.
template <int K>
__device__ __forceinline__ bool lane_fit_sample(const int (&x)[K], const int (&v)[K], double* model,
                                                double* s_out) {
    int ns = 0;
#pragma unroll
    for (int i = 0; i < K; ++i) {
        bool dup = false;
#pragma unroll
        for (int j = 0; j < i; ++j) dup |= v[j] == v[i];
        ns += !dup;
    }
    if (ns < K) return false;  // "needs three / five distinct rows"
    double s = 1.0;
#pragma unroll
    for (int i = 0; i < K; ++i) s = fmax(s, fabs((double)v[i]));
    double A[K][K], b[K];
#pragma unroll
    for (int i = 0; i < K; ++i) {
        b[i] = 0.0;
#pragma unroll
        for (int j = 0; j < K; ++j) A[i][j] = 0.0;
    }
#pragma unroll
    for (int p = 0; p < K; ++p) {
        const double t = (double)v[p] / s;
        double ph[K];
#pragma unroll
        for (int i = 0; i < K; ++i) ph[i] = phi_k<K>(i, t);
#pragma unroll
        for (int i = 0; i < K; ++i)
#pragma unroll
            for (int j = 0; j < K; ++j) A[i][j] = A[i][j] + ph[i] * ph[j];
        const double xd = (double)x[p];
#pragma unroll
        for (int i = 0; i < K; ++i) b[i] = b[i] + xd * ph[i];
    }
    solve_model<K>(A, b, s, model);
    *s_out = s;
    return true;
}

// Least-squares fit of the points idx[0..n) (indices into px/pv). Whole warp:
// lane e < K*K accumulates a(e/K, e%K), lane K*K+i accumulates b(i), each
// sequentially in point order. Result in st.fit_model / st.fit_s.
// The basis values are first tabulated lane-parallel (tbuf rows: 1, phi_1 ..
// phi_{K-1}, x; (K+1)*n doubles), so each accumulation chain is only loads,
// an independent product and the dependent add: the reference's per-entry
// summation order is unchanged.
template <int K>
__device__ bool warp_fit(const int* px, const int* pv, const int* idx, int n, double* tbuf,
                         RansacState& st) {
    const int lane = threadIdx.x & 31;
    int ok = 0;
    if (lane == 0) {
        int seen[K];
        int ns = 0;
        for (int i = 0; i < n && ns < K; ++i) {
            const int r = pv[idx[i]];
            bool dup = false;
            for (int j = 0; j < ns; ++j) dup |= seen[j] == r;
            if (!dup) seen[ns++] = r;
        }
        ok = ns >= K;
    }
    ok = __shfl_sync(0xffffffffu, ok, 0);
    if (!ok) return false;
    double s = 1.0;  // max(1, max|v|): exact and order independent
    for (int i = lane; i < n; i += 32) s = fmax(s, fabs((double)pv[idx[i]]));
    for (int o = 16; o; o >>= 1) s = fmax(s, __shfl_xor_sync(0xffffffffu, s, o));
    for (int p = lane; p < n; p += 32) {
        const int id = idx[p];
        const double t = (double)pv[id] / s;
        tbuf[p] = 1.0;
#pragma unroll
        for (int i = 1; i < K; ++i) tbuf[i * n + p] = phi_k<K>(i, t);
        tbuf[K * n + p] = (double)px[id];
    }
    __syncwarp();
    if (lane < K * K + K) {
        // a(i, j) = sum phi_i * phi_j; b(i) = sum x * phi_i (vanish.hpp:226-229)
        const int fa = lane < K * K ? lane / K : K, fb = lane < K * K ? lane % K : lane - K * K;
        const double* ra = tbuf + fa * n;
        const double* rb = tbuf + fb * n;
        double acc = 0.0;
        int p = 0;
        for (; p + 8 <= n; p += 8) {
            double pr[8];
#pragma unroll
            for (int q = 0; q < 8; ++q) pr[q] = ra[p + q] * rb[p + q];
#pragma unroll
            for (int q = 0; q < 8; ++q) acc = acc + pr[q];
        }
        for (; p < n; ++p) acc = acc + ra[p] * rb[p];
        st.ab[lane] = acc;
    }
    __syncwarp();
    if (lane == 0) {
        double A[K][K], b[K];
#pragma unroll
        for (int i = 0; i < K; ++i) {
            b[i] = st.ab[K * K + i];
#pragma unroll
            for (int j = 0; j < K; ++j) A[i][j] = st.ab[i * K + j];
        }
        solve_model<K>(A, b, s, st.fit_model);
        st.fit_s = s;
    }
    __syncwarp();
    return true;
}

// Order-preserving filter: out <- {src[i] : res2(model, p) < tol}, whole warp.
template <int K>
__device__ int warp_classify(const int* px, const int* pv, const int* src, int n,
                             const double* model, double tol, int* out) {
    const int lane = threadIdx.x & 31;
    int cnt = 0;
    for (int base = 0; base < n; base += 32) {
        const int i = base + lane;
        bool in = false;
        int id = 0;
        if (i < n) {
            id = src ? src[i] : i;
            in = res2<K>(model, px[id], pv[id]) < tol;
        }
        const unsigned bal = __ballot_sync(0xffffffffu, in);
        if (in) out[cnt + __popc(bal & ((1u << lane) - 1u))] = id;
        cnt += __popc(bal);
    }
    __syncwarp();
    return cnt;
}

// ransac_trim over points 0..n-1 by the first NW warps of the CTA (NW >= 3).
// bufs: NW + 2 index lists of capacity n; tbuf: (K + 1) * n doubles; all shared memory.
// Every thread of the CTA must call this (it contains __syncthreads).
template <int K, int NW>
__device__ void block_ransac(const int* px, const int* pv, int n, double tol, double eps,
                             int max_iter, const uint64_t* rng, int* const* bufs, double* tbuf,
                             RansacState& st) {
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    if (tid == 0) {
        st.msg = 0;
        st.iterations = 0;
        st.degraded = 0;
        st.fraction = 0;
        st.n_inl = 0;
        st.inl = bufs[0];
        st.m_buf = 0;
        st.msz = n;
        st.it0 = 0;
        st.done = n < K;
        st.iterations_run = 0;
        st.best = -1.0;
        st.have = 0;
        for (int w = 0; w < NW; ++w) st.w_buf[w] = 1 + w;
        if (n < K) st.msg = LK_MSG_RANSAC_FEW_POINTS;  // ransac.hpp:41-42
    }
    __syncthreads();
#ifdef LK_GAMMA_PROF
    if (tid == 0) { st.t_fit = st.t_cls = st.t_commit = 0; st.rounds = 0; }
#endif
    if (st.done) return;
    for (int i = tid; i < n; i += blockDim.x) bufs[0][i] = i;
    __syncthreads();
    while (!st.done) {
#ifdef LK_GAMMA_PROF
        const long long r0 = clock64();
#endif
        const int it = st.it0 + warp;
        const int msz = st.msz;
        if (warp < NW && it < max_iter && msz >= K) {
            const int* m = bufs[st.m_buf];
            int ok = 0;
            if (lane == 0) {  // partial Fisher-Yates on an identity index (ransac.hpp:58-64)
                int opos[2 * K], oval[2 * K], no = 0;
                int sx[K], sv[K];
                const uint64_t* r = rng + (size_t)it * K;
#pragma unroll
                for (int i = 0; i < K; ++i) {
                    const int j = i + (int)mod64_small(r[i], (unsigned)(msz - i));
                    int vi = i, vj = j;
                    for (int q = 0; q < no; ++q) {
                        if (opos[q] == i) vi = oval[q];
                        if (opos[q] == j) vj = oval[q];
                    }
                    bool fi = false, fj = false;
                    for (int q = 0; q < no; ++q) {
                        if (opos[q] == i) { oval[q] = vj; fi = true; }
                        if (opos[q] == j) { oval[q] = vi; fj = true; }
                    }
                    if (!fi) { opos[no] = i; oval[no] = vj; ++no; }
                    if (!fj && j != i) { opos[no] = j; oval[no] = vi; ++no; }
                    const int pid = m[vj];
                    sx[i] = px[pid];
                    sv[i] = pv[pid];
                }
                double mdl[5] = {0, 0, 0, 0, 0}, s = 0;
                ok = lane_fit_sample<K>(sx, sv, mdl, &s);
                for (int k = 0; k < K; ++k) st.w_model[warp][k] = mdl[k];
                st.w_s[warp] = s;
                st.w_ok[warp] = ok;
            }
            ok = __shfl_sync(0xffffffffu, ok, 0);
            __syncwarp();
#ifdef LK_GAMMA_PROF
            if (warp == 0 && lane == 0) st.t_fit += clock64() - r0;
            const long long r1 = clock64();
#endif
            if (ok) {
                double mdl[5];
                for (int k = 0; k < K; ++k) mdl[k] = st.w_model[warp][k];
                const int cnt =
                    warp_classify<K>(px, pv, m, msz, mdl, tol, bufs[st.w_buf[warp]]);
                if (lane == 0) {  // the fraction is computed here, not in the serial commit
                    st.w_cnt[warp] = cnt;
                    st.w_frac[warp] = (double)cnt / (double)msz;
                }
            }
#ifdef LK_GAMMA_PROF
            if (warp == 0 && lane == 0) st.t_cls += clock64() - r1;
#endif
        }
        __syncthreads();
#ifdef LK_GAMMA_PROF
        const long long r2 = clock64();
#endif
        if (tid == 0) {  // commit in iteration order (ransac.hpp:54-87)
            int next_it0 = st.it0 + NW;
            for (int w = 0; w < NW; ++w) {
                const int it2 = st.it0 + w;
                if (it2 >= max_iter) {
                    st.done = 1;
                    break;
                }
                st.iterations_run = it2 + 1;
                if (st.msz < K) {
                    st.done = 1;
                    break;
                }
                if (!st.w_ok[w]) continue;  // degenerate sample, iteration consumed
                const int cnt = st.w_cnt[w];
                const double fraction = st.w_frac[w];  // = cnt / st.msz (same msz this round)
                if (fraction > st.best) {
                    st.best = fraction;
                    for (int k = 0; k < K; ++k) st.best_model[k] = st.w_model[w][k];
                    st.best_s = st.w_s[w];
                    st.have = 1;
                }
                bool trimmed = false;
                if (fraction >= st.best && fraction > 0.5 && cnt >= K) {
                    const int b = st.m_buf;
                    st.m_buf = st.w_buf[w];
                    st.w_buf[w] = b;
                    st.msz = cnt;
                    trimmed = true;
                }
                if (st.best >= eps) {
                    st.done = 1;
                    break;
                }
                if (trimmed) {
                    next_it0 = it2 + 1;
                    break;
                }
            }
            st.it0 = next_it0;
            if (st.it0 >= max_iter) st.done = 1;
        }
        __syncthreads();
#ifdef LK_GAMMA_PROF
        if (tid == 0) { st.t_commit += clock64() - r2; ++st.rounds; }
#endif
    }
#ifdef LK_GAMMA_PROF
    if (tid == 0) st.t_loop = clock64();
#endif
    // final model and refits (ransac.hpp:88-118), warp 0
    if (warp == 0) {
        const int iterations = st.iterations_run;
        if (!st.have) {
            if (lane == 0) {
                st.msg = LK_MSG_RANSAC_NO_FIT;  // ransac.hpp:90
                st.iterations = iterations;
            }
        } else {
            // two free lists besides m
            int fa = -1, fb = -1;
            for (int i = 0; i < NW + 2; ++i)
                if (i != st.m_buf) {
                    if (fa < 0) fa = i;
                    else if (fb < 0) fb = i;
                }
            const int* m = bufs[st.m_buf];
            const int msz = st.msz;
            int* inl = bufs[fa];
            int* nxt = bufs[fb];
            double bm[5];
            for (int k = 0; k < K; ++k) bm[k] = st.best_model[k];
            int ninl = warp_classify<K>(px, pv, m, msz, bm, tol, inl);
            if (lane == 0) {
                for (int k = 0; k < K; ++k) st.model[k] = bm[k];
                st.s = st.best_s;
            }
            for (int round = 0; round < 3 && ninl >= K; ++round) {
                if (!warp_fit<K>(px, pv, inl, ninl, tbuf, st)) break;
                double rm[5];
                for (int k = 0; k < K; ++k) rm[k] = st.fit_model[k];
                if (lane == 0) {
                    for (int k = 0; k < K; ++k) st.model[k] = rm[k];
                    st.s = st.fit_s;
                }
                // next = {p in all points : res2 < tol}
                const int cnt = warp_classify<K>(px, pv, nullptr, n, rm, tol, nxt);
                bool same = cnt == ninl;  // next == inl as (x, v) value sequences
                if (same) {
                    bool diff = false;
                    for (int i = lane; i < cnt; i += 32) {
                        const int a = nxt[i], b = inl[i];
                        diff |= px[a] != px[b] || pv[a] != pv[b];
                    }
                    same = !__any_sync(0xffffffffu, diff);
                }
                int* tmp = inl;
                inl = nxt;
                nxt = tmp;
                ninl = cnt;
                if (same) break;
            }
            if (lane == 0) {
                if (ninl == 0) {
                    st.inl = m;
                    st.n_inl = msz;
                } else {
                    st.inl = inl;
                    st.n_inl = ninl;
                }
                st.iterations = iterations;
                st.fraction = st.best;
                st.degraded = st.best < eps;
            }
        }
    }
    __syncthreads();
}

}  // namespace lkg
