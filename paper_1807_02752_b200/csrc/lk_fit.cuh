// lk_fit.cuh — one-warp trimming RANSAC with least-squares refits.
//
// Restates, on one warp per frame:
//   detail::ransac_trim         ransac.hpp:36-119
//   fit_parabola_lsq            road_profile.hpp:86-111   (K = 3)
//   fit_quartic (kappa = 1)     vanish.hpp:201-243        (K = 5)
//   Eigen LDLT + solve
// Sequential semantics are kept exactly: the sample sequence comes from a
// host-built table of mt19937_64(seed) outputs (iteration `it` consumes
// outputs it*K .. it*K+K-1, ransac.hpp:54-64); classification is
// lane-parallel with ORDER-PRESERVING ballot compaction; every normal-equation
// entry is summed sequentially in point order by its own lane.
#pragma once

#include "lk_device.cuh"

namespace lkg {

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
    double best_model[5];
    double best_s;
    double fit_model[5];
    double fit_s;
    double ab[32];     // normal-equation entries gathered for lane 0
    int sidx[5];
    int fit_ok;
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

// ---- LDLT (Appendix B), serial on one lane, row-major N x N, lower used.
template <int N>
__device__ void ldlt_factor(double* A, int* t) {
    double temp[N];
    for (int k = 0; k < N; ++k) {
        int p = k;
        double big = fabs(A[k * N + k]);
        for (int i = k + 1; i < N; ++i) {
            const double c = fabs(A[i * N + i]);
            if (c > big) {
                big = c;
                p = i;
            }
        }
        t[k] = p;
        if (p != k) {
            for (int j = 0; j < k; ++j) {
                double x = A[k * N + j]; A[k * N + j] = A[p * N + j]; A[p * N + j] = x;
            }
            for (int i = p + 1; i < N; ++i) {
                double x = A[i * N + k]; A[i * N + k] = A[i * N + p]; A[i * N + p] = x;
            }
            { double x = A[k * N + k]; A[k * N + k] = A[p * N + p]; A[p * N + p] = x; }
            for (int i = k + 1; i < p; ++i) {
                double x = A[i * N + k]; A[i * N + k] = A[p * N + i]; A[p * N + i] = x;
            }
        }
        if (k > 0) {
            for (int j = 0; j < k; ++j) temp[j] = A[j * N + j] * A[k * N + j];
            double dot = A[k * N] * temp[0];
            for (int j = 1; j < k; ++j) dot = dot + A[k * N + j] * temp[j];
            A[k * N + k] = A[k * N + k] - dot;
            for (int i = k + 1; i < N; ++i) {
                double s = A[i * N] * temp[0];
                for (int j = 1; j < k; ++j) s = s + A[i * N + j] * temp[j];
                A[i * N + k] = A[i * N + k] - s;
            }
        }
        const double akk = A[k * N + k];
        const bool valid = fabs(akk) > 0.0;
        if (k == 0 && !valid) {
            for (int j = 0; j < N; ++j) t[j] = j;
            break;
        }
        if (valid)
            for (int i = k + 1; i < N; ++i) A[i * N + k] = A[i * N + k] / akk;
    }
}

template <int N>
__device__ void ldlt_solve(const double* A, const int* t, const double* b, double* x) {
    for (int i = 0; i < N; ++i) x[i] = b[i];
    for (int k = 0; k < N; ++k) {
        double s = x[k]; x[k] = x[t[k]]; x[t[k]] = s;
    }
    for (int i = 0; i < N; ++i)
        for (int s = i + 1; s < N; ++s) x[s] = x[s] - x[i] * A[s * N + i];
    for (int i = 0; i < N; ++i) {
        const double d = A[i * N + i];
        if (fabs(d) > 2.2250738585072014e-308)  // DBL_MIN
            x[i] = x[i] / d;
        else
            x[i] = 0.0;
    }
    for (int i = N - 2; i >= 0; --i) {
        double s = A[(i + 1) * N + i] * x[i + 1];
        for (int j = i + 2; j < N; ++j) s = s + A[j * N + i] * x[j];
        x[i] = x[i] - s;
    }
    for (int k = N - 1; k >= 0; --k) {
        double s = x[k]; x[k] = x[t[k]]; x[t[k]] = s;
    }
}

// Least-squares fit of the points idx[0..n) (indices into px/pv). Whole warp.
// Returns false for a degenerate set (the reference throws: "needs three /
// five distinct rows"). Result in st.fit_model / st.fit_s.
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
    // s = max(1, max|v|): exact and order independent
    double s = 1.0;
    for (int i = lane; i < n; i += 32) s = fmax(s, fabs((double)pv[idx[i]]));
    for (int o = 16; o; o >>= 1) s = fmax(s, __shfl_xor_sync(0xffffffffu, s, o));
    for (int i = lane; i < n; i += 32) tbuf[i] = (double)pv[idx[i]] / s;
    __syncwarp();
    // lane e < K*K: a(e/K, e%K); K*K <= e < K*K+K: b(e-K*K). Sequential in point order.
    double acc = 0.0;
    if (lane < K * K) {
        const int ii = lane / K, jj = lane % K;
        for (int p = 0; p < n; ++p) {
            const double t = tbuf[p];
            acc = acc + phi_k<K>(ii, t) * phi_k<K>(jj, t);
        }
    } else if (lane < K * K + K) {
        const int ii = lane - K * K;
        for (int p = 0; p < n; ++p) {
            const double t = tbuf[p];
            acc = acc + (double)px[idx[p]] * phi_k<K>(ii, t);
        }
    }
    if (lane < K * K + K) st.ab[lane] = acc;
    __syncwarp();
    if (lane == 0) {
        double A[K * K], L[K * K], b[K], x[K];
        int t[K];
        for (int e = 0; e < K * K; ++e) A[e] = L[e] = st.ab[e];
        for (int i = 0; i < K; ++i) b[i] = st.ab[K * K + i];
        ldlt_factor<K>(L, t);
        ldlt_solve<K>(L, t, b, x);
        if (K == 5) {  // x += solve(b - a*x)  (vanish.hpp:230-232)
            double r[K], dx[K];
            for (int i = 0; i < K; ++i) {
                double ax = A[i * K] * x[0];
                for (int j = 1; j < K; ++j) ax = ax + A[i * K + j] * x[j];
                r[i] = b[i] - ax;
            }
            ldlt_solve<K>(L, t, r, dx);
            for (int i = 0; i < K; ++i) x[i] = x[i] + dx[i];
            double sk = 1.0;
            for (int k = 0; k < K; ++k) {
                st.fit_model[k] = x[k] / sk;
                sk *= s;
            }
        } else {
            st.fit_model[0] = x[0];
            st.fit_model[1] = x[1] / s;
            st.fit_model[2] = x[2] / (s * s);
        }
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
            id = src[i];
            in = res2<K>(model, px[id], pv[id]) < tol;
        }
        const unsigned bal = __ballot_sync(0xffffffffu, in);
        if (in) out[cnt + __popc(bal & ((1u << lane) - 1u))] = id;
        cnt += __popc(bal);
    }
    __syncwarp();
    return cnt;
}

// ransac_trim over points 0..n-1. bufs: three index lists of capacity n,
// tbuf: n doubles. All in shared memory; called by exactly one full warp.
template <int K>
__device__ void warp_ransac(const int* px, const int* pv, int n, double tol, double eps,
                            int max_iter, const uint64_t* rng, int* bufA, int* bufB, int* bufC,
                            double* tbuf, RansacState& st) {
    const int lane = threadIdx.x & 31;
    if (lane == 0) {
        st.msg = 0;
        st.iterations = 0;
        st.degraded = 0;
        st.fraction = 0;
        st.n_inl = 0;
        st.inl = bufA;
    }
    __syncwarp();
    if (n < K) {  // ransac.hpp:41-42
        if (lane == 0) st.msg = LK_MSG_RANSAC_FEW_POINTS;
        __syncwarp();
        return;
    }
    for (int i = lane; i < n; i += 32) bufA[i] = i;
    __syncwarp();
    int* m = bufA;
    int* inl = bufB;
    int msz = n;
    double best = -1.0;
    bool have = false;
    int iterations = 0;
    for (int it = 0; it < max_iter; ++it) {
        iterations = it + 1;
        if (msz < K) break;
        if (lane == 0) {  // partial Fisher-Yates on an identity index (ransac.hpp:58-64)
            int opos[2 * K], oval[2 * K], no = 0;
            auto get = [&](int p) {
                for (int q = 0; q < no; ++q)
                    if (opos[q] == p) return oval[q];
                return p;
            };
            auto set = [&](int p, int v) {
                for (int q = 0; q < no; ++q)
                    if (opos[q] == p) {
                        oval[q] = v;
                        return;
                    }
                opos[no] = p;
                oval[no] = v;
                ++no;
            };
            const uint64_t* r = rng + (size_t)it * K;
            for (int i = 0; i < K; ++i) {
                const int j = i + (int)(r[i] % (uint64_t)(msz - i));
                const int vi = get(i), vj = get(j);
                set(i, vj);
                set(j, vi);
                st.sidx[i] = m[vj];
            }
        }
        __syncwarp();
        if (!warp_fit<K>(px, pv, st.sidx, K, tbuf, st)) continue;  // iteration consumed
        double model[5];
        for (int k = 0; k < K; ++k) model[k] = st.fit_model[k];
        const double ms = st.fit_s;
        const int cnt = warp_classify<K>(px, pv, m, msz, model, tol, inl);
        const double fraction = (double)cnt / (double)msz;
        if (fraction > best) {
            best = fraction;
            if (lane == 0) {
                for (int k = 0; k < K; ++k) st.best_model[k] = model[k];
                st.best_s = ms;
            }
            have = true;
        }
        if (fraction >= best && fraction > 0.5 && cnt >= K) {
            int* tmp = m;
            m = inl;
            inl = tmp;
            msz = cnt;
        }
        __syncwarp();
        if (best >= eps) break;
    }
    if (!have) {  // ransac.hpp:90
        if (lane == 0) {
            st.msg = LK_MSG_RANSAC_NO_FIT;
            st.iterations = iterations;
        }
        __syncwarp();
        return;
    }
    double bm[5];
    for (int k = 0; k < K; ++k) bm[k] = st.best_model[k];
    int ninl = warp_classify<K>(px, pv, m, msz, bm, tol, inl);
    if (lane == 0) {
        for (int k = 0; k < K; ++k) st.model[k] = bm[k];
        st.s = st.best_s;
    }
    // third list: whichever of bufA/B/C is neither m nor inl
    int* nxt = (m != bufA && inl != bufA) ? bufA : (m != bufB && inl != bufB) ? bufB : bufC;
    for (int round = 0; round < 3 && ninl >= K; ++round) {
        if (!warp_fit<K>(px, pv, inl, ninl, tbuf, st)) break;
        double rm[5];
        for (int k = 0; k < K; ++k) rm[k] = st.fit_model[k];
        if (lane == 0) {
            for (int k = 0; k < K; ++k) st.model[k] = rm[k];
            st.s = st.fit_s;
        }
        // next = {p in all points : res2 < tol}; the identity source is implicit
        int cnt = 0;
        for (int base = 0; base < n; base += 32) {
            const int i = base + lane;
            const bool in = i < n && res2<K>(rm, px[i], pv[i]) < tol;
            const unsigned bal = __ballot_sync(0xffffffffu, in);
            if (in) nxt[cnt + __popc(bal & ((1u << lane) - 1u))] = i;
            cnt += __popc(bal);
        }
        __syncwarp();
        // settled: next == inl compared as (x, v) value sequences
        bool same = cnt == ninl;
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
        st.fraction = best;
        st.degraded = best < eps;
    }
    __syncwarp();
}

}  // namespace lkg
