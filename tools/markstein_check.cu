// Exhaustive-style check that q = RN(q0 + r*y), q0 = RN(a*y), r = fma(-q0, b, a),
// y = RN(1/b) equals the IEEE quotient RN(a/b) (the k_energy track division).
// usage: markstein_check [n_per_thread]; prints mismatches per test family.
#include <cstdio>
#include <cstdint>
#include <cstdlib>

__device__ __forceinline__ uint64_t mix(uint64_t x) {
    x ^= x >> 33; x *= 0xff51afd7ed558ccdULL; x ^= x >> 33; x *= 0xc4ceb9fe1a85ec53ULL; x ^= x >> 33;
    return x;
}

__global__ void k(int family, long long n_per, unsigned long long* bad, double* ex) {
    const uint64_t tid = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x;
    unsigned long long nb = 0;
    for (long long it = 0; it < n_per; ++it) {
        const uint64_t h1 = mix(tid * 0x9E3779B97F4A7C15ULL + it * 2 + 1 + family * 0x1234567ULL);
        const uint64_t h2 = mix(h1 + 0x632BE59BD9B4E019ULL);
        double a, b;
        if (family == 0) {  // the pipeline's ranges: |b| in [0.5, 4096], |a| up to 2^24
            b = __longlong_as_double((long long)((h1 & 0x000FFFFFFFFFFFFFULL) |
                                                 ((uint64_t)(1022 + (h1 >> 60) % 13) << 52)));
            a = __longlong_as_double((long long)((h2 & 0x000FFFFFFFFFFFFFULL) |
                                                 ((uint64_t)(1000 + (h2 >> 58) % 48) << 52)));
        } else if (family == 1) {  // b with all-ones / near-ones significands
            const uint64_t m = 0x000FFFFFFFFFFFFFULL ^ (h1 & 0xF);
            b = __longlong_as_double((long long)(m | ((uint64_t)(1023 + (h1 >> 60) % 8) << 52)));
            a = __longlong_as_double((long long)((h2 & 0x000FFFFFFFFFFFFFULL) |
                                                 ((uint64_t)(1010 + (h2 >> 58) % 30) << 52)));
        } else {  // wide exponents, away from overflow / underflow
            b = __longlong_as_double((long long)((h1 & 0x000FFFFFFFFFFFFFULL) |
                                                 ((uint64_t)(523 + (h1 >> 53) % 1000) << 52)));
            a = __longlong_as_double((long long)((h2 & 0x000FFFFFFFFFFFFFULL) |
                                                 ((uint64_t)(523 + (h2 >> 53) % 1000) << 52)));
        }
        if (h1 & (1ULL << 31)) a = -a;
        if (h2 & (1ULL << 31)) b = -b;
        const double y = __ddiv_rn(1.0, b);
        const double q0 = __dmul_rn(a, y);
        const double r = __fma_rn(-q0, b, a);
        const double q = __fma_rn(r, y, q0);
        const double ref = __ddiv_rn(a, b);
        if (__double_as_longlong(q) != __double_as_longlong(ref)) {
            if (nb == 0) { ex[0] = a; ex[1] = b; }
            ++nb;
        }
    }
    if (nb) atomicAdd(bad, nb);
}

int main(int argc, char** argv) {
    const long long n_per = argc > 1 ? atoll(argv[1]) : 4096;
    unsigned long long* bad;
    double* ex;
    cudaMalloc(&bad, 8);
    cudaMalloc(&ex, 16);
    const int blocks = 148 * 16, threads = 256;
    for (int fam = 0; fam < 3; ++fam) {
        cudaMemset(bad, 0, 8);
        k<<<blocks, threads>>>(fam, n_per, bad, ex);
        unsigned long long h = 0;
        double e[2] = {0, 0};
        cudaMemcpy(&h, bad, 8, cudaMemcpyDeviceToHost);
        cudaMemcpy(e, ex, 16, cudaMemcpyDeviceToHost);
        printf("family %d: %lld cases, %llu mismatches%s", fam, (long long)blocks * threads * n_per, h,
               h ? "" : "\n");
        if (h) printf(" (e.g. a=%.17g b=%.17g)\n", e[0], e[1]);
    }
    return cudaDeviceSynchronize() != cudaSuccess;
}
