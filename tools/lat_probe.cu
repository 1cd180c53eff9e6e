// Latency probe: dependent FP64 add chain, dependent double shuffle chain and
// the k_integral step pattern, in clock cycles per operation (one warp).
#include <cstdio>

__global__ void k(double* out, long long* cyc, int n, double a) {
    const int lane = threadIdx.x & 31;
    double x = a + lane, y = 1.0, m1 = 0.0, m2 = 0.0;
    long long t0 = clock64();
    for (int i = 0; i < n; ++i) x = x + a;  // dependent DADD chain
    long long t1 = clock64();
    for (int i = 0; i < n; ++i) y = __shfl_up_sync(0xffffffffu, y, 1) + 1e-30;  // shfl + dadd
    long long t2 = clock64();
    for (int i = 0; i < n; ++i) {  // the integral step: 2 shuffles + 3 dependent adds
        double up = __shfl_up_sync(0xffffffffu, m1, 1), dg = __shfl_up_sync(0xffffffffu, m2, 1);
        const double val = ((up + m1) - dg) + a;
        m2 = m1;
        m1 = val;
    }
    long long t3 = clock64();
    if (lane == 0) {
        cyc[0] = (t1 - t0) / n;
        cyc[1] = (t2 - t1) / n;
        cyc[2] = (t3 - t2) / n;
    }
    out[threadIdx.x] = x + y + m1;
}

int main() {
    double* o;
    long long* c;
    cudaMalloc(&o, 32 * 8);
    cudaMalloc(&c, 3 * 8);
    k<<<1, 32>>>(o, c, 100000, 1e-9);
    long long h[3];
    cudaMemcpy(h, c, sizeof h, cudaMemcpyDeviceToHost);
    printf("cycles per: dadd %lld, shfl.f64+dadd %lld, integral step %lld\n", h[0], h[1], h[2]);
    return 0;
}
