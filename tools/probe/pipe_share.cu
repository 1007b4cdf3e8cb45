// Does FP64 work on other SM sub-partitions slow a dependent DADD chain?
// warp 0: dependent chain (clock64); warps 1..W-1: independent DMUL streams.
#include <cstdio>
#include <cstdlib>
#include <cuda_runtime.h>
__global__ void k(const double* in, double* out, long long* cyc, int n, int busy_iters) {
    const int w = threadIdx.x >> 5, lane = threadIdx.x & 31;
    if (w == 0) {
        double a = in[lane], b = in[lane + 1];
        long long t0 = clock64();
#pragma unroll 16
        for (int i = 0; i < n; ++i) a = __dadd_rn(a, b);
        long long t1 = clock64();
        out[lane] = a;
        if (lane == 0) cyc[0] = t1 - t0;
    } else {
        double x0 = in[lane] + 1, x1 = x0 + 1, x2 = x0 + 2, x3 = x0 + 3, m = 1.0000001;
        for (int i = 0; i < busy_iters; ++i) {
            x0 = __dmul_rn(x0, m); x1 = __dmul_rn(x1, m); x2 = __dmul_rn(x2, m); x3 = __dmul_rn(x3, m);
        }
        out[threadIdx.x] = x0 + x1 + x2 + x3;
    }
}
int main() {
    double *in, *out; long long* cyc;
    cudaMalloc(&in, 4096 * 8); cudaMalloc(&out, 4096 * 8); cudaMalloc(&cyc, 64);
    cudaMemset(in, 0, 4096 * 8);
    const int n = 1728 * 4;
    for (int nw : {1, 2, 4, 8, 16}) {
        long long h = 0;
        for (int r = 0; r < 3; ++r) k<<<1, 32 * nw>>>(in, out, cyc, n, 20000);
        cudaMemcpy(&h, cyc, 8, cudaMemcpyDeviceToHost);
        printf("warps %2d: chain cycles/add %.2f\n", nw, (double)h / n);
    }
    return 0;
}
