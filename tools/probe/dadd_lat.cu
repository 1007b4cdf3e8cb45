// Dependent-latency probe: cycles per dependent DADD / DMUL / LDS->DADD
// chains on one warp (clock64), to size the latency-mode M2L floor
// (1728 ordered adds per target, compiled.py:443-446).
#include <cstdio>
#include <cuda_runtime.h>
__global__ void chain(const double* in, double* out, long long* cyc, int n) {
    __shared__ double s[2048];
    for (int i = threadIdx.x; i < 2048; i += blockDim.x) s[i] = in[i];
    __syncthreads();
    double a = in[threadIdx.x], b = in[threadIdx.x + 1];
    long long t0 = clock64();
#pragma unroll 16
    for (int i = 0; i < n; ++i) a = __dadd_rn(a, b);
    long long t1 = clock64();
    double m = a;
#pragma unroll 16
    for (int i = 0; i < n; ++i) m = __dmul_rn(m, b);
    long long t2 = clock64();
    double c = 0.0;
#pragma unroll 16
    for (int i = 0; i < n; ++i) c = __dadd_rn(c, s[(i * 8 + threadIdx.x) & 2047]);
    long long t3 = clock64();
    out[threadIdx.x] = a + m + c;
    if (threadIdx.x == 0) { cyc[0] = t1 - t0; cyc[1] = t2 - t1; cyc[2] = t3 - t2; }
}
int main() {
    const int n = 1728 * 4;
    double *in, *out; long long* cyc;
    cudaMalloc(&in, 4096 * 8); cudaMalloc(&out, 4096 * 8); cudaMalloc(&cyc, 64);
    cudaMemset(in, 0, 4096 * 8);
    for (int w = 0; w < 3; ++w) chain<<<1, 32>>>(in, out, cyc, n);
    long long h[3];
    cudaMemcpy(h, cyc, sizeof h, cudaMemcpyDeviceToHost);
    printf("cycles per dependent op: dadd %.2f dmul %.2f lds+dadd %.2f\n", (double)h[0] / n, (double)h[1] / n,
           (double)h[2] / n);
    cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
    // empty-kernel launch-to-launch time on one stream
    for (int k = 0; k < 2; ++k) {
        cudaEventRecord(e0);
        for (int i = 0; i < 100; ++i) chain<<<1, 32>>>(in, out, cyc, 1);
        cudaEventRecord(e1); cudaEventSynchronize(e1);
        float ms; cudaEventElapsedTime(&ms, e0, e1);
        if (k) printf("back-to-back tiny launch: %.2f us each\n", ms * 10);
    }
    return 0;
}
