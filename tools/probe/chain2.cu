// Dependent DADD chain variants (cycles per add): constant operand, 24
// distinct register operands, and operands arriving by LDS.128 one batch
// ahead (the latency-mode consumer's pattern).
#include <cstdio>
#include <cstdlib>
#include <cuda_runtime.h>
__global__ void k(const double* in, double* out, long long* cyc, int iters, double getenv_fill) {
    __shared__ double2 s[32 * 64];
    const double fill = getenv_fill;
    for (int i = threadIdx.x; i < 32 * 64; i += blockDim.x) s[i] = make_double2(in[i % 100] + fill, in[(i + 7) % 100] + fill);
    __syncthreads();
    if (threadIdx.x >= 32) return;
    const int lane = threadIdx.x;
    double r[24];
#pragma unroll
    for (int j = 0; j < 24; ++j) r[j] = in[j + lane];
    double a = 0.0;
    long long t0 = clock64();
    for (int it = 0; it < iters; ++it) {
#pragma unroll
        for (int j = 0; j < 24; ++j) a = __dadd_rn(a, r[j]);
    }
    long long t1 = clock64();
    double b = 0.0;
    double2 va[12], vb[12];
#pragma unroll
    for (int j = 0; j < 12; ++j) va[j] = s[(j * 32 + lane) & 2047];
    for (int it = 0; it < iters; it += 2) {
#pragma unroll
        for (int j = 0; j < 12; ++j) vb[j] = s[((it + 1) * 97 + j * 32 + lane) & 2047];
#pragma unroll
        for (int j = 0; j < 12; ++j) { b = __dadd_rn(b, va[j].x); b = __dadd_rn(b, va[j].y); }
#pragma unroll
        for (int j = 0; j < 12; ++j) va[j] = s[((it + 2) * 97 + j * 32 + lane) & 2047];
#pragma unroll
        for (int j = 0; j < 12; ++j) { b = __dadd_rn(b, vb[j].x); b = __dadd_rn(b, vb[j].y); }
    }
    long long t2 = clock64();
    double c = 0.0;
    for (int it = 0; it < iters; ++it) {
#pragma unroll
        for (int j = 0; j < 24; ++j) c = c + r[j];  // plain +, same thing
    }
    long long t3 = clock64();
    // rolling: reload each register right after its two adds
    double d = 0.0;
    double2 w[12];
#pragma unroll
    for (int j = 0; j < 12; ++j) w[j] = s[(j * 32 + lane) & 2047];
    for (int it = 0; it < iters; ++it) {
        const int base = ((it + 1) * 97) & 2047;
#pragma unroll
        for (int j = 0; j < 12; ++j) {
            d = __dadd_rn(d, w[j].x);
            d = __dadd_rn(d, w[j].y);
            w[j] = s[(base + j * 32 + lane) & 2047];
        }
    }
    long long t4 = clock64();
    out[lane] = a + b + c + d;
    if (lane == 0) { cyc[0] = t1 - t0; cyc[1] = t2 - t1; cyc[2] = t3 - t2; cyc[3] = t4 - t3; }
}
int main() {
    double *in, *out; long long* cyc;
    cudaMalloc(&in, 4096 * 8); cudaMalloc(&out, 4096 * 8); cudaMalloc(&cyc, 64);
    cudaMemset(in, 0, 4096 * 8);
    const int iters = 72;
    const int nt = getenv("NT") ? atoi(getenv("NT")) : 32;
    for (int w = 0; w < 3; ++w) k<<<1, nt>>>(in, out, cyc, iters, getenv("FILL") ? atof(getenv("FILL")) : 0.0);
    long long h[4];
    cudaMemcpy(h, cyc, sizeof h, cudaMemcpyDeviceToHost);
    const double n = 24.0 * iters;
    printf("threads %d cycles/add: distinct regs %.2f, lds.128-fed %.2f, plain + %.2f, rolling %.2f\n", nt, h[0] / n, h[1] / n, h[2] / n, h[3] / n);
    return 0;
}
