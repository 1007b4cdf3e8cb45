// Fixed cost of a latency-shaped launch on B200: event-to-event time of an
// (almost) empty kernel after a busy kernel, by grid / dynamic shared memory /
// carveout preference -- what the latency-mode M2L pays outside its own work.
#include <cstdio>
#include <cuda_runtime.h>

__global__ void spin(long long cycles) {
    const long long t0 = clock64();
    while (clock64() - t0 < cycles) { }
}

__global__ void __launch_bounds__(512, 1) empty(int* out) {
    extern __shared__ int sm[];
    if (threadIdx.x == 0) sm[0] = blockIdx.x;
    __syncthreads();
    if (threadIdx.x == 0 && sm[0] < 0) out[0] = 1;
}

int main() {
    int* out;
    cudaMalloc(&out, 4);
    cudaEvent_t a, b;
    cudaEventCreate(&a);
    cudaEventCreate(&b);
    cudaFuncSetAttribute(empty, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024);
    const int grids[] = {64, 128};
    const int smems[] = {16, 100 * 1024, 200 * 1024};
    for (int carve = 0; carve < 2; ++carve) {
        if (carve) cudaFuncSetAttribute(spin, cudaFuncAttributePreferredSharedMemoryCarveout, 100);
        for (int g : grids)
            for (int s : smems) {
                float best = 1e9, sum = 0;
                for (int it = 0; it < 20; ++it) {
                    spin<<<1, 32>>>(200000);
                    cudaEventRecord(a);
                    empty<<<g, 512, s>>>(out);
                    cudaEventRecord(b);
                    cudaEventSynchronize(b);
                    float ms;
                    cudaEventElapsedTime(&ms, a, b);
                    if (it >= 4) {
                        best = ms < best ? ms : best;
                        sum += ms;
                    }
                }
                printf("spin carveout %s  grid %3d  smem %6d B: min %.2f us  mean %.2f us\n", carve ? "max-smem" : "default",
                       g, s, best * 1e3, sum / 16 * 1e3);
            }
    }
    printf("%s\n", cudaGetErrorString(cudaGetLastError()));
    return 0;
}
