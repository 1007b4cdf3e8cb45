// Host round trip of a one-subgrid call: launch a tiny kernel that writes one
// double into mapped pinned memory, then wait for it by
//   (a) cudaStreamSynchronize, (b) polling cudaStreamQuery, (c) spinning on the
//   mapped result word (the kernel fences system-wide before the flag store),
//   (d) cudaEventSynchronize on an event recorded after the kernel.
#include <chrono>
#include <cstdio>
#include <cuda_runtime.h>

__global__ void tiny(double* out, volatile unsigned* flag, unsigned seq) {
    if (threadIdx.x == 0) {
        out[0] = 1.0 + seq;
        __threadfence_system();
        *flag = seq;
    }
}

int main() {
    char* h;
    cudaHostAlloc((void**)&h, 4096, cudaHostAllocMapped);
    char* hd;
    cudaHostGetDevicePointer((void**)&hd, h, 0);
    cudaStream_t st;
    cudaStreamCreateWithFlags(&st, cudaStreamNonBlocking);
    cudaEvent_t ev;
    cudaEventCreateWithFlags(&ev, cudaEventDisableTiming);
    volatile unsigned* flag = reinterpret_cast<volatile unsigned*>(h + 64);
    unsigned seq = 0;
    for (int mode = 0; mode < 4; ++mode) {
        double best = 1e9, sum = 0;
        const int n = 2000;
        for (int it = 0; it < n + 100; ++it) {
            ++seq;
            const auto t0 = std::chrono::steady_clock::now();
            tiny<<<1, 32, 0, st>>>(reinterpret_cast<double*>(hd), reinterpret_cast<volatile unsigned*>(hd + 64), seq);
            if (mode == 0) cudaStreamSynchronize(st);
            if (mode == 1) while (cudaStreamQuery(st) == cudaErrorNotReady) { }
            if (mode == 2) while (*flag != seq) { }
            if (mode == 3) {
                cudaEventRecord(ev, st);
                cudaEventSynchronize(ev);
            }
            const double us = std::chrono::duration<double, std::micro>(std::chrono::steady_clock::now() - t0).count();
            if (it >= 100) {
                sum += us;
                best = us < best ? us : best;
            }
        }
        if (mode == 2) cudaStreamSynchronize(st);
        const char* names[] = {"cudaStreamSynchronize", "cudaStreamQuery spin", "mapped flag spin", "event sync"};
        printf("%-22s launch+wait: mean %.2f us  min %.2f us\n", names[mode], sum / n, best);
    }
    printf("%s\n", cudaGetErrorString(cudaGetLastError()));
    return 0;
}
