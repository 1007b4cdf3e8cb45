// Phase split of the deduplicated fused hydro (clock64 per CTA): X = slopes +
// faces (faces on 8 warps), S = distinct states (all 16 warps), config-5 L=4
// state (uniform-ish U), summed over the CTA's leaves.
#define SG_DD_PROBE
#include "../../paper_2210_06439_b200/csrc/sg_hydro.cu"
#include <cstdio>
#include <vector>
int main() {
    const int L = 4, n = 8 << L, B = 1 << (3 * L), pad = 2;
    const int64_t P = n + 2 * pad, vol = P * P * P;
    std::vector<double> h(5 * vol);
    for (int64_t i = 0; i < vol; ++i) {
        h[i] = 1.0 + 0.3 * ((i * 2654435761u) % 1000) / 1000.0;
        h[vol + i] = h[2 * vol + i] = h[3 * vol + i] = 0.01;
        h[4 * vol + i] = 2.5;
    }
    std::vector<int> lv(3 * B);
    for (int b = 0; b < B; ++b) { lv[3 * b] = b % (n / 8); lv[3 * b + 1] = (b / (n / 8)) % (n / 8); lv[3 * b + 2] = b / ((n / 8) * (n / 8)); }
    double *U, *FX, *FY, *FZ, *smax; uint32_t* err; int* dl;
    cudaMalloc(&U, sizeof(double) * 5 * vol);
    cudaMalloc(&FX, sizeof(double) * B * 5 * 576); cudaMalloc(&FY, sizeof(double) * B * 5 * 576);
    cudaMalloc(&FZ, sizeof(double) * B * 5 * 576); cudaMalloc(&smax, 8 * B); cudaMalloc(&err, 4 * B);
    cudaMalloc(&dl, 4 * 3 * B);
    cudaMemcpy(U, h.data(), sizeof(double) * 5 * vol, cudaMemcpyHostToDevice);
    cudaMemcpy(dl, lv.data(), 4 * 3 * B, cudaMemcpyHostToDevice);
    for (int it = 0; it < 3; ++it) {
        long long z[148][4] = {};
        cudaMemcpyToSymbol(g_dd_probe, z, sizeof z);
        sg_hydro_fused(U, n, n, n, pad, 0, dl, B, 1e-12, 1.4, FX, FY, FZ, smax, err, nullptr, nullptr, 0, nullptr);
        cudaDeviceSynchronize();
        long long p[148][4];
        cudaMemcpyFromSymbol(p, g_dd_probe, sizeof p);
        double x = 0, s = 0, xf = 0;
        for (int b = 0; b < 148; ++b) { x += p[b][0] / 148.0; s += p[b][1] / 148.0; xf += p[b][2] / 148.0; }
        printf("per CTA: X %.0f cycles (planes with faces %.0f), S %.0f cycles; X share %.1f%%\n", x, xf, s, 100 * x / (x + s));
    }
    printf("%s\n", cudaGetErrorString(cudaGetLastError()));
    return 0;
}
