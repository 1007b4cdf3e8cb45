// Timeline probe of the fused latency M2L kernel (clock64 marks per CTA):
// producer row 0 / row 143 done, consumer first row, half-way, end.
#define SG_FL_PROBE
#include "../../paper_2210_06439_b200/csrc/sg_gravity.cu"
#include <cstdio>
#include <vector>
int main(int argc, char** argv) {
    // argv[1] = CTA stride of the consumer CTAs (2 under SG_M2L_FL_SPLIT=1/2: rank 0 = even CTAs)
    const int cs = argc > 1 ? atoi(argv[1]) : 1;
    const int n = 24;
    std::vector<double> h(n * n * n);
    for (int i = 0; i < n * n * n; ++i) h[i] = 1.0 + (i % 7) * 0.1;
    double *mass, *cl, *out;
    cudaMalloc(&mass, sizeof(double) * n * n * n);
    cudaMalloc(&cl, sizeof(double) * 12 * 12 * 12 * 4);
    cudaMalloc(&out, sizeof(double) * 4 * 512);
    cudaMemcpy(mass, h.data(), sizeof(double) * h.size(), cudaMemcpyHostToDevice);
    const double dx = 1.0 / 64, rad = dx / 0.34, eps = 0.5 * dx;
    sg_cluster_aggregate(mass, n, n, n, 1, dx, cl, nullptr);
    std::vector<double> ws(1);
    double* wsd;
    const int64_t wb = sg_m2l_workspace_bytes(1);
    cudaMalloc(&wsd, wb);
    for (int it = 0; it < 5; ++it)
        sg_m2l(mass, 8, 8, 8, 8, 0, cl, 0, nullptr, 1, dx, rad * rad, eps * eps, 1, 0, 512, out, 8, 8, 8, 0, wsd, wb,
               SG_PREC_EXACT, nullptr);
    cudaDeviceSynchronize();
    long long z[256][8] = {};
    cudaMemcpyToSymbol(g_fl_probe, z, sizeof z);
    sg_m2l(mass, 8, 8, 8, 8, 0, cl, 0, nullptr, 1, dx, rad * rad, eps * eps, 1, 0, 512, out, 8, 8, 8, 0, wsd, wb,
           SG_PREC_EXACT, nullptr);
    cudaDeviceSynchronize();
    long long p[256][8];
    cudaMemcpyFromSymbol(p, g_fl_probe, sizeof p);
    double a[8] = {0};
    for (int b = 0; b < 64 * cs; b += cs)
        for (int i = 1; i < 7; ++i) a[i] += (double)(i == 6 ? p[b][6] : p[b][i] - p[b][0]) / 64;
    printf("cycles after start (avg over 64 CTAs): prod row0 %.0f, prod row143 %.0f, cons row0 %.0f, (unused) %.0f, cons end %.0f, cons spin %.0f\n",
           a[1], a[2], a[3], a[4], a[5], a[6]);
    double sw = 0;
    for (int b = 0; b < 64 * cs; b += cs) sw += p[b][7] / 64.0;
    printf("producer 0 ring-slot wait %.0f cycles (12 rows)\n", sw);
    if (cs == 2) {  // rank-1 CTAs: producers of the odd cz planes
        double r143 = 0, w1 = 0, r1 = 0;
        for (int b = 1; b < 128; b += 2) {
            r143 += (double)(p[b][2] - p[b - 1][0]) / 64;
            r1 += (double)(p[b][1] - p[b - 1][0]) / 64;
            w1 += p[b][7] / 64.0;
        }
        printf("rank 1: first row issued %.0f, row 143 issued %.0f cycles after rank 0's start; producer 0 wait %.0f\n",
               r1, r143, w1);
    }
    printf("%s\n", cudaGetErrorString(cudaGetLastError()));
    return 0;
}
