// FP64 pipe microbenchmark used by bench.py to measure the roofline
// denominator on the box (MEASURED_PEAKS.json carries no FP64 entry).
// mode 0: DFMA chains (FLOP = 2 per op); mode 1: DADD chains (1 per op).
// 8 independent chains per thread, grid = 4 CTAs x 256 threads per SM.
#include "sg_common.cuh"
#include "../../include/sg.h"

namespace sg {

template <int MODE>
__global__ void __launch_bounds__(256) fp64_peak_kernel(int iters, double a, double b, double* sink) {
    double v[8];
#pragma unroll
    for (int i = 0; i < 8; ++i) v[i] = a + (double)(threadIdx.x + i);
#pragma unroll 1
    for (int it = 0; it < iters; ++it) {
#pragma unroll
        for (int k = 0; k < 16; ++k) {
#pragma unroll
            for (int i = 0; i < 8; ++i) {
                if (MODE == 0) v[i] = __fma_rn(v[i], b, a);
                else v[i] = __dadd_rn(v[i], b);
            }
        }
    }
    double s = 0.0;
#pragma unroll
    for (int i = 0; i < 8; ++i) s += v[i];
    if (s == 1234.5) sink[0] = s;  // practically never taken; defeats DCE
}

}  // namespace sg

extern "C" int sg_fp64_peak(int mode, int iters, double* sink, int64_t* flops_out, void* stream) {
    SG_TRY(sg_check_ptr("sg_fp64_peak", "sink", sink));
    SG_TRY(sg_check_ptr("sg_fp64_peak", "flops_out", flops_out));
    if (iters < 0 || (mode != 0 && mode != 1)) {
        sg_set_error("sg_fp64_peak: mode must be 0 or 1 and iters >= 0");
        return SG_EINVAL;
    }
    const int grid = 4 * sg_device_sm_count();
    sg_count_launch(1);
    if (mode == 0)
        sg::fp64_peak_kernel<0><<<grid, 256, 0, (cudaStream_t)stream>>>(iters, 1e-3, 0.999999, sink);
    else
        sg::fp64_peak_kernel<1><<<grid, 256, 0, (cudaStream_t)stream>>>(iters, 1e-3, 1e-9, sink);
    *flops_out = (int64_t)grid * 256 * 8 * 16 * (int64_t)iters * (mode == 0 ? 2 : 1);
    return sg_check_launch("sg_fp64_peak");
}
