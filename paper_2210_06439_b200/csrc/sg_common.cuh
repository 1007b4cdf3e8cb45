// Shared helpers for the sm_100a subgrid kernels.
//
// Arithmetic contract (reference pkg/src/simdgrid/kernels/compiled.py:1-17):
// every FP64 operation on the data path is written with the explicit
// round-to-nearest intrinsics below, so no multiply-add can ever be
// contracted into a DFMA (the library is also built with -fmad=false), IEEE
// sqrt/div are the CUDA FP64 defaults, expressions keep the reference's
// association, and every per-output accumulation runs in the reference's
// sequential order.  Together this makes the CUDA results bit-identical to
// the reference (tests/test_gpu_*.py check it against golden digests).
#pragma once

#include <cuda_runtime.h>
#include <stdint.h>
#ifdef SG_DEBUG_BOUNDS
#include <cstdio>
#endif

namespace sg {

constexpr int NIN = 8;    // interior cells per subgrid axis
constexpr int NRC = 10;   // reconstruction region width (interior + 1 ring)
constexpr int NDIR = 26;  // lattice directions
constexpr int NVAR = 5;   // rho, sx, sy, sz, E

__device__ __forceinline__ double add(double a, double b) { return __dadd_rn(a, b); }
__device__ __forceinline__ double sub(double a, double b) { return __dsub_rn(a, b); }
__device__ __forceinline__ double mul(double a, double b) { return __dmul_rn(a, b); }
__device__ __forceinline__ double dvd(double a, double b) { return __ddiv_rn(a, b); }
__device__ __forceinline__ double dsqrt(double a) { return __dsqrt_rn(a); }

// A strided view of one or more cell-centred fields.
//   element(b, comp, z, y, x) = base[b*leaf_stride + comp*comp_stride
//                                     + (oz+z)*sz + (oy+y)*sy + (ox+x)]
// where (ox, oy, oz) = pad + 8*(cx, cy, cz) - halo for leaf b with
// coordinates leaves[3b..3b+2] (or (0,0,0) when leaves is null).  A global
// padded field (batched path) uses leaf_stride = 0 and leaf coordinates; a
// stack of per-subgrid blocks (drop-in path) uses leaf_stride = block volume
// and no coordinates.
struct FieldView {
    const double* base;
    int64_t sy, sz, comp_stride, leaf_stride;
    int32_t pad;
};

__host__ inline FieldView make_view(const double* base, int64_t nx, int64_t ny, int64_t nz,
                                    int32_t pad, int64_t leaf_stride) {
    FieldView v;
    v.base = base;
    v.sy = nx + 2 * pad;
    v.sz = v.sy * (ny + 2 * pad);
    v.comp_stride = v.sz * (nz + 2 * pad);
    v.leaf_stride = leaf_stride;
    v.pad = pad;
    return v;
}

// Debug builds (-DSG_DEBUG_BOUNDS, tools/debug_bounds.sh) trap on any
// violated index precondition: the compute-sanitizer stand-in on pools
// where the sanitizer is unavailable.  Release builds compile them out.
#ifdef SG_DEBUG_BOUNDS
#define SG_DASSERT(c)                                                                  \
    do {                                                                               \
        if (!(c)) {                                                                    \
            printf("sg bounds check failed: %s (%s:%d)\n", #c, __FILE__, __LINE__);   \
            __trap();                                                                  \
        }                                                                              \
    } while (0)
#else
#define SG_DASSERT(c) \
    do {              \
    } while (0)
#endif

// Pointer to cell (0,0,0) of the box starting `halo` cells before leaf b's
// interior origin.
__device__ __forceinline__ const double* leaf_origin(const FieldView& v, const int32_t* leaves,
                                                     int64_t b, int halo) {
    int64_t cx = 0, cy = 0, cz = 0;
    if (leaves) {
        cx = leaves[3 * b + 0];
        cy = leaves[3 * b + 1];
        cz = leaves[3 * b + 2];
    }
    int64_t ox = v.pad + NIN * cx - halo, oy = v.pad + NIN * cy - halo, oz = v.pad + NIN * cz - halo;
    // the (8 + 2 halo)^3 box lies inside the padded view (padded dims from the pitches)
    SG_DASSERT(ox >= 0 && oy >= 0 && oz >= 0);
    SG_DASSERT(ox + NIN + 2 * halo <= v.sy);
    SG_DASSERT(oy + NIN + 2 * halo <= v.sz / v.sy);
    SG_DASSERT(oz + NIN + 2 * halo <= v.comp_stride / v.sz);
    return v.base + b * v.leaf_stride + oz * v.sz + oy * v.sy + ox;
}

__device__ __forceinline__ bool signbit_d(double v) {
    return __double_as_longlong(v) < 0;
}

int sm_count();  // SMs of the current device (cached, sg_gravity.cu)

}  // namespace sg

// error reporting shared by every C-ABI entry point
void sg_set_error(const char* fmt, ...);
void sg_count_launch(int n);
int sg_check_launch(const char* what);
int sg_check_view(const char* fn, const char* name, const void* base, int64_t nx, int64_t ny, int64_t nz,
                  int32_t pad, int64_t leaf_stride);
int sg_check_ptr(const char* fn, const char* name, const void* p);
#define SG_TRY(expr)          \
    do {                      \
        int sg_rc_ = (expr);  \
        if (sg_rc_) return sg_rc_; \
    } while (0)
