// Per-subgrid drop-in entry points (the reference's Python kernel API,
// kernels/__init__.py:122-267, one SubGrid per call).  Host arrays in and
// out, staged through per-thread MAPPED pinned memory: inputs that a kernel
// reads once (max_wavespeed, hydro_update, the P2P cube) and every small
// output (gravity interiors, smax, status words) are read / written by the
// kernel in place over the host link (zero-copy: no copy launches); inputs
// read many times (the 24^3 M2L cube, reconstruct's stencil) get one H2D
// copy into per-thread device staging.  One stream synchronisation per call
// (none for reconstruct, whose output stays on the device).  The kernels are
// the batched ones (nleaves = 1): the same bits as the batched path.
#include <cstring>

#include "sg_common.cuh"
#include "../../include/sg.h"

namespace sg {
namespace {

constexpr int64_t U_DOUBLES = 5 * 12 * 12 * 12;        // stacked (rho, sx, sy, sz, E) block
constexpr int64_t OUT_DOUBLES = 4 * 512;               // phi, gx, gy, gz interiors

// grow-only staging owned by the calling thread, one set per device
struct Stage {
    int dev = -1;
    char* h = nullptr;   // pinned, mapped
    char* hd = nullptr;  // its device alias
    size_t hcap = 0;
    char* d = nullptr;
    size_t dcap = 0;
    cudaEvent_t pending = nullptr;  // last async use of h (reconstruct's H2D)
    bool armed = false;
    ~Stage() {
        // process teardown may already have unloaded the runtime: ignore errors
        if (h) cudaFreeHost(h);
        if (d) cudaFree(d);
        if (pending) cudaEventDestroy(pending);
    }
};
constexpr int MAX_DEV = 16;
thread_local Stage g_stage[MAX_DEV];

int stage_for(size_t hbytes, size_t dbytes, Stage** out) {
    int dev = 0;
    if (cudaGetDevice(&dev) != cudaSuccess || dev < 0 || dev >= MAX_DEV) {
        sg_set_error("sg_dropin: no usable CUDA device");
        return SG_ECUDA;
    }
    Stage& s = g_stage[dev];
    s.dev = dev;
    if (s.armed) {  // the previous call's async H2D must have read h
        cudaEventSynchronize(s.pending);
        s.armed = false;
    }
    if (!s.pending && cudaEventCreateWithFlags(&s.pending, cudaEventDisableTiming) != cudaSuccess) {
        cudaGetLastError();
        sg_set_error("sg_dropin: event creation failed");
        return SG_ECUDA;
    }
    if (s.hcap < hbytes) {
        if (s.h) cudaFreeHost(s.h);
        s.h = s.hd = nullptr;
        s.hcap = 0;
        if (cudaHostAlloc(reinterpret_cast<void**>(&s.h), hbytes, cudaHostAllocMapped) != cudaSuccess ||
            cudaHostGetDevicePointer(reinterpret_cast<void**>(&s.hd), s.h, 0) != cudaSuccess) {
            cudaGetLastError();
            sg_set_error("sg_dropin: mapped pinned staging of %zu bytes failed", hbytes);
            return SG_ECUDA;
        }
        s.hcap = hbytes;
    }
    if (dbytes && s.dcap < dbytes) {
        if (s.d) cudaFree(s.d);  // synchronises the device: only when growing
        s.d = nullptr;
        s.dcap = 0;
        if (cudaMalloc(reinterpret_cast<void**>(&s.d), dbytes) != cudaSuccess) {
            cudaGetLastError();
            sg_set_error("sg_dropin: device staging of %zu bytes failed", dbytes);
            return SG_ECUDA;
        }
        s.dcap = dbytes;
    }
    *out = &s;
    return SG_OK;
}

size_t up(size_t b) { return (b + 255) & ~size_t(255); }

int finish(const char* fn, cudaStream_t st) {
    const cudaError_t e = cudaStreamSynchronize(st);
    if (e != cudaSuccess) {
        sg_set_error("%s: %s", fn, cudaGetErrorString(e));
        return SG_ECUDA;
    }
    return SG_OK;
}

#define SG_CU(fn, expr)                                                   \
    do {                                                                  \
        const cudaError_t e_ = (expr);                                    \
        if (e_ != cudaSuccess) {                                          \
            sg_set_error("%s: %s", fn, cudaGetErrorString(e_));           \
            return SG_ECUDA;                                              \
        }                                                                 \
    } while (0)

}  // namespace
}  // namespace sg

using namespace sg;

// the 8^3 interiors of the 5 stacked (12, 12, 12) blocks, row by row:
// what max_wavespeed reads and hydro_update reads and writes (20 KB of 69 KB)
static void copy_interiors(double* dst, const double* src) {
    for (int v = 0; v < 5; ++v)
        for (int z = 2; z < 10; ++z)
            for (int y = 2; y < 10; ++y) {
                const int64_t o = ((int64_t)(v * 12 + z) * 12 + y) * 12 + 2;
                std::memcpy(dst + o, src + o, 8 * sizeof(double));
            }
}

extern "C" {

int sg_dropin_max_wavespeed(const double* U, double gamma, double pfloor, double* smax, void* stream) {
    SG_TRY(sg_check_ptr("sg_dropin_max_wavespeed", "U", U));
    SG_TRY(sg_check_ptr("sg_dropin_max_wavespeed", "smax", smax));
    const cudaStream_t st = (cudaStream_t)stream;
    const size_t ub = sizeof(double) * U_DOUBLES;
    Stage* s;
    SG_TRY(stage_for(up(ub) + 64, 0, &s));
    copy_interiors(reinterpret_cast<double*>(s->h), U);
    // zero-copy: the kernel reads each interior cell once from the mapped
    // buffer and writes the one result there
    double* hS = reinterpret_cast<double*>(s->h + up(ub));
    SG_TRY(sg_max_wavespeed(reinterpret_cast<double*>(s->hd), 8, 8, 8, 2, 0, nullptr, 1, gamma, pfloor,
                            reinterpret_cast<double*>(s->hd + up(ub)), stream));
    SG_TRY(finish("sg_dropin_max_wavespeed", st));
    *smax = *reinterpret_cast<volatile double*>(hS);
    return SG_OK;
}

int sg_dropin_monopole(const double* cube, int32_t halo, double dx, double rad2, double eps2, int32_t precision,
                       double* out, void* stream) {
    SG_TRY(sg_check_ptr("sg_dropin_monopole", "cube", cube));
    SG_TRY(sg_check_ptr("sg_dropin_monopole", "out", out));
    if (halo < 0 || halo > 8) {
        sg_set_error("sg_dropin_monopole: halo %d must be in [0, 8]", halo);
        return SG_EINVAL;
    }
    const cudaStream_t st = (cudaStream_t)stream;
    const int64_t S = 8 + 2 * halo;
    const size_t cb = sizeof(double) * S * S * S, ob = sizeof(double) * OUT_DOUBLES;
    Stage* s;
    SG_TRY(stage_for(up(cb) + ob, 0, &s));
    std::memcpy(s->h, cube, cb);
    // zero-copy both ways: the kernel stages the cube into shared memory once
    // and writes each output once
    SG_TRY(sg_p2p(reinterpret_cast<double*>(s->hd), 8, 8, 8, halo, 0, nullptr, 1, dx, rad2, eps2, halo,
                  reinterpret_cast<double*>(s->hd + up(cb)), 8, 8, 8, 0, precision, stream));
    SG_TRY(finish("sg_dropin_monopole", st));
    std::memcpy(out, s->h + up(cb), ob);
    return SG_OK;
}

int sg_dropin_multipole(const double* cube, double dx, double rad2, double eps2, int32_t order, int32_t i0,
                        int32_t i1, int32_t precision, double* out, void* stream) {
    SG_TRY(sg_check_ptr("sg_dropin_multipole", "cube", cube));
    SG_TRY(sg_check_ptr("sg_dropin_multipole", "out", out));
    const cudaStream_t st = (cudaStream_t)stream;
    const size_t cb = sizeof(double) * 24 * 24 * 24, clb = sizeof(double) * 12 * 12 * 12 * 4,
                 ob = sizeof(double) * OUT_DOUBLES;
    const int64_t wsb = sg_m2l_workspace_bytes(1);
    Stage* s;
    SG_TRY(stage_for(up(cb) + ob, up(cb) + up(clb) + (size_t)wsb, &s));
    std::memcpy(s->h, cube, cb);
    // the near-field masses are re-read by many CTAs: one H2D copy; the
    // outputs are written once, straight into the mapped buffer
    double* dC = reinterpret_cast<double*>(s->d);
    double* dCl = reinterpret_cast<double*>(s->d + up(cb));
    double* dW = reinterpret_cast<double*>(s->d + up(cb) + up(clb));
    double* hO = reinterpret_cast<double*>(s->hd + up(cb));
    SG_CU("sg_dropin_multipole", cudaMemcpyAsync(dC, s->h, cb, cudaMemcpyHostToDevice, st));
    SG_TRY(sg_cluster_aggregate(dC, 24, 24, 24, 1, dx, dCl, stream));
    SG_TRY(sg_m2l(dC, 8, 8, 8, 8, 0, dCl, 0, nullptr, 1, dx, rad2, eps2, order, i0, i1, hO, 8, 8, 8, 0, dW, wsb,
                  precision, stream));
    SG_TRY(finish("sg_dropin_multipole", st));
    // only the computed range is an output (the reference's run(i0, i1))
    const int a = i0 < 0 ? 0 : i0, b = i1 > 512 ? 512 : i1;
    const double* h = reinterpret_cast<const double*>(s->h + up(cb));
    for (int c = 0; c < 4 && a < b; ++c)
        std::memcpy(out + c * 512 + a, h + c * 512 + a, sizeof(double) * (size_t)(b - a));
    return SG_OK;
}

int sg_dropin_reconstruct(const double* U, double floor_, double* Q, void* stream) {
    SG_TRY(sg_check_ptr("sg_dropin_reconstruct", "U", U));
    SG_TRY(sg_check_ptr("sg_dropin_reconstruct", "Q", Q));
    const cudaStream_t st = (cudaStream_t)stream;
    const size_t ub = sizeof(double) * U_DOUBLES;
    Stage* s;
    SG_TRY(stage_for(ub, ub, &s));
    std::memcpy(s->h, U, ub);
    double* dU = reinterpret_cast<double*>(s->d);
    SG_CU("sg_dropin_reconstruct", cudaMemcpyAsync(dU, s->h, ub, cudaMemcpyHostToDevice, st));
    SG_TRY(sg_reconstruct(dU, 8, 8, 8, 2, 0, nullptr, 1, floor_, Q, stream));
    // no synchronisation: Q stays on the device (stream-ordered for the
    // following flux); the next call on this thread waits for the H2D before
    // reusing the staging buffers
    SG_CU("sg_dropin_reconstruct", cudaEventRecord(s->pending, st));
    s->armed = true;
    return SG_OK;
}

int sg_dropin_flux(const double* Q, double gamma, double* FX, double* FY, double* FZ, double* smax, uint32_t* err,
                   void* stream) {
    SG_TRY(sg_check_ptr("sg_dropin_flux", "Q", Q));
    SG_TRY(sg_check_ptr("sg_dropin_flux", "smax", smax));
    SG_TRY(sg_check_ptr("sg_dropin_flux", "err", err));
    const cudaStream_t st = (cudaStream_t)stream;
    Stage* s;
    SG_TRY(stage_for(16, 0, &s));
    SG_TRY(sg_flux(Q, 1, gamma, FX, FY, FZ, reinterpret_cast<double*>(s->hd), reinterpret_cast<uint32_t*>(s->hd + 8),
                   nullptr, nullptr, 0, stream));
    SG_TRY(finish("sg_dropin_flux", st));
    std::memcpy(smax, s->h, 8);
    std::memcpy(err, s->h + 8, 4);
    return SG_OK;
}

int sg_dropin_hydro_update(double* U, const double* FX, const double* FY, const double* FZ, double dt, double dx,
                           double cfl, uint32_t* status, void* stream) {
    SG_TRY(sg_check_ptr("sg_dropin_hydro_update", "U", U));
    SG_TRY(sg_check_ptr("sg_dropin_hydro_update", "status", status));
    const cudaStream_t st = (cudaStream_t)stream;
    const size_t ub = sizeof(double) * U_DOUBLES;
    Stage* s;
    SG_TRY(stage_for(up(ub) + 16, 0, &s));
    copy_interiors(reinterpret_cast<double*>(s->h), U);
    // zero-copy: every interior value is read and rewritten once in place
    SG_TRY(sg_hydro_update(reinterpret_cast<double*>(s->hd), 8, 8, 8, 2, 0, nullptr, 1, FX, FY, FZ, nullptr,
                           nullptr, dt, dx, cfl, reinterpret_cast<uint32_t*>(s->hd + up(ub)), nullptr, nullptr, 0,
                           nullptr, stream));
    SG_TRY(finish("sg_dropin_hydro_update", st));
    copy_interiors(U, reinterpret_cast<const double*>(s->h));
    std::memcpy(status, s->h + up(ub), 4);
    return SG_OK;
}

}  // extern "C"
