/*
 * sg.h -- C ABI of the B200-native (sm_100a) FP64 subgrid kernels (libsg.so).
 *
 * Drop-in boundary for the reference package's kernel layer
 * (reference pkg/src/simdgrid/kernels/compiled.py: the seven numba array
 * kernels).  Every entry point is a batched, stream-ordered mirror of one
 * reference array kernel: plain device pointers, sizes and a cudaStream_t
 * passed as void*; no torch or framework types.  The Python front end
 * (paper_2210_06439_b200/kernels.py) mirrors the reference's Python entry
 * points (kernels/__init__.py:122-267) on top of this ABI; INTEGRATION.md
 * shows the ctypes binding a reference maintainer would add.
 *
 * Conventions
 *  - Return value: SG_OK (0) or an error code; sg_last_error() gives a
 *    thread-local message.  Launches are asynchronous on `stream`.
 *  - Re-entrant: no global mutable state besides read-only constant tables;
 *    concurrent calls on distinct outputs (e.g. one stream per caller) are safe.
 *  - Field views.  A "view" of a cell-centred field is (base, nx, ny, nz, pad,
 *    leaf_stride): `ncomp` components, each a C-contiguous array of dims
 *    (nz+2*pad, ny+2*pad, nx+2*pad) indexed [z][y][x], component stride =
 *    that volume.  Leaf b's interior starts at (pad + 8*cz, pad + 8*cy,
 *    pad + 8*cx) of block b (address base + b*leaf_stride), where (cx,cy,cz)
 *    = leaves[3b..3b+2] (int32, device) or (0,0,0) when leaves == NULL.
 *      batched path : one global padded field, leaf_stride 0, leaf coords;
 *      drop-in path : a stack of per-subgrid blocks, leaf_stride = block
 *                     volume * ncomp, leaves == NULL.
 *  - Validation (before any CUDA call): NULL required pointers, negative or
 *    zero interior dims, negative pads/strides, bad halo/order/precision ->
 *    SG_EINVAL with the argument named in sg_last_error().  An empty batch
 *    (nleaves <= 0) is a no-op.  Preconditions the library cannot check
 *    without reading device memory: leaf coordinates lie inside the view
 *    (0 <= 8*c < interior dim per axis) and buffers have the documented sizes.
 *  - Arithmetic is FP64, IEEE round-to-nearest, no FMA contraction, the
 *    reference's association and accumulation order: bit-identical results.
 */
#ifndef SG_H
#define SG_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define SG_ABI_VERSION 4

/* precision modes of the gravity kernels:
 *  SG_PREC_EXACT  bit-identical to the reference (no FMA, reference order)
 *  SG_PREC_FMA    FMA-contracted / re-associated far terms (north_star's
 *                 FP64 FMA design); within 1e-12 max-norm relative per output
 *                 component of the exact results (tests/test_gpu_fma.py) */
#define SG_PREC_EXACT 0
#define SG_PREC_FMA 1

#define SG_OK 0
#define SG_EINVAL 1
#define SG_ECUDA 2

int sg_abi_version(void);
const char *sg_last_error(void);
int sg_device_sm_count(void);
/* kernels launched by this library so far (all threads, monotonic) */
unsigned long long sg_launch_count(void);

/* ---------------------------------------------------------------- gravity */

/* Replaces compiled.cluster_aggregate (compiled.py:324-352).
 * mass: `nleaf` stacked C-contiguous arrays of dims (mnz, mny, mnx) (all
 * even); clusters: matching (mnz/2, mny/2, mnx/2, 4) arrays of
 * {M, Dx, Dy, Dz}.  Run on a whole padded global mass field (nleaf = 1) the
 * result is bitwise equal to the reference's per-neighbourhood aggregation. */
int sg_cluster_aggregate(const double *mass, int64_t mnx, int64_t mny, int64_t mnz, int64_t nleaf,
                         double dx, double *clusters, void *stream);

/* Replaces compiled.monopole_kernel_impl (compiled.py:281-321) called by
 * kernels.monopole_kernel (kernels/__init__.py:205-221).
 * mass view (pad >= halo), halo = gravity_halo(theta) <= 8; rad2 and eps2
 * computed as kernels/__init__.py:215-218.  out view: 4 components
 * (phi, gx, gy, gz), pad 0, dims (onx, ony, onz). */
int sg_p2p(const double *mass, int64_t nx, int64_t ny, int64_t nz, int32_t pad, int64_t leaf_stride,
           const int32_t *leaves, int64_t nleaves, double dx, double rad2, double eps2, int32_t halo,
           double *out, int64_t onx, int64_t ony, int64_t onz, int64_t out_leaf_stride, int32_t precision,
           void *stream);

/* Replaces compiled.multipole_kernel_impl (compiled.py:355-451) called by
 * kernels.multipole_prepare/multipole_kernel (kernels/__init__.py:224-261).
 * mass view with even pad >= 8 (near-field cells), clusters from
 * sg_cluster_aggregate over the same padded array (cluster_leaf_stride in
 * doubles for stacked blocks, else 0), order in {0,1}, flat interior target
 * range [i0, i1) (the reference's run(i0, i1) chunk), out view as sg_p2p.
 * workspace: device scratch of >= sg_m2l_workspace_bytes(nleaves) bytes
 * (near-field partial sums, or for nleaves <= 4 the per-(target, cluster)
 * terms of the latency mode, 28 MB per subgrid; contents are not an output).
 * One workspace per concurrently running call (per stream).  Results are
 * independent of the launch shape: batches of <= 12 subgrids run a latency
 * mode (a fused producer / ordered-chain kernel, 64 CTAs per subgrid -- 64
 * two-CTA clusters when a launch carries one subgrid -- with a
 * per-device cached geometry table built on first use of a (dx, rad2, eps2)
 * key -- that first call synchronises `stream`; while `stream` is being
 * captured, or outside the small-near regime, batches of <= 4 run a term
 * kernel over 144 CTAs per subgrid plus an ordered reduction instead).  The fused kernel is
 * launched with programmatic dependent launch: it may begin while the
 * previous kernel on `stream` drains and reads no input before that kernel
 * has completed.  Larger batches run a persistent kernel (two mirror-paired
 * targets per thread in the exact mode); all give the same bits. */
int64_t sg_m2l_workspace_bytes(int64_t nleaves);
int sg_m2l(const double *mass, int64_t nx, int64_t ny, int64_t nz, int32_t pad, int64_t leaf_stride,
           const double *clusters, int64_t cluster_leaf_stride, const int32_t *leaves, int64_t nleaves,
           double dx, double rad2, double eps2, int32_t order, int32_t i0, int32_t i1, double *out,
           int64_t onx, int64_t ony, int64_t onz, int64_t out_leaf_stride, double *workspace,
           int64_t workspace_bytes, int32_t precision, void *stream);

/* ------------------------------------------------------------------ hydro */

/* Replaces compiled.reconstruct_kernel (compiled.py:31-102) called by
 * kernels.reconstruct (kernels/__init__.py:122-136).  U view: 5 components
 * (rho, sx, sy, sz, E), pad >= 2 with ghosts filled.  Q: [nleaves][5][26][10][10][10]. */
int sg_reconstruct(const double *U, int64_t nx, int64_t ny, int64_t nz, int32_t pad, int64_t leaf_stride,
                   const int32_t *leaves, int64_t nleaves, double floor_, double *Q, void *stream);

/* Replaces compiled.flux_kernel (compiled.py:105-262) called by kernels.flux
 * (kernels/__init__.py:150-162).  FX [B][5][8][8][9], FY [B][5][8][9][8],
 * FZ [B][5][9][8][8], smax[B]; err[B] = 0xFFFFFFFF or the reference's first
 * error in loop order packed as key<<12 | code<<10 | cell (code 1 density,
 * 2 pressure; cell = (z*10+y)*10+x in Q coordinates).  latch (nullable):
 * latch[b] = min(latch[b], err[b]) so multi-iteration device runs can be
 * checked once.  gate (nullable) + iter: first-failing-iteration gating for
 * multi-iteration runs (the reference raises after the first failing hydro
 * iteration, driver.py:83-88 / 173-174): a failing leaf does
 * prev = atomicMin(gate, iter) and latches only if prev >= iter, so once an
 * iteration has failed, later iterations (stream-ordered launches with a
 * larger iter) record nothing and *gate names the failing iteration. */
int sg_flux(const double *Q, int64_t nleaves, double gamma, double *FX, double *FY, double *FZ,
            double *smax, uint32_t *err, uint32_t *latch, int32_t *gate, int32_t iter, void *stream);

/* Replaces the legacy straight-line flux (kernels/legacy.py:63-146; the
 * reference's legacy reconstruct is value-identical to reconstruct_kernel).
 * Outputs as sg_flux; err packs ((((axis*8+i)*9+j)*9+k)*9+q)*2 + check with
 * the LEFT cell, the legacy kernel's convention. */
int sg_flux_legacy(const double *Q, int64_t nleaves, double gamma, double *FX, double *FY, double *FZ,
                   double *smax, uint32_t *err, uint32_t *latch, int32_t *gate, int32_t iter, void *stream);

/* Fused reconstruct + flux for the batched step: same outputs, smax, err and
 * latch as sg_reconstruct followed by sg_flux (bit-identical), without
 * materialising Q.  U view as sg_reconstruct. */
int sg_hydro_fused(const double *U, int64_t nx, int64_t ny, int64_t nz, int32_t pad, int64_t leaf_stride,
                   const int32_t *leaves, int64_t nleaves, double floor_, double gamma, double *FX, double *FY,
                   double *FZ, double *smax, uint32_t *err, uint32_t *latch, int32_t *gate, int32_t iter,
                   void *stream);

/* Replaces compiled.hydro_update_kernel (compiled.py:265-278) plus the checks
 * of kernels.hydro_update (kernels/__init__.py:165-188), in place on the U
 * view.  dt from *dt_dev when non-NULL (device-computed, graph-capturable),
 * else `dt`; dtdx = dt/dx on device.  smax (flux max speed) may be NULL to
 * skip the CFL check.  status[b] = 0xFFFFFFFF ok, else kind<<16 | detail:
 * kind 0 dt<=0, 1 CFL violation, 2 rho<=0/NaN at interior cell detail,
 * 3 E<=0/NaN at cell detail (first in (z,y,x) order, rho before E).
 * latch, gate, iter (nullable) as for sg_flux.  err_info (nullable,
 * [B][2]): when leaf b latches, err_info[b] = {smax[b], dt} of that
 * iteration, so the reference's CFL message can be rebuilt after later
 * iterations have overwritten smax and dt. */
int sg_hydro_update(double *U, int64_t nx, int64_t ny, int64_t nz, int32_t pad, int64_t leaf_stride,
                    const int32_t *leaves, int64_t nleaves, const double *FX, const double *FY,
                    const double *FZ, const double *smax, const double *dt_dev, double dt, double dx,
                    double cfl, uint32_t *status, uint32_t *latch, int32_t *gate, int32_t iter,
                    double *err_info, void *stream);

/* Replaces compiled.max_wavespeed_kernel (compiled.py:454-480) called by
 * kernels.max_wavespeed (kernels/__init__.py:264-267): smax[b] per leaf. */
int sg_max_wavespeed(const double *U, int64_t nx, int64_t ny, int64_t nz, int32_t pad, int64_t leaf_stride,
                     const int32_t *leaves, int64_t nleaves, double gamma, double pfloor, double *smax,
                     void *stream);

/* driver.py:170-171: s_pre = max over leaves (values >= 0), then
 * dt = cfl*dx/(3*s_pre), both on device. */
int sg_max_reduce(const double *vals, int64_t n, double *out, void *stream);
int sg_dt_from_smax(const double *s_pre, double cfl, double dx, double *dt, void *stream);

/* ------------------------------------------------------------------- grid */

/* octree.exchange_ghosts / source_cube on a device-resident padded global
 * field (octree.py:149-214): fill pad cells of `ncomp` components from the
 * periodic image along the axes in wrap_mask (bit0 x, bit1 y, bit2 z).  In
 * z-slab mode (wrap_mask = 3) z-halo planes come from the neighbour ranks
 * and only their x/y pads are filled here. */
int sg_fill_periodic(double *field, int64_t ncomp, int64_t nx, int64_t ny, int64_t nz, int32_t pad,
                     int32_t wrap_mask, void *stream);

/* Batched octree.source_cube (octree.py:186-214) / ghost-filled 12^3 blocks:
 * out[b][c][z][y][x] for the (8+2*halo)^3 box around leaf b's interior,
 * from any field view with pad >= halo (pads filled). */
int sg_gather_blocks(const double *field, int64_t nx, int64_t ny, int64_t nz, int32_t pad, int64_t leaf_stride,
                     const int32_t *leaves, int64_t nleaves, int64_t ncomp, int32_t halo, double *out,
                     void *stream);

/* driver.py:165-166: dst interior (pad dst_pad) = src component 0 interior
 * (pad src_pad) * scale, with scale = dx**3. */
int sg_scale_copy(double *dst, int32_t dst_pad, const double *src, int32_t src_pad, int64_t nx, int64_t ny,
                  int64_t nz, double scale, void *stream);

/* --------------------------------------------------- per-subgrid drop-in */

/* One SubGrid per call, HOST arrays in and out (the reference's Python entry
 * points, kernels/__init__.py:122-267, take and fill numpy arrays).  Each
 * call stages through per-thread pinned and device buffers: one memcpy into
 * pinned memory, one H2D copy, the batched kernel(s) with nleaves = 1, one
 * D2H copy and one synchronisation of `stream`.  Same bits as the batched
 * entry points.  U: (rho, sx, sy, sz, E) stacked (5, 12, 12, 12) blocks with
 * ghost width 2; out: (phi, gx, gy, gz) interiors as (4, 8, 8, 8). */

/* kernels.max_wavespeed (kernels/__init__.py:264-267). */
int sg_dropin_max_wavespeed(const double *U, double gamma, double pfloor, double *smax, void *stream);
/* kernels.monopole_kernel (kernels/__init__.py:205-221): cube = source_cube(sources, "mass", halo),
 * (8+2*halo)^3. */
int sg_dropin_monopole(const double *cube, int32_t halo, double dx, double rad2, double eps2, int32_t precision,
                       double *out, void *stream);
/* kernels.multipole_prepare + run(i0, i1) (kernels/__init__.py:224-261): cube = source_cube(sources, "mass", 8),
 * 24^3; clusters are aggregated on the device; only targets [i0, i1) of out are written. */
int sg_dropin_multipole(const double *cube, double dx, double rad2, double eps2, int32_t order, int32_t i0,
                        int32_t i1, int32_t precision, double *out, void *stream);
/* kernels.reconstruct (kernels/__init__.py:122-136): Q is a DEVICE buffer of 5*26*10^3 doubles (it stays on
 * the device for the following flux call). */
int sg_dropin_reconstruct(const double *U, double floor_, double *Q, void *stream);
/* kernels.flux (kernels/__init__.py:150-162): Q, FX, FY, FZ DEVICE buffers; *smax and *err (sg_flux's
 * status word) returned on the host. */
int sg_dropin_flux(const double *Q, double gamma, double *FX, double *FY, double *FZ, double *smax, uint32_t *err,
                   void *stream);
/* kernels.hydro_update (kernels/__init__.py:165-188) without the CFL check (done by the caller on the host):
 * U (host, in/out), FX/FY/FZ DEVICE buffers; *status as sg_hydro_update's. */
int sg_dropin_hydro_update(double *U, const double *FX, const double *FY, const double *FZ, double dt, double dx,
                           double cfl, uint32_t *status, void *stream);

/* ------------------------------------------------------------ measurement */

/* FP64 pipe microbenchmark (roofline denominator): mode 0 DFMA chains,
 * mode 1 DADD chains; *flops_out = FLOPs issued (DFMA counted as 2). */
int sg_fp64_peak(int mode, int iters, double *sink, int64_t *flops_out, void *stream);

#ifdef __cplusplus
}
#endif

#endif /* SG_H */
