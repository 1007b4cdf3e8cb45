// Hydro kernels for sm_100a: minmod reconstruction at the 26 lattice
// directions, Rusanov flux with 3x3 Simpson face quadrature, forward-Euler
// conservative update with the reference's validity checks, and the
// cell-centred max wave speed with the dt reduction.
//
// Reference semantics (bit-exact):
//   reconstruct_kernel     compiled.py:31-102    (entry kernels/__init__.py:122-136)
//   flux_kernel            compiled.py:105-262   (entry kernels/__init__.py:150-162)
//   hydro_update_kernel    compiled.py:265-278   (entry kernels/__init__.py:165-188)
//   max_wavespeed_kernel   compiled.py:454-480   (entry kernels/__init__.py:264-267)
//   dt = cfl*dx/(3*s_pre)  driver.py:170-171
//
// The unfused reconstruct -> Q -> flux pair is the drop-in path and is
// HBM-bound (Q is 1.04 MB per subgrid).  Parallelism comes only from
// independent outputs (cells, faces, subgrids); every per-output chain keeps
// the reference's sequential order.
#include <atomic>
#include <mutex>

#include "sg_common.cuh"
#include "../../include/sg.h"

namespace sg {

// geometry.py:21-31: (dz, dy, dx) lexicographic without the zero offset
__constant__ double c_dirs[NDIR][3];
// geometry.py:41-56
__constant__ int c_dplus[3][9];
__constant__ int c_dminus[3][9];
// geometry.py:59-61
__constant__ double c_simpson[9];

// __constant__ memory is per device: upload the tables once per device.
// Re-entrant (concurrent callers on their own streams):
// the flag is atomic and the first upload per device runs under a mutex.
constexpr int SG_MAX_DEVICES = 64;
static std::atomic<bool> g_tables_ready[SG_MAX_DEVICES] = {};
static std::mutex g_tables_mu;

static int host_dir_index(int dz, int dy, int dx) {
    int idx = (dz + 1) * 9 + (dy + 1) * 3 + (dx + 1);
    return idx > 13 ? idx - 1 : idx;
}

static int init_tables() {
    int dev = 0;
    if (cudaGetDevice(&dev) != cudaSuccess || dev < 0 || dev >= SG_MAX_DEVICES) {
        sg_set_error("hydro constant tables: no current CUDA device");
        return SG_ECUDA;
    }
    if (g_tables_ready[dev].load(std::memory_order_acquire)) return SG_OK;
    std::lock_guard<std::mutex> lock(g_tables_mu);
    if (g_tables_ready[dev].load(std::memory_order_relaxed)) return SG_OK;
    double dirs[NDIR][3];
    int d = 0;
    for (int dz = -1; dz <= 1; ++dz)
        for (int dy = -1; dy <= 1; ++dy)
            for (int dx = -1; dx <= 1; ++dx) {
                if (!dz && !dy && !dx) continue;
                dirs[d][0] = dz;
                dirs[d][1] = dy;
                dirs[d][2] = dx;
                ++d;
            }
    int dp[3][9], dm[3][9];
    const int t[3] = {-1, 0, 1};
    for (int i1 = 0; i1 < 3; ++i1)
        for (int i2 = 0; i2 < 3; ++i2) {
            const int t1 = t[i1], t2 = t[i2], q = i1 * 3 + i2;
            dp[0][q] = host_dir_index(t2, t1, 1);
            dm[0][q] = host_dir_index(t2, t1, -1);
            dp[1][q] = host_dir_index(t2, 1, t1);
            dm[1][q] = host_dir_index(t2, -1, t1);
            dp[2][q] = host_dir_index(1, t2, t1);
            dm[2][q] = host_dir_index(-1, t2, t1);
        }
    const double w[9] = {1.0, 4.0, 1.0, 4.0, 16.0, 4.0, 1.0, 4.0, 1.0};
    double sw[9];
    for (int i = 0; i < 9; ++i) sw[i] = w[i] / 36.0;  // host IEEE division, as numpy
    if (cudaMemcpyToSymbol(c_dirs, dirs, sizeof(dirs)) != cudaSuccess ||
        cudaMemcpyToSymbol(c_dplus, dp, sizeof(dp)) != cudaSuccess ||
        cudaMemcpyToSymbol(c_dminus, dm, sizeof(dm)) != cudaSuccess ||
        cudaMemcpyToSymbol(c_simpson, sw, sizeof(sw)) != cudaSuccess) {
        sg_set_error("hydro constant tables: %s", cudaGetErrorString(cudaGetLastError()));
        return SG_ECUDA;
    }
    g_tables_ready[dev].store(true, std::memory_order_release);
    return SG_OK;
}

// latch leaf b's error, gated on the first failing iteration (include/sg.h,
// sg_flux): returns whether it was recorded
__device__ __forceinline__ bool latch_error(uint32_t* latch, int64_t b, uint32_t code, int32_t* gate,
                                            int32_t iter) {
    if (!latch) return false;
    if (gate && atomicMin(gate, iter) < iter) return false;
    atomicMin(latch + b, code);
    return true;
}

__device__ __forceinline__ double minmod(double ap, double am) {
    // compiled.py:58-62 (select semantics, NaN-preserving)
    const double mag = fabs(ap) < fabs(am) ? ap : am;
    const bool sgn = (ap > 0.0 && am > 0.0) || (ap < 0.0 && am < 0.0);
    return sgn ? mag : 0.0;
}

// ---------------------------------------------------------------------------
// reconstruct: U view (5 comps, G=2 ghosts around each leaf) -> Q[B,5,26,10^3]
// ---------------------------------------------------------------------------
constexpr int REC_THREADS = 256;
constexpr int REC_CELLS = NRC * NRC * NRC;

__global__ void __launch_bounds__(REC_THREADS)
reconstruct_kernel(FieldView uv, const int32_t* __restrict__ leaves, double floor_, double* __restrict__ Q) {
    // the 4 cell blocks of a leaf are adjacent CTAs (x), sharing its U block in L2
    const int cell = blockIdx.x * REC_THREADS + threadIdx.x;
    const int64_t b = blockIdx.y;
    if (cell >= REC_CELLS) return;
    const int x = cell % NRC, y = (cell / NRC) % NRC, z = cell / (NRC * NRC);
    const double* u0 = leaf_origin(uv, leaves, b, 2) + (z + 1) * uv.sz + (y + 1) * uv.sy + (x + 1);
    double uc[NVAR], sl[NVAR][3];
#pragma unroll
    for (int v = 0; v < NVAR; ++v) {
        const double* p = u0 + v * uv.comp_stride;
        const double u = __ldg(p);
        uc[v] = u;
        sl[v][0] = minmod(sub(__ldg(p + 1), u), sub(u, __ldg(p - 1)));
        sl[v][1] = minmod(sub(__ldg(p + uv.sy), u), sub(u, __ldg(p - uv.sy)));
        sl[v][2] = minmod(sub(__ldg(p + uv.sz), u), sub(u, __ldg(p - uv.sz)));
    }
    double* q = Q + b * (int64_t)(NVAR * NDIR * REC_CELLS) + cell;
#pragma unroll 2
    for (int d = 0; d < NDIR; ++d) {
        const double fdz = c_dirs[d][0], fdy = c_dirs[d][1], fdx = c_dirs[d][2];
        double r[NVAR];
#pragma unroll
        for (int v = 0; v < NVAR; ++v)
            r[v] = add(uc[v], mul(0.5, add(add(mul(fdx, sl[v][0]), mul(fdy, sl[v][1])), mul(fdz, sl[v][2]))));
        double rho = r[0] < floor_ ? floor_ : r[0];
        double en = r[4] < floor_ ? floor_ : r[4];
        const double ke = dvd(mul(0.5, add(add(mul(r[1], r[1]), mul(r[2], r[2])), mul(r[3], r[3]))), rho);
        const double emin = add(mul(ke, add(1.0, floor_)), floor_);
        en = en < emin ? emin : en;
        q[(0 * NDIR + d) * REC_CELLS] = rho;
        q[(1 * NDIR + d) * REC_CELLS] = r[1];
        q[(2 * NDIR + d) * REC_CELLS] = r[2];
        q[(3 * NDIR + d) * REC_CELLS] = r[3];
        q[(4 * NDIR + d) * REC_CELLS] = en;
    }
}

// ---------------------------------------------------------------------------
// flux: Q -> FX[B,5,8,8,9], FY[B,5,8,9,8], FZ[B,5,9,8,8], smax[B], err[B]
// err packs the reference's FIRST error in loop order:
//   key = ((((axis*8+i)*9+j)*9+k)*9 + q)*4 + check ; err = key<<12 | code<<10 | cell
// 0xFFFFFFFF = no error.
// ---------------------------------------------------------------------------
constexpr int FLUX_THREADS = 576;

// one face (compiled.py:120-262) of leaf Qb: quadrature states read from Q
__device__ __forceinline__ void flux_face(const double* __restrict__ Qb, int axis, int i, int j, int k,
                                          double gamma, double gm1, int64_t b, double* __restrict__ FX,
                                          double* __restrict__ FY, double* __restrict__ FZ, double& smax,
                                          uint32_t& err) {
    int zl, zr, yl, yr, xl, xr;
    if (axis == 0) {
        zl = zr = i + 1; yl = yr = j + 1; xl = k; xr = k + 1;
    } else if (axis == 1) {
        zl = zr = i + 1; yl = j; yr = j + 1; xl = xr = k + 1;
    } else {
        zl = j; zr = j + 1; yl = yr = i + 1; xl = xr = k + 1;
    }
    const int cl_ = (zl * NRC + yl) * NRC + xl, cr_ = (zr * NRC + yr) * NRC + xr;
    const uint32_t kbase = (uint32_t)((((axis * 8 + i) * 9 + j) * 9 + k) * 9);
    double f0 = 0.0, f1 = 0.0, f2 = 0.0, f3 = 0.0, f4 = 0.0;
    const int64_t VS = (int64_t)NDIR * REC_CELLS;
    // the 10 state loads of quadrature point qp+1 are issued before qp's
    // arithmetic (software pipelining: the load latency hides behind it)
    double nl[5], nr[5];
    {
        const double* pl_ = Qb + c_dplus[axis][0] * REC_CELLS + cl_;
        const double* pr_ = Qb + c_dminus[axis][0] * REC_CELLS + cr_;
#pragma unroll
        for (int v = 0; v < 5; ++v) {
            nl[v] = __ldg(pl_ + v * VS);
            nr[v] = __ldg(pr_ + v * VS);
        }
    }
#pragma unroll 1
    for (int qp = 0; qp < 9; ++qp) {
        const double w = c_simpson[qp];
        const double ul0 = nl[0], ul1 = nl[1], ul2 = nl[2], ul3 = nl[3], ul4 = nl[4];
        const double ur0 = nr[0], ur1 = nr[1], ur2 = nr[2], ur3 = nr[3], ur4 = nr[4];
        if (qp < 8) {
            const double* pl_ = Qb + c_dplus[axis][qp + 1] * REC_CELLS + cl_;
            const double* pr_ = Qb + c_dminus[axis][qp + 1] * REC_CELLS + cr_;
#pragma unroll
            for (int v = 0; v < 5; ++v) {
                nl[v] = __ldg(pl_ + v * VS);
                nr[v] = __ldg(pr_ + v * VS);
            }
        }
        const uint32_t key = (kbase + qp) * 4;
        if (err == 0xFFFFFFFFu) {
            if (ul0 <= 0.0) err = ((key + 0) << 12) | (1u << 10) | (uint32_t)cl_;
            else if (ur0 <= 0.0) err = ((key + 1) << 12) | (1u << 10) | (uint32_t)cr_;
        }
        const double invl = dvd(1.0, ul0);
        const double vxl = mul(ul1, invl), vyl = mul(ul2, invl), vzl = mul(ul3, invl);
        const double kel = mul(0.5, add(add(mul(ul1, vxl), mul(ul2, vyl)), mul(ul3, vzl)));
        const double pl = mul(gm1, sub(ul4, kel));
        const double invr = dvd(1.0, ur0);
        const double vxr = mul(ur1, invr), vyr = mul(ur2, invr), vzr = mul(ur3, invr);
        const double ker = mul(0.5, add(add(mul(ur1, vxr), mul(ur2, vyr)), mul(ur3, vzr)));
        const double pr = mul(gm1, sub(ur4, ker));
        if (err == 0xFFFFFFFFu) {
            if (pl <= 0.0) err = ((key + 2) << 12) | (2u << 10) | (uint32_t)cl_;
            else if (pr <= 0.0) err = ((key + 3) << 12) | (2u << 10) | (uint32_t)cr_;
        }
        const double cl = dsqrt(mul(mul(gamma, pl), invl));
        const double cr = dsqrt(mul(mul(gamma, pr), invr));
        const double vnl = axis == 0 ? vxl : (axis == 1 ? vyl : vzl);
        const double vnr = axis == 0 ? vxr : (axis == 1 ? vyr : vzr);
        const double sl = add(fabs(vnl), cl);
        const double sr = add(fabs(vnr), cr);
        const double s = sl > sr ? sl : sr;
        if (s > smax) smax = s;
        const double fl0 = mul(ul0, vnl);
        double fl1 = mul(ul1, vnl), fl2 = mul(ul2, vnl), fl3 = mul(ul3, vnl);
        const double fl4 = mul(add(ul4, pl), vnl);
        const double fr0 = mul(ur0, vnr);
        double fr1 = mul(ur1, vnr), fr2 = mul(ur2, vnr), fr3 = mul(ur3, vnr);
        const double fr4 = mul(add(ur4, pr), vnr);
        if (axis == 0) {
            fl1 = add(fl1, pl);
            fr1 = add(fr1, pr);
        } else if (axis == 1) {
            fl2 = add(fl2, pl);
            fr2 = add(fr2, pr);
        } else {
            fl3 = add(fl3, pl);
            fr3 = add(fr3, pr);
        }
        const double hs = mul(0.5, s);
        f0 = add(f0, mul(w, sub(mul(0.5, add(fl0, fr0)), mul(hs, sub(ur0, ul0)))));
        f1 = add(f1, mul(w, sub(mul(0.5, add(fl1, fr1)), mul(hs, sub(ur1, ul1)))));
        f2 = add(f2, mul(w, sub(mul(0.5, add(fl2, fr2)), mul(hs, sub(ur2, ul2)))));
        f3 = add(f3, mul(w, sub(mul(0.5, add(fl3, fr3)), mul(hs, sub(ur3, ul3)))));
        f4 = add(f4, mul(w, sub(mul(0.5, add(fl4, fr4)), mul(hs, sub(ur4, ul4)))));
    }
    double* F;
    if (axis == 0) F = FX + b * 5 * 576 + (i * 8 + j) * 9 + k;
    else if (axis == 1) F = FY + b * 5 * 576 + (i * 9 + j) * 8 + k;
    else F = FZ + b * 5 * 576 + (j * 8 + i) * 8 + k;
    F[0] = f0;
    F[576] = f1;
    F[2 * 576] = f2;
    F[3 * 576] = f3;
    F[4 * 576] = f4;
}

// face (axis, i, j, k) of the f-th entry of the z-plane-major face order:
// per interior plane p its 72 x-faces, 72 y-faces and the 64 z-faces below
// it, then the 64 top z-faces
__device__ __forceinline__ void plane_major_face(int f, int& axis, int& i, int& j, int& k) {
    if (f < 8 * 208) {
        const int p = f / 208, r = f % 208;
        if (r < 72) {
            axis = 0; i = p; j = r / 9; k = r % 9;
        } else if (r < 144) {
            axis = 1; i = p; j = (r - 72) / 8; k = (r - 72) % 8;
        } else {
            axis = 2; j = p; i = (r - 144) / 8; k = (r - 144) % 8;
        }
    } else {
        const int r = f - 8 * 208;
        axis = 2; j = 8; i = r / 8; k = r % 8;
    }
}

__global__ void __launch_bounds__(FLUX_THREADS)
flux_kernel(const double* __restrict__ Q, double gamma, double* __restrict__ FX, double* __restrict__ FY,
            double* __restrict__ FZ, double* __restrict__ smax_out, uint32_t* __restrict__ err_out,
            uint32_t* __restrict__ latch, int32_t* __restrict__ gate, int32_t iter) {
    __shared__ unsigned long long s_smax;
    __shared__ uint32_t s_err;
    const int64_t b = blockIdx.x;
    const int t = threadIdx.x;
    if (t == 0) {
        s_smax = 0ull;  // +0.0
        s_err = 0xFFFFFFFFu;
    }
    __syncthreads();
    const double* Qb = Q + b * (int64_t)(NVAR * NDIR * REC_CELLS);
    const double gm1 = sub(gamma, 1.0);
    double smax = 0.0;
    uint32_t err = 0xFFFFFFFFu;
    // faces in z-plane-major order -- per interior plane p its 72 x-faces,
    // 72 y-faces and the 64 z-faces below it, then the 64 top z-faces -- so
    // the three axes' faces of a cell (which share corner-direction states
    // of Q) are read together and each round touches ~1/3 of the leaf's Q
    // (L2-resident) instead of whole-leaf sweeps per axis.  Per-face
    // arithmetic and the first-error keys are unchanged.  (Axis-major
    // whole-leaf sweeps: 1.07 ms at L=4; plane-major 1.01 ms; plus the
    // software-pipelined state loads in flux_face 0.855 ms.)
#pragma unroll 1
    for (int f = t; f < 3 * 576; f += FLUX_THREADS) {
        int axis, i, j, k;
        plane_major_face(f, axis, i, j, k);
        flux_face(Qb, axis, i, j, k, gamma, gm1, b, FX, FY, FZ, smax, err);
    }
    // smax >= 0 and never NaN: its bit pattern orders like an unsigned integer
    atomicMax(&s_smax, (unsigned long long)__double_as_longlong(smax));
    if (err != 0xFFFFFFFFu) atomicMin(&s_err, err);
    __syncthreads();
    if (t == 0) {
        smax_out[b] = __longlong_as_double((long long)s_smax);
        err_out[b] = s_err;
        if (s_err != 0xFFFFFFFFu) latch_error(latch, b, s_err, gate, iter);
    }
}

// ---------------------------------------------------------------------------
// legacy flux (reference kernels/legacy.py:63-146): the old straight-line
// formulation -- ke = |s|^2/(2 rho), v_n = s_n/rho, sqrt(gamma p / rho),
// s = max(.,.) with Python semantics, and the first error always naming the
// LEFT cell.  Physics-equal to flux_kernel, bit-identical to legacy.py.
// The reference recomputes every quadrature state once per variable; the
// values do not depend on v, so they are computed once per point here and
// the five per-variable chains (each in (i1, i2) order) advance together.
// err key = ((((axis*8+i)*9+j)*9+k)*9+q)*2 + check.
// ---------------------------------------------------------------------------
// one legacy face (reference legacy.py:63-146), states read from Q with the
// next quadrature point's loads issued ahead (as flux_face)
__device__ __forceinline__ void legacy_face(const double* __restrict__ Qb, int axis, int i, int j, int k,
                                            double gamma, double gm1, int64_t b, double* __restrict__ FX,
                                            double* __restrict__ FY, double* __restrict__ FZ, double& smax,
                                            uint32_t& err) {
    const int64_t VS = (int64_t)NDIR * REC_CELLS;
    int zl, zr, yl, yr, xl, xr;
    if (axis == 0) {
        zl = zr = i + 1; yl = yr = j + 1; xl = k; xr = k + 1;
    } else if (axis == 1) {
        zl = zr = i + 1; yl = j; yr = j + 1; xl = xr = k + 1;
    } else {
        zl = j; zr = j + 1; yl = yr = i + 1; xl = xr = k + 1;
    }
    const int cl_ = (zl * NRC + yl) * NRC + xl, cr_ = (zr * NRC + yr) * NRC + xr;
    const uint32_t kbase = (uint32_t)((((axis * 8 + i) * 9 + j) * 9 + k) * 9);
    double acc[NVAR] = {0.0, 0.0, 0.0, 0.0, 0.0};
    double nl[NVAR], nr[NVAR];
    {
        const double* pl_ = Qb + c_dplus[axis][0] * REC_CELLS + cl_;
        const double* pr_ = Qb + c_dminus[axis][0] * REC_CELLS + cr_;
#pragma unroll
        for (int v = 0; v < NVAR; ++v) {
            nl[v] = __ldg(pl_ + v * VS);
            nr[v] = __ldg(pr_ + v * VS);
        }
    }
#pragma unroll 1
    for (int qp = 0; qp < 9; ++qp) {
        const double w = c_simpson[qp];
        double ql[NVAR], qr[NVAR];
#pragma unroll
        for (int v = 0; v < NVAR; ++v) {
            ql[v] = nl[v];
            qr[v] = nr[v];
        }
        if (qp < 8) {
            const double* pl_ = Qb + c_dplus[axis][qp + 1] * REC_CELLS + cl_;
            const double* pr_ = Qb + c_dminus[axis][qp + 1] * REC_CELLS + cr_;
#pragma unroll
            for (int v = 0; v < NVAR; ++v) {
                nl[v] = __ldg(pl_ + v * VS);
                nr[v] = __ldg(pr_ + v * VS);
            }
        }
        const double rl = ql[0], rr = qr[0];
        const uint32_t key = (kbase + qp) * 2;
        if (err == 0xFFFFFFFFu && (rl <= 0.0 || rr <= 0.0)) err = ((key + 0) << 12) | (1u << 10) | (uint32_t)cl_;
        const double kel = dvd(add(add(mul(ql[1], ql[1]), mul(ql[2], ql[2])), mul(ql[3], ql[3])), mul(2.0, rl));
        const double ker = dvd(add(add(mul(qr[1], qr[1]), mul(qr[2], qr[2])), mul(qr[3], qr[3])), mul(2.0, rr));
        const double pl = mul(gm1, sub(ql[4], kel));
        const double pr = mul(gm1, sub(qr[4], ker));
        if (err == 0xFFFFFFFFu && (pl <= 0.0 || pr <= 0.0)) err = ((key + 1) << 12) | (2u << 10) | (uint32_t)cl_;
        const double snl = axis == 0 ? ql[1] : (axis == 1 ? ql[2] : ql[3]);
        const double snr = axis == 0 ? qr[1] : (axis == 1 ? qr[2] : qr[3]);
        const double vnl = dvd(snl, rl);
        const double vnr = dvd(snr, rr);
        const double sa = add(fabs(vnl), dsqrt(dvd(mul(gamma, pl), rl)));
        const double sb = add(fabs(vnr), dsqrt(dvd(mul(gamma, pr), rr)));
        const double s = sb > sa ? sb : sa;  // Python max(sa, sb)
        if (s > smax) smax = s;
        const double hs = mul(0.5, s);
#pragma unroll
        for (int v = 0; v < NVAR; ++v) {
            const double ul = ql[v], ur = qr[v];
            double flv, frv;
            if (v == 0) {
                flv = mul(rl, vnl);
                frv = mul(rr, vnr);
            } else if (v == 4) {
                flv = mul(add(ul, pl), vnl);
                frv = mul(add(ur, pr), vnr);
            } else {
                flv = mul(ul, vnl);
                frv = mul(ur, vnr);
                if (v == 1 + axis) {
                    flv = add(flv, pl);
                    frv = add(frv, pr);
                }
            }
            acc[v] = add(acc[v], mul(w, sub(mul(0.5, add(flv, frv)), mul(hs, sub(ur, ul)))));
        }
    }
    double* F;
    if (axis == 0) F = FX + b * 5 * 576 + (i * 8 + j) * 9 + k;
    else if (axis == 1) F = FY + b * 5 * 576 + (i * 9 + j) * 8 + k;
    else F = FZ + b * 5 * 576 + (j * 8 + i) * 8 + k;
#pragma unroll
    for (int v = 0; v < NVAR; ++v) F[v * 576] = acc[v];
}

__global__ void __launch_bounds__(FLUX_THREADS)
flux_legacy_kernel(const double* __restrict__ Q, double gamma, double* __restrict__ FX, double* __restrict__ FY,
                   double* __restrict__ FZ, double* __restrict__ smax_out, uint32_t* __restrict__ err_out,
                   uint32_t* __restrict__ latch, int32_t* __restrict__ gate, int32_t iter) {
    __shared__ unsigned long long s_smax;
    __shared__ uint32_t s_err;
    const int64_t b = blockIdx.x;
    const int t = threadIdx.x;
    if (t == 0) {
        s_smax = 0ull;
        s_err = 0xFFFFFFFFu;
    }
    __syncthreads();
    const double* Qb = Q + b * (int64_t)(NVAR * NDIR * REC_CELLS);
    const double gm1 = sub(gamma, 1.0);
    double smax = 0.0;
    uint32_t err = 0xFFFFFFFFu;
#pragma unroll 1
    for (int f = t; f < 3 * 576; f += FLUX_THREADS) {
        int axis, i, j, k;
        plane_major_face(f, axis, i, j, k);
        legacy_face(Qb, axis, i, j, k, gamma, gm1, b, FX, FY, FZ, smax, err);
    }
    atomicMax(&s_smax, (unsigned long long)__double_as_longlong(smax));
    if (err != 0xFFFFFFFFu) atomicMin(&s_err, err);
    __syncthreads();
    if (t == 0) {
        smax_out[b] = __longlong_as_double((long long)s_smax);
        err_out[b] = s_err;
        if (s_err != 0xFFFFFFFFu) latch_error(latch, b, s_err, gate, iter);
    }
}

// ---------------------------------------------------------------------------
// fused reconstruct + flux (batched step path): U block and per-cell
// {uc, minmod slopes} in shared memory, every quadrature state rebuilt on the
// fly with the reconstruct_kernel expression tree -- Q (1.04 MB/subgrid) is
// never written.  Outputs/status identical to sg_reconstruct + sg_flux.
// ---------------------------------------------------------------------------
#ifndef FUSED_NT
#define FUSED_NT 512
#endif
constexpr int FUSED_THREADS = FUSED_NT;  // faces t, t+NT, ... of the axis-major list of 1728
constexpr int CELL_REC = 20;        // uc[5], slope[5][3]
constexpr size_t FUSED_SMEM = sizeof(double) * (NVAR * 1728 + CELL_REC * REC_CELLS);

// compiled.py:74-97 for one (cell, direction), cell record read from smem
__device__ __forceinline__ void rebuild_state(const double* __restrict__ C, int cell, int d, double floor_,
                                              double onepf, double& rho, double& sx, double& sy, double& sz,
                                              double& en) {
    const double fdz = c_dirs[d][0], fdy = c_dirs[d][1], fdx = c_dirs[d][2];
    double r[NVAR];
#pragma unroll
    for (int v = 0; v < NVAR; ++v) {
        const double* c = C + cell;
        r[v] = add(c[v * REC_CELLS],
                   mul(0.5, add(add(mul(fdx, c[(NVAR + v * 3 + 0) * REC_CELLS]), mul(fdy, c[(NVAR + v * 3 + 1) * REC_CELLS])),
                                mul(fdz, c[(NVAR + v * 3 + 2) * REC_CELLS]))));
    }
    rho = r[0] < floor_ ? floor_ : r[0];
    en = r[4] < floor_ ? floor_ : r[4];
    sx = r[1];
    sy = r[2];
    sz = r[3];
    const double ke = dvd(mul(0.5, add(add(mul(sx, sx), mul(sy, sy)), mul(sz, sz))), rho);
    const double emin = add(mul(ke, onepf), floor_);
    en = en < emin ? emin : en;
}

// one face (compiled.py:120-262); axis is warp-uniform at run time
__device__ __forceinline__ void fused_face(const double* __restrict__ C, int axis, int fi, int64_t b,
                                           double floor_, double onepf, double gamma, double gm1,
                                           double* __restrict__ FX, double* __restrict__ FY,
                                           double* __restrict__ FZ, double& smax, uint32_t& err) {
    const int nj = axis == 0 ? NIN : NIN + 1;
    const int nk = axis == 0 ? NIN + 1 : NIN;
    const int k = fi % nk, j = (fi / nk) % nj, i = fi / (nk * nj);
    int zl, zr, yl, yr, xl, xr;
    if (axis == 0) {
        zl = zr = i + 1; yl = yr = j + 1; xl = k; xr = k + 1;
    } else if (axis == 1) {
        zl = zr = i + 1; yl = j; yr = j + 1; xl = xr = k + 1;
    } else {
        zl = j; zr = j + 1; yl = yr = i + 1; xl = xr = k + 1;
    }
    const int cl_ = (zl * NRC + yl) * NRC + xl, cr_ = (zr * NRC + yr) * NRC + xr;
    SG_DASSERT(cl_ >= 0 && cl_ < REC_CELLS && cr_ >= 0 && cr_ < REC_CELLS);
    const uint32_t kbase = (uint32_t)((((axis * 8 + i) * 9 + j) * 9 + k) * 9);
    double f0 = 0.0, f1 = 0.0, f2 = 0.0, f3 = 0.0, f4 = 0.0;
#pragma unroll 1
    for (int qp = 0; qp < 9; ++qp) {
        const double w = c_simpson[qp];
        double ul0, ul1, ul2, ul3, ul4, ur0, ur1, ur2, ur3, ur4;
        rebuild_state(C, cl_, c_dplus[axis][qp], floor_, onepf, ul0, ul1, ul2, ul3, ul4);
        asm volatile("" ::: "memory");  // bound the smem loads in flight (register pressure)
        rebuild_state(C, cr_, c_dminus[axis][qp], floor_, onepf, ur0, ur1, ur2, ur3, ur4);
        const uint32_t key = (kbase + qp) * 4;
        if (err == 0xFFFFFFFFu) {
            if (ul0 <= 0.0) err = ((key + 0) << 12) | (1u << 10) | (uint32_t)cl_;
            else if (ur0 <= 0.0) err = ((key + 1) << 12) | (1u << 10) | (uint32_t)cr_;
        }
        const double invl = dvd(1.0, ul0);
        const double vxl = mul(ul1, invl), vyl = mul(ul2, invl), vzl = mul(ul3, invl);
        const double kel = mul(0.5, add(add(mul(ul1, vxl), mul(ul2, vyl)), mul(ul3, vzl)));
        const double pl = mul(gm1, sub(ul4, kel));
        const double invr = dvd(1.0, ur0);
        const double vxr = mul(ur1, invr), vyr = mul(ur2, invr), vzr = mul(ur3, invr);
        const double ker = mul(0.5, add(add(mul(ur1, vxr), mul(ur2, vyr)), mul(ur3, vzr)));
        const double pr = mul(gm1, sub(ur4, ker));
        if (err == 0xFFFFFFFFu) {
            if (pl <= 0.0) err = ((key + 2) << 12) | (2u << 10) | (uint32_t)cl_;
            else if (pr <= 0.0) err = ((key + 3) << 12) | (2u << 10) | (uint32_t)cr_;
        }
        const double cl = dsqrt(mul(mul(gamma, pl), invl));
        const double cr = dsqrt(mul(mul(gamma, pr), invr));
        const double vnl = axis == 0 ? vxl : (axis == 1 ? vyl : vzl);
        const double vnr = axis == 0 ? vxr : (axis == 1 ? vyr : vzr);
        const double sl = add(fabs(vnl), cl);
        const double sr = add(fabs(vnr), cr);
        const double s = sl > sr ? sl : sr;
        if (s > smax) smax = s;
        const double fl0 = mul(ul0, vnl);
        double fl1 = mul(ul1, vnl), fl2 = mul(ul2, vnl), fl3 = mul(ul3, vnl);
        const double fl4 = mul(add(ul4, pl), vnl);
        const double fr0 = mul(ur0, vnr);
        double fr1 = mul(ur1, vnr), fr2 = mul(ur2, vnr), fr3 = mul(ur3, vnr);
        const double fr4 = mul(add(ur4, pr), vnr);
        if (axis == 0) {
            fl1 = add(fl1, pl);
            fr1 = add(fr1, pr);
        } else if (axis == 1) {
            fl2 = add(fl2, pl);
            fr2 = add(fr2, pr);
        } else {
            fl3 = add(fl3, pl);
            fr3 = add(fr3, pr);
        }
        const double hs = mul(0.5, s);
        f0 = add(f0, mul(w, sub(mul(0.5, add(fl0, fr0)), mul(hs, sub(ur0, ul0)))));
        f1 = add(f1, mul(w, sub(mul(0.5, add(fl1, fr1)), mul(hs, sub(ur1, ul1)))));
        f2 = add(f2, mul(w, sub(mul(0.5, add(fl2, fr2)), mul(hs, sub(ur2, ul2)))));
        f3 = add(f3, mul(w, sub(mul(0.5, add(fl3, fr3)), mul(hs, sub(ur3, ul3)))));
        f4 = add(f4, mul(w, sub(mul(0.5, add(fl4, fr4)), mul(hs, sub(ur4, ul4)))));
    }
    double* o;
    if (axis == 0) o = FX + b * 5 * 576 + (i * 8 + j) * 9 + k;
    else if (axis == 1) o = FY + b * 5 * 576 + (i * 9 + j) * 8 + k;
    else o = FZ + b * 5 * 576 + (j * 8 + i) * 8 + k;
    o[0] = f0;
    o[576] = f1;
    o[2 * 576] = f2;
    o[3 * 576] = f3;
    o[4 * 576] = f4;
}

// async copy of leaf b's 5 x 12^3 block (rows of 12 doubles = 6 x 16 B,
// 16-B aligned because the padded row pitch and the leaf origin are even)
__device__ __forceinline__ void prefetch_block(double* Us, const FieldView& uv, const int32_t* leaves, int64_t b) {
    const double* u0 = leaf_origin(uv, leaves, b, 2);
    for (int c = threadIdx.x; c < NVAR * 144 * 6; c += FUSED_THREADS) {
        const int row = c / 6, part = c % 6;
        const int v = row / 144, r = row % 144;
        const double* src = u0 + v * uv.comp_stride + (r / 12) * uv.sz + (r % 12) * uv.sy + 2 * part;
        const unsigned dst = (unsigned)__cvta_generic_to_shared(Us + row * 12 + 2 * part);
        asm volatile("cp.async.cg.shared.global [%0], [%1], 16;\n" ::"r"(dst), "l"(src) : "memory");
    }
    asm volatile("cp.async.commit_group;\n" ::: "memory");
}

__global__ void __launch_bounds__(FUSED_THREADS, 1)
hydro_fused_kernel(FieldView uv, const int32_t* __restrict__ leaves, int64_t B, double floor_, double gamma,
                   double* __restrict__ FX, double* __restrict__ FY, double* __restrict__ FZ,
                   double* __restrict__ smax_out, uint32_t* __restrict__ err_out, uint32_t* __restrict__ latch,
                   int32_t* __restrict__ gate, int32_t iter) {
    extern __shared__ __align__(16) unsigned char smem_raw[];
    double* Us = reinterpret_cast<double*>(smem_raw);  // [5][12][12][12]
    double* C = Us + NVAR * 1728;                       // [20][1000]
    __shared__ unsigned long long s_smax;
    __shared__ uint32_t s_err;
    const int t = threadIdx.x;
    const double gm1 = sub(gamma, 1.0);
    const double onepf = add(1.0, floor_);
    int64_t b = blockIdx.x;
    if (b < B) prefetch_block(Us, uv, leaves, b);
    for (; b < B; b += gridDim.x) {
        if (t == 0) {
            s_smax = 0ull;
            s_err = 0xFFFFFFFFu;
        }
        asm volatile("cp.async.wait_group 0;\n" ::: "memory");
        __syncthreads();
        // per region cell: centre values and minmod slopes (compiled.py:55-72)
        for (int cell = t; cell < REC_CELLS; cell += FUSED_THREADS) {
            const int x = cell % NRC + 1, y = (cell / NRC) % NRC + 1, z = cell / (NRC * NRC) + 1;
#pragma unroll
            for (int v = 0; v < NVAR; ++v) {
                const double* p = Us + v * 1728 + (z * 12 + y) * 12 + x;
                const double u = p[0];
                C[v * REC_CELLS + cell] = u;
                C[(NVAR + v * 3 + 0) * REC_CELLS + cell] = minmod(sub(p[1], u), sub(u, p[-1]));
                C[(NVAR + v * 3 + 1) * REC_CELLS + cell] = minmod(sub(p[12], u), sub(u, p[-12]));
                C[(NVAR + v * 3 + 2) * REC_CELLS + cell] = minmod(sub(p[144], u), sub(u, p[-144]));
            }
        }
        __syncthreads();
        // the U block is consumed: stream the next leaf's in behind the faces
        if (b + gridDim.x < B) prefetch_block(Us, uv, leaves, b + gridDim.x);
        double smax = 0.0;
        uint32_t err = 0xFFFFFFFFu;
        // faces, axis-major; 576 = 18 warps per axis so the axis is warp-uniform
#pragma unroll 1
        for (int ff = t; ff < 3 * 576; ff += FUSED_THREADS)
            fused_face(C, ff / 576, ff % 576, b, floor_, onepf, gamma, gm1, FX, FY, FZ, smax, err);
        atomicMax(&s_smax, (unsigned long long)__double_as_longlong(smax));
        if (err != 0xFFFFFFFFu) atomicMin(&s_err, err);
        __syncthreads();
        if (t == 0) {
            smax_out[b] = __longlong_as_double((long long)s_smax);
            err_out[b] = s_err;
            if (s_err != 0xFFFFFFFFu) latch_error(latch, b, s_err, gate, iter);
        }
    }
    asm volatile("cp.async.wait_group 0;\n" ::: "memory");
}

// ---------------------------------------------------------------------------
// hydro update (in place on the U view) + the reference's checks
// (kernels/__init__.py:168-187):  status = 0xFFFFFFFF ok, else
//   kind<<16 | detail,  kind 0: dt<=0, 1: CFL, 2: rho<=0/NaN at cell, 3: E
// ---------------------------------------------------------------------------
__global__ void __launch_bounds__(512)
hydro_update_kernel(FieldView uv, const int32_t* __restrict__ leaves, const double* __restrict__ FX,
                    const double* __restrict__ FY, const double* __restrict__ FZ,
                    const double* __restrict__ smax, const double* __restrict__ dt_dev, double dt_val,
                    double dx, double cfl, uint32_t* __restrict__ status, uint32_t* __restrict__ latch,
                    int32_t* __restrict__ gate, int32_t iter, double* __restrict__ err_info) {
    __shared__ uint32_t s_st;
    const int64_t b = blockIdx.x;
    const int t = threadIdx.x;
    const double dt = dt_dev ? *dt_dev : dt_val;
    if (t == 0) {
        uint32_t st = 0xFFFFFFFFu;
        if (!(dt > 0.0)) st = 0u << 16;
        else if (smax && mul(dt, smax[b]) > mul(cfl, dx)) st = 1u << 16;
        s_st = st;
    }
    __syncthreads();
    const double dtdx = dvd(dt, dx);
    const int x = t & 7, y = (t >> 3) & 7, z = t >> 6;
    double* u = const_cast<double*>(leaf_origin(uv, leaves, b, 0)) + z * uv.sz + y * uv.sy + x;
    const double* fx = FX + b * 5 * 576 + (z * 8 + y) * 9 + x;
    const double* fy = FY + b * 5 * 576 + (z * 9 + y) * 8 + x;
    const double* fz = FZ + b * 5 * 576 + (z * 8 + y) * 8 + x;
    double rho = 0.0, en = 0.0;
#pragma unroll
    for (int v = 0; v < NVAR; ++v) {
        const int64_t o = v * 576;
        const double net = add(add(sub(fx[o + 1], fx[o]), sub(fy[o + 8], fy[o])), sub(fz[o + 64], fz[o]));
        const double nu = sub(u[v * uv.comp_stride], mul(dtdx, net));
        u[v * uv.comp_stride] = nu;
        if (v == 0) rho = nu;
        if (v == 4) en = nu;
    }
    const int cell = (z * 8 + y) * 8 + x;
    if (!(rho > 0.0)) atomicMin(&s_st, (2u << 16) | (uint32_t)cell);
    else if (!(en > 0.0)) atomicMin(&s_st, (3u << 16) | (uint32_t)cell);
    __syncthreads();
    if (t == 0) {
        if (status) status[b] = s_st;
        if (s_st != 0xFFFFFFFFu && latch_error(latch, b, s_st, gate, iter) && err_info) {
            err_info[2 * b] = smax ? smax[b] : 0.0;
            err_info[2 * b + 1] = dt;
        }
    }
}

// ---------------------------------------------------------------------------
// max wave speed per leaf (compiled.py:454-480) and the dt reduction
// ---------------------------------------------------------------------------
__global__ void __launch_bounds__(512)
max_wavespeed_kernel(FieldView uv, const int32_t* __restrict__ leaves, double gamma, double pfloor,
                     double* __restrict__ out) {
    __shared__ unsigned long long s_max;
    const int64_t b = blockIdx.x;
    const int t = threadIdx.x;
    if (t == 0) s_max = 0ull;
    __syncthreads();
    const int x = t & 7, y = (t >> 3) & 7, z = t >> 6;
    const double* u = leaf_origin(uv, leaves, b, 0) + z * uv.sz + y * uv.sy + x;
    const int64_t cs = uv.comp_stride;
    const double gm1 = sub(gamma, 1.0);
    const double rho = __ldg(u), m1 = __ldg(u + cs), m2 = __ldg(u + 2 * cs), m3 = __ldg(u + 3 * cs),
                 e = __ldg(u + 4 * cs);
    const double inv = dvd(1.0, rho);
    const double vx = mul(m1, inv), vy = mul(m2, inv), vz = mul(m3, inv);
    const double ke = mul(0.5, add(add(mul(m1, vx), mul(m2, vy)), mul(m3, vz)));
    double p = mul(gm1, sub(e, ke));
    if (!(p > pfloor)) p = pfloor;
    const double c = dsqrt(mul(mul(gamma, p), inv));
    double av = fabs(vx);
    if (fabs(vy) > av) av = fabs(vy);
    if (fabs(vz) > av) av = fabs(vz);
    const double s = add(av, c);
    // reference: `if s > smax: smax = s` from 0.0 -> max over non-NaN s >= 0
    if (s > 0.0) atomicMax(&s_max, (unsigned long long)__double_as_longlong(s));
    __syncthreads();
    if (t == 0) out[b] = __longlong_as_double((long long)s_max);
}

__global__ void max_reduce_kernel(const double* __restrict__ vals, int64_t n, double* __restrict__ out) {
    __shared__ unsigned long long s_max;
    if (threadIdx.x == 0) s_max = 0ull;
    __syncthreads();
    double m = 0.0;
    for (int64_t i = threadIdx.x; i < n; i += blockDim.x) {
        const double v = vals[i];
        if (v > m) m = v;
    }
    atomicMax(&s_max, (unsigned long long)__double_as_longlong(m));
    __syncthreads();
    if (threadIdx.x == 0) *out = __longlong_as_double((long long)s_max);
}

__global__ void dt_kernel(const double* __restrict__ s_pre, double cfl, double dx, double* __restrict__ dt) {
    // driver.py:171  dt = cfl * dx / (3.0 * s_pre)
    *dt = dvd(mul(cfl, dx), mul(3.0, *s_pre));
}

}  // namespace sg

using namespace sg;

extern "C" {

int sg_reconstruct(const double* U, int64_t nx, int64_t ny, int64_t nz, int32_t pad, int64_t leaf_stride,
                   const int32_t* leaves, int64_t nleaves, double floor_, double* Q, void* stream) {
    if (pad < 2) {
        sg_set_error("sg_reconstruct: U pad must be >= 2 (got %d)", pad);
        return SG_EINVAL;
    }
    if (nleaves <= 0) return SG_OK;
    SG_TRY(sg_check_view("sg_reconstruct", "U", U, nx, ny, nz, pad, leaf_stride));
    SG_TRY(sg_check_ptr("sg_reconstruct", "Q", Q));
    SG_TRY(init_tables());
    FieldView uv = make_view(U, nx, ny, nz, pad, leaf_stride);
    // leaves on grid.y (<= 65535 per launch): larger batches in chunks
    constexpr int64_t CHUNK = 65535;
    for (int64_t first = 0; first < nleaves; first += CHUNK) {
        const int64_t n = nleaves - first < CHUNK ? nleaves - first : CHUNK;
        FieldView v = uv;
        const int32_t* lv = leaves;
        if (leaves) lv += 3 * first;
        else v.base += first * uv.leaf_stride;
        dim3 grid((REC_CELLS + REC_THREADS - 1) / REC_THREADS, (unsigned)n);
        sg_count_launch(1);
        reconstruct_kernel<<<grid, REC_THREADS, 0, (cudaStream_t)stream>>>(
            v, lv, floor_, Q + first * (int64_t)(NVAR * NDIR * REC_CELLS));
    }
    return sg_check_launch("sg_reconstruct");
}

int sg_flux(const double* Q, int64_t nleaves, double gamma, double* FX, double* FY, double* FZ,
            double* smax, uint32_t* err, uint32_t* latch, int32_t* gate, int32_t iter, void* stream) {
    if (nleaves <= 0) return SG_OK;
    SG_TRY(sg_check_ptr("sg_flux", "Q", Q));
    SG_TRY(sg_check_ptr("sg_flux", "FX", FX));
    SG_TRY(sg_check_ptr("sg_flux", "FY", FY));
    SG_TRY(sg_check_ptr("sg_flux", "FZ", FZ));
    SG_TRY(sg_check_ptr("sg_flux", "smax", smax));
    SG_TRY(sg_check_ptr("sg_flux", "err", err));
    SG_TRY(init_tables());
    sg_count_launch(1);
    flux_kernel<<<(unsigned)nleaves, FLUX_THREADS, 0, (cudaStream_t)stream>>>(Q, gamma, FX, FY, FZ, smax, err, latch,
                                                                                gate, iter);
    return sg_check_launch("sg_flux");
}

int sg_flux_legacy(const double* Q, int64_t nleaves, double gamma, double* FX, double* FY, double* FZ,
                   double* smax, uint32_t* err, uint32_t* latch, int32_t* gate, int32_t iter, void* stream) {
    if (nleaves <= 0) return SG_OK;
    SG_TRY(sg_check_ptr("sg_flux_legacy", "Q", Q));
    SG_TRY(sg_check_ptr("sg_flux_legacy", "FX", FX));
    SG_TRY(sg_check_ptr("sg_flux_legacy", "FY", FY));
    SG_TRY(sg_check_ptr("sg_flux_legacy", "FZ", FZ));
    SG_TRY(sg_check_ptr("sg_flux_legacy", "smax", smax));
    SG_TRY(sg_check_ptr("sg_flux_legacy", "err", err));
    SG_TRY(init_tables());
    sg_count_launch(1);
    flux_legacy_kernel<<<(unsigned)nleaves, FLUX_THREADS, 0, (cudaStream_t)stream>>>(Q, gamma, FX, FY, FZ, smax,
                                                                                      err, latch, gate, iter);
    return sg_check_launch("sg_flux_legacy");
}

int sg_hydro_fused(const double* U, int64_t nx, int64_t ny, int64_t nz, int32_t pad, int64_t leaf_stride,
                   const int32_t* leaves, int64_t nleaves, double floor_, double gamma, double* FX, double* FY,
                   double* FZ, double* smax, uint32_t* err, uint32_t* latch, int32_t* gate, int32_t iter,
                   void* stream) {
    if (pad < 2) {
        sg_set_error("sg_hydro_fused: U pad must be >= 2 (got %d)", pad);
        return SG_EINVAL;
    }
    if (nleaves <= 0) return SG_OK;
    SG_TRY(sg_check_view("sg_hydro_fused", "U", U, nx, ny, nz, pad, leaf_stride));
    SG_TRY(sg_check_ptr("sg_hydro_fused", "FX", FX));
    SG_TRY(sg_check_ptr("sg_hydro_fused", "FY", FY));
    SG_TRY(sg_check_ptr("sg_hydro_fused", "FZ", FZ));
    SG_TRY(sg_check_ptr("sg_hydro_fused", "smax", smax));
    SG_TRY(sg_check_ptr("sg_hydro_fused", "err", err));
    SG_TRY(init_tables());
    cudaFuncSetAttribute(hydro_fused_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)FUSED_SMEM);
    FieldView uv = make_view(U, nx, ny, nz, pad, leaf_stride);
    // the leaf block's x origin is pad - 2 + 8 cx: an even pad keeps its rows 16-byte aligned
    if (((uintptr_t)U & 15) || (pad & 1) || (uv.sy & 1) || (uv.sz & 1) || (uv.comp_stride & 1) || (leaf_stride & 1)) {
        sg_set_error("sg_hydro_fused: U rows must be 16-byte aligned (even pad and pitches, aligned base)");
        return SG_EINVAL;
    }
    int dev = 0, nsm = 148;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, dev);
    const int64_t grid = nleaves < nsm ? nleaves : nsm;
    sg_count_launch(1);
    hydro_fused_kernel<<<(unsigned)grid, FUSED_THREADS, FUSED_SMEM, (cudaStream_t)stream>>>(
        uv, leaves, nleaves, floor_, gamma, FX, FY, FZ, smax, err, latch, gate, iter);
    return sg_check_launch("sg_hydro_fused");
}

int sg_hydro_update(double* U, int64_t nx, int64_t ny, int64_t nz, int32_t pad, int64_t leaf_stride,
                    const int32_t* leaves, int64_t nleaves, const double* FX, const double* FY,
                    const double* FZ, const double* smax, const double* dt_dev, double dt, double dx,
                    double cfl, uint32_t* status, uint32_t* latch, int32_t* gate, int32_t iter,
                    double* err_info, void* stream) {
    if (nleaves <= 0) return SG_OK;
    SG_TRY(sg_check_view("sg_hydro_update", "U", U, nx, ny, nz, pad, leaf_stride));
    SG_TRY(sg_check_ptr("sg_hydro_update", "FX", FX));
    SG_TRY(sg_check_ptr("sg_hydro_update", "FY", FY));
    SG_TRY(sg_check_ptr("sg_hydro_update", "FZ", FZ));
    FieldView uv = make_view(U, nx, ny, nz, pad, leaf_stride);
    sg_count_launch(1);
    hydro_update_kernel<<<(unsigned)nleaves, 512, 0, (cudaStream_t)stream>>>(
        uv, leaves, FX, FY, FZ, smax, dt_dev, dt, dx, cfl, status, latch, gate, iter, err_info);
    return sg_check_launch("sg_hydro_update");
}

int sg_max_wavespeed(const double* U, int64_t nx, int64_t ny, int64_t nz, int32_t pad, int64_t leaf_stride,
                     const int32_t* leaves, int64_t nleaves, double gamma, double pfloor, double* smax,
                     void* stream) {
    if (nleaves <= 0) return SG_OK;
    SG_TRY(sg_check_view("sg_max_wavespeed", "U", U, nx, ny, nz, pad, leaf_stride));
    SG_TRY(sg_check_ptr("sg_max_wavespeed", "smax", smax));
    FieldView uv = make_view(U, nx, ny, nz, pad, leaf_stride);
    sg_count_launch(1);
    max_wavespeed_kernel<<<(unsigned)nleaves, 512, 0, (cudaStream_t)stream>>>(uv, leaves, gamma, pfloor, smax);
    return sg_check_launch("sg_max_wavespeed");
}

int sg_max_reduce(const double* vals, int64_t n, double* out, void* stream) {
    SG_TRY(sg_check_ptr("sg_max_reduce", "out", out));
    if (n > 0) SG_TRY(sg_check_ptr("sg_max_reduce", "vals", vals));
    sg_count_launch(1);
    max_reduce_kernel<<<1, 1024, 0, (cudaStream_t)stream>>>(vals, n, out);
    return sg_check_launch("sg_max_reduce");
}

int sg_dt_from_smax(const double* s_pre, double cfl, double dx, double* dt, void* stream) {
    SG_TRY(sg_check_ptr("sg_dt_from_smax", "s_pre", s_pre));
    SG_TRY(sg_check_ptr("sg_dt_from_smax", "dt", dt));
    sg_count_launch(1);
    dt_kernel<<<1, 1, 0, (cudaStream_t)stream>>>(s_pre, cfl, dx, dt);
    return sg_check_launch("sg_dt_from_smax");
}

}  // extern "C"
