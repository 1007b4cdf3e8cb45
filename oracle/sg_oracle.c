/*
 * sg_oracle.c -- CPU ORACLE (test infrastructure only; never shipped, never
 * the thing measured except as bench.py's `cpu_baseline` / `--impl reference`
 * leg).  Only tests/, __graft_entry__.smoke() and bench.py may load it.
 *
 * A plain-C restatement of the reference's production kernels
 * (reference pkg/src/simdgrid/kernels/compiled.py), operation for operation:
 * same expression association, same loop/accumulation order, masked terms
 * added as literal 0.0, ternary selects (NaN semantics preserved).  Compiled
 * with -ffp-contract=off and no fast-math, so no FMA contraction and IEEE
 * sqrt/div: each function is bit-identical to the numba kernel it restates
 * (pinned by tests/test_oracle_golden.py against fixtures generated from the
 * reference itself by tests/golden/make_golden.py).
 *
 * The W (lane count) argument of the reference kernels is dropped: results
 * are W-independent by the reference's own contract (compiled.py:3-6), and
 * this is the W=1 (scalar backend) order.
 *
 * Batched helpers at the bottom gather each leaf's inputs from periodic
 * global fields exactly like octree.source_cube / exchange_ghosts
 * (reference octree.py:149-214) and run leaves in parallel on a pthread pool (the
 * analogue of the reference WorkerPool, one task per leaf).
 */
#define _GNU_SOURCE  /* sched_getaffinity / CPU_COUNT */
#include <math.h>
#include <sched.h>
#include <stdint.h>
#include <stdlib.h>
#include <string.h>
#include <pthread.h>
#include <unistd.h>

#define EXT 12
#define NIN 8
#define NRC 10
#define NDIR 26

/* Build flavours (oracle/Makefile): liboracle.so is portable x86-64 (the
 * test checker); liboracle_native.so adds -march=native for timing the CPU
 * baseline on the host it runs on.  Vectorisation never changes a rounding:
 * no reassociation, no contraction (-ffp-contract=off), IEEE sqrt/div. */
#define MP_CLONES

/* geometry.py:21-31 -- (dz, dy, dx) lexicographic, zero offset skipped */
static double DIRS_F[NDIR][3];
/* geometry.py:41-56 */
static int64_t DPLUS[3][3][3], DMINUS[3][3][3];
/* geometry.py:59-61 */
static double SIMPSON[3][3];
static int tables_ready = 0;

static int64_t dir_index(int dz, int dy, int dx) {
    int idx = (dz + 1) * 9 + (dy + 1) * 3 + (dx + 1);
    return idx > 13 ? idx - 1 : idx;
}

static void init_tables(void) {
    if (tables_ready) return;
    int d = 0;
    for (int dz = -1; dz <= 1; ++dz)
        for (int dy = -1; dy <= 1; ++dy)
            for (int dx = -1; dx <= 1; ++dx) {
                if (dz == 0 && dy == 0 && dx == 0) continue;
                DIRS_F[d][0] = (double)dz;
                DIRS_F[d][1] = (double)dy;
                DIRS_F[d][2] = (double)dx;
                ++d;
            }
    const int t[3] = {-1, 0, 1};
    for (int i1 = 0; i1 < 3; ++i1)
        for (int i2 = 0; i2 < 3; ++i2) {
            int t1 = t[i1], t2 = t[i2];
            DPLUS[0][i1][i2] = dir_index(t2, t1, 1);
            DMINUS[0][i1][i2] = dir_index(t2, t1, -1);
            DPLUS[1][i1][i2] = dir_index(t2, 1, t1);
            DMINUS[1][i1][i2] = dir_index(t2, -1, t1);
            DPLUS[2][i1][i2] = dir_index(1, t2, t1);
            DMINUS[2][i1][i2] = dir_index(-1, t2, t1);
        }
    const double w[3][3] = {{1.0, 4.0, 1.0}, {4.0, 16.0, 4.0}, {1.0, 4.0, 1.0}};
    for (int a = 0; a < 3; ++a)
        for (int b = 0; b < 3; ++b) SIMPSON[a][b] = w[a][b] / 36.0;
    tables_ready = 1;
}

#define U5(U, v, z, y, x) (U)[(((v) * EXT + (z)) * EXT + (y)) * EXT + (x)]
#define Q5(Q, v, d, z, y, x) (Q)[((((v) * NDIR + (d)) * NRC + (z)) * NRC + (y)) * NRC + (x)]

static double minmod(double ap, double am) {
    /* compiled.py:58-62 */
    double mag = fabs(ap) < fabs(am) ? ap : am;
    int sgn = (ap > 0.0 && am > 0.0) || (ap < 0.0 && am < 0.0);
    return sgn ? mag : 0.0;
}

/* compiled.py:31-102 */
MP_CLONES
void or_reconstruct(const double *U, double floor_, double *Q) {
    init_tables();
    double slopes[5][3], uc[5];
    for (int z = 0; z < NRC; ++z) {
        int ze = z + 1;
        for (int y = 0; y < NRC; ++y) {
            int ye = y + 1;
            for (int x = 0; x < NRC; ++x) {
                int xe = x + 1;
                for (int v = 0; v < 5; ++v) {
                    double u = U5(U, v, ze, ye, xe);
                    uc[v] = u;
                    slopes[v][0] = minmod(U5(U, v, ze, ye, xe + 1) - u, u - U5(U, v, ze, ye, xe - 1));
                    slopes[v][1] = minmod(U5(U, v, ze, ye + 1, xe) - u, u - U5(U, v, ze, ye - 1, xe));
                    slopes[v][2] = minmod(U5(U, v, ze + 1, ye, xe) - u, u - U5(U, v, ze - 1, ye, xe));
                }
                for (int d = 0; d < NDIR; ++d) {
                    double fdz = DIRS_F[d][0], fdy = DIRS_F[d][1], fdx = DIRS_F[d][2];
                    double rho = uc[0] + 0.5 * ((fdx * slopes[0][0] + fdy * slopes[0][1]) + fdz * slopes[0][2]);
                    rho = rho < floor_ ? floor_ : rho;
                    double sx = uc[1] + 0.5 * ((fdx * slopes[1][0] + fdy * slopes[1][1]) + fdz * slopes[1][2]);
                    double sy = uc[2] + 0.5 * ((fdx * slopes[2][0] + fdy * slopes[2][1]) + fdz * slopes[2][2]);
                    double sz = uc[3] + 0.5 * ((fdx * slopes[3][0] + fdy * slopes[3][1]) + fdz * slopes[3][2]);
                    double en = uc[4] + 0.5 * ((fdx * slopes[4][0] + fdy * slopes[4][1]) + fdz * slopes[4][2]);
                    en = en < floor_ ? floor_ : en;
                    double ke = (0.5 * ((sx * sx + sy * sy) + sz * sz)) / rho;
                    double emin = ke * (1.0 + floor_) + floor_;
                    en = en < emin ? emin : en;
                    Q5(Q, 0, d, z, y, x) = rho;
                    Q5(Q, 1, d, z, y, x) = sx;
                    Q5(Q, 2, d, z, y, x) = sy;
                    Q5(Q, 3, d, z, y, x) = sz;
                    Q5(Q, 4, d, z, y, x) = en;
                }
            }
        }
    }
}

/* compiled.py:105-262.  FX (5,8,8,9) [v,z,y,s]; FY (5,8,9,8); FZ (5,9,8,8).
 * out3 = {smax, err_code, err_cell} (codes returned as doubles' integer
 * values through separate pointers to keep the ABI plain). */
MP_CLONES
void or_flux(const double *Q, double gamma, double *FX, double *FY, double *FZ,
             double *smax_out, int64_t *err_code_out, int64_t *err_cell_out) {
    init_tables();
    double gm1 = gamma - 1.0;
    double smax = 0.0;
    int64_t err_code = 0, err_cell = -1;
    for (int axis = 0; axis < 3; ++axis) {
        for (int i = 0; i < NIN; ++i) {
            int nj = axis == 0 ? NIN : NIN + 1;
            for (int j = 0; j < nj; ++j) {
                int nk = axis == 0 ? NIN + 1 : NIN;
                for (int k = 0; k < nk; ++k) {
                    int zl, zr, yl, yr, xl, xr;
                    if (axis == 0) {
                        zl = zr = i + 1; yl = yr = j + 1; xl = k; xr = k + 1;
                    } else if (axis == 1) {
                        zl = zr = i + 1; yl = j; yr = j + 1; xl = xr = k + 1;
                    } else {
                        zl = j; zr = j + 1; yl = yr = i + 1; xl = xr = k + 1;
                    }
                    double f0 = 0.0, f1 = 0.0, f2 = 0.0, f3 = 0.0, f4 = 0.0;
                    for (int i1 = 0; i1 < 3; ++i1) {
                        for (int i2 = 0; i2 < 3; ++i2) {
                            double w = SIMPSON[i1][i2];
                            int64_t dl = DPLUS[axis][i1][i2];
                            int64_t dr = DMINUS[axis][i1][i2];
                            double ul0 = Q5(Q, 0, dl, zl, yl, xl), ul1 = Q5(Q, 1, dl, zl, yl, xl);
                            double ul2 = Q5(Q, 2, dl, zl, yl, xl), ul3 = Q5(Q, 3, dl, zl, yl, xl);
                            double ul4 = Q5(Q, 4, dl, zl, yl, xl);
                            double ur0 = Q5(Q, 0, dr, zr, yr, xr), ur1 = Q5(Q, 1, dr, zr, yr, xr);
                            double ur2 = Q5(Q, 2, dr, zr, yr, xr), ur3 = Q5(Q, 3, dr, zr, yr, xr);
                            double ur4 = Q5(Q, 4, dr, zr, yr, xr);
                            if (ul0 <= 0.0 && err_code == 0) { err_code = 1; err_cell = (zl * NRC + yl) * NRC + xl; }
                            if (ur0 <= 0.0 && err_code == 0) { err_code = 1; err_cell = (zr * NRC + yr) * NRC + xr; }
                            double invl = 1.0 / ul0;
                            double vxl = ul1 * invl, vyl = ul2 * invl, vzl = ul3 * invl;
                            double kel = 0.5 * ((ul1 * vxl + ul2 * vyl) + ul3 * vzl);
                            double pl = gm1 * (ul4 - kel);
                            double invr = 1.0 / ur0;
                            double vxr = ur1 * invr, vyr = ur2 * invr, vzr = ur3 * invr;
                            double ker = 0.5 * ((ur1 * vxr + ur2 * vyr) + ur3 * vzr);
                            double pr = gm1 * (ur4 - ker);
                            if (pl <= 0.0 && err_code == 0) { err_code = 2; err_cell = (zl * NRC + yl) * NRC + xl; }
                            if (pr <= 0.0 && err_code == 0) { err_code = 2; err_cell = (zr * NRC + yr) * NRC + xr; }
                            double cl = sqrt((gamma * pl) * invl);
                            double cr = sqrt((gamma * pr) * invr);
                            double vnl, vnr;
                            if (axis == 0) { vnl = vxl; vnr = vxr; }
                            else if (axis == 1) { vnl = vyl; vnr = vyr; }
                            else { vnl = vzl; vnr = vzr; }
                            double sl = fabs(vnl) + cl;
                            double sr = fabs(vnr) + cr;
                            double s = sl > sr ? sl : sr;
                            if (s > smax) smax = s;
                            double fl0 = ul0 * vnl, fl1 = ul1 * vnl, fl2 = ul2 * vnl, fl3 = ul3 * vnl;
                            double fl4 = (ul4 + pl) * vnl;
                            double fr0 = ur0 * vnr, fr1 = ur1 * vnr, fr2 = ur2 * vnr, fr3 = ur3 * vnr;
                            double fr4 = (ur4 + pr) * vnr;
                            if (axis == 0) { fl1 = fl1 + pl; fr1 = fr1 + pr; }
                            else if (axis == 1) { fl2 = fl2 + pl; fr2 = fr2 + pr; }
                            else { fl3 = fl3 + pl; fr3 = fr3 + pr; }
                            double hs = 0.5 * s;
                            f0 = f0 + w * (0.5 * (fl0 + fr0) - hs * (ur0 - ul0));
                            f1 = f1 + w * (0.5 * (fl1 + fr1) - hs * (ur1 - ul1));
                            f2 = f2 + w * (0.5 * (fl2 + fr2) - hs * (ur2 - ul2));
                            f3 = f3 + w * (0.5 * (fl3 + fr3) - hs * (ur3 - ul3));
                            f4 = f4 + w * (0.5 * (fl4 + fr4) - hs * (ur4 - ul4));
                        }
                    }
                    double f[5] = {f0, f1, f2, f3, f4};
                    for (int v = 0; v < 5; ++v) {
                        if (axis == 0) FX[((v * 8 + i) * 8 + j) * 9 + k] = f[v];
                        else if (axis == 1) FY[((v * 8 + i) * 9 + j) * 8 + k] = f[v];
                        else FZ[((v * 9 + j) * 8 + i) * 8 + k] = f[v];
                    }
                }
            }
        }
    }
    *smax_out = smax;
    *err_code_out = err_code;
    *err_cell_out = err_cell;
}

/* compiled.py:265-278 (U in place, 5 variables) */
void or_hydro_update(double *U, const double *FX, const double *FY, const double *FZ, double dtdx) {
    for (int v = 0; v < 5; ++v)
        for (int z = 0; z < NIN; ++z)
            for (int y = 0; y < NIN; ++y)
                for (int x = 0; x < NIN; ++x) {
                    double net = ((FX[((v * 8 + z) * 8 + y) * 9 + x + 1] - FX[((v * 8 + z) * 8 + y) * 9 + x])
                                  + (FY[((v * 8 + z) * 9 + y + 1) * 8 + x] - FY[((v * 8 + z) * 9 + y) * 8 + x]))
                                 + (FZ[((v * 9 + z + 1) * 8 + y) * 8 + x] - FZ[((v * 9 + z) * 8 + y) * 8 + x]);
                    double *u = &U5(U, v, z + 2, y + 2, x + 2);
                    *u = *u - dtdx * net;
                }
}

/* compiled.py:281-321.  cube (8+2h)^3; outputs contiguous (8,8,8). */
MP_CLONES
void or_monopole(const double *cube, int64_t halo, double dx, double rad2, double eps2,
                 double *phi, double *gx, double *gy, double *gz) {
    int64_t S = NIN + 2 * halo;
    for (int z = 0; z < NIN; ++z)
        for (int y = 0; y < NIN; ++y)
            for (int x = 0; x < NIN; ++x) {
                double acc_p = 0.0, acc_x = 0.0, acc_y = 0.0, acc_z = 0.0;
                for (int64_t oz = -halo; oz <= halo; ++oz) {
                    double rz = (-(double)oz) * dx;
                    for (int64_t oy = -halo; oy <= halo; ++oy) {
                        double ry = (-(double)oy) * dx;
                        for (int64_t ox = -halo; ox <= halo; ++ox) {
                            double rx = (-(double)ox) * dx;
                            double m = cube[((z + oz + halo) * S + (y + oy + halo)) * S + (x + ox + halo)];
                            double r2 = (rx * rx + ry * ry) + rz * rz;
                            int ok = r2 <= rad2 && !(ox == 0 && oy == 0 && oz == 0);
                            double rt = sqrt(r2 + eps2);
                            double inv = 1.0 / rt;
                            double pt = -(m * inv);
                            double inv3 = (inv * inv) * inv;
                            double com = m * inv3;
                            acc_p = acc_p + (ok ? pt : 0.0);
                            acc_x = acc_x + (ok ? -(com * rx) : 0.0);
                            acc_y = acc_y + (ok ? -(com * ry) : 0.0);
                            acc_z = acc_z + (ok ? -(com * rz) : 0.0);
                        }
                    }
                }
                int o = (z * 8 + y) * 8 + x;
                phi[o] = acc_p; gx[o] = acc_x; gy[o] = acc_y; gz[o] = acc_z;
            }
}

/* compiled.py:324-352.  cube (n,n,n) -> 4 x (n/2)^3 */
void or_cluster_aggregate(const double *cube, int64_t n, double dx,
                          double *M, double *Dx, double *Dy, double *Dz) {
    int64_t nc = n / 2;
    for (int64_t cz = 0; cz < nc; ++cz)
        for (int64_t cy = 0; cy < nc; ++cy)
            for (int64_t cx = 0; cx < nc; ++cx) {
                double m_tot = 0.0, dxa = 0.0, dya = 0.0, dza = 0.0;
                for (int oz = 0; oz < 2; ++oz)
                    for (int oy = 0; oy < 2; ++oy)
                        for (int ox = 0; ox < 2; ++ox) {
                            double m = cube[((2 * cz + oz) * n + (2 * cy + oy)) * n + (2 * cx + ox)];
                            m_tot = m_tot + m;
                            dxa = dxa + m * (((double)ox - 0.5) * dx);
                            dya = dya + m * (((double)oy - 0.5) * dx);
                            dza = dza + m * (((double)oz - 0.5) * dx);
                        }
                int64_t c = (cz * nc + cy) * nc + cx;
                M[c] = m_tot; Dx[c] = dxa; Dy[c] = dya; Dz[c] = dza;
            }
}

/* compiled.py:355-451.  cube 24^3, clusters 12^3; flat interior range [i0,i1);
 * outputs contiguous (8,8,8) (only cells in range written).
 *
 * Restated row by row so the compiler can vectorise the per-cluster work
 * (both branches are still evaluated for every cluster, as the reference
 * does): loop A computes the far terms of the 12 clusters of a (cz,cy) row,
 * loop B the 96 near cell terms, loop C accumulates them sequentially in
 * the reference's order.  Every value is produced by the same expression
 * tree as compiled.py, so results are bit-identical (pinned by the tests). */
#define MP_NC 12
MP_CLONES
void or_multipole(const double *cube, const double *M, const double *Dx, const double *Dy,
                  const double *Dz, int64_t nc, double dx, double rad2, double eps2, int64_t order,
                  int64_t i0, int64_t i1, double *phi, double *gx, double *gy, double *gz) {
    if (nc != MP_NC) return;
    const int64_t n = 2 * MP_NC;
    double pf[MP_NC], gxf[MP_NC], gyf[MP_NC], gzf[MP_NC];
    int far_[MP_NC];
    double pn[MP_NC * 8], gxn[MP_NC * 8], gyn[MP_NC * 8], gzn[MP_NC * 8];
    for (int64_t f = i0; f < i1; ++f) {
        int64_t z = f / 64, y = (f % 64) / 8, x = f % 8;
        double tx = (double)x + 0.5, ty = (double)y + 0.5, tz = (double)z + 0.5;
        double acc_p = 0.0, acc_x = 0.0, acc_y = 0.0, acc_z = 0.0;
        for (int64_t cz = 0; cz < MP_NC; ++cz) {
            double bz = (double)(2 * cz - 8);
            for (int64_t cy = 0; cy < MP_NC; ++cy) {
                double by = (double)(2 * cy - 8);
                const int64_t c0 = (cz * MP_NC + cy) * MP_NC;
                /* A: far terms (compiled.py:394-418) */
                for (int cx = 0; cx < MP_NC; ++cx) {
                    double bx = (double)(2 * cx - 8);
                    double rx = (tx - (bx + 1.0)) * dx;
                    double ry = (ty - (by + 1.0)) * dx;
                    double rz = (tz - (bz + 1.0)) * dx;
                    double r2 = (rx * rx + ry * ry) + rz * rz;
                    far_[cx] = r2 > rad2;
                    double mt = M[c0 + cx];
                    double rt = sqrt(r2 + eps2);
                    double inv = 1.0 / rt;
                    double inv3 = (inv * inv) * inv;
                    double p_f = -(mt * inv);
                    double gcom = mt * inv3;
                    double gx_f = -(gcom * rx), gy_f = -(gcom * ry), gz_f = -(gcom * rz);
                    if (order == 1) {
                        double dxa = Dx[c0 + cx], dya = Dy[c0 + cx], dza = Dz[c0 + cx];
                        double dr = (dxa * rx + dya * ry) + dza * rz;
                        p_f = p_f - dr * inv3;
                        double inv5 = (inv3 * inv) * inv;
                        double t3 = (3.0 * dr) * inv5;
                        gx_f = (gx_f + dxa * inv3) - t3 * rx;
                        gy_f = (gy_f + dya * inv3) - t3 * ry;
                        gz_f = (gz_f + dza * inv3) - t3 * rz;
                    }
                    pf[cx] = p_f; gxf[cx] = gx_f; gyf[cx] = gy_f; gzf[cx] = gz_f;
                }
                /* B: near cell terms, masked as literal 0.0 (compiled.py:423-442) */
                for (int e = 0; e < MP_NC * 8; ++e) {
                    int cx = e >> 3, o = e & 7;
                    int ox = o & 1, oy = (o >> 1) & 1, oz = o >> 2;
                    double bx = (double)(2 * cx - 8);
                    double m = cube[((2 * cz + oz) * n + (2 * cy + oy)) * n + (2 * cx + ox)];
                    double sx = (tx - ((bx + (double)ox) + 0.5)) * dx;
                    double sy = (ty - ((by + (double)oy) + 0.5)) * dx;
                    double sz = (tz - ((bz + (double)oz) + 0.5)) * dx;
                    double r2s = (sx * sx + sy * sy) + sz * sz;
                    int ok = r2s > 0.0;
                    double rts = sqrt(r2s + eps2);
                    double invs = 1.0 / rts;
                    double pt = -(m * invs);
                    double invs3 = (invs * invs) * invs;
                    double coms = m * invs3;
                    pn[e] = ok ? pt : 0.0;
                    gxn[e] = ok ? -(coms * sx) : 0.0;
                    gyn[e] = ok ? -(coms * sy) : 0.0;
                    gzn[e] = ok ? -(coms * sz) : 0.0;
                }
                /* C: sequential accumulation (compiled.py:419-446) */
                for (int cx = 0; cx < MP_NC; ++cx) {
                    double p_n = 0.0, gx_n = 0.0, gy_n = 0.0, gz_n = 0.0;
                    for (int o = 0; o < 8; ++o) {
                        p_n = p_n + pn[cx * 8 + o];
                        gx_n = gx_n + gxn[cx * 8 + o];
                        gy_n = gy_n + gyn[cx * 8 + o];
                        gz_n = gz_n + gzn[cx * 8 + o];
                    }
                    acc_p = acc_p + (far_[cx] ? pf[cx] : p_n);
                    acc_x = acc_x + (far_[cx] ? gxf[cx] : gx_n);
                    acc_y = acc_y + (far_[cx] ? gyf[cx] : gy_n);
                    acc_z = acc_z + (far_[cx] ? gzf[cx] : gz_n);
                }
            }
        }
        int64_t o = (z * 8 + y) * 8 + x;
        phi[o] = acc_p; gx[o] = acc_x; gy[o] = acc_y; gz[o] = acc_z;
    }
}

/* compiled.py:454-480 */
double or_max_wavespeed(const double *U, double gamma, double pfloor) {
    double gm1 = gamma - 1.0;
    double smax = 0.0;
    for (int z = 2; z < 2 + NIN; ++z)
        for (int y = 2; y < 2 + NIN; ++y)
            for (int x = 2; x < 2 + NIN; ++x) {
                double rho = U5(U, 0, z, y, x);
                double inv = 1.0 / rho;
                double vx = U5(U, 1, z, y, x) * inv;
                double vy = U5(U, 2, z, y, x) * inv;
                double vz = U5(U, 3, z, y, x) * inv;
                double ke = 0.5 * ((U5(U, 1, z, y, x) * vx + U5(U, 2, z, y, x) * vy) + U5(U, 3, z, y, x) * vz);
                double p = gm1 * (U5(U, 4, z, y, x) - ke);
                if (!(p > pfloor)) p = pfloor;
                double c = sqrt((gamma * p) * inv);
                double av = fabs(vx);
                if (fabs(vy) > av) av = fabs(vy);
                if (fabs(vz) > av) av = fabs(vz);
                double s = av + c;
                if (s > smax) smax = s;
            }
    return smax;
}

/* ------------------------------------------------------------------------ */
/* Batched drivers over periodic global fields (n,n,n) [z,y,x].              */
/* leaves: B x 3 int64 (cx, cy, cz) leaf coordinates.                        */

static inline int64_t wrap(int64_t i, int64_t n) { i %= n; return i < 0 ? i + n : i; }

static void gather_cube(const double *g, int64_t n, const int64_t *leaf, int64_t halo, double *cube) {
    /* octree.source_cube (octree.py:186-214) on a periodic unigrid */
    int64_t S = NIN + 2 * halo;
    int64_t ox = leaf[0] * NIN - halo, oy = leaf[1] * NIN - halo, oz = leaf[2] * NIN - halo;
    for (int64_t z = 0; z < S; ++z)
        for (int64_t y = 0; y < S; ++y)
            for (int64_t x = 0; x < S; ++x)
                cube[(z * S + y) * S + x] = g[(wrap(oz + z, n) * n + wrap(oy + y, n)) * n + wrap(ox + x, n)];
}

/* Parallel-for over leaves: worker threads pull leaf indices from an atomic
 * counter (dynamic schedule, one leaf per grab -- like the reference's one
 * pool task per leaf).  Results never depend on the thread count. */
typedef void (*leaf_fn)(void *ctx, int64_t b, void *scratch);
typedef struct {
    leaf_fn fn; void *ctx; int64_t B; size_t scratch_bytes; int64_t next;
} pool_job;

static void *pool_worker(void *arg) {
    pool_job *job = (pool_job *)arg;
    void *scratch = malloc(job->scratch_bytes);
    for (;;) {
        int64_t b = __atomic_fetch_add(&job->next, 1, __ATOMIC_RELAXED);
        if (b >= job->B) break;
        job->fn(job->ctx, b, scratch);
    }
    free(scratch);
    return NULL;
}

int or_max_threads(void) {
    /* the CPUs this process may run on (affinity / cgroup cpusets), not
     * every online CPU of the host */
    cpu_set_t set;
    if (sched_getaffinity(0, sizeof set, &set) == 0) {
        int c = CPU_COUNT(&set);
        if (c > 0) return c;
    }
    long n = sysconf(_SC_NPROCESSORS_ONLN);
    return n > 0 ? (int)n : 1;
}

static void parallel_leaves(leaf_fn fn, void *ctx, int64_t B, size_t scratch_bytes, int nthreads) {
    if (nthreads <= 0) nthreads = or_max_threads();
    if (nthreads > B) nthreads = (int)(B > 0 ? B : 1);
    pool_job job = {fn, ctx, B, scratch_bytes, 0};
    if (nthreads == 1) { pool_worker(&job); return; }
    pthread_t *tid = (pthread_t *)malloc(sizeof(pthread_t) * nthreads);
    for (int t = 0; t < nthreads; ++t) pthread_create(&tid[t], NULL, pool_worker, &job);
    for (int t = 0; t < nthreads; ++t) pthread_join(tid[t], NULL);
    free(tid);
}

typedef struct {
    const double *g; int64_t n, halo; double dx, rad2, eps2, floor_, gamma, dtdx; int64_t order;
    const int64_t *leaves; double *out, *Unew, *smax; int64_t *err_code, *err_cell;
} batch_ctx;

static void p2p_leaf(void *c, int64_t b, void *scratch) {
    batch_ctx *k = (batch_ctx *)c;
    double *cube = (double *)scratch;
    gather_cube(k->g, k->n, k->leaves + 3 * b, k->halo, cube);
    double *o = k->out + b * 4 * 512;
    or_monopole(cube, k->halo, k->dx, k->rad2, k->eps2, o, o + 512, o + 1024, o + 1536);
}

/* out: B x 4 x 512 (phi, gx, gy, gz), interior order [z,y,x] */
void or_p2p_batch(const double *mass, int64_t n, int64_t halo, double dx, double rad2, double eps2,
                  const int64_t *leaves, int64_t B, double *out, int nthreads) {
    batch_ctx k = {0};
    k.g = mass; k.n = n; k.halo = halo; k.dx = dx; k.rad2 = rad2; k.eps2 = eps2;
    k.leaves = leaves; k.out = out;
    int64_t S = NIN + 2 * halo;
    parallel_leaves(p2p_leaf, &k, B, sizeof(double) * S * S * S, nthreads);
}

static void m2l_leaf(void *c, int64_t b, void *scratch) {
    batch_ctx *k = (batch_ctx *)c;
    double *cube = (double *)scratch, *cl = cube + 24 * 24 * 24;
    gather_cube(k->g, k->n, k->leaves + 3 * b, 8, cube);
    or_cluster_aggregate(cube, 24, k->dx, cl, cl + 1728, cl + 3456, cl + 5184);
    double *o = k->out + b * 4 * 512;
    or_multipole(cube, cl, cl + 1728, cl + 3456, cl + 5184, 12, k->dx, k->rad2, k->eps2, k->order, 0, 512,
                 o, o + 512, o + 1024, o + 1536);
}

void or_m2l_batch(const double *mass, int64_t n, double dx, double rad2, double eps2, int64_t order,
                  const int64_t *leaves, int64_t B, double *out, int nthreads) {
    batch_ctx k = {0};
    k.g = mass; k.n = n; k.dx = dx; k.rad2 = rad2; k.eps2 = eps2; k.order = order;
    k.leaves = leaves; k.out = out;
    parallel_leaves(m2l_leaf, &k, B, sizeof(double) * (24 * 24 * 24 + 4 * 1728), nthreads);
}

static void hydro_leaf(void *c, int64_t b, void *scratch) {
    batch_ctx *k = (batch_ctx *)c;
    int64_t n = k->n, nn = n * n * n;
    double *Ub = (double *)scratch;
    double *Q = Ub + 5 * 1728;
    double *FX = Q + 5 * NDIR * 1000, *FY = FX + 5 * 576, *FZ = FY + 5 * 576;
    for (int v = 0; v < 5; ++v) gather_cube(k->g + v * nn, n, k->leaves + 3 * b, 2, Ub + v * 1728);
    or_reconstruct(Ub, k->floor_, Q);
    or_flux(Q, k->gamma, FX, FY, FZ, k->smax + b, k->err_code + b, k->err_cell + b);
    if (k->dtdx > 0.0 && k->Unew) {
        or_hydro_update(Ub, FX, FY, FZ, k->dtdx);
        const int64_t *lf = k->leaves + 3 * b;
        for (int v = 0; v < 5; ++v)
            for (int z = 0; z < NIN; ++z)
                for (int y = 0; y < NIN; ++y)
                    for (int x = 0; x < NIN; ++x)
                        k->Unew[v * nn + ((lf[2] * NIN + z) * n + lf[1] * NIN + y) * n + lf[0] * NIN + x] =
                            U5(Ub, v, z + 2, y + 2, x + 2);
    }
}

/* One hydro iteration over the listed leaves of a periodic state U (5,n,n,n):
 * ghost exchange (gather with G=2), reconstruct, flux, and -- if dtdx > 0 --
 * the forward-Euler update written into Unew (5,n,n,n).  Per-leaf smax and
 * (err_code, err_cell) are returned.  Mirrors driver.hydro_job
 * (driver.py:141-160) minus the Python-level checks. */
void or_hydro_batch(const double *U, int64_t n, double floor_, double gamma, double dtdx,
                    const int64_t *leaves, int64_t B, double *Unew, double *smax,
                    int64_t *err_code, int64_t *err_cell, int nthreads) {
    batch_ctx k = {0};
    k.g = U; k.n = n; k.floor_ = floor_; k.gamma = gamma; k.dtdx = dtdx; k.leaves = leaves;
    k.Unew = Unew; k.smax = smax; k.err_code = err_code; k.err_cell = err_cell;
    parallel_leaves(hydro_leaf, &k, B, sizeof(double) * (5 * 1728 + 5 * NDIR * 1000 + 15 * 576), nthreads);
}

static void ws_leaf(void *c, int64_t b, void *scratch) {
    batch_ctx *k = (batch_ctx *)c;
    int64_t nn = k->n * k->n * k->n;
    double *Ub = (double *)scratch;
    for (int v = 0; v < 5; ++v) gather_cube(k->g + v * nn, k->n, k->leaves + 3 * b, 2, Ub + v * 1728);
    k->smax[b] = or_max_wavespeed(Ub, k->gamma, k->rad2 /* pfloor */);
}

/* Per-leaf max_wavespeed over a periodic state. */
void or_wavespeed_batch(const double *U, int64_t n, double gamma, double pfloor,
                        const int64_t *leaves, int64_t B, double *smax, int nthreads) {
    batch_ctx k = {0};
    k.g = U; k.n = n; k.gamma = gamma; k.rad2 = pfloor; k.leaves = leaves; k.smax = smax;
    parallel_leaves(ws_leaf, &k, B, sizeof(double) * 5 * 1728, nthreads);
}
