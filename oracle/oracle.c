/*
 * oracle.c -- CPU restatement of the reference gridding kernels.
 *
 * TEST INFRASTRUCTURE ONLY.  This file is the parity checker for the CUDA
 * path and the CPU baseline timed by bench.py (`cpu_baseline` leg and
 * `--impl reference`).  Nothing in the product package links or calls it.
 *
 * It restates /root/reference/pkg/src/voxmol/_kernels.py function by
 * function, with the same argument meaning (packed CSR layout built by
 * voxelizer._run_batch, voxelizer.py:372-435) and the same IEEE evaluation
 * order.  Build with -ffp-contract=off and without -ffast-math: numba runs
 * these kernels with fastmath off (_kernels.py:9), so a*b+c is never fused.
 *
 * Parallelism mirrors numba's prange: over packed sets in the forward
 * (_kernels.py:40,124) and over atoms in the backward (_kernels.py:216,268).
 * Every work item owns a disjoint output block and sums in atom order in f64,
 * so the result is independent of the OpenMP thread count, like the reference.
 *
 * Pinning: tests/test_oracle_golden.py checks every function here against
 * fixtures produced by the live reference (tests/golden/make_golden.py).
 */
#include <math.h>
#include <stdint.h>
#include <stdlib.h>
#include <string.h>
#ifdef _OPENMP
#include <omp.h>
#endif

/* _kernels.py:22-30 */
static inline void axis_bounds(double x, double cut, double origin, double res,
                               int64_t npts, int64_t *lo_out, int64_t *hi_out) {
    int64_t lo = (int64_t)ceil(((x - cut) - origin) / res);
    int64_t hi = (int64_t)floor(((x + cut) - origin) / res);
    if (lo < 0) lo = 0;
    if (hi > npts - 1) hi = npts - 1;
    *lo_out = lo;
    *hi_out = hi;
}

static inline int64_t imin(int64_t a, int64_t b) { return a < b ? a : b; }
static inline int64_t imax(int64_t a, int64_t b) { return a > b ? a : b; }

int oracle_num_threads(void) {
#ifdef _OPENMP
    return omp_get_max_threads();
#else
    return 1;
#endif
}

void oracle_set_num_threads(int n) {
#ifdef _OPENMP
    if (n > 0) omp_set_num_threads(n);
#else
    (void)n;
#endif
}

/* _kernels.py:33-113 forward_index_sets.
 * out: (nex, nch, npts, npts, npts) f32, pre-zeroed by the caller
 * (voxelizer.py:320-333).  coords (natoms,3) f64, radii f64 (already scaled),
 * tidx i64, set_* i64 (nsets), origins (nex,3) f64. */
void oracle_forward_index_sets(float *out, int64_t nch, int64_t npts,
                               const double *coords, const double *radii,
                               const int64_t *tidx, const int64_t *set_start,
                               const int64_t *set_end, const int64_t *set_example,
                               const int64_t *set_choff, const int64_t *set_t,
                               int64_t nsets, const double *origins, double res,
                               double grm, double rmult, int binary) {
    const int64_t D = npts;
    const int64_t D3 = D * D * D;
#pragma omp parallel for schedule(dynamic, 1)
    for (int64_t s = 0; s < nsets; s++) {
        int64_t a0 = set_start[s], a1 = set_end[s];
        if (a1 <= a0) continue;
        int64_t e = set_example[s];
        int64_t off = set_choff[s];
        int64_t nt = set_t[s];
        double ox = origins[e * 3 + 0], oy = origins[e * 3 + 1], oz = origins[e * 3 + 2];

        /* union box of atom footprints (_kernels.py:49-65) */
        int64_t bi0 = D, bi1 = -1, bj0 = D, bj1 = -1, bk0 = D, bk1 = -1;
        for (int64_t a = a0; a < a1; a++) {
            double r = radii[a];
            double cut = binary ? r : r * rmult;
            int64_t i0, i1, j0, j1, k0, k1;
            axis_bounds(coords[a * 3 + 0], cut, ox, res, D, &i0, &i1);
            axis_bounds(coords[a * 3 + 1], cut, oy, res, D, &j0, &j1);
            axis_bounds(coords[a * 3 + 2], cut, oz, res, D, &k0, &k1);
            if (i0 > i1 || j0 > j1 || k0 > k1) continue;
            bi0 = imin(bi0, i0); bi1 = imax(bi1, i1);
            bj0 = imin(bj0, j0); bj1 = imax(bj1, j1);
            bk0 = imin(bk0, k0); bk1 = imax(bk1, k1);
        }
        if (bi1 < bi0) continue;
        int64_t ni = bi1 - bi0 + 1, nj = bj1 - bj0 + 1, nk = bk1 - bk0 + 1;
        double *tmp = (double *)calloc((size_t)(nt * ni * nj * nk), sizeof(double));
        unsigned char *touched = (unsigned char *)calloc((size_t)nt, 1);

        for (int64_t a = a0; a < a1; a++) {
            double x = coords[a * 3 + 0], y = coords[a * 3 + 1], z = coords[a * 3 + 2];
            double r = radii[a];
            int64_t c = tidx[a];
            double cut = binary ? r : r * rmult;
            int64_t i0, i1, j0, j1, k0, k1;
            axis_bounds(x, cut, ox, res, D, &i0, &i1);
            axis_bounds(y, cut, oy, res, D, &j0, &j1);
            axis_bounds(z, cut, oz, res, D, &k0, &k1);
            if (i0 > i1 || j0 > j1 || k0 > k1) continue;
            touched[c] = 1;
            double r2 = r * r;
            double inv_r2 = 1.0 / r2;
            double gr = grm * r;
            double d02 = gr * gr;
            double dzr = rmult * r;
            double q0 = (2.0 * grm) / r;
            double qa = exp((-2.0 * grm) * grm) * (q0 * q0);
            for (int64_t i = i0; i <= i1; i++) {
                double dx = (ox + (double)i * res) - x;
                double dx2 = dx * dx;
                for (int64_t j = j0; j <= j1; j++) {
                    double dy = (oy + (double)j * res) - y;
                    double dxy2 = dx2 + dy * dy;
                    double *row = tmp + ((c * ni + (i - bi0)) * nj + (j - bj0)) * nk - bk0;
                    for (int64_t k = k0; k <= k1; k++) {
                        double dz = (oz + (double)k * res) - z;
                        double d2 = dxy2 + dz * dz;
                        if (binary) {
                            if (d2 <= r2) row[k] = 1.0;
                            continue;
                        }
                        if (d2 <= d02) {
                            row[k] += exp((-2.0 * d2) * inv_r2);
                        } else {
                            double d = sqrt(d2);
                            if (d < dzr) {
                                double t = d - dzr;
                                row[k] += (qa * t) * t;
                            }
                        }
                    }
                }
            }
        }
        /* writeback of touched channels over the union box (_kernels.py:107-113) */
        for (int64_t c = 0; c < nt; c++) {
            if (!touched[c]) continue;
            float *oc = out + (e * nch + off + c) * D3;
            for (int64_t i = bi0; i <= bi1; i++)
                for (int64_t j = bj0; j <= bj1; j++) {
                    const double *row = tmp + ((c * ni + (i - bi0)) * nj + (j - bj0)) * nk - bk0;
                    float *orow = oc + (i * D + j) * D;
                    for (int64_t k = bk0; k <= bk1; k++) orow[k] = (float)row[k];
                }
        }
        free(tmp);
        free(touched);
    }
}

/* _kernels.py:116-206 forward_vector_sets.  weights_flat f64 packed per set
 * at w_start[s] (row-major atoms x nt), atom_radii f64 (scaled), type_radii_flat
 * f64 (already scaled when radius_type_indexed) at tr_start[s]. */
void oracle_forward_vector_sets(float *out, int64_t nch, int64_t npts,
                                const double *coords, const double *weights_flat,
                                const int64_t *w_start, const double *atom_radii,
                                const double *type_radii_flat, const int64_t *tr_start,
                                int radius_type_indexed, const int64_t *set_start,
                                const int64_t *set_end, const int64_t *set_example,
                                const int64_t *set_choff, const int64_t *set_t,
                                int64_t nsets, const double *origins, double res,
                                double grm, double rmult, int binary) {
    const int64_t D = npts;
    const int64_t D3 = D * D * D;
#pragma omp parallel for schedule(dynamic, 1)
    for (int64_t s = 0; s < nsets; s++) {
        int64_t a0 = set_start[s], a1 = set_end[s];
        if (a1 <= a0) continue;
        int64_t e = set_example[s];
        int64_t off = set_choff[s];
        int64_t nt = set_t[s];
        double ox = origins[e * 3 + 0], oy = origins[e * 3 + 1], oz = origins[e * 3 + 2];

        double rmax = 0.0; /* _kernels.py:134-138 */
        if (radius_type_indexed) {
            for (int64_t c = 0; c < nt; c++)
                if (type_radii_flat[tr_start[s] + c] > rmax) rmax = type_radii_flat[tr_start[s] + c];
        }
        int64_t bi0 = D, bi1 = -1, bj0 = D, bj1 = -1, bk0 = D, bk1 = -1;
        for (int64_t a = a0; a < a1; a++) {
            double r = radius_type_indexed ? rmax : atom_radii[a];
            double cut = binary ? r : r * rmult;
            int64_t i0, i1, j0, j1, k0, k1;
            axis_bounds(coords[a * 3 + 0], cut, ox, res, D, &i0, &i1);
            axis_bounds(coords[a * 3 + 1], cut, oy, res, D, &j0, &j1);
            axis_bounds(coords[a * 3 + 2], cut, oz, res, D, &k0, &k1);
            if (i0 > i1 || j0 > j1 || k0 > k1) continue;
            bi0 = imin(bi0, i0); bi1 = imax(bi1, i1);
            bj0 = imin(bj0, j0); bj1 = imax(bj1, j1);
            bk0 = imin(bk0, k0); bk1 = imax(bk1, k1);
        }
        if (bi1 < bi0) continue;
        int64_t ni = bi1 - bi0 + 1, nj = bj1 - bj0 + 1, nk = bk1 - bk0 + 1;
        double *tmp = (double *)calloc((size_t)(nt * ni * nj * nk), sizeof(double));
        unsigned char *touched = (unsigned char *)calloc((size_t)nt, 1);

        for (int64_t a = a0; a < a1; a++) {
            double x = coords[a * 3 + 0], y = coords[a * 3 + 1], z = coords[a * 3 + 2];
            int64_t wrow = w_start[s] + (a - a0) * nt;
            for (int64_t c = 0; c < nt; c++) {
                double w = weights_flat[wrow + c];
                if (w == 0.0) continue;
                double r = radius_type_indexed ? type_radii_flat[tr_start[s] + c] : atom_radii[a];
                double cut = binary ? r : r * rmult;
                int64_t i0, i1, j0, j1, k0, k1;
                axis_bounds(x, cut, ox, res, D, &i0, &i1);
                axis_bounds(y, cut, oy, res, D, &j0, &j1);
                axis_bounds(z, cut, oz, res, D, &k0, &k1);
                if (i0 > i1 || j0 > j1 || k0 > k1) continue;
                touched[c] = 1;
                double r2 = r * r;
                double inv_r2 = 1.0 / r2;
                double gr = grm * r;
                double d02 = gr * gr;
                double dzr = rmult * r;
                double q0 = (2.0 * grm) / r;
                double qa = exp((-2.0 * grm) * grm) * (q0 * q0);
                for (int64_t i = i0; i <= i1; i++) {
                    double dx = (ox + (double)i * res) - x;
                    double dx2 = dx * dx;
                    for (int64_t j = j0; j <= j1; j++) {
                        double dy = (oy + (double)j * res) - y;
                        double dxy2 = dx2 + dy * dy;
                        double *row = tmp + ((c * ni + (i - bi0)) * nj + (j - bj0)) * nk - bk0;
                        for (int64_t k = k0; k <= k1; k++) {
                            double dz = (oz + (double)k * res) - z;
                            double d2 = dxy2 + dz * dz;
                            if (binary) {
                                if (d2 <= r2 && w > row[k]) row[k] = w;
                                continue;
                            }
                            if (d2 <= d02) {
                                row[k] += w * exp((-2.0 * d2) * inv_r2);
                            } else {
                                double d = sqrt(d2);
                                if (d < dzr) {
                                    double t = d - dzr;
                                    row[k] += ((w * qa) * t) * t;
                                }
                            }
                        }
                    }
                }
            }
        }
        for (int64_t c = 0; c < nt; c++) {
            if (!touched[c]) continue;
            float *oc = out + (e * nch + off + c) * D3;
            for (int64_t i = bi0; i <= bi1; i++)
                for (int64_t j = bj0; j <= bj1; j++) {
                    const double *row = tmp + ((c * ni + (i - bi0)) * nj + (j - bj0)) * nk - bk0;
                    float *orow = oc + (i * D + j) * D;
                    for (int64_t k = bk0; k <= bk1; k++) orow[k] = (float)row[k];
                }
        }
        free(tmp);
        free(touched);
    }
}

/* _kernels.py:209-255 backward_index.  grid_grad (ntypes, npts^3) f32 of ONE
 * set's channel block; coord_grad (n,3) f64 output. */
void oracle_backward_index(double *coord_grad, const double *coords, const double *radii,
                           const int64_t *tidx, int64_t n, const float *grid_grad,
                           int64_t npts, const double *origin, double res, double grm,
                           double rmult) {
    const int64_t D = npts;
    const double ox = origin[0], oy = origin[1], oz = origin[2];
#pragma omp parallel for schedule(dynamic, 8)
    for (int64_t a = 0; a < n; a++) {
        double x = coords[a * 3 + 0], y = coords[a * 3 + 1], z = coords[a * 3 + 2];
        double r = radii[a];
        int64_t c = tidx[a];
        double inv_r2 = 1.0 / (r * r);
        double d0 = grm * r;
        double d02 = d0 * d0;
        double dzr = rmult * r;
        double q0 = (2.0 * grm) / r;
        double qa = exp((-2.0 * grm) * grm) * (q0 * q0);
        int64_t i0, i1, j0, j1, k0, k1;
        axis_bounds(x, dzr, ox, res, D, &i0, &i1);
        axis_bounds(y, dzr, oy, res, D, &j0, &j1);
        axis_bounds(z, dzr, oz, res, D, &k0, &k1);
        double gx = 0.0, gy = 0.0, gz = 0.0;
        const float *gc = grid_grad + c * D * D * D;
        for (int64_t i = i0; i <= i1; i++) {
            double dx = x - (ox + (double)i * res);
            for (int64_t j = j0; j <= j1; j++) {
                double dy = y - (oy + (double)j * res);
                for (int64_t k = k0; k <= k1; k++) {
                    double dz = z - (oz + (double)k * res);
                    double d2 = (dx * dx + dy * dy) + dz * dz;
                    if (d2 <= 0.0 || d2 >= dzr * dzr) continue;
                    double g = (double)gc[(i * D + j) * D + k];
                    if (g == 0.0) continue;
                    double d = sqrt(d2);
                    double slope;
                    if (d2 <= d02)
                        slope = exp((-2.0 * d2) * inv_r2) * ((-4.0 * d) * inv_r2);
                    else
                        slope = (2.0 * qa) * (d - dzr);
                    double scale = (g * slope) / d;
                    gx += scale * dx;
                    gy += scale * dy;
                    gz += scale * dz;
                }
            }
        }
        coord_grad[a * 3 + 0] = gx;
        coord_grad[a * 3 + 1] = gy;
        coord_grad[a * 3 + 2] = gz;
    }
}

/* _kernels.py:258-314 backward_vector.  weights (n,nt) f64; type_radii (nt)
 * f64 (scaled); coord_grad (n,3) and type_grad (n,nt) f64 outputs. */
void oracle_backward_vector(double *coord_grad, double *type_grad, const double *coords,
                            const double *atom_radii, const double *weights, int64_t n,
                            int64_t nt, const float *grid_grad, int64_t npts,
                            const double *type_radii, int radius_type_indexed,
                            const double *origin, double res, double grm, double rmult) {
    const int64_t D = npts;
    const double ox = origin[0], oy = origin[1], oz = origin[2];
#pragma omp parallel for schedule(dynamic, 4)
    for (int64_t a = 0; a < n; a++) {
        double x = coords[a * 3 + 0], y = coords[a * 3 + 1], z = coords[a * 3 + 2];
        double gx = 0.0, gy = 0.0, gz = 0.0;
        for (int64_t c = 0; c < nt; c++) {
            double r = radius_type_indexed ? type_radii[c] : atom_radii[a];
            double w = weights[a * nt + c];
            double inv_r2 = 1.0 / (r * r);
            double gr = grm * r;
            double d02 = gr * gr;
            double dzr = rmult * r;
            double q0 = (2.0 * grm) / r;
            double qa = exp((-2.0 * grm) * grm) * (q0 * q0);
            int64_t i0, i1, j0, j1, k0, k1;
            axis_bounds(x, dzr, ox, res, D, &i0, &i1);
            axis_bounds(y, dzr, oy, res, D, &j0, &j1);
            axis_bounds(z, dzr, oz, res, D, &k0, &k1);
            double tg = 0.0;
            const float *gc = grid_grad + c * D * D * D;
            for (int64_t i = i0; i <= i1; i++) {
                double dx = x - (ox + (double)i * res);
                for (int64_t j = j0; j <= j1; j++) {
                    double dy = y - (oy + (double)j * res);
                    for (int64_t k = k0; k <= k1; k++) {
                        double dz = z - (oz + (double)k * res);
                        double d2 = (dx * dx + dy * dy) + dz * dz;
                        if (d2 >= dzr * dzr) continue;
                        double g = (double)gc[(i * D + j) * D + k];
                        if (g == 0.0) continue;
                        double dens, slope;
                        if (d2 <= d02) {
                            dens = exp((-2.0 * d2) * inv_r2);
                            slope = dens * ((-4.0 * sqrt(d2)) * inv_r2);
                        } else {
                            double d = sqrt(d2);
                            double t = d - dzr;
                            dens = (qa * t) * t;
                            slope = (2.0 * qa) * t;
                        }
                        tg += g * dens;
                        if (d2 > 0.0 && w != 0.0) {
                            double scale = ((w * g) * slope) / sqrt(d2);
                            gx += scale * dx;
                            gy += scale * dy;
                            gz += scale * dz;
                        }
                    }
                }
            }
            type_grad[a * nt + c] = tg;
        }
        coord_grad[a * 3 + 0] = gx;
        coord_grad[a * 3 + 1] = gy;
        coord_grad[a * 3 + 2] = gz;
    }
}
