// backward.cu -- grid gradients -> atom coordinate (and type) gradients.
//
// Reference: _kernels.py:209-255 (backward_index), 258-314 (backward_vector):
// per atom, a float64 sum over its voxel box (cut = rmult * r) of
// g * slope(d) / d * (x - v), and for vector types sum g * density per channel.
//
// B200 design: one warp per atom, batched over every set of every example.
//  * The Gaussian core is separable, exp(-2 d^2/r^2) = Ex(i) Ey(j) Ez(k): a
//    warp fills per-axis tables (offset and f64 exp factor) in shared memory,
//    ~3 x 13 f64 exps per atom instead of one per voxel.  Boxes wider than the
//    tables are walked in sub-boxes.
//  * Lanes own (i, j) rows of the box; each row visits only its k span inside
//    the cutoff sphere (rows outside the sphere's disc are skipped), four
//    voxels at a time with the loads issued first.
//  * Geometry and accumulation stay in f64 (f32 terms fail the
//    1e-6 gate on near-cancelling components).  The quadratic tail needs 1/d:
//    an f32 MUFU estimate refined by one f64 Newton step.  Two accumulator
//    chains per lane, then a warp-shuffle reduction: no atomics, deterministic.
#include "common.cuh"

namespace {

constexpr int kMaxN = 32;   // table entries per axis (sub-box edge)
constexpr int kMaxT = 16;   // channels kept in registers by the shared-geometry vector path
constexpr int kWarps = 8;

struct BwdArgs {
    gm_params p;
    gm_batch b;
    const double *pos;
    const float *grid_grad;
    float *coord_grad;
    float *type_grad;
};

struct Tables {
    double dx[kMaxN], ex[kMaxN], dy[kMaxN], ey[kMaxN], dz[kMaxN], ez[kMaxN];
};

// One atom (for one channel radius): position, origin, full voxel box.
struct Atom {
    double x, y, z, ox, oy, oz;
    double dzr, dzr2, m2inv_r2;
    int i0, i1, j0, j1, k0, k1;
};

__device__ __forceinline__ double offs(double x, double o, int i, double res) {
    // _kernels.py:232-236: x - (o + i*res), same association, no contraction
    return __dsub_rn(x, __dadd_rn(o, __dmul_rn((double)i, res)));
}

__device__ __forceinline__ float approx_rsqrt(float x) {
    float y;
    asm("rsqrt.approx.ftz.f32 %0, %1;" : "=f"(y) : "f"(x));
    return y;
}

// 1/sqrt(d2) to ~1e-13 relative: f32 MUFU estimate + one f64 Newton step.
__device__ __forceinline__ double rsqrt_d(double d2) {
    const double y0 = (double)approx_rsqrt((float)d2);
    const double e = fma(-d2 * y0, y0, 1.0);
    return fma(0.5 * y0, e, y0);
}

// floor(a / b) for 0 <= a < 2^16, 1 <= b <= 64 (float reciprocal, exact here).
__device__ __forceinline__ int idiv(int a, float inv_b) {
    return (int)(((float)a + 0.5f) * inv_b);
}

// Walk the box of atom A (cutoff A.dzr) over grid channel gbase.  For every
// voxel with d2 < dzr2 (and d2 > 0 when SKIP_CENTER) -- and, when LOAD,
// g != 0 -- calls f(slot, d2, dx, dy, dz, Exyz, g_or_voxel_offset) in a fixed
// order per lane.  Lanes own (i, j) rows of the box; a row visits only the k
// span inside the cutoff sphere, four voxels at a time (loads first).  With
// LOAD the walk passes g; otherwise the voxel offset (as double) and the
// callee loads.  `slot` alternates between two accumulator chains.
template <bool SKIP_CENTER, bool LOAD, typename F>
__device__ __forceinline__ void walk(const Atom &A, Tables &T, const float *gbase, int D,
                                     double res, float inv_res, int lane, F &&f) {
    for (int si = A.i0; si <= A.i1; si += kMaxN)
        for (int sj = A.j0; sj <= A.j1; sj += kMaxN)
            for (int sk = A.k0; sk <= A.k1; sk += kMaxN) {
                const int ni = min(kMaxN, A.i1 - si + 1), nj = min(kMaxN, A.j1 - sj + 1),
                          nk = min(kMaxN, A.k1 - sk + 1);
                __syncwarp();
                if (lane < ni) {
                    const double d = offs(A.x, A.ox, si + lane, res);
                    T.dx[lane] = d;
                    T.ex[lane] = exp(A.m2inv_r2 * (d * d));
                }
                if (lane < nj) {
                    const double d = offs(A.y, A.oy, sj + lane, res);
                    T.dy[lane] = d;
                    T.ey[lane] = exp(A.m2inv_r2 * (d * d));
                }
                if (lane < nk) {
                    const double d = offs(A.z, A.oz, sk + lane, res);
                    T.dz[lane] = d;
                    T.ez[lane] = exp(A.m2inv_r2 * (d * d));
                }
                __syncwarp();
                const float inv_nj = __frcp_rn((float)nj);
                const float dz0 = (float)T.dz[0];
                const int nrows = ni * nj;
                for (int row = lane; row < nrows; row += 32) {
                    const int ii = idiv(row, inv_nj), jj = row - ii * nj;
                    const double dx = T.dx[ii], dy = T.dy[jj];
                    const double b2 = fma(dy, dy, dx * dx);
                    const double rem = A.dzr2 - b2;
                    if (rem <= 0.0) continue;  // the whole row is at or beyond the cutoff
                    const float rho = fmaf(sqrtf((float)rem), 1.0001f, 1e-5f * (float)A.dzr);
                    const int klo = max(0, (int)ceilf(fmaxf((dz0 - rho) * inv_res, -1.0f)));
                    const int khi = min(nk - 1, (int)floorf(fminf((dz0 + rho) * inv_res, (float)nk)));
                    const double exy = T.ex[ii] * T.ey[jj];
                    const size_t rbase = ((size_t)(si + ii) * D + (sj + jj)) * D + sk;
                    for (int k0 = klo; k0 <= khi; k0 += 4) {
                        float g[4];
                        double d2[4];
#pragma unroll
                        for (int u = 0; u < 4; u++) {
                            const int kk = k0 + u;
                            bool in = false;
                            d2[u] = A.dzr2;
                            if (kk <= khi) {
                                const double dz = T.dz[kk];
                                d2[u] = fma(dz, dz, b2);
                                in = (SKIP_CENTER ? d2[u] > 0.0 : true) && d2[u] < A.dzr2;
                            }
                            if (LOAD) g[u] = in ? __ldg(gbase + rbase + kk) : 0.0f;
                            else g[u] = in ? 1.0f : 0.0f;
                        }
#pragma unroll
                        for (int u = 0; u < 4; u++) {
                            if (g[u] != 0.0f) {
                                const int kk = k0 + u;
                                const double gv = LOAD ? (double)g[u] : (double)(rbase + kk);
                                f(u & 1, d2[u], dx, dy, T.dz[kk], exy * T.ez[kk], gv);
                            }
                        }
                    }
                }
            }
}

__device__ __forceinline__ void load_atom(const BwdArgs &P, int a, Atom &A, int &s, int &e) {
    const gm_batch &b = P.b;
    s = b.atom_set[a];
    e = b.set_example[s];
    A.x = P.pos[3 * a];
    A.y = P.pos[3 * a + 1];
    A.z = P.pos[3 * a + 2];
    A.ox = b.origins[3 * e];
    A.oy = b.origins[3 * e + 1];
    A.oz = b.origins[3 * e + 2];
}

// Box for cutoff rmult*r (_kernels.py:225-227); false when it misses the grid.
__device__ __forceinline__ bool set_radius(Atom &A, double r, double rmult, double res, int D) {
    A.dzr = rmult * r;
    A.dzr2 = A.dzr * A.dzr;
    A.m2inv_r2 = -2.0 / (r * r);
    axis_bounds(A.x, A.dzr, A.ox, res, D, A.i0, A.i1);
    axis_bounds(A.y, A.dzr, A.oy, res, D, A.j0, A.j1);
    axis_bounds(A.z, A.dzr, A.oz, res, D, A.k0, A.k1);
    return A.i0 <= A.i1 && A.j0 <= A.j1 && A.k0 <= A.k1;
}

__device__ __forceinline__ void store_coord(const BwdArgs &P, int a, int lane, double gx,
                                            double gy, double gz) {
    gx = warp_sum(gx);
    gy = warp_sum(gy);
    gz = warp_sum(gz);
    if (lane == 0) {
        P.coord_grad[3 * a + 0] = (float)gx;
        P.coord_grad[3 * a + 1] = (float)gy;
        P.coord_grad[3 * a + 2] = (float)gz;
    }
}

// ---------------------------------------------------------------------------
// Index types: kLPA lanes per atom.  The lanes of an atom share per-axis
// tables (offset, f64 Gaussian factor; kSub entries per axis, sub-boxes for
// larger boxes) and split its (i, j) rows round-robin; each row walks only
// its k span inside the cutoff sphere, two voxels at a time, branch-free
// (voxels outside the sphere load nothing and add an exact 0).
// ---------------------------------------------------------------------------
constexpr int kLPA = 4;                 // lanes per atom
constexpr int kSub = 16;                // table entries per axis
constexpr int kAtomsPerBlock = 256 / kLPA;

struct SmallTables {
    double dx[kSub], ex[kSub], dy[kSub], ey[kSub], dz[kSub], ez[kSub], ezdz[kSub];
};

__global__ void __launch_bounds__(256, 2) k_backward_index(const BwdArgs P) {
    __shared__ SmallTables tabs[kAtomsPerBlock];
    const int sub = threadIdx.x & (kLPA - 1);
    const int slot = threadIdx.x / kLPA;
    const int a = blockIdx.x * kAtomsPerBlock + slot;
    const gm_batch &b = P.b;
    const bool live = a < b.natoms;
    const int D = P.p.npts;
    const double res = P.p.resolution, grm = P.p.gaussian_radius_multiple;
    const float inv_res = (float)(1.0 / res);
    SmallTables &T = tabs[slot];
    // the lanes of one atom (they share T); atoms of a warp may run different
    // sub-box loops, so synchronise only the group
    const unsigned gmask = ((1u << kLPA) - 1u) << ((threadIdx.x & 31) & ~(kLPA - 1));
    double ax0 = 0.0, ay0 = 0.0, az0 = 0.0, ax1 = 0.0, ay1 = 0.0, az1 = 0.0;
    Atom A;
    bool any = false;
    int e = 0, c = 0;
    double d02 = 0.0, qa2 = 0.0, m4inv_r2 = 0.0;
    if (live) {
        int s;
        load_atom(P, a, A, s, e);
        c = b.set_choff[s] + b.atom_type[a];
        const double r = b.atom_radius[a];
        const double d0 = grm * r;
        d02 = d0 * d0;
        const double q0 = (2.0 * grm) / r;
        qa2 = 2.0 * (exp((-2.0 * grm) * grm) * (q0 * q0));
        m4inv_r2 = -4.0 / (r * r);
        any = set_radius(A, r, P.p.radius_multiple, res, D);
    }
    const size_t D3 = (size_t)D * D * D;
    const float *gbase = P.grid_grad + ((size_t)e * b.nchannels + c) * D3;
    // sub-box loop bounds are uniform across the atom's lanes
    const int si_end = any ? A.i1 : -1;
    for (int si = any ? A.i0 : 0; si <= si_end; si += kSub)
        for (int sj = A.j0; sj <= A.j1; sj += kSub)
            for (int sk = A.k0; sk <= A.k1; sk += kSub) {
                const int ni = min(kSub, A.i1 - si + 1), nj = min(kSub, A.j1 - sj + 1),
                          nk = min(kSub, A.k1 - sk + 1);
                __syncwarp(gmask);
                for (int l = sub; l < 3 * kSub; l += kLPA) {
                    const int ax = l / kSub, q = l - ax * kSub;
                    const int n = ax == 0 ? ni : (ax == 1 ? nj : nk);
                    if (q < n) {
                        const double x = ax == 0 ? A.x : (ax == 1 ? A.y : A.z);
                        const double o = ax == 0 ? A.ox : (ax == 1 ? A.oy : A.oz);
                        const int i0 = ax == 0 ? si : (ax == 1 ? sj : sk);
                        const double d = offs(x, o, i0 + q, res);
                        const double E = exp(A.m2inv_r2 * (d * d));
                        double *dt = ax == 0 ? T.dx : (ax == 1 ? T.dy : T.dz);
                        double *et = ax == 0 ? T.ex : (ax == 1 ? T.ey : T.ez);
                        dt[q] = d;
                        et[q] = E;
                        if (ax == 2) T.ezdz[q] = E * d;
                    }
                }
                __syncwarp(gmask);
                const float inv_nj = __frcp_rn((float)nj);
                const float dz0 = (float)T.dz[0];
                const float *gsub = gbase + ((size_t)si * D + sj) * D + sk;
                for (int row = sub; row < ni * nj; row += kLPA) {
                    const int ii = idiv(row, inv_nj), jj = row - ii * nj;
                    const double dx = T.dx[ii], dy = T.dy[jj];
                    const double b2 = fma(dy, dy, dx * dx);
                    const double rem = A.dzr2 - b2;
                    if (rem <= 0.0) continue;
                    const float rho = fmaf(sqrtf((float)rem), 1.0001f, 1e-5f * (float)A.dzr);
                    const int klo = max(0, (int)ceilf(fmaxf((dz0 - rho) * inv_res, -1.0f)));
                    const int khi =
                        min(nk - 1, (int)floorf(fminf((dz0 + rho) * inv_res, (float)nk)));
                    const double exy = T.ex[ii] * T.ey[jj] * m4inv_r2;
                    const float *gr = gsub + ((size_t)ii * D + jj) * D;
                    // Gaussian core of the row: voxels certainly within d0 (shrunk
                    // span; the separable factors reduce them to two FMAs each)
                    int kc0 = khi + 1, kc1 = khi;
                    const double remc = d02 - b2;
                    if (remc > 0.0) {
                        const float rc = fmaf(sqrtf((float)remc), 0.99999f, -1e-4f * (float)res);
                        if (rc > 0.0f) {
                            kc0 = max(klo, (int)ceilf((dz0 - rc) * inv_res));
                            kc1 = min(khi, (int)floorf((dz0 + rc) * inv_res));
                            if (kc0 > kc1) {
                                kc0 = khi + 1;
                                kc1 = khi;
                            }
                        }
                    }
                    // the whole row span first (<= kSub loads in flight), then the math
                    float g[kSub];
#pragma unroll
                    for (int q = 0; q < kSub; q++)
                        g[q] = (klo + q <= khi) ? __ldg(gr + klo + q) : 0.0f;
                    double cs = 0.0, csz = 0.0, ts = 0.0, tsz = 0.0;
#pragma unroll
                    for (int q = 0; q < kSub; q++) {
                        const int kk = klo + q;
                        if (kk > khi) break;
                        const double gq = (double)g[q];
                        if (kk >= kc0 && kk <= kc1) {
                            cs = fma(gq, T.ez[kk], cs);
                            csz = fma(gq, T.ezdz[kk], csz);
                        } else {
                            // shell and boundary voxels: exact f64 classification
                            const double dz = T.dz[kk];
                            const double d2 = fma(dz, dz, b2);
                            const bool in = d2 > 0.0 && d2 < A.dzr2;
                            const double gv = in ? gq : 0.0;
                            const double rd = rsqrt_d(d2);
                            const double sq = gv * qa2 * fma(-A.dzr, rd, 1.0);
                            const double sg = gv * (exy * T.ez[kk]);
                            const double sc = d2 <= d02 ? sg : sq;
                            ts += sc;
                            tsz = fma(sc, dz, tsz);
                        }
                    }
                    // slope/d * offset summed over the row: core terms share exy
                    const double srow = fma(exy, cs, ts);
                    ax0 = fma(srow, dx, ax0);
                    ay0 = fma(srow, dy, ay0);
                    az0 = fma(exy, csz, az0 + tsz);
                }
            }
    double gx = ax0 + ax1, gy = ay0 + ay1, gz = az0 + az1;
#pragma unroll
    for (int o = 1; o < kLPA; o <<= 1) {
        gx += __shfl_xor_sync(0xffffffffu, gx, o);
        gy += __shfl_xor_sync(0xffffffffu, gy, o);
        gz += __shfl_xor_sync(0xffffffffu, gz, o);
    }
    if (live && sub == 0) {
        P.coord_grad[3 * a + 0] = (float)gx;
        P.coord_grad[3 * a + 1] = (float)gy;
        P.coord_grad[3 * a + 2] = (float)gz;
    }
}

// Vector types (_kernels.py:258-314).  With per-atom radii and <= kMaxT
// channels the geometry is shared by all channels of the set: one walk, all
// channel gradients per voxel, the coordinate term from sum_c w_c g_c.  With
// type-indexed radii (or more channels) each channel walks its own box.
__global__ void __launch_bounds__(256) k_backward_vector(const BwdArgs P) {
    __shared__ Tables tabs[kWarps];
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    const int a = blockIdx.x * kWarps + warp;
    const gm_batch &b = P.b;
    if (a >= b.natoms) return;
    const int D = P.p.npts;
    const double res = P.p.resolution, grm = P.p.gaussian_radius_multiple,
                 rmult = P.p.radius_multiple;
    const float inv_res = (float)(1.0 / res);
    Atom A;
    int s, e;
    load_atom(P, a, A, s, e);
    const int Tn = b.set_t[s];
    const int row = b.set_wstart[s] + (a - b.set_start[s]) * Tn;
    const size_t D3 = (size_t)D * D * D;
    const double eg = exp((-2.0 * grm) * grm);
    const float *gset = P.grid_grad + ((size_t)e * b.nchannels + b.set_choff[s]) * D3;
    double gx = 0.0, gy = 0.0, gz = 0.0;

    if (!P.p.radius_type_indexed && Tn <= kMaxT) {
        const double r = b.atom_radius[a];
        const double gr = grm * r, d02 = gr * gr;
        const double q0 = (2.0 * grm) / r;
        const double qa = eg * (q0 * q0);
        const double m4inv_r2 = -4.0 / (r * r);
        double w[kMaxT], tg[kMaxT];
#pragma unroll
        for (int c = 0; c < kMaxT; c++) {
            w[c] = c < Tn ? (double)b.weights[row + c] : 0.0;
            tg[c] = 0.0;
        }
        if (set_radius(A, r, rmult, res, D)) {
            const double dzr = A.dzr;
            walk<false, false>(A, tabs[warp], gset, D, res, inv_res, lane,
                               [&](int, double d2, double dx, double dy, double dz, double exyz,
                                   double voff) {
                                   double dens, sod;  // density, slope / d
                                   if (d2 <= d02) {
                                       dens = exyz;
                                       sod = dens * m4inv_r2;
                                   } else {
                                       const double rd = rsqrt_d(d2);
                                       const double t = fma(d2, rd, -dzr);
                                       dens = (qa * t) * t;
                                       sod = (2.0 * qa) * t * rd;
                                   }
                                   const float *gv = gset + (size_t)voff;
                                   double sw = 0.0;
#pragma unroll
                                   for (int c = 0; c < kMaxT; c++) {
                                       if (c < Tn) {
                                           const double g = (double)__ldg(gv + c * D3);
                                           tg[c] = fma(g, dens, tg[c]);
                                           sw = fma(w[c], g, sw);
                                       }
                                   }
                                   if (d2 > 0.0) {
                                       const double sc = sw * sod;
                                       gx = fma(sc, dx, gx);
                                       gy = fma(sc, dy, gy);
                                       gz = fma(sc, dz, gz);
                                   }
                               });
        }
#pragma unroll
        for (int c = 0; c < kMaxT; c++) {
            if (c < Tn) {
                const double v = warp_sum(tg[c]);
                if (lane == 0 && P.type_grad) P.type_grad[row + c] = (float)v;
            }
        }
    } else {
        for (int c = 0; c < Tn; c++) {
            const double r = P.p.radius_type_indexed ? b.type_radius[b.set_trstart[s] + c]
                                                     : b.atom_radius[a];
            const double w = (double)b.weights[row + c];
            const double gr = grm * r, d02 = gr * gr;
            const double q0 = (2.0 * grm) / r;
            const double qa = eg * (q0 * q0);
            const double m4inv_r2 = -4.0 / (r * r);
            double tg = 0.0;
            if (set_radius(A, r, rmult, res, D)) {
                const double dzr = A.dzr;
                walk<false, true>(A, tabs[warp], gset + (size_t)c * D3, D, res, inv_res, lane,
                                  [&](int, double d2, double dx, double dy, double dz, double exyz,
                                      double g) {
                                      double dens, sod;
                                      if (d2 <= d02) {
                                          dens = exyz;
                                          sod = dens * m4inv_r2;
                                      } else {
                                          const double rd = rsqrt_d(d2);
                                          const double t = fma(d2, rd, -dzr);
                                          dens = (qa * t) * t;
                                          sod = (2.0 * qa) * t * rd;
                                      }
                                      tg = fma(g, dens, tg);
                                      if (d2 > 0.0 && w != 0.0) {
                                          const double sc = (w * g) * sod;
                                          gx = fma(sc, dx, gx);
                                          gy = fma(sc, dy, gy);
                                          gz = fma(sc, dz, gz);
                                      }
                                  });
            }
            tg = warp_sum(tg);
            if (lane == 0 && P.type_grad) P.type_grad[row + c] = (float)tg;
        }
    }
    store_coord(P, a, lane, gx, gy, gz);
}

}  // namespace

gm_status backward_impl(const gm_params *p, const gm_batch *b, const Workspace &ws,
                        const float *grid_grad, float *coord_grad, float *type_grad,
                        cudaStream_t s) {
    BwdArgs P;
    P.p = *p;
    P.b = *b;
    P.pos = ws.pos;
    P.grid_grad = grid_grad;
    P.coord_grad = coord_grad;
    P.type_grad = type_grad;
    if (b->vector_mode)
        k_backward_vector<<<(b->natoms + kWarps - 1) / kWarps, 256, 0, s>>>(P);
    else
        k_backward_index<<<(b->natoms + kAtomsPerBlock - 1) / kAtomsPerBlock, 256, 0, s>>>(P);
    LAUNCH_CHECK();
    return GM_OK;
}
