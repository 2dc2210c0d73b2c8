// backward.cu -- grid gradients -> atom coordinate (and type) gradients.
//
// Reference: _kernels.py:209-255 (backward_index), 258-314 (backward_vector):
// per atom, a float64 sum over its voxel box (cut = rmult * r) of
// g * slope(d) / d * (x - v), and for vector types sum g * density per channel.
//
// B200 design: one warp per atom, batched over every set of every example.
// The Gaussian core is separable, exp(-2 d^2/r^2) = Ex(i) Ey(j) Ez(k), so a
// warp first fills per-axis tables (offset and f64 exp factor, <= 64 entries
// per axis, in shared memory): ~40 f64 exps per atom instead of one per voxel.
// Lanes then own (row, column) pairs of the box's j-k face -- column fixed per
// lane -- and walk the i axis with four independent loads in flight.  Geometry
// and accumulation stay in f64 (f32 terms fail the 1e-6 gate on
// near-cancelling components); the quadratic tail uses one f64 rsqrt.  Lane
// partial sums are reduced with warp shuffles: no atomics, deterministic.
#include "common.cuh"

namespace {

constexpr int kMaxN = 64;   // table capacity per axis (box edge in voxels)
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

struct AtomGeom {
    double x, y, z, ox, oy, oz, m2inv_r2, res;
    int i0, j0, k0, ni, nj, nk;
    bool direct;
};

// Box (_kernels.py:225-227) and per-axis tables: d = x - (o + i*res) in the
// reference's association, E = exp(-2 d^2 / r^2) in f64.  Returns false for an
// empty box; sets G.direct when an edge exceeds the table capacity (the walk
// then evaluates offsets and exponentials per voxel).
__device__ __forceinline__ bool build_tables(AtomGeom &G, double cut, double m2inv_r2, double res,
                                             int D, Tables &T, int lane) {
    int i1, j1, k1;
    axis_bounds(G.x, cut, G.ox, res, D, G.i0, i1);
    axis_bounds(G.y, cut, G.oy, res, D, G.j0, j1);
    axis_bounds(G.z, cut, G.oz, res, D, G.k0, k1);
    if (G.i0 > i1 || G.j0 > j1 || G.k0 > k1) return false;
    G.ni = i1 - G.i0 + 1;
    G.nj = j1 - G.j0 + 1;
    G.nk = k1 - G.k0 + 1;
    G.m2inv_r2 = m2inv_r2;
    G.res = res;
    G.direct = G.ni > kMaxN || G.nj > kMaxN || G.nk > kMaxN;
    if (G.direct) return true;
    __syncwarp();
    for (int l = lane; l < G.ni; l += 32) {
        const double d = __dsub_rn(G.x, __dadd_rn(G.ox, __dmul_rn((double)(G.i0 + l), res)));
        T.dx[l] = d;
        T.ex[l] = exp(m2inv_r2 * (d * d));
    }
    for (int l = lane; l < G.nj; l += 32) {
        const double d = __dsub_rn(G.y, __dadd_rn(G.oy, __dmul_rn((double)(G.j0 + l), res)));
        T.dy[l] = d;
        T.ey[l] = exp(m2inv_r2 * (d * d));
    }
    for (int l = lane; l < G.nk; l += 32) {
        const double d = __dsub_rn(G.z, __dadd_rn(G.oz, __dmul_rn((double)(G.k0 + l), res)));
        T.dz[l] = d;
        T.ez[l] = exp(m2inv_r2 * (d * d));
    }
    __syncwarp();
    return true;
}

__device__ __forceinline__ double offs(double x, double o, int i, double res) {
    return __dsub_rn(x, __dadd_rn(o, __dmul_rn((double)i, res)));
}

// 1/sqrt(d2) to ~1e-13: f32 MUFU estimate + one f64 Newton step.
__device__ __forceinline__ double rsqrt_d(double d2) {
    const double y0 = (double)rsqrtf((float)d2);
    const double e = fma(-d2 * y0, y0, 1.0);
    return fma(0.5 * y0, e, y0);
}

// Walk the box of one atom for one channel.  f(slot, d2, dx, dy, dz, Exyz, g)
// is called for every voxel with 0 <= d2 < dzr2 (d2 > 0 when SKIP_CENTER)
// and g != 0, in a fixed order per lane; `slot` alternates so callers can keep
// two independent accumulator chains.  Eight loads per lane are issued before
// any is consumed.
template <bool SKIP_CENTER, typename F>
__device__ __forceinline__ void walk_box(const AtomGeom &G, const Tables &T, const float *gbase,
                                         int D, double dzr2, int lane, F &&f) {
    const size_t plane = (size_t)D * D;
    for (int kb = 0; kb < G.nk; kb += 32) {
        const int nks = min(32, G.nk - kb);
        const float inv = __frcp_rn((float)nks);
        const int rpi = small_div(32, inv);
        const int r = small_div(lane, inv), kk = kb + lane - r * nks;
        if (r >= rpi) continue;
        const double dz = G.direct ? offs(G.z, G.oz, G.k0 + kk, G.res) : T.dz[kk];
        const double ez = G.direct ? 1.0 : T.ez[kk];
        const double dz2 = dz * dz;
        for (int jj = r; jj < G.nj; jj += rpi) {
            const double dy = G.direct ? offs(G.y, G.oy, G.j0 + jj, G.res) : T.dy[jj];
            const double dyz2 = fma(dy, dy, dz2);
            const double eyz = G.direct ? 1.0 : T.ey[jj] * ez;
            const float *gp = gbase + ((size_t)G.i0 * D + (G.j0 + jj)) * D + (G.k0 + kk);
            for (int i0 = 0; i0 < G.ni; i0 += 8) {
                float g[8];
#pragma unroll
                for (int q = 0; q < 8; q++) {
                    const int ii = i0 + q;
                    bool in = false;
                    if (ii < G.ni) {
                        const double dx = G.direct ? offs(G.x, G.ox, G.i0 + ii, G.res) : T.dx[ii];
                        const double d2 = fma(dx, dx, dyz2);
                        in = (SKIP_CENTER ? d2 > 0.0 : true) && d2 < dzr2;
                    }
                    g[q] = in ? __ldg(gp + (size_t)ii * plane) : 0.0f;
                }
#pragma unroll
                for (int q = 0; q < 8; q++) {
                    if (g[q] != 0.0f) {
                        const int ii = i0 + q;
                        const double dx = G.direct ? offs(G.x, G.ox, G.i0 + ii, G.res) : T.dx[ii];
                        const double d2 = fma(dx, dx, dyz2);
                        const double exyz = G.direct ? exp(G.m2inv_r2 * d2) : T.ex[ii] * eyz;
                        f(q & 1, d2, dx, dy, dz, exyz, (double)g[q]);
                    }
                }
            }
        }
    }
}

__global__ void __launch_bounds__(256, 3) k_backward_index(const BwdArgs A) {
    __shared__ Tables tabs[kWarps];
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    const int a = blockIdx.x * kWarps + warp;
    const gm_batch &b = A.b;
    if (a >= b.natoms) return;
    const int D = A.p.npts;
    const double res = A.p.resolution, grm = A.p.gaussian_radius_multiple,
                 rmult = A.p.radius_multiple;
    const int s = b.atom_set[a];
    const int e = b.set_example[s];
    const int c = b.set_choff[s] + b.atom_type[a];
    AtomGeom G;
    G.x = A.pos[3 * a];
    G.y = A.pos[3 * a + 1];
    G.z = A.pos[3 * a + 2];
    G.ox = b.origins[3 * e];
    G.oy = b.origins[3 * e + 1];
    G.oz = b.origins[3 * e + 2];
    const double r = b.atom_radius[a];
    const double inv_r2 = 1.0 / (r * r);
    const double d0 = grm * r, d02 = d0 * d0;
    const double dzr = rmult * r, dzr2 = dzr * dzr;
    const double q0 = (2.0 * grm) / r;
    const double qa2 = 2.0 * (exp((-2.0 * grm) * grm) * (q0 * q0));
    const double m4inv_r2 = -4.0 * inv_r2;
    double ax0 = 0.0, ay0 = 0.0, az0 = 0.0, ax1 = 0.0, ay1 = 0.0, az1 = 0.0;
    Tables &T = tabs[warp];
    if (build_tables(G, dzr, -2.0 * inv_r2, res, D, T, lane)) {
        const float *gbase = A.grid_grad + ((size_t)e * b.nchannels + c) * ((size_t)D * D * D);
        walk_box<true>(G, T, gbase, D, dzr2, lane,
                       [&](int slot, double d2, double dx, double dy, double dz, double exyz,
                           double g) {
                           // slope / d: Gaussian exp(-2 d^2/r^2) * (-4/r^2) (no sqrt);
                           // tail 2 qa (d - dzr) / d
                           const double rd = rsqrt_d(d2);
                           const double sq = g * (qa2 * fma(d2, rd, -dzr)) * rd;
                           const double sg = g * exyz * m4inv_r2;
                           const double sc = d2 <= d02 ? sg : sq;
                           if (slot) {
                               ax1 = fma(sc, dx, ax1);
                               ay1 = fma(sc, dy, ay1);
                               az1 = fma(sc, dz, az1);
                           } else {
                               ax0 = fma(sc, dx, ax0);
                               ay0 = fma(sc, dy, ay0);
                               az0 = fma(sc, dz, az0);
                           }
                       });
    }
    double gx = ax0 + ax1, gy = ay0 + ay1, gz = az0 + az1;
    gx = warp_sum(gx);
    gy = warp_sum(gy);
    gz = warp_sum(gz);
    if (lane == 0) {
        A.coord_grad[3 * a + 0] = (float)gx;
        A.coord_grad[3 * a + 1] = (float)gy;
        A.coord_grad[3 * a + 2] = (float)gz;
    }
}

// Vector types (_kernels.py:258-314).  With per-atom radii and <= kMaxT
// channels the geometry is shared by all channels of the set: one walk, all
// channel gradients per voxel, the coordinate term from sum_c w_c g_c.  With
// type-indexed radii (or many channels) each channel has its own box.
__global__ void __launch_bounds__(256) k_backward_vector(const BwdArgs A) {
    __shared__ Tables tabs[kWarps];
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    const int a = blockIdx.x * kWarps + warp;
    const gm_batch &b = A.b;
    if (a >= b.natoms) return;
    const int D = A.p.npts;
    const double res = A.p.resolution, grm = A.p.gaussian_radius_multiple,
                 rmult = A.p.radius_multiple;
    const int s = b.atom_set[a];
    const int e = b.set_example[s];
    const int Tn = b.set_t[s];
    const int row = b.set_wstart[s] + (a - b.set_start[s]) * Tn;
    AtomGeom G;
    G.x = A.pos[3 * a];
    G.y = A.pos[3 * a + 1];
    G.z = A.pos[3 * a + 2];
    G.ox = b.origins[3 * e];
    G.oy = b.origins[3 * e + 1];
    G.oz = b.origins[3 * e + 2];
    const size_t D3 = (size_t)D * D * D;
    const double eg = exp((-2.0 * grm) * grm);
    const float *gset = A.grid_grad + ((size_t)e * b.nchannels + b.set_choff[s]) * D3;
    double gx = 0.0, gy = 0.0, gz = 0.0;
    Tables &T = tabs[warp];

    if (!A.p.radius_type_indexed && Tn <= kMaxT) {
        const double r = b.atom_radius[a];
        const double inv_r2 = 1.0 / (r * r);
        const double gr = grm * r, d02 = gr * gr;
        const double dzr = rmult * r, dzr2 = dzr * dzr;
        const double q0 = (2.0 * grm) / r;
        const double qa = eg * (q0 * q0);
        const double m4inv_r2 = -4.0 * inv_r2;
        double w[kMaxT], tg[kMaxT];
#pragma unroll
        for (int c = 0; c < kMaxT; c++) {
            w[c] = c < Tn ? (double)b.weights[row + c] : 0.0;
            tg[c] = 0.0;
        }
        if (build_tables(G, dzr, -2.0 * inv_r2, res, D, T, lane)) {
            const size_t plane = (size_t)D * D;
            for (int kb = 0; kb < G.nk; kb += 32) {
                const int nks = min(32, G.nk - kb);
                const float inv = __frcp_rn((float)nks);
                const int rpi = small_div(32, inv);
                const int rr = small_div(lane, inv), kk = kb + lane - rr * nks;
                if (rr >= rpi) continue;
                const double dz = G.direct ? offs(G.z, G.oz, G.k0 + kk, res) : T.dz[kk];
                const double ez = G.direct ? 1.0 : T.ez[kk];
                for (int jj = rr; jj < G.nj; jj += rpi) {
                    const double dy = G.direct ? offs(G.y, G.oy, G.j0 + jj, res) : T.dy[jj];
                    const double dyz2 = fma(dy, dy, dz * dz);
                    const double eyz = G.direct ? 1.0 : T.ey[jj] * ez;
                    const float *gp = gset + ((size_t)G.i0 * D + (G.j0 + jj)) * D + (G.k0 + kk);
                    for (int ii = 0; ii < G.ni; ii++) {
                        const double dx = G.direct ? offs(G.x, G.ox, G.i0 + ii, res) : T.dx[ii];
                        const double d2 = fma(dx, dx, dyz2);
                        if (d2 >= dzr2) continue;
                        double dens, sod;  // density, slope / d
                        if (d2 <= d02) {
                            dens = G.direct ? exp(G.m2inv_r2 * d2) : T.ex[ii] * eyz;
                            sod = dens * m4inv_r2;
                        } else {
                            const double rd = rsqrt_d(d2);
                            const double t = fma(d2, rd, -dzr);
                            dens = (qa * t) * t;
                            sod = (2.0 * qa) * t * rd;
                        }
                        const float *gv = gp + (size_t)ii * plane;
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
                    }
                }
            }
        }
#pragma unroll
        for (int c = 0; c < kMaxT; c++) {
            if (c < Tn) {
                const double v = warp_sum(tg[c]);
                if (lane == 0 && A.type_grad) A.type_grad[row + c] = (float)v;
            }
        }
    } else {
        for (int c = 0; c < Tn; c++) {
            const double r = A.p.radius_type_indexed ? b.type_radius[b.set_trstart[s] + c]
                                                     : b.atom_radius[a];
            const double w = (double)b.weights[row + c];
            const double inv_r2 = 1.0 / (r * r);
            const double gr = grm * r, d02 = gr * gr;
            const double dzr = rmult * r, dzr2 = dzr * dzr;
            const double q0 = (2.0 * grm) / r;
            const double qa = eg * (q0 * q0);
            const double m4inv_r2 = -4.0 * inv_r2;
            double tg = 0.0;
            if (build_tables(G, dzr, -2.0 * inv_r2, res, D, T, lane)) {
                walk_box<false>(G, T, gset + (size_t)c * D3, D, dzr2, lane,
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
            if (lane == 0 && A.type_grad) A.type_grad[row + c] = (float)tg;
        }
    }
    gx = warp_sum(gx);
    gy = warp_sum(gy);
    gz = warp_sum(gz);
    if (lane == 0) {
        A.coord_grad[3 * a + 0] = (float)gx;
        A.coord_grad[3 * a + 1] = (float)gy;
        A.coord_grad[3 * a + 2] = (float)gz;
    }
}

}  // namespace

gm_status backward_impl(const gm_params *p, const gm_batch *b, const Workspace &ws,
                        const float *grid_grad, float *coord_grad, float *type_grad,
                        cudaStream_t s) {
    BwdArgs A;
    A.p = *p;
    A.b = *b;
    A.pos = ws.pos;
    A.grid_grad = grid_grad;
    A.coord_grad = coord_grad;
    A.type_grad = type_grad;
    const int blocks = (b->natoms + kWarps - 1) / kWarps;
    if (b->vector_mode) k_backward_vector<<<blocks, 256, 0, s>>>(A);
    else k_backward_index<<<blocks, 256, 0, s>>>(A);
    LAUNCH_CHECK();
    return GM_OK;
}
