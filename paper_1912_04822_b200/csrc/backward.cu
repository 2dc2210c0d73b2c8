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
#include <stdlib.h>

#include <type_traits>

#include "common.cuh"

namespace {

constexpr int kMaxT = 16;   // channels kept in registers by the shared-geometry vector path

struct BwdArgs {
    gm_params p;
    gm_batch b;
    const double *pos;
    const float *grid_grad;
    float *coord_grad;
    float *type_grad;
    double *coord_grad64;  // optional f64 outputs (the reference-shaped *_host entry
    double *type_grad64;   // points return the f64 sums like _kernels.py:214,265)
    const BwdAtom *batoms; // index mode: per-atom records of the prepare pass
    const int32_t *atom_order; // vector mode: atom of each launch slot (bwd_slot inverse)
    const VBwdAtom *vbatoms;   // vector mode: per-slot records of the prepare pass
    double eg;             // exp(-2 grm^2), a batch constant (_kernels.py:224)
    int early;             // 1: the records may be read before the PDL wait (the
                           // previous launch on this workspace was the forward)
};


// One atom (for one channel radius): position, origin, full voxel box.
struct Atom {
    double x, y, z, ox, oy, oz;
    double r;  // radius * radius_scale (vector walk)
    double dzr, dzr2, m2inv_r2;
    int i0, i1, j0, j1, k0, k1;
};

__device__ __forceinline__ double offs(double x, double o, int i, double res) {
    // _kernels.py:232-236: x - (o + i*res), same association, no contraction
    return __dsub_rn(x, __dadd_rn(o, __dmul_rn((double)i, res)));
}

__device__ __forceinline__ float approx_sqrt(float x) {
    float y;
    asm("sqrt.approx.ftz.f32 %0, %1;" : "=f"(y) : "f"(x));
    return y;
}

// 1/sqrt(d2) to ~1e-13 relative: the f64 MUFU estimate (MUFU.RSQ64H, ~2^-22)
// + one f64 Newton step -- one XU op, no f32 <-> f64 conversions.
__device__ __forceinline__ double rsqrt_d(double d2) {
    double y0;
    asm("rsqrt.approx.ftz.f64 %0, %1;" : "=d"(y0) : "d"(d2));
    const double e = fma(-d2 * y0, y0, 1.0);
    return fma(0.5 * y0, e, y0);
}

// exp(x) for x <= 0 (the per-axis Gaussian factors exp(-2 d^2 / r^2)):
// x = n ln2 + r with |r| <= ln2/2 (fdlibm's split ln2, exact n ln2_hi), a
// degree-11 Taylor polynomial (relative error < 1e-14), scaled by 2^n
// through the exponent field.  Branch-free, ~17 instructions instead of the
// general libm path.
__device__ __forceinline__ double exp_nonpos(double x) {
    x = fmax(x, -700.0);
    const double n = rint(x * 1.4426950408889634);
    double r = fma(-n, 6.93147180369123816490e-01, x);
    r = fma(-n, 1.90821492927058770002e-10, r);
    double p = 2.5052108385441720e-08;  // 1/11!
    p = fma(p, r, 2.7557319223985893e-07);
    p = fma(p, r, 2.7557319223985888e-06);
    p = fma(p, r, 2.4801587301587302e-05);
    p = fma(p, r, 1.9841269841269841e-04);
    p = fma(p, r, 1.3888888888888889e-03);
    p = fma(p, r, 8.3333333333333332e-03);
    p = fma(p, r, 4.1666666666666664e-02);
    p = fma(p, r, 1.6666666666666666e-01);
    p = fma(p, r, 0.5);
    p = fma(p, r, 1.0);
    p = fma(p, r, 1.0);
    return p * __hiloint2double(((int)n + 1023) << 20, 0);
}

// Exact float -> double widening on the integer pipe (F2F.F64.F32 runs on the
// XU).  Zeros and denormals map to signed zero (grid gradients below 1e-38
// contribute nothing at f32 output precision); inf / NaN are not expected in
// gradients.  The index walk converts with F2F (measured faster there).
__device__ __forceinline__ double widen(float f) {
    const unsigned u = __float_as_uint(f);
    const bool nz = (u & 0x7f800000u) != 0u;
    const unsigned hi = (u & 0x80000000u) | (nz ? ((u >> 3) & 0x0fffffffu) + (896u << 20) : 0u);
    const unsigned lo = nz ? (u << 29) : 0u;
    return __hiloint2double((int)hi, (int)lo);
}

// floor(a / b) for 0 <= a < 2^16, 1 <= b <= 64 (float reciprocal, exact here).
__device__ __forceinline__ int idiv(int a, float inv_b) {
    return (int)(((float)a + 0.5f) * inv_b);
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
#if GM_BWD_SPLITSUM
    double v[4] = {gx, gy, gz, 0.0};
    int idx;
    const double s = warp_sum_split<4>(v, lane, idx);  // lanes 8 idx .. 8 idx + 7
    if ((lane & 7) == 0 && idx < 3) {
        if (P.coord_grad64) P.coord_grad64[3 * a + idx] = s;
        else P.coord_grad[3 * a + idx] = (float)s;
    }
#else
    gx = warp_sum(gx);
    gy = warp_sum(gy);
    gz = warp_sum(gz);
    if (lane == 0 && P.coord_grad64) {
        P.coord_grad64[3 * a + 0] = gx;
        P.coord_grad64[3 * a + 1] = gy;
        P.coord_grad64[3 * a + 2] = gz;
    } else if (lane == 0) {
        P.coord_grad[3 * a + 0] = (float)gx;
        P.coord_grad[3 * a + 1] = (float)gy;
        P.coord_grad[3 * a + 2] = (float)gz;
    }
#endif
}

// ---------------------------------------------------------------------------
// One warp per atom, flattened walk (index and vector types).
//
// The atom's box is cut into sub-boxes of <= kTab voxels per axis and chunks
// of <= kIRows / kRows (i, j) rows (index / vector walk).  Phase 1: lanes
// compute each row's k span inside the cutoff sphere and a warp scan lays the
// non-empty rows out back to back
// (row table in shared memory: start offset, k origin, b2 = dx^2 + dy^2, dx,
// dy, Gaussian factor Ex*Ey).  Phase 2: the warp walks the flattened list in
// windows of 32 voxels, kU windows per step -- every lane has a voxel (no
// lane idles on short rows); a lane finds its row from a bit mask of the row
// starts inside its window (REDUX + popc).  Geometry and accumulation in
// f64; the tail's 1/d from MUFU.RSQ64H + one Newton step.
// ---------------------------------------------------------------------------
#ifndef GM_BWD_WARPS
#define GM_BWD_WARPS 1
#endif
constexpr int kBwdWarps = GM_BWD_WARPS;
#ifndef GM_BWD_ROWS
// rows per chunk of the index walk: two phase-1 passes of 32 rows exactly
// (GM_BWD_P1X2), and 4.9 KB of shared memory per warp lets all 32 one-warp CTAs
// reside.  C2 / C5 backward: 48 rows 100.6 / 458 us, 64 92.6 / 433, 72 96.6 /
// 454, 80 96.0 / 446, 88 94.5 / 441, 96 94.5 / 435, 128 94.7 / 433, 192 106 / 455
#define GM_BWD_ROWS 64
#endif
#ifndef GM_BWDV_ROWS
#define GM_BWDV_ROWS 96  // rows per chunk of the vector walk (64: C4 backward 303.5 -> 305.6 us)
#endif
#ifndef GM_BWD_KU
#define GM_BWD_KU 4
#endif
#ifndef GM_BWD_CHAINS
#define GM_BWD_CHAINS 1
#endif
#ifndef GM_BWD_P1X2
#define GM_BWD_P1X2 2  // index walk, phase 1: rows per lane per pass (1 or 2)
#endif
#ifndef GM_BWD_PREFETCH
// L2 prefetch of each row span in phase 1: 0 none, 1 prefetch.global.L2 of the
// span's first / last line, 2 cp.async.bulk.prefetch of exactly its 16-B
// granules.  C2 / C5 backward: 102.7 / 479.6 us, 94.5 / 436.6 us, 123.1 / 512.5
// us; DRAM reads equal in all three (83.5 / 550 MB: HBM fills whole 128-B
// lines, tools/pf_ab.sh)
#define GM_BWD_PREFETCH 1
#endif
#ifndef GM_BWD_GGHINT
#define GM_BWD_GGHINT 0  // cache hint of the index-mode grid_grad loads (see ld_gg)
#endif
#ifndef GM_BWDV_GGHINT
#define GM_BWDV_GGHINT 3  // cache hint of the shared-walk vector grid_grad loads
#endif
#ifndef GM_BWD_SPLITSUM
#define GM_BWD_SPLITSUM 1  // multi-value warp sums for the per-atom gradient epilogues
#endif
#ifndef GM_BWDV_D48
#define GM_BWDV_D48 1  // vector backward specialised for 14 channels on 48^3 grids
#endif
#ifndef GM_BWDV_PTR
#define GM_BWDV_PTR 1  // vector walk: stepped 64-bit channel pointers (vs 32-bit offsets)
#endif
#ifndef GM_BWDV_MINB
#define GM_BWDV_MINB 16  // vector-mode backward: resident one-warp CTAs per SM
#endif
#ifndef GM_BWD_MINB
#define GM_BWD_MINB 32
#endif
// grid_grad loads (read-only for the kernel's lifetime) with a cache hint:
// 0 plain ld.global.nc, 1 L1::no_allocate, 2 L2 evict_last, 3 L1::evict_last.
// Measured: index mode is best plain (C2 89.3 us; 1: 94.9, 2: 90.6, 3: 90.1);
// the vector walk's 14-channel loads gain from L1::evict_last (C4 319 -> 314 us).
template <int HINT>
__device__ __forceinline__ float ld_gg(const float *p) {
    float v;
    if (HINT == 1) {
        asm("ld.global.nc.L1::no_allocate.f32 %0, [%1];" : "=f"(v) : "l"(p));
    } else if (HINT == 2) {
        uint64_t pol;
        asm("createpolicy.fractional.L2::evict_last.b64 %0, 1.0;" : "=l"(pol));
        asm("ld.global.nc.L2::cache_hint.f32 %0, [%1], %2;" : "=f"(v) : "l"(p), "l"(pol));
    } else if (HINT == 3) {
        asm("ld.global.nc.L1::evict_last.f32 %0, [%1];" : "=f"(v) : "l"(p));
    } else {
        v = __ldg(p);
    }
    return v;
}

constexpr int kRows = GM_BWDV_ROWS;  // rows per chunk (vector walk)
constexpr int kIRows = GM_BWD_ROWS;  // rows per chunk (index walk)
constexpr int kTab = 32;      // table entries per axis (sub-box edge)
constexpr int kU = GM_BWD_KU;  // 32-voxel windows per step (loads in flight per lane)

struct __align__(8) RowEntry {
    int voff;    // grid offset of the row's voxel k minus its flattened index:
                 // voxel v of the row sits at gbase + voff + v
    int kz;      // table index of voxel v: kz + v
    double b2;   // dx^2 + dy^2
    double exy;  // Ex * Ey * exy_scale
    double dx, dy;
};

struct WarpBwd {
    double dz[kTab], ez[kTab], dx[kTab], ex[kTab], dy[kTab], ey[kTab];
    double wt[kMaxT];  // vector mode: the atom's type weights (broadcast reads)
    RowEntry rows[kRows];
    unsigned starts[kRows * kTab / 32 + kU];  // bit v: a row starts at flattened voxel v
};

// f(slot, d2, R, dz, ez, voxel_offset, g): every voxel of the box with
// d2 < dzr2 (others get g = 0 / are skipped), g loaded by the walk when LOADG.
template <bool LOADG, int KU = kU, typename F>
__device__ __forceinline__ void flat_walk(const Atom &A, WarpBwd &W, const float *gbase, int D,
                                          double res, float inv_res, int lane, double exy_scale,
                                          F &&f) {
    const unsigned lt = (1u << lane) - 1u;
    const double dzr = A.dzr, dzr2 = A.dzr2;
    for (int si = A.i0; si <= A.i1; si += kTab)
        for (int sj = A.j0; sj <= A.j1; sj += kTab)
            for (int sk = A.k0; sk <= A.k1; sk += kTab) {
                const int ni = min(kTab, A.i1 - si + 1), nj = min(kTab, A.j1 - sj + 1),
                          nk = min(kTab, A.k1 - sk + 1);
                __syncwarp();
                for (int l = lane; l < ni + nj + nk; l += 32) {
                    const int ax = l < ni ? 0 : (l < ni + nj ? 1 : 2);
                    const int q = l - (ax == 0 ? 0 : (ax == 1 ? ni : ni + nj));
                    const double d = ax == 0 ? offs(A.x, A.ox, si + q, res)
                                             : (ax == 1 ? offs(A.y, A.oy, sj + q, res)
                                                        : offs(A.z, A.oz, sk + q, res));
                    const double E = exp_nonpos(A.m2inv_r2 * (d * d));
                    double *dt = ax == 0 ? W.dx : (ax == 1 ? W.dy : W.dz);
                    double *et = ax == 0 ? W.ex : (ax == 1 ? W.ey : W.ez);
                    dt[q] = d;
                    et[q] = E;
                }
                __syncwarp();
                const float dz0 = (float)W.dz[0];
                const float inv_nj = __frcp_rn((float)nj);
                const size_t sbase = ((size_t)si * D + sj) * D + sk;
                const int nrows_all = ni * nj;
                for (int rb = 0; rb < nrows_all; rb += kRows) {
                    // ---- phase 1: row spans, compacted with a warp scan ----
                    int nrow = 0, total = 0;
                    const int nwords = (min(nrows_all - rb, kRows) * nk + 31) >> 5;
                    for (int w = lane; w < nwords + KU; w += 32) W.starts[w] = 0u;
                    __syncwarp();
                    const int rend = min(nrows_all, rb + kRows);
                    for (int r0 = rb; r0 < rend; r0 += 32) {
                        const int row = r0 + lane;
                        int len = 0, klo = 0, ii = 0, jj = 0;
                        double b2 = 0.0, dx = 0.0, dy = 0.0;
                        if (row < rend) {
                            ii = idiv(row, inv_nj);
                            jj = row - ii * nj;
                            dx = W.dx[ii];
                            dy = W.dy[jj];
                            b2 = fma(dy, dy, dx * dx);
                            const double rem = dzr2 - b2;
                            if (rem > 0.0) {
                                const float rho =
                                    fmaf(approx_sqrt((float)rem), 1.0001f, 1e-5f * (float)dzr);
                                klo = max(0, __float2int_ru(fmaxf((dz0 - rho) * inv_res, -1.0f)));
                                const int khi = min(
                                    nk - 1, __float2int_rd(fminf((dz0 + rho) * inv_res, (float)nk)));
                                len = max(0, khi - klo + 1);
                            }
                        }
                        int sc = len;  // inclusive scan of the span lengths
#pragma unroll
                        for (int o = 1; o < 32; o <<= 1) {
                            const int t = __shfl_up_sync(0xffffffffu, sc, o);
                            if (lane >= o) sc += t;
                        }
                        const unsigned m = __ballot_sync(0xffffffffu, len > 0);
                        if (len > 0) {
                            RowEntry &R = W.rows[nrow + __popc(m & lt)];
                            const int st = total + sc - len;
                            atomicOr(&W.starts[st >> 5], 1u << (st & 31));
                            R.voff = (int)sbase + (ii * D + jj) * D + klo - st;
                            R.kz = klo - st;
                            R.b2 = b2;
                            R.exy = (W.ex[ii] * W.ey[jj]) * exy_scale;
                            R.dx = dx;
                            R.dy = dy;
                        }
                        nrow += __popc(m);
                        total += __shfl_sync(0xffffffffu, sc, 31);
                    }
                    __syncwarp();
                    // ---- phase 2: KU windows of 32 voxels per step ----
                    // voxel v's row = (row starts <= v) - 1: one bitmap word per window
                    const unsigned le = 0xffffffffu >> (31 - lane);
                    int cur = -1;  // rows started before the next window, minus one
                    for (int base = 0; base < total; base += 32 * KU) {
                        int myrow[KU];
#pragma unroll
                        for (int u = 0; u < KU; u++) {
                            const unsigned M = W.starts[(base >> 5) + u];
                            myrow[u] = cur + __popc(M & le);
                            cur += __popc(M);
                        }
                        float g[KU];
                        int kk[KU];
                        int vo[KU];
#pragma unroll
                        for (int u = 0; u < KU; u++) {
                            const int v = base + 32 * u + lane;
                            g[u] = 0.0f;
                            kk[u] = 0;
                            vo[u] = 0;
                            if (v < total) {
                                const RowEntry &R = W.rows[myrow[u]];
                                kk[u] = R.kz + v;
                                vo[u] = R.voff + v;
                                if (LOADG) g[u] = ld_gg<GM_BWD_GGHINT>(gbase + vo[u]);
                            }
                        }
#pragma unroll
                        for (int u = 0; u < KU; u++) {
                            const int v = base + 32 * u + lane;
                            if (v < total) {
                                const RowEntry &R = W.rows[myrow[u]];
                                const double dz = W.dz[kk[u]];
                                const double d2 = fma(dz, dz, R.b2);
                                f(GM_BWD_CHAINS > 1 ? (u & 1) : 0, d2, R, dz, W.ez[kk[u]], (size_t)vo[u], g[u]);
                            }
                        }
                    }
                    __syncwarp();
                }
            }
}

// ---------------------------------------------------------------------------
// Index types: the same flattened walk, specialised.  Row records carry the
// f64 row constants (dx, dy, b2 = dx^2 + dy^2, Ex Ey (-4/r^2)) and the grid
// offset; phase 2 is branch-free: voxels past the end of the list clamp their
// addresses to the last voxel and contribute zero, so every lane issues the
// same instruction stream (loads for all kU windows first, then the math).
// ---------------------------------------------------------------------------
struct __align__(16) IRow {
    double dx, dy;   // row offsets x - (o + i res), y - (o + j res)
    double b2, exy;  // dx^2 + dy^2; Ex Ey (-4 / r^2)
    const float *gp; // grid_grad address of the row's voxel v, minus v
    int kz;          // table index of voxel v, minus v
    int pad;
};
static_assert(sizeof(IRow) == 48, "IRow must be 48 bytes");

struct WarpIdx {
    double2 zt[kTab];  // per k: offset z - (o + k res), Gaussian factor Ez
    double dx[kTab], ex[kTab], dy[kTab], ey[kTab];
    IRow rows[kIRows];
    unsigned starts[kIRows * kTab / 32 + kU];  // bit v: a row starts at flattened voxel v
};

__global__ void __launch_bounds__(kBwdWarps * 32, GM_BWD_MINB) k_backward_index(const BwdArgs P) {
    // the next prepare pass may launch now: it waits for this grid before
    // writing the workspace this kernel reads
    pdl_trigger();
    __shared__ WarpIdx wsm[kBwdWarps];
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    const int rec = blockIdx.x * kBwdWarps + warp;  // record slot (launch order)
    if (rec >= P.b.natoms) return;
    WarpIdx &W = wsm[warp];
    const int D = P.p.npts;
    const double res = P.p.resolution;
    const float inv_res = (float)(1.0 / res);
    // right after a prepare pass (which triggers its dependents before its
    // stores) the records are only valid after the wait
    if (!P.early) pdl_wait();
    // the prepare pass's record: position relative to the origin, constants,
    // and the forward item's box (_kernels.py:225-227) -- one load level
    const BwdAtom B = P.batoms[rec];
    const int a = B.atom;
    const int i0 = box_lo(B.ibox), i1 = box_hi(B.ibox), j0 = box_lo(B.jbox),
              j1 = box_hi(B.jbox), k0 = box_lo(B.kbox), k1 = box_hi(B.kbox);
    const double dzr = B.dzr, dzr2 = B.dzr2, d02 = B.d02, qa2 = B.qa2;
    const double qa2dzr = qa2 * dzr;
    double gx = 0.0, gy = 0.0, gz = 0.0;
    if (i0 <= i1 && j0 <= j1 && k0 <= k1) {
        const float *gbase = P.grid_grad + (size_t)B.slab * ((size_t)D * D * D);
        const unsigned lt = (1u << lane) - 1u, le = 0xffffffffu >> (31 - lane);
        for (int si = i0; si <= i1; si += kTab)
            for (int sj = j0; sj <= j1; sj += kTab)
                for (int sk = k0; sk <= k1; sk += kTab) {
                    const int ni = min(kTab, i1 - si + 1), nj = min(kTab, j1 - sj + 1),
                              nk = min(kTab, k1 - sk + 1);
                    __syncwarp();
                    // per-axis tables: offsets (_kernels.py:232-236) and Gaussian factors
                    for (int l = lane; l < ni + nj + nk; l += 32) {
                        const int ax = l < ni ? 0 : (l < ni + nj ? 1 : 2);
                        const int q = l - (ax == 0 ? 0 : (ax == 1 ? ni : ni + nj));
                        const double d = ax == 0 ? offs(B.lx, 0.0, si + q, res)
                                                 : (ax == 1 ? offs(B.ly, 0.0, sj + q, res)
                                                            : offs(B.lz, 0.0, sk + q, res));
                        const double E = exp_nonpos(B.m2inv_r2 * (d * d));
                        if (ax == 2) {
                            W.zt[q] = make_double2(d, E);
                        } else {
                            (ax == 0 ? W.dx : W.dy)[q] = d;
                            (ax == 0 ? W.ex : W.ey)[q] = E;
                        }
                    }
                    __syncwarp();
                    const float dz0 = (float)W.zt[0].x;
                    const float inv_nj = __frcp_rn((float)nj);
                    const unsigned sbase = (unsigned)((si * D + sj) * D + sk);
                    const int nrows_all = ni * nj;
                    for (int rb = 0; rb < nrows_all; rb += kIRows) {
                        // ---- phase 1: row spans, compacted with a warp scan ----
                        int nrow = 0, total = 0;
                        const int rend = min(nrows_all, rb + kIRows);
                        const int nwords = ((rend - rb) * nk + 31) >> 5;
                        for (int w = lane; w < nwords + kU; w += 32) W.starts[w] = 0u;
                        __syncwarp();
                        // rows r0 + lane and (GM_BWD_P1X2) r0 + 32 + lane per pass:
                        // two independent span / scan chains in flight
                        struct Span {
                            int len, klo, ii, jj;
                            double dx, dy, b2;
                        };
                        auto span_of = [&](int row) {
                            Span q{0, 0, 0, 0, 0.0, 0.0, 0.0};
                            q.ii = idiv(row, inv_nj);
                            q.jj = row - q.ii * nj;
                            if (row < rend) {
                                q.dx = W.dx[q.ii];
                                q.dy = W.dy[q.jj];
                                q.b2 = fma(q.dy, q.dy, q.dx * q.dx);
                                const double rem = dzr2 - q.b2;
                                if (rem > 0.0) {
                                    const float rho = fmaf(approx_sqrt((float)rem), 1.0001f,
                                                           1e-5f * (float)dzr);
                                    q.klo = max(0, __float2int_ru(fmaxf((dz0 - rho) * inv_res, -1.0f)));
                                    const int khi = min(nk - 1, __float2int_rd(fminf(
                                                                    (dz0 + rho) * inv_res, (float)nk)));
                                    q.len = max(0, khi - q.klo + 1);
                                }
                            }
                            return q;
                        };
                        auto place = [&](const Span &q, int rowidx, int st) {
                            IRow &R = W.rows[rowidx];
                            atomicOr(&W.starts[st >> 5], 1u << (st & 31));
                            R.dx = q.dx;
                            R.dy = q.dy;
                            R.b2 = q.b2;
                            R.exy = (W.ex[q.ii] * W.ey[q.jj]) * B.m4inv_r2;
                            R.gp = gbase + (sbase + (unsigned)((q.ii * D + q.jj) * D + q.klo)) - st;
                            R.kz = q.klo - st;
#if GM_BWD_PREFETCH == 1
                            // the row's grid_grad span into L2 now: phase 2's
                            // loads then hit (a hint only, no ordering)
                            const float *rp = R.gp + st;
                            asm volatile("prefetch.global.L2 [%0];" ::"l"(rp));
                            if ((((uintptr_t)rp) & 127u) + 4u * (unsigned)q.len > 128u)
                                asm volatile("prefetch.global.L2 [%0];" ::"l"(rp + q.len - 1));
#elif GM_BWD_PREFETCH == 2
                            // the same as a bulk L2 prefetch of exactly the
                            // span's 16-B granules (no whole-line fetches)
                            {
                                const uintptr_t p0 = (uintptr_t)(R.gp + st) & ~(uintptr_t)15;
                                const uintptr_t p1 = ((uintptr_t)(R.gp + st + q.len) + 15) & ~(uintptr_t)15;
                                asm volatile("cp.async.bulk.prefetch.L2.global [%0], %1;" ::"l"(p0),
                                             "r"((unsigned)(p1 - p0))
                                             : "memory");
                            }
#endif
                        };
                        for (int r0 = rb; r0 < rend; r0 += 32 * GM_BWD_P1X2) {
                            const Span qa = span_of(r0 + lane);
                            Span qb{0, 0, 0, 0, 0.0, 0.0, 0.0};
                            if (GM_BWD_P1X2 > 1) qb = span_of(r0 + 32 + lane);
                            int sa = qa.len, sb = qb.len;  // inclusive scans of the span lengths
#pragma unroll
                            for (int o = 1; o < 32; o <<= 1) {
                                const int ta = __shfl_up_sync(0xffffffffu, sa, o);
                                const int tb = GM_BWD_P1X2 > 1 ? __shfl_up_sync(0xffffffffu, sb, o) : 0;
                                if (lane >= o) {
                                    sa += ta;
                                    sb += tb;
                                }
                            }
                            const unsigned ma = __ballot_sync(0xffffffffu, qa.len > 0);
                            const int tota = __shfl_sync(0xffffffffu, sa, 31);
                            if (qa.len > 0) place(qa, nrow + __popc(ma & lt), total + sa - qa.len);
                            nrow += __popc(ma);
                            total += tota;
                            if (GM_BWD_P1X2 > 1) {
                                const unsigned mb = __ballot_sync(0xffffffffu, qb.len > 0);
                                const int totb = __shfl_sync(0xffffffffu, sb, 31);
                                if (qb.len > 0) place(qb, nrow + __popc(mb & lt), total + sb - qb.len);
                                nrow += __popc(mb);
                                total += totb;
                            }
                        }
                        __syncwarp();
                        // ---- phase 2: kU windows of 32 voxels per step ----
                        // grid_grad may come from the previous kernel (PDL launch):
                        // the prologue above overlapped it, the loads must not
                        pdl_wait();
                        int cur = -1;  // rows started before the next window, minus one
                        const int last = total - 1;
                        // U windows from base; the loop's tail runs one window
                        // at a time (no clamped dead windows).  Lane l still
                        // visits voxels l, l+32, ... in order: same sums.
                        // FULL: every voxel of the U windows exists (no clamp, no mask)
                        auto step = [&](auto Uc, auto Fc, int base) {
                            constexpr int U = decltype(Uc)::value;
                            constexpr bool FULL = decltype(Fc)::value;
                            int myrow[U];
#pragma unroll
                            for (int u = 0; u < U; u++) {
                                const unsigned M = W.starts[(base >> 5) + u];
                                myrow[u] = cur + __popc(M & le);
                                cur += __popc(M);
                            }
                            float g[U];
#pragma unroll
                            for (int u = 0; u < U; u++) {
                                const int v = FULL ? base + 32 * u + lane : min(base + 32 * u + lane, last);
                                g[u] = ld_gg<GM_BWD_GGHINT>(W.rows[myrow[u]].gp + v);
                            }
#pragma unroll
                            for (int u = 0; u < U; u++) {
                                const int vr = base + 32 * u + lane;
                                const int v = FULL ? vr : min(vr, last);
                                const IRow &R = W.rows[myrow[u]];
                                const double2 zt = W.zt[R.kz + v];
                                const double dz = zt.x;
                                const double d2 = fma(dz, dz, R.b2);
                                const double rd = rsqrt_d(d2);
                                // slope/d (_kernels.py:244-251): Gaussian core
                                // Ex Ey Ez (-4/r^2), tail 2 qa (d - dzr) / d; d2 = 0
                                // takes the core branch and contributes 0 (dx=dy=dz=0)
                                const double t = d2 <= d02 ? R.exy * zt.y : fma(-qa2dzr, rd, qa2);
                                const double scl =
                                    (double)(((FULL || vr <= last) && d2 < dzr2) ? g[u] : 0.0f) * t;
                                gx = fma(scl, R.dx, gx);
                                gy = fma(scl, R.dy, gy);
                                gz = fma(scl, dz, gz);
                            }
                        };
                        int base = 0;
                        for (; base + 32 * kU <= total; base += 32 * kU)
                            step(std::integral_constant<int, kU>{}, std::true_type{}, base);
                        for (; base < total; base += 32)
                            step(std::integral_constant<int, 1>{}, std::false_type{}, base);
                        __syncwarp();
                    }
                }
    }
    store_coord(P, a, lane, gx, gy, gz);
}

// Vector types with per-atom radii: one geometry walk, every channel of the
// set per voxel (type gradients, _kernels.py:296-313) and the coordinate
// term from sum_c w_c g_c.  NT > 0: compile-time channel count (no
// predicates, 32-bit channel offsets); NT = 0: up to kMaxT, predicated.
template <int NT, int DC>
__device__ __forceinline__ void vector_shared_walk(const BwdArgs &P, WarpBwd &W, Atom &A, int a,
                                                   int row, int Tn, const float *gset, int D,
                                                   double res, float inv_res, int lane,
                                                   double &gx, double &gy, double &gz) {
    constexpr int NC = NT > 0 ? NT : kMaxT;
    const gm_batch &b = P.b;
    const double grm = P.p.gaussian_radius_multiple, rmult = P.p.radius_multiple;
    const double r = A.r;
    const double gr = grm * r, d02 = gr * gr;
    const double q0 = (2.0 * grm) / r;
    const double qa = P.eg * (q0 * q0);
    const double m4inv_r2 = -4.0 / (r * r);
    const unsigned D3 = (unsigned)D * D * D;
    const size_t D3l = D3;
    double tg[NC];
#pragma unroll
    for (int c = 0; c < NC; c++) tg[c] = 0.0;
    // the weights live in shared memory (broadcast reads): registers go to
    // the per-channel type-gradient accumulators
    double *w = W.wt;
    if (lane < kMaxT) w[lane] = lane < Tn ? (double)b.weights[row + lane] : 0.0;
    __syncwarp();
    if (set_radius(A, r, rmult, res, D)) {
        const double dzr = A.dzr, dzr2 = A.dzr2;
        flat_walk<false, 1>(A, W, gset, D, res, inv_res, lane, 1.0,
                            [&](int, double d2, const RowEntry &R, double dz, double ez,
                                size_t voff, float) {
                                if (d2 >= dzr2) return;
                                double dens, sod;  // density, slope / d
                                if (d2 <= d02) {
                                    dens = R.exy * ez;
                                    sod = dens * m4inv_r2;
                                } else {
                                    const double rd = rsqrt_d(d2);
                                    const double t = fma(d2, rd, -dzr);
                                    dens = (qa * t) * t;
                                    sod = (2.0 * qa) * t * rd;
                                }
                                float gc[NC];
#if GM_BWDV_PTR
                                if (DC > 0) {
                                    // compile-time channel stride: one address,
                                    // the channel offsets are load immediates
                                    const float *gp = gset + voff;
#pragma unroll
                                    for (int c = 0; c < NC; c++)
                                        gc[c] = ld_gg<GM_BWDV_GGHINT>(gp + (size_t)c * DC * DC * DC);
                                } else {
                                    // one 64-bit pointer stepped by the channel stride
                                    const float *gp = gset + voff;
#pragma unroll
                                    for (int c = 0; c < NC; c++, gp += D3l)
                                        gc[c] = (NT > 0 || c < Tn) ? ld_gg<GM_BWDV_GGHINT>(gp) : 0.0f;
                                }
#else
                                unsigned off = (unsigned)voff;
#pragma unroll
                                for (int c = 0; c < NC; c++, off += D3)
                                    gc[c] = (NT > 0 || c < Tn) ? ld_gg<GM_BWDV_GGHINT>(gset + off) : 0.0f;
#endif
                                double sw = 0.0;
#pragma unroll
                                for (int c = 0; c < NC; c++) {
                                    if (NT > 0 || c < Tn) {
                                        const double g = (double)gc[c];
                                        tg[c] = fma(g, dens, tg[c]);
                                        sw = fma(w[c], g, sw);
                                    }
                                }
                                if (d2 > 0.0) {
                                    const double sc = sw * sod;
                                    gx = fma(sc, R.dx, gx);
                                    gy = fma(sc, R.dy, gy);
                                    gz = fma(sc, dz, gz);
                                }
                            });
    }
#if GM_BWD_SPLITSUM
    static_assert(NC <= 16, "type gradients: at most 16 channels per split sum");
    double v[16];
#pragma unroll
    for (int c = 0; c < 16; c++) v[c] = (c < NC && (NT > 0 || c < Tn)) ? tg[c] : 0.0;
    int idx;
    const double sum = warp_sum_split<16>(v, lane, idx);  // lanes 2 idx, 2 idx + 1
    if ((lane & 1) == 0 && idx < Tn) {
        if (P.type_grad64) P.type_grad64[row + idx] = sum;
        else if (P.type_grad) P.type_grad[row + idx] = (float)sum;
    }
#else
#pragma unroll
    for (int c = 0; c < NC; c++) {
        if (NT > 0 || c < Tn) {
            const double v = warp_sum(tg[c]);
            if (lane == 0 && P.type_grad64) P.type_grad64[row + c] = v;
            else if (lane == 0 && P.type_grad) P.type_grad[row + c] = (float)v;
        }
    }
#endif
}

// Vector types (_kernels.py:258-314).  With per-atom radii and <= kMaxT
// channels the geometry is shared by all channels of the set: one walk, all
// channel gradients per voxel, the coordinate term from sum_c w_c g_c.  With
// type-indexed radii (or more channels) each channel walks its own box.
__global__ void __launch_bounds__(kBwdWarps * 32, GM_BWDV_MINB) k_backward_vector(const BwdArgs P) {
    __shared__ WarpBwd wsm[kBwdWarps];
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    const int slot = blockIdx.x * kBwdWarps + warp;
    const gm_batch &b = P.b;
    if (slot >= b.natoms) return;
    // the prepare pass's record at this launch slot (heaviest atoms first when
    // the batch carries a launch order): one load level
    const VBwdAtom V = P.vbatoms[slot];
    const int a = V.atom, s = V.set;
    const int D = P.p.npts;
    const double res = P.p.resolution, grm = P.p.gaussian_radius_multiple,
                 rmult = P.p.radius_multiple;
    const float inv_res = (float)(1.0 / res);
    Atom A;
    A.x = V.x;
    A.y = V.y;
    A.z = V.z;
    A.ox = V.ox;
    A.oy = V.oy;
    A.oz = V.oz;
    A.r = V.r;
    const int Tn = V.T;
    const int row = V.row;
    const size_t D3 = (size_t)D * D * D;
    const float *gset = P.grid_grad + (size_t)V.slab * D3;
    double gx = 0.0, gy = 0.0, gz = 0.0;

    if (!P.p.radius_type_indexed && Tn <= kMaxT) {
        // channel loops fully unrolled without predicates for the common
        // 14-type table, predicated up to kMaxT otherwise
        if (Tn == 14 && D == 48 && GM_BWDV_D48)  // the default 0.5 A / 23.5 A grid
            vector_shared_walk<14, 48>(P, wsm[warp], A, a, row, Tn, gset, D, res, inv_res, lane, gx, gy, gz);
        else if (Tn == 14)
            vector_shared_walk<14, 0>(P, wsm[warp], A, a, row, Tn, gset, D, res, inv_res, lane, gx, gy, gz);
        else
            vector_shared_walk<0, 0>(P, wsm[warp], A, a, row, Tn, gset, D, res, inv_res, lane, gx, gy, gz);
    } else {
        for (int c = 0; c < Tn; c++) {
            const double r = P.p.radius_type_indexed ? b.type_radius[b.set_trstart[s] + c]
                                                     : A.r;
            const double w = (double)b.weights[row + c];
            const double gr = grm * r, d02 = gr * gr;
            const double q0 = (2.0 * grm) / r;
            const double qa = P.eg * (q0 * q0);
            const double m4inv_r2 = -4.0 / (r * r);
            double tg = 0.0;
            if (set_radius(A, r, rmult, res, D)) {
                const double dzr = A.dzr, dzr2 = A.dzr2;
                flat_walk<true>(A, wsm[warp], gset + (size_t)c * D3, D, res, inv_res, lane, 1.0,
                                [&](int, double d2, const RowEntry &R, double dz, double ez,
                                    size_t, float gf) {
                                    if (d2 >= dzr2 || gf == 0.0f) return;
                                    const double g = widen(gf);
                                    double dens, sod;
                                    if (d2 <= d02) {
                                        dens = R.exy * ez;
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
                                        gx = fma(sc, R.dx, gx);
                                        gy = fma(sc, R.dy, gy);
                                        gz = fma(sc, dz, gz);
                                    }
                                });
            }
            tg = warp_sum(tg);
            if (lane == 0 && P.type_grad64) P.type_grad64[row + c] = tg;
            else if (lane == 0 && P.type_grad) P.type_grad[row + c] = (float)tg;
        }
    }
    store_coord(P, a, lane, gx, gy, gz);
}

}  // namespace

gm_status backward_impl(const gm_params *p, const gm_batch *b, const Workspace &ws,
                        const float *grid_grad, float *coord_grad, float *type_grad,
                        cudaStream_t s, bool early_prologue, double *coord_grad64,
                        double *type_grad64) {
    BwdArgs P;
    P.coord_grad64 = coord_grad64;
    P.type_grad64 = type_grad64;
    P.early = early_prologue ? 1 : 0;
    P.p = *p;
    P.b = *b;
    P.pos = ws.pos;
    P.grid_grad = grid_grad;
    P.coord_grad = coord_grad;
    P.type_grad = type_grad;
    P.batoms = ws.batoms;
    P.atom_order = ws.atom_order;
    P.vbatoms = ws.vbatoms;
    P.eg = exp((-2.0 * p->gaussian_radius_multiple) * p->gaussian_radius_multiple);
    if (b->vector_mode)
        k_backward_vector<<<(b->natoms + kBwdWarps - 1) / kBwdWarps, kBwdWarps * 32, 0, s>>>(P);
    else
        CUDA_TRY(gm_launch_pdl(k_backward_index, dim3((b->natoms + kBwdWarps - 1) / kBwdWarps),
                               dim3(kBwdWarps * 32), 0, s, P));
    LAUNCH_CHECK();
    return GM_OK;
}
