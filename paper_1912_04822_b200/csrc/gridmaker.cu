// gridmaker.cu -- B200 (sm_100a) kernels of the GridMaker hot path + C ABI.
//
// Reference path: /root/reference/pkg/src/voxmol/_kernels.py (numba CPU) driven
// by voxelizer.py:203-301,335-435 and geom.py:99-112.  See DESIGN.md for the
// data layout and the roofline of each kernel.
//
// Kernels
//   k_prepare_atoms   fused Transform (geom.py:105) in numpy's FMA order -> f64 positions
//   k_prepare_items   per forward item: integer voxel box (_kernels.py:22-30),
//                     grid-local hi/lo f32 coordinates, density constants
//   k_forward<...>    one CTA per (example, tile of TI x TJ full k-rows, channel chunk):
//                     ordered culling of the example's items into smem, warp-patch
//                     gather with ballot culling, smem accumulation in item order,
//                     coalesced float4 streaming stores of every voxel (zeros included)
//   k_backward_index  one warp per atom, f64 geometry, warp-shuffle reduction
//   k_backward_vector one warp per atom, all channels (type + coordinate gradients)
//
// Determinism: every output voxel is owned by one lane that adds contributions
// in ascending item order; no atomics anywhere, so results are bitwise
// reproducible and independent of batching (reference property, _kernels.py:3-9).

#include <cuda_runtime.h>
#include <stdarg.h>
#include <math_constants.h>
#include <stdint.h>
#include <stdio.h>
#include <string.h>

#include <algorithm>
#include <atomic>
#include <mutex>
#include <string>
#include <vector>

#include "../../include/gridmaker_b200.h"

#define GM_VERSION "gridmaker_b200 0.1.0 (sm_100a)"

// ----------------------------------------------------------------------------
// error plumbing
// ----------------------------------------------------------------------------
static thread_local std::string g_err;
static std::atomic<int64_t> g_launches{0};

static gm_status fail(gm_status code, const char *fmt, ...) {
    char buf[512];
    va_list ap;
    va_start(ap, fmt);
    vsnprintf(buf, sizeof buf, fmt, ap);
    va_end(ap);
    g_err = buf;
    return code;
}

#define CUDA_TRY(expr)                                                                  \
    do {                                                                                \
        cudaError_t _e = (expr);                                                        \
        if (_e != cudaSuccess)                                                          \
            return fail(GM_ERR_CUDA, "%s failed: %s (%s:%d)", #expr, cudaGetErrorString(_e), \
                        __FILE__, __LINE__);                                            \
    } while (0)

#define LAUNCH_CHECK()                                                                  \
    do {                                                                                \
        g_launches.fetch_add(1, std::memory_order_relaxed);                             \
        cudaError_t _e = cudaGetLastError();                                            \
        if (_e != cudaSuccess)                                                          \
            return fail(GM_ERR_CUDA, "kernel launch failed: %s (%s:%d)",                \
                        cudaGetErrorString(_e), __FILE__, __LINE__);                    \
    } while (0)

// ----------------------------------------------------------------------------
// device records
// ----------------------------------------------------------------------------
// One forward item (index mode: an atom; vector mode: an (atom, channel) pair
// with nonzero weight).  64 bytes = 4 x LDS.128 when broadcast from smem.
struct __align__(16) FwdItem {
    float xh, yh, zh, cexp;  // grid-local coordinate (hi part); -2 log2(e) / r^2
    float xl, yl, zl, d02;   // lo parts; (grm r)^2
    float dzr, qa, w;        // cutoff rmult*r; quadratic coefficient; weight
    int ch;                  // absolute output channel
    int ibox, jbox, kbox;    // lo | hi << 16 (valid boxes only)
    int atom;
};
static_assert(sizeof(FwdItem) == 64, "FwdItem must be 64 bytes");

// Exact binary-mode record: transformed f64 position and r^2.
struct __align__(16) BinItem {
    double x, y, z, r2;
};

static constexpr int kWarps = 8;
static constexpr int kThreads = kWarps * 32;
static constexpr int kCap = 2 * kThreads;  // smem item-list capacity per round

struct Workspace {
    double *pos;      // natoms*3
    FwdItem *items;   // nitems
    BinItem *bitems;  // nitems
    int4 *cull;       // nitems: {ch or -1, ibox, jbox, kbox}
};

static size_t align_up(size_t x, size_t a) { return (x + a - 1) / a * a; }

static void carve(void *base, int32_t natoms, int32_t nitems, Workspace *w) {
    char *p = (char *)base;
    size_t off = 0;
    w->pos = (double *)(p + off);
    off = align_up(off + sizeof(double) * 3 * (size_t)std::max(natoms, 1), 256);
    w->items = (FwdItem *)(p + off);
    off = align_up(off + sizeof(FwdItem) * (size_t)std::max(nitems, 1), 256);
    w->bitems = (BinItem *)(p + off);
    off = align_up(off + sizeof(BinItem) * (size_t)std::max(nitems, 1), 256);
    w->cull = (int4 *)(p + off);
}

extern "C" size_t gm_workspace_bytes(int32_t natoms, int32_t nitems) {
    size_t off = 0;
    off = align_up(off + sizeof(double) * 3 * (size_t)std::max(natoms, 1), 256);
    off = align_up(off + sizeof(FwdItem) * (size_t)std::max(nitems, 1), 256);
    off = align_up(off + sizeof(BinItem) * (size_t)std::max(nitems, 1), 256);
    off = align_up(off + sizeof(int4) * (size_t)std::max(nitems, 1), 256);
    return off + 256;
}

extern "C" const double *gm_workspace_positions(const void *workspace) {
    return (const double *)workspace;
}

// ----------------------------------------------------------------------------
// shared device helpers
// ----------------------------------------------------------------------------
// _kernels.py:22-30 in f64 with the reference's operation order:
//   lo = ceil(((x - cut) - origin) / res), hi = floor(((x + cut) - origin) / res),
// clamped to [0, D-1].  Clamping keeps lo > hi for empty boxes.
__device__ __forceinline__ void axis_bounds(double x, double cut, double origin, double res,
                                            int D, int &lo, int &hi) {
    double l = ceil(__ddiv_rn(__dsub_rn(__dsub_rn(x, cut), origin), res));
    double h = floor(__ddiv_rn(__dsub_rn(__dadd_rn(x, cut), origin), res));
    l = fmin(fmax(l, 0.0), (double)D);
    h = fmax(fmin(h, (double)(D - 1)), -1.0);
    lo = (int)l;
    hi = (int)h;
}

// One output coordinate of (x - c) @ R.T with the 3-term dot product evaluated
// in the FMA order numpy/BLAS uses on the host (codes: geom.py matmul_order).
__device__ __forceinline__ double dot3(const double a[3], const double *b, int order) {
    switch (order) {
        case 1: return __fma_rn(a[2], b[2], __fma_rn(a[0], b[0], __dmul_rn(a[1], b[1])));
        case 2: return __fma_rn(a[1], b[1], __fma_rn(a[2], b[2], __dmul_rn(a[0], b[0])));
        case 3: return __fma_rn(a[1], b[1], __fma_rn(a[0], b[0], __dmul_rn(a[2], b[2])));
        case 4: return __fma_rn(a[0], b[0], __fma_rn(a[2], b[2], __dmul_rn(a[1], b[1])));
        case 5: return __fma_rn(a[0], b[0], __fma_rn(a[1], b[1], __dmul_rn(a[2], b[2])));
        case 6: return __dadd_rn(__dadd_rn(__dmul_rn(a[0], b[0]), __dmul_rn(a[1], b[1])),
                                 __dmul_rn(a[2], b[2]));
        case 7: return __dadd_rn(__dadd_rn(__dmul_rn(a[0], b[0]), __dmul_rn(a[2], b[2])),
                                 __dmul_rn(a[1], b[1]));
        case 8: return __dadd_rn(__dadd_rn(__dmul_rn(a[1], b[1]), __dmul_rn(a[2], b[2])),
                                 __dmul_rn(a[0], b[0]));
        default: return __fma_rn(a[2], b[2], __fma_rn(a[1], b[1], __dmul_rn(a[0], b[0])));
    }
}

__device__ __forceinline__ double warp_sum(double v) {
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
    return v;
}

// ----------------------------------------------------------------------------
// prepare: transform + localise
// ----------------------------------------------------------------------------
struct PrepArgs {
    gm_params p;
    gm_batch b;
    Workspace ws;
};

// geom.py:99-112: x' = ((x - c) @ R.T + c) + t in float64.  Without a transform
// the f32 input is widened exactly (voxelizer.py:366).
__global__ void __launch_bounds__(256) k_prepare_atoms(const PrepArgs A) {
    const gm_batch &b = A.b;
    for (int a = blockIdx.x * blockDim.x + threadIdx.x; a < b.natoms;
         a += gridDim.x * blockDim.x) {
        double x[3];
        if (b.coords64) {
            x[0] = b.coords64[3 * a + 0];
            x[1] = b.coords64[3 * a + 1];
            x[2] = b.coords64[3 * a + 2];
        } else {
            x[0] = (double)b.coords32[3 * a + 0];
            x[1] = (double)b.coords32[3 * a + 1];
            x[2] = (double)b.coords32[3 * a + 2];
        }
        if (b.xforms) {
            const int s = b.atom_set[a];
            const int e = b.set_example[s];
            const double *X = b.xforms + 15 * (size_t)e;
            const int nset = b.set_end[s] - b.set_start[s];
            const int order = nset == 1 ? A.p.matmul_order_1 : A.p.matmul_order_n;
            double d[3] = {__dsub_rn(x[0], X[9]), __dsub_rn(x[1], X[10]), __dsub_rn(x[2], X[11])};
#pragma unroll
            for (int j = 0; j < 3; j++) {
                double r = dot3(d, X + 3 * j, order);
                x[j] = __dadd_rn(__dadd_rn(r, X[9 + j]), X[12 + j]);
            }
        }
        A.ws.pos[3 * a + 0] = x[0];
        A.ws.pos[3 * a + 1] = x[1];
        A.ws.pos[3 * a + 2] = x[2];
    }
}

__device__ __forceinline__ void split_hilo(double v, float &hi, float &lo) {
    hi = (float)v;
    lo = (float)(v - (double)hi);
}

__global__ void __launch_bounds__(256) k_prepare_items(const PrepArgs A) {
    const gm_batch &b = A.b;
    const gm_params &p = A.p;
    const int D = p.npts;
    const double res = p.resolution, grm = p.gaussian_radius_multiple, rmult = p.radius_multiple;
    for (int it = blockIdx.x * blockDim.x + threadIdx.x; it < b.nitems;
         it += gridDim.x * blockDim.x) {
        const int a = b.item_atom ? b.item_atom[it] : it;
        const int s = b.atom_set[a];
        const int e = b.set_example[s];
        const int ch = b.set_choff[s] + (b.item_channel ? b.item_channel[it] : b.atom_type[a]);
        const double r = b.item_radius ? b.item_radius[it] : b.atom_radius[a];
        const float w = b.item_weight ? b.item_weight[it] : 1.0f;
        const double x = A.ws.pos[3 * a + 0], y = A.ws.pos[3 * a + 1], z = A.ws.pos[3 * a + 2];
        const double ox = b.origins[3 * e + 0], oy = b.origins[3 * e + 1],
                     oz = b.origins[3 * e + 2];
        // _kernels.py:55/74 (index) and 144/167 (vector): cut = r (binary) or r*rmult
        const double cut = p.binary ? r : __dmul_rn(r, rmult);
        int i0, i1, j0, j1, k0, k1;
        axis_bounds(x, cut, ox, res, D, i0, i1);
        axis_bounds(y, cut, oy, res, D, j0, j1);
        axis_bounds(z, cut, oz, res, D, k0, k1);
        const bool valid = i0 <= i1 && j0 <= j1 && k0 <= k1;
        FwdItem f;
        split_hilo(x - ox, f.xh, f.xl);
        split_hilo(y - oy, f.yh, f.yl);
        split_hilo(z - oz, f.zh, f.zl);
        const double r2 = r * r;
        f.cexp = (float)((-2.0 * CUDART_L2E) / r2);
        const double gr = grm * r;
        f.d02 = (float)(gr * gr);
        f.dzr = (float)(rmult * r);
        const double q0 = (2.0 * grm) / r;
        f.qa = (float)(exp((-2.0 * grm) * grm) * (q0 * q0));
        f.w = w;
        f.ch = ch;
        f.ibox = i0 | (i1 << 16);
        f.jbox = j0 | (j1 << 16);
        f.kbox = k0 | (k1 << 16);
        f.atom = a;
        A.ws.items[it] = f;
        if (p.binary) A.ws.bitems[it] = BinItem{x, y, z, __dmul_rn(r, r)};
        A.ws.cull[it] = make_int4(valid ? ch : -1, f.ibox, f.jbox, f.kbox);
    }
}

// ----------------------------------------------------------------------------
// forward
// ----------------------------------------------------------------------------
struct FwdArgs {
    const FwdItem *items;
    const BinItem *bitems;
    const int4 *cull;
    const int32_t *ex_item_start, *ex_item_end;
    const double *origins;
    float *out;
    double res;
    int D, C;
    int TI, TJ, CC, SJ;   // tile rows, channel chunk, padded row stride
    int ntj, nchunks;
};

__device__ __forceinline__ int box_lo(int b) { return b & 0xffff; }
__device__ __forceinline__ int box_hi(int b) { return b >> 16; }

template <int PI, int PJ, int PK, bool BINARY, bool VECTOR>
__global__ void __launch_bounds__(kThreads, 2) k_forward(const FwdArgs A) {
    extern __shared__ __align__(16) unsigned char smem[];
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    const int e = blockIdx.y;
    const int chunk = blockIdx.x % A.nchunks;
    const int tij = blockIdx.x / A.nchunks;
    const int i0 = (tij / A.ntj) * A.TI, j0 = (tij % A.ntj) * A.TJ;
    const int D = A.D, TI = A.TI, TJ = A.TJ, SJ = A.SJ;
    const int c0 = chunk * A.CC, c1 = min(A.C, c0 + A.CC), ncc = c1 - c0;
    const int SC = TI * TJ * SJ;  // channel stride in acc
    const int acc_elems = A.CC * SC;

    float *acc = reinterpret_cast<float *>(smem);
    FwdItem *list = reinterpret_cast<FwdItem *>(smem + (size_t)acc_elems * 4);
    BinItem *blist = reinterpret_cast<BinItem *>(list + kCap);
    int *wcount = reinterpret_cast<int *>(BINARY ? (unsigned char *)(blist + kCap)
                                                 : (unsigned char *)blist);

    const float4 z4 = make_float4(0.f, 0.f, 0.f, 0.f);
    for (int q = tid; q < acc_elems / 4; q += kThreads) reinterpret_cast<float4 *>(acc)[q] = z4;

    const int ti_hi = min(i0 + TI, D) - 1, tj_hi = min(j0 + TJ, D) - 1;
    const int is = A.ex_item_start[e], ie = A.ex_item_end[e];
    const double ox = A.origins[3 * e + 0], oy = A.origins[3 * e + 1], oz = A.origins[3 * e + 2];

    // per-lane voxel within a warp patch
    const int lk = lane % PK, lj = (lane / PK) % PJ, li = lane / (PK * PJ);
    const int npi = TI / PI, npj = TJ / PJ, npk = (D + PK - 1) / PK;
    const int npatch = npi * npj * npk;

    int count = 0;
    __syncthreads();
    for (int base = is; base < ie; base += kThreads) {
        const int it = base + tid;
        bool keep = false;
        if (it < ie) {
            const int4 cr = A.cull[it];
            keep = cr.x >= c0 && cr.x < c1 && box_lo(cr.y) <= ti_hi && box_hi(cr.y) >= i0 &&
                   box_lo(cr.z) <= tj_hi && box_hi(cr.z) >= j0;
        }
        const unsigned m = __ballot_sync(0xffffffffu, keep);
        if (lane == 0) wcount[warp] = __popc(m);
        __syncthreads();
        int before = 0, total = 0;
#pragma unroll
        for (int w = 0; w < kWarps; w++) {
            const int c = wcount[w];
            before += (w < warp) ? c : 0;
            total += c;
        }
        if (keep) {
            const int pos = count + before + __popc(m & ((1u << lane) - 1u));
            list[pos] = A.items[it];
            if (BINARY) blist[pos] = A.bitems[it];
        }
        count += total;
        __syncthreads();
        if (count > kCap - kThreads || base + kThreads >= ie) {
            // ---- process the ordered candidate list ----
            for (int pch = warp; pch < npatch; pch += kWarps) {
                const int pk = pch % npk, pj = (pch / npk) % npj, pi = pch / (npk * npj);
                const int pil = i0 + pi * PI, pjl = j0 + pj * PJ, pkl = pk * PK;
                if (pil >= D || pjl >= D) continue;  // warp-uniform
                const int pih = min(pil + PI - 1, D - 1), pjh = min(pjl + PJ - 1, D - 1),
                          pkh = min(pkl + PK - 1, D - 1);
                const int i = pil + li, j = pjl + lj, k = pkl + lk;
                const bool lvalid = i < D && j < D && k < D;
                const int off = ((i - i0) * TJ + (j - j0)) * SJ + k;
                float vxh, vxl, vyh, vyl, vzh, vzl;
                double vx64 = 0, vy64 = 0, vz64 = 0;
                if (BINARY) {
                    vx64 = __dadd_rn(ox, __dmul_rn((double)i, A.res));
                    vy64 = __dadd_rn(oy, __dmul_rn((double)j, A.res));
                    vz64 = __dadd_rn(oz, __dmul_rn((double)k, A.res));
                } else {
                    split_hilo((double)i * A.res, vxh, vxl);
                    split_hilo((double)j * A.res, vyh, vyl);
                    split_hilo((double)k * A.res, vzh, vzl);
                }
                for (int b0 = 0; b0 < count; b0 += 32) {
                    const int idx = b0 + lane;
                    bool hit = false;
                    if (idx < count) {
                        const FwdItem &c = list[idx];
                        hit = box_lo(c.ibox) <= pih && box_hi(c.ibox) >= pil &&
                              box_lo(c.jbox) <= pjh && box_hi(c.jbox) >= pjl &&
                              box_lo(c.kbox) <= pkh && box_hi(c.kbox) >= pkl;
                    }
                    unsigned hm = __ballot_sync(0xffffffffu, hit);
                    while (hm) {
                        const int t = __ffs(hm) - 1;
                        hm &= hm - 1;
                        const FwdItem &c = list[b0 + t];
                        const bool inb = lvalid && i >= box_lo(c.ibox) && i <= box_hi(c.ibox) &&
                                         j >= box_lo(c.jbox) && j <= box_hi(c.jbox) &&
                                         k >= box_lo(c.kbox) && k <= box_hi(c.kbox);
                        if (!inb) continue;
                        float *dst = acc + (c.ch - c0) * SC + off;
                        if (BINARY) {
                            // _kernels.py:87-98 / 180-192: exact f64, no contraction
                            const BinItem &bi = blist[b0 + t];
                            const double dx = __dsub_rn(vx64, bi.x);
                            const double dy = __dsub_rn(vy64, bi.y);
                            const double dz = __dsub_rn(vz64, bi.z);
                            const double d2 = __dadd_rn(__dadd_rn(__dmul_rn(dx, dx), __dmul_rn(dy, dy)),
                                                        __dmul_rn(dz, dz));
                            if (d2 <= bi.r2) {
                                if (VECTOR) *dst = fmaxf(*dst, c.w);
                                else *dst = 1.0f;
                            }
                        } else {
                            // _kernels.py:99-106: Gaussian core, quadratic tail
                            const float dx = (vxh - c.xh) + (vxl - c.xl);
                            const float dy = (vyh - c.yh) + (vyl - c.yl);
                            const float dz = (vzh - c.zh) + (vzl - c.zl);
                            const float d2 = fmaf(dz, dz, fmaf(dy, dy, dx * dx));
                            const float g = exp2f(d2 * c.cexp);
                            const float d = sqrtf(d2);
                            const float t2 = d - c.dzr;
                            const float q = c.qa * t2 * t2;
                            const float v = d2 <= c.d02 ? g : (d < c.dzr ? q : 0.0f);
                            *dst = fmaf(c.w, v, *dst);
                        }
                    }
                }
            }
            __syncthreads();
            count = 0;
        }
    }
    __syncthreads();

    // ---- coalesced streaming stores of the whole tile (zeros included) ----
    const int TIv = min(TI, D - i0), TJv = min(TJ, D - j0);
    const int nrows = ncc * TIv * TJv;
    const size_t D3 = (size_t)D * D * D;
    float *obase = A.out + ((size_t)e * A.C + c0) * D3 + ((size_t)i0 * D + j0) * D;
    if ((D & 3) == 0) {
        const int nq = D >> 2;
        for (int q = tid; q < nrows * nq; q += kThreads) {
            const int row = q / nq, qq = q - row * nq;
            const int jj = row % TJv, ii = (row / TJv) % TIv, cc = row / (TJv * TIv);
            const float4 v = *reinterpret_cast<const float4 *>(acc + cc * SC + (ii * TJ + jj) * SJ + 4 * qq);
            __stcs(reinterpret_cast<float4 *>(obase + cc * D3 + ((size_t)ii * D + jj) * D) + qq, v);
        }
    } else {
        for (int q = tid; q < nrows * D; q += kThreads) {
            const int row = q / D, k = q - row * D;
            const int jj = row % TJv, ii = (row / TJv) % TIv, cc = row / (TJv * TIv);
            __stcs(obase + cc * D3 + ((size_t)ii * D + jj) * D + k, acc[cc * SC + (ii * TJ + jj) * SJ + k]);
        }
    }
}

// ----------------------------------------------------------------------------
// backward
// ----------------------------------------------------------------------------
struct BwdArgs {
    gm_params p;
    gm_batch b;
    const double *pos;
    const float *grid_grad;
    float *coord_grad;
    float *type_grad;
};

// Box of one atom split into row segments of <= 32 voxels along k; lane l of
// the warp serves segment (l / L) of each step, voxel (l % L) in it.
struct BoxWalk {
    int i0, j0, k0, nj, nk, L, nseg, spi, total;
};

__device__ __forceinline__ bool make_walk(double x, double y, double z, double cut, double ox,
                                          double oy, double oz, double res, int D, BoxWalk &w) {
    int i1, j1, k1;
    axis_bounds(x, cut, ox, res, D, w.i0, i1);
    axis_bounds(y, cut, oy, res, D, w.j0, j1);
    axis_bounds(z, cut, oz, res, D, w.k0, k1);
    if (w.i0 > i1 || w.j0 > j1 || w.k0 > k1) return false;
    const int ni = i1 - w.i0 + 1;
    w.nj = j1 - w.j0 + 1;
    w.nk = k1 - w.k0 + 1;
    w.L = min(w.nk, 32);
    w.nseg = (w.nk + w.L - 1) / w.L;
    w.spi = 32 / w.L;
    w.total = ni * w.nj * w.nseg;
    return true;
}

// _kernels.py:209-255: coordinate gradient of every index-typed atom of the batch.
__global__ void __launch_bounds__(256) k_backward_index(const BwdArgs A) {
    const int lane = threadIdx.x & 31;
    const int a = blockIdx.x * 8 + (threadIdx.x >> 5);
    const gm_batch &b = A.b;
    if (a >= b.natoms) return;
    const int D = A.p.npts;
    const double res = A.p.resolution, grm = A.p.gaussian_radius_multiple,
                 rmult = A.p.radius_multiple;
    const int s = b.atom_set[a];
    const int e = b.set_example[s];
    const int c = b.set_choff[s] + b.atom_type[a];
    const double x = A.pos[3 * a], y = A.pos[3 * a + 1], z = A.pos[3 * a + 2];
    const double ox = b.origins[3 * e], oy = b.origins[3 * e + 1], oz = b.origins[3 * e + 2];
    const double r = b.atom_radius[a];
    const double inv_r2 = 1.0 / (r * r);
    const double d0 = grm * r, d02 = d0 * d0;
    const double dzr = rmult * r, dzr2 = dzr * dzr;
    const double q0 = (2.0 * grm) / r;
    const double qa2 = 2.0 * (exp((-2.0 * grm) * grm) * (q0 * q0));
    const double m4inv_r2 = -4.0 * inv_r2;
    const float cexp = (float)(-2.0 * inv_r2);
    double gx = 0.0, gy = 0.0, gz = 0.0;
    BoxWalk w;
    if (make_walk(x, y, z, dzr, ox, oy, oz, res, D, w)) {
        const float *g_base = A.grid_grad + ((size_t)e * b.nchannels + c) * ((size_t)D * D * D);
        const int seg_off = lane / w.L, kin = lane - seg_off * w.L;
        if (seg_off < w.spi) {
            for (int sg = seg_off; sg < w.total; sg += w.spi) {
                const int row = sg / w.nseg, sk = sg - row * w.nseg;
                const int k = w.k0 + sk * w.L + kin;
                if (k - w.k0 >= w.nk) continue;
                const int ii = row / w.nj, jj = row - ii * w.nj;
                const int i = w.i0 + ii, j = w.j0 + jj;
                // _kernels.py:232-237 (same association, no contraction)
                const double dx = __dsub_rn(x, __dadd_rn(ox, __dmul_rn((double)i, res)));
                const double dy = __dsub_rn(y, __dadd_rn(oy, __dmul_rn((double)j, res)));
                const double dz = __dsub_rn(z, __dadd_rn(oz, __dmul_rn((double)k, res)));
                const double d2 = __dadd_rn(__dadd_rn(__dmul_rn(dx, dx), __dmul_rn(dy, dy)),
                                            __dmul_rn(dz, dz));
                if (d2 <= 0.0 || d2 >= dzr2) continue;
                const float g = __ldg(g_base + ((size_t)i * D + j) * D + k);
                if (g == 0.0f) continue;
                double scale;
                if (d2 <= d02) {
                    // slope / d = exp(-2 d^2/r^2) * (-4/r^2): no sqrt needed
                    scale = (double)g * (double)expf((float)d2 * cexp) * m4inv_r2;
                } else {
                    const double d = sqrt(d2);
                    scale = ((double)g * (qa2 * (d - dzr))) / d;
                }
                gx = fma(scale, dx, gx);
                gy = fma(scale, dy, gy);
                gz = fma(scale, dz, gz);
            }
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

// _kernels.py:258-314: type gradients for every channel of the atom's set and
// coordinate gradients weighted by the atom's type vector.
__global__ void __launch_bounds__(256) k_backward_vector(const BwdArgs A) {
    const int lane = threadIdx.x & 31;
    const int a = blockIdx.x * 8 + (threadIdx.x >> 5);
    const gm_batch &b = A.b;
    if (a >= b.natoms) return;
    const int D = A.p.npts;
    const double res = A.p.resolution, grm = A.p.gaussian_radius_multiple,
                 rmult = A.p.radius_multiple;
    const int s = b.atom_set[a];
    const int e = b.set_example[s];
    const int T = b.set_t[s];
    const int row_off = b.set_wstart[s] + (a - b.set_start[s]) * T;
    const double x = A.pos[3 * a], y = A.pos[3 * a + 1], z = A.pos[3 * a + 2];
    const double ox = b.origins[3 * e], oy = b.origins[3 * e + 1], oz = b.origins[3 * e + 2];
    const size_t D3 = (size_t)D * D * D;
    const double eg = exp((-2.0 * grm) * grm);
    double gx = 0.0, gy = 0.0, gz = 0.0;
    for (int c = 0; c < T; c++) {
        const double r = A.p.radius_type_indexed ? b.type_radius[b.set_trstart[s] + c]
                                                 : b.atom_radius[a];
        const double w = (double)b.weights[row_off + c];
        const double inv_r2 = 1.0 / (r * r);
        const double gr = grm * r, d02 = gr * gr;
        const double dzr = rmult * r, dzr2 = dzr * dzr;
        const double q0 = (2.0 * grm) / r;
        const double qa = eg * (q0 * q0);
        const float cexp = (float)(-2.0 * inv_r2);
        const double m4inv_r2 = -4.0 * inv_r2;
        double tg = 0.0;
        BoxWalk wk;
        if (make_walk(x, y, z, dzr, ox, oy, oz, res, D, wk)) {
            const float *g_base = A.grid_grad + ((size_t)e * b.nchannels + b.set_choff[s] + c) * D3;
            const int seg_off = lane / wk.L, kin = lane - seg_off * wk.L;
            if (seg_off < wk.spi) {
                for (int sg = seg_off; sg < wk.total; sg += wk.spi) {
                    const int row = sg / wk.nseg, sk = sg - row * wk.nseg;
                    const int k = wk.k0 + sk * wk.L + kin;
                    if (k - wk.k0 >= wk.nk) continue;
                    const int ii = row / wk.nj, jj = row - ii * wk.nj;
                    const int i = wk.i0 + ii, j = wk.j0 + jj;
                    const double dx = __dsub_rn(x, __dadd_rn(ox, __dmul_rn((double)i, res)));
                    const double dy = __dsub_rn(y, __dadd_rn(oy, __dmul_rn((double)j, res)));
                    const double dz = __dsub_rn(z, __dadd_rn(oz, __dmul_rn((double)k, res)));
                    const double d2 = __dadd_rn(__dadd_rn(__dmul_rn(dx, dx), __dmul_rn(dy, dy)),
                                                __dmul_rn(dz, dz));
                    if (d2 >= dzr2) continue;
                    const float g = __ldg(g_base + ((size_t)i * D + j) * D + k);
                    if (g == 0.0f) continue;
                    double dens, scale = 0.0;
                    if (d2 <= d02) {
                        dens = (double)expf((float)d2 * cexp);
                        scale = (w * (double)g) * dens * m4inv_r2;
                    } else {
                        const double d = sqrt(d2);
                        const double t = d - dzr;
                        dens = (qa * t) * t;
                        scale = ((w * (double)g) * ((2.0 * qa) * t)) / d;
                    }
                    tg = fma((double)g, dens, tg);
                    if (d2 > 0.0 && w != 0.0) {
                        gx = fma(scale, dx, gx);
                        gy = fma(scale, dy, gy);
                        gz = fma(scale, dz, gz);
                    }
                }
            }
        }
        tg = warp_sum(tg);
        if (lane == 0 && A.type_grad) A.type_grad[row_off + c] = (float)tg;
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

// ----------------------------------------------------------------------------
// host-side launch logic
// ----------------------------------------------------------------------------
static gm_status check_params(const gm_params *p) {
    if (!p) return fail(GM_ERR_INVALID, "params is NULL");
    if (!(p->resolution > 0)) return fail(GM_ERR_INVALID, "resolution must be > 0");
    if (p->npts < 1 || p->npts > 4096) return fail(GM_ERR_INVALID, "npts %d out of range", p->npts);
    if (!(p->radius_multiple > 0)) return fail(GM_ERR_INVALID, "radius_multiple must be > 0");
    return GM_OK;
}

static gm_status check_batch(const gm_batch *b) {
    if (!b) return fail(GM_ERR_INVALID, "batch is NULL");
    if (b->nexamples < 0 || b->nsets < 0 || b->natoms < 0 || b->nitems < 0 || b->nchannels < 0)
        return fail(GM_ERR_INVALID, "negative batch size");
    if (b->natoms > 0 && !b->coords32 && !b->coords64)
        return fail(GM_ERR_INVALID, "batch has atoms but no coordinates");
    if (b->natoms > 0 && (!b->atom_set || !b->atom_radius || !b->set_example || !b->set_choff ||
                          !b->set_start || !b->set_end || !b->set_t))
        return fail(GM_ERR_INVALID, "batch is missing atom/set arrays");
    if (b->nexamples > 0 && (!b->origins || !b->ex_item_start || !b->ex_item_end))
        return fail(GM_ERR_INVALID, "batch is missing per-example arrays");
    if (b->nexamples > 65535) return fail(GM_ERR_INVALID, "too many examples per launch");
    return GM_OK;
}

extern "C" gm_status gm_prepare(const gm_params *p, const gm_batch *b, void *workspace,
                                size_t workspace_bytes, void *stream) {
    gm_status st = check_params(p);
    if (st) return st;
    if ((st = check_batch(b))) return st;
    if (!workspace || workspace_bytes < gm_workspace_bytes(b->natoms, b->nitems))
        return fail(GM_ERR_INVALID, "workspace too small (%zu < %zu)", workspace_bytes,
                    gm_workspace_bytes(b->natoms, b->nitems));
    if (!b->vector_mode && b->nitems != b->natoms)
        return fail(GM_ERR_INVALID, "index mode needs one item per atom");
    if (b->nitems > 0 && !b->item_channel && !b->atom_type)
        return fail(GM_ERR_INVALID, "items need item_channel or atom_type");
    PrepArgs A;
    A.p = *p;
    A.b = *b;
    carve(workspace, b->natoms, b->nitems, &A.ws);
    cudaStream_t s = (cudaStream_t)stream;
    if (b->natoms > 0) {
        int blocks = std::min((b->natoms + 255) / 256, 148 * 16);
        k_prepare_atoms<<<blocks, 256, 0, s>>>(A);
        LAUNCH_CHECK();
    }
    if (b->nitems > 0) {
        int blocks = std::min((b->nitems + 255) / 256, 148 * 16);
        k_prepare_items<<<blocks, 256, 0, s>>>(A);
        LAUNCH_CHECK();
    }
    return GM_OK;
}

struct FwdConfig {
    int TI, TJ, CC, SJ, nchunks, patch;  // patch: 0 = 2x4x4, 1 = 2x2x8, 2 = 1x1x32
    size_t smem;
};

static int padded_row(int D) {
    int s = (D + 3) & ~3;
    // 4*odd mod 32 keeps the 2x4x4 warp patch conflict-free on the 32 banks
    while ((s % 32) != 4 && (s % 32) != 12 && (s % 32) != 20 && (s % 32) != 28) s += 4;
    return s;
}

static FwdConfig choose_config(int D, int C, bool binary) {
    static const int tiles[][3] = {{4, 4, 0}, {4, 2, 1}, {2, 2, 1}, {1, 1, 2}};
    const size_t budget = 72 * 1024;
    const size_t list_bytes = (size_t)kCap * (sizeof(FwdItem) + (binary ? sizeof(BinItem) : 0)) + 64;
    FwdConfig cfg{};
    cfg.SJ = padded_row(D);
    const int want = std::min(C, 14) > 0 ? std::min(C, 14) : 1;
    for (int t = 0; t < 4; t++) {
        const size_t per_ch = (size_t)tiles[t][0] * tiles[t][1] * cfg.SJ * 4;
        int fit = (int)(budget / per_ch);
        if (fit >= want || t == 3) {
            fit = std::max(fit, 1);
            cfg.TI = tiles[t][0];
            cfg.TJ = tiles[t][1];
            cfg.patch = tiles[t][2];
            cfg.nchunks = (std::max(C, 1) + fit - 1) / fit;
            cfg.CC = (std::max(C, 1) + cfg.nchunks - 1) / cfg.nchunks;
            cfg.smem = (size_t)cfg.CC * per_ch + list_bytes;
            break;
        }
    }
    return cfg;
}

template <int PI, int PJ, int PK, bool BIN, bool VEC>
static gm_status launch_forward_t(const FwdArgs &A, const FwdConfig &cfg, int nex, cudaStream_t s) {
    auto kern = k_forward<PI, PJ, PK, BIN, VEC>;
    static thread_local int smem_set = 0;  // per instantiation, per thread (per device context)
    if ((int)cfg.smem > smem_set) {
        CUDA_TRY(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)cfg.smem));
        smem_set = (int)cfg.smem;
    }
    const int ntiles = ((A.D + cfg.TI - 1) / cfg.TI) * ((A.D + cfg.TJ - 1) / cfg.TJ) * cfg.nchunks;
    dim3 grid(ntiles, nex);
    kern<<<grid, kThreads, cfg.smem, s>>>(A);
    LAUNCH_CHECK();
    return GM_OK;
}

template <bool BIN, bool VEC>
static gm_status launch_forward_mode(const FwdArgs &A, const FwdConfig &cfg, int nex, cudaStream_t s) {
    switch (cfg.patch) {
        case 0: return launch_forward_t<2, 4, 4, BIN, VEC>(A, cfg, nex, s);
        case 1: return launch_forward_t<2, 2, 8, BIN, VEC>(A, cfg, nex, s);
        default: return launch_forward_t<1, 1, 32, BIN, VEC>(A, cfg, nex, s);
    }
}

extern "C" gm_status gm_forward(const gm_params *p, const gm_batch *b, const void *workspace,
                                float *out, void *stream) {
    gm_status st = check_params(p);
    if (st) return st;
    if ((st = check_batch(b))) return st;
    if (b->nexamples == 0 || b->nchannels == 0) return GM_OK;
    if (!out) return fail(GM_ERR_INVALID, "out is NULL");
    if (!workspace) return fail(GM_ERR_INVALID, "workspace is NULL");
    Workspace ws;
    carve(const_cast<void *>(workspace), b->natoms, b->nitems, &ws);
    const FwdConfig cfg = choose_config(p->npts, b->nchannels, p->binary != 0);
    FwdArgs A;
    A.items = ws.items;
    A.bitems = ws.bitems;
    A.cull = ws.cull;
    A.ex_item_start = b->ex_item_start;
    A.ex_item_end = b->ex_item_end;
    A.origins = b->origins;
    A.out = out;
    A.res = p->resolution;
    A.D = p->npts;
    A.C = b->nchannels;
    A.TI = cfg.TI;
    A.TJ = cfg.TJ;
    A.CC = cfg.CC;
    A.SJ = cfg.SJ;
    A.ntj = (A.D + cfg.TJ - 1) / cfg.TJ;
    A.nchunks = cfg.nchunks;
    cudaStream_t s = (cudaStream_t)stream;
    if (p->binary) {
        return b->vector_mode ? launch_forward_mode<true, true>(A, cfg, b->nexamples, s)
                              : launch_forward_mode<true, false>(A, cfg, b->nexamples, s);
    }
    return launch_forward_mode<false, false>(A, cfg, b->nexamples, s);
}

extern "C" gm_status gm_backward(const gm_params *p, const gm_batch *b, const void *workspace,
                                 const float *grid_grad, float *coord_grad, float *type_grad,
                                 void *stream) {
    gm_status st = check_params(p);
    if (st) return st;
    if ((st = check_batch(b))) return st;
    if (b->natoms == 0) return GM_OK;
    if (!coord_grad) return fail(GM_ERR_INVALID, "coord_grad is NULL");
    cudaStream_t s = (cudaStream_t)stream;
    if (p->binary) {
        // voxelizer.py:284-289: binary grids are flat almost everywhere
        CUDA_TRY(cudaMemsetAsync(coord_grad, 0, sizeof(float) * 3 * (size_t)b->natoms, s));
        if (b->vector_mode && type_grad && b->nweights > 0)
            CUDA_TRY(cudaMemsetAsync(type_grad, 0, sizeof(float) * (size_t)b->nweights, s));
        return GM_OK;
    }
    if (!grid_grad || !workspace) return fail(GM_ERR_INVALID, "grid_grad/workspace is NULL");
    if (!b->vector_mode && !b->atom_type) return fail(GM_ERR_INVALID, "atom_type is NULL");
    if (b->vector_mode && (!b->weights || !b->set_wstart))
        return fail(GM_ERR_INVALID, "vector backward needs weights and set_wstart");
    if (b->vector_mode && p->radius_type_indexed && (!b->type_radius || !b->set_trstart))
        return fail(GM_ERR_INVALID, "radius_type_indexed needs type_radius and set_trstart");
    BwdArgs A;
    A.p = *p;
    A.b = *b;
    A.pos = (const double *)workspace;
    A.grid_grad = grid_grad;
    A.coord_grad = coord_grad;
    A.type_grad = type_grad;
    const int blocks = (b->natoms + 7) / 8;
    if (b->vector_mode) k_backward_vector<<<blocks, 256, 0, s>>>(A);
    else k_backward_index<<<blocks, 256, 0, s>>>(A);
    LAUNCH_CHECK();
    return GM_OK;
}

// ----------------------------------------------------------------------------
// reference-shaped host entry points (numpy buffers in, numpy buffers out)
// ----------------------------------------------------------------------------
namespace {

struct DevBuf {
    void *ptr = nullptr;
    size_t bytes = 0;
    ~DevBuf() {
        if (ptr) cudaFree(ptr);
    }
    cudaError_t reserve(size_t n) {
        if (n <= bytes) return cudaSuccess;
        if (ptr) cudaFree(ptr);
        ptr = nullptr;
        bytes = 0;
        cudaError_t e = cudaMalloc(&ptr, n);
        if (e == cudaSuccess) bytes = n;
        return e;
    }
};

// Staging arena for the *_host entry points: one growable device buffer per
// thread, carved into the arrays of one call.
struct Arena {
    DevBuf buf;
};

thread_local Arena t_arena;

struct HostPlan {
    std::vector<std::pair<size_t, std::pair<const void *, size_t>>> uploads;
    size_t used = 0;
    size_t add(const void *src, size_t bytes) {
        size_t off = used;
        used = align_up(used + std::max<size_t>(bytes, 1), 256);
        if (src) uploads.push_back({off, {src, bytes}});
        return off;
    }
};

}  // namespace

static gm_status run_host_forward(float *out, int64_t nexamples, int64_t nch, int64_t npts,
                                  const double *coords, int64_t natoms,
                                  const std::vector<int32_t> &atom_set,
                                  const std::vector<int32_t> &atom_type,
                                  const std::vector<double> &atom_radius,
                                  const std::vector<int32_t> &item_atom,
                                  const std::vector<int32_t> &item_channel,
                                  const std::vector<float> &item_weight,
                                  const std::vector<double> &item_radius, bool vector_mode,
                                  const std::vector<int32_t> *sets /* 5 arrays */,
                                  const std::vector<int32_t> &ex_start,
                                  const std::vector<int32_t> &ex_end, const double *origins,
                                  const gm_params &p) {
    const int32_t nsets = (int32_t)sets[0].size();
    const int32_t nitems = vector_mode ? (int32_t)item_atom.size() : (int32_t)natoms;
    HostPlan plan;
    const size_t o_coords = plan.add(coords, sizeof(double) * 3 * natoms);
    const size_t o_aset = plan.add(atom_set.data(), 4 * atom_set.size());
    const size_t o_atype = plan.add(atom_type.data(), 4 * atom_type.size());
    const size_t o_arad = plan.add(atom_radius.data(), 8 * atom_radius.size());
    size_t o_sets[5];
    for (int k = 0; k < 5; k++) o_sets[k] = plan.add(sets[k].data(), 4 * sets[k].size());
    const size_t o_iatom = plan.add(item_atom.data(), 4 * item_atom.size());
    const size_t o_ich = plan.add(item_channel.data(), 4 * item_channel.size());
    const size_t o_iw = plan.add(item_weight.data(), 4 * item_weight.size());
    const size_t o_irad = plan.add(item_radius.data(), 8 * item_radius.size());
    const size_t o_exs = plan.add(ex_start.data(), 4 * ex_start.size());
    const size_t o_exe = plan.add(ex_end.data(), 4 * ex_end.size());
    const size_t o_orig = plan.add(origins, sizeof(double) * 3 * nexamples);
    const size_t ws_bytes = gm_workspace_bytes((int32_t)natoms, nitems);
    const size_t o_ws = plan.add(nullptr, ws_bytes);
    const size_t out_bytes = sizeof(float) * (size_t)nexamples * nch * npts * npts * npts;
    const size_t o_out = plan.add(nullptr, out_bytes);

    Arena &ar = t_arena;
    CUDA_TRY(ar.buf.reserve(plan.used));
    char *d = (char *)ar.buf.ptr;
    for (auto &u : plan.uploads)
        CUDA_TRY(cudaMemcpy(d + u.first, u.second.first, u.second.second, cudaMemcpyHostToDevice));
    gm_batch b;
    memset(&b, 0, sizeof b);
    b.nexamples = (int32_t)nexamples;
    b.nsets = nsets;
    b.natoms = (int32_t)natoms;
    b.nitems = nitems;
    b.nchannels = (int32_t)nch;
    b.vector_mode = vector_mode;
    b.coords64 = (const double *)(d + o_coords);
    b.atom_set = (const int32_t *)(d + o_aset);
    b.atom_type = atom_type.empty() ? nullptr : (const int32_t *)(d + o_atype);
    b.atom_radius = (const double *)(d + o_arad);
    b.set_start = (const int32_t *)(d + o_sets[0]);
    b.set_end = (const int32_t *)(d + o_sets[1]);
    b.set_example = (const int32_t *)(d + o_sets[2]);
    b.set_choff = (const int32_t *)(d + o_sets[3]);
    b.set_t = (const int32_t *)(d + o_sets[4]);
    if (vector_mode) {
        b.item_atom = (const int32_t *)(d + o_iatom);
        b.item_channel = (const int32_t *)(d + o_ich);
        b.item_weight = (const float *)(d + o_iw);
        b.item_radius = (const double *)(d + o_irad);
    }
    b.ex_item_start = (const int32_t *)(d + o_exs);
    b.ex_item_end = (const int32_t *)(d + o_exe);
    b.origins = (const double *)(d + o_orig);
    gm_status st = gm_prepare(&p, &b, d + o_ws, ws_bytes, nullptr);
    if (st) return st;
    st = gm_forward(&p, &b, d + o_ws, (float *)(d + o_out), nullptr);
    if (st) return st;
    CUDA_TRY(cudaMemcpy(out, d + o_out, out_bytes, cudaMemcpyDeviceToHost));
    return GM_OK;
}

static gm_params host_params(int64_t npts, double res, double grm, double rmult, int32_t binary,
                             int32_t rti) {
    gm_params p;
    memset(&p, 0, sizeof p);
    p.resolution = res;
    p.dimension = res * (double)(npts - 1);
    p.radius_scale = 1.0;
    p.gaussian_radius_multiple = grm;
    p.radius_multiple = rmult;
    p.npts = (int32_t)npts;
    p.binary = binary;
    p.radius_type_indexed = rti;
    p.matmul_order_1 = -1;
    p.matmul_order_n = -1;
    return p;
}

// Validates the reference's packing invariants (voxelizer.py:372-388): sets of
// one example are consecutive and atoms are packed in set order.
static gm_status pack_sets(int64_t nsets, int64_t nexamples, int64_t natoms,
                           const int64_t *set_start, const int64_t *set_end,
                           const int64_t *set_example, const int64_t *set_choff,
                           const int64_t *set_t, std::vector<int32_t> *sets,
                           std::vector<int32_t> &atom_set) {
    for (int k = 0; k < 5; k++) sets[k].resize(nsets);
    atom_set.assign(natoms, 0);
    int64_t prev_e = 0;
    for (int64_t s = 0; s < nsets; s++) {
        if (set_start[s] < 0 || set_end[s] > natoms || set_end[s] < set_start[s])
            return fail(GM_ERR_INVALID, "set %lld has a bad atom range", (long long)s);
        if (set_example[s] < prev_e || set_example[s] >= nexamples)
            return fail(GM_ERR_INVALID, "sets must be grouped by example in order");
        prev_e = set_example[s];
        sets[0][s] = (int32_t)set_start[s];
        sets[1][s] = (int32_t)set_end[s];
        sets[2][s] = (int32_t)set_example[s];
        sets[3][s] = (int32_t)set_choff[s];
        sets[4][s] = (int32_t)set_t[s];
        for (int64_t a = set_start[s]; a < set_end[s]; a++) atom_set[a] = (int32_t)s;
    }
    return GM_OK;
}

extern "C" gm_status gm_forward_index_sets_host(
    float *out, int64_t nexamples, int64_t nch, int64_t npts, const double *coords,
    const double *radii, const int64_t *tidx, int64_t natoms, const int64_t *set_start,
    const int64_t *set_end, const int64_t *set_example, const int64_t *set_choff,
    const int64_t *set_t, int64_t nsets, const double *origins, double res, double grm,
    double rmult, int32_t binary) {
    if (!out || (natoms && (!coords || !radii || !tidx)) || !origins)
        return fail(GM_ERR_INVALID, "NULL argument");
    std::vector<int32_t> sets[5], atom_set;
    gm_status st = pack_sets(nsets, nexamples, natoms, set_start, set_end, set_example, set_choff,
                             set_t, sets, atom_set);
    if (st) return st;
    std::vector<int32_t> atom_type(natoms);
    for (int64_t a = 0; a < natoms; a++) atom_type[a] = (int32_t)tidx[a];
    std::vector<double> atom_radius(radii, radii + natoms);
    std::vector<int32_t> ex_start(nexamples, 0), ex_end(nexamples, 0);
    for (int64_t s = 0; s < nsets; s++) {
        const int64_t e = set_example[s];
        if (ex_end[e] == ex_start[e]) ex_start[e] = (int32_t)set_start[s];
        ex_end[e] = (int32_t)set_end[s];
    }
    gm_params p = host_params(npts, res, grm, rmult, binary, 0);
    static const std::vector<int32_t> ei;
    static const std::vector<float> ef;
    static const std::vector<double> ed;
    return run_host_forward(out, nexamples, nch, npts, coords, natoms, atom_set, atom_type,
                            atom_radius, ei, ei, ef, ed, false, sets, ex_start, ex_end, origins, p);
}

extern "C" gm_status gm_forward_vector_sets_host(
    float *out, int64_t nexamples, int64_t nch, int64_t npts, const double *coords,
    int64_t natoms, const double *weights_flat, int64_t nweights, const int64_t *w_start,
    const double *atom_radii, const double *type_radii_flat, int64_t ntype_radii,
    const int64_t *tr_start, int32_t radius_type_indexed, const int64_t *set_start,
    const int64_t *set_end, const int64_t *set_example, const int64_t *set_choff,
    const int64_t *set_t, int64_t nsets, const double *origins, double res, double grm,
    double rmult, int32_t binary) {
    if (!out || !origins || (natoms && (!coords || !weights_flat || !atom_radii)))
        return fail(GM_ERR_INVALID, "NULL argument");
    std::vector<int32_t> sets[5], atom_set;
    gm_status st = pack_sets(nsets, nexamples, natoms, set_start, set_end, set_example, set_choff,
                             set_t, sets, atom_set);
    if (st) return st;
    std::vector<int32_t> item_atom, item_channel;
    std::vector<float> item_weight;
    std::vector<double> item_radius;
    std::vector<int32_t> ex_start(nexamples, 0), ex_end(nexamples, 0);
    std::vector<char> seen(nexamples, 0);
    for (int64_t s = 0; s < nsets; s++) {
        const int64_t e = set_example[s], nt = set_t[s];
        if (!seen[e]) {
            ex_start[e] = (int32_t)item_atom.size();
            seen[e] = 1;
        }
        for (int64_t a = set_start[s]; a < set_end[s]; a++) {
            for (int64_t c = 0; c < nt; c++) {
                const int64_t wi = w_start[s] + (a - set_start[s]) * nt + c;
                if (wi < 0 || wi >= nweights) return fail(GM_ERR_INVALID, "weight index out of range");
                const double w = weights_flat[wi];
                if (w == 0.0) continue;  // _kernels.py:164
                double r = atom_radii[a];
                if (radius_type_indexed) {
                    const int64_t ti = tr_start[s] + c;
                    if (!type_radii_flat || ti < 0 || ti >= ntype_radii)
                        return fail(GM_ERR_INVALID, "type radius index out of range");
                    r = type_radii_flat[ti];
                }
                item_atom.push_back((int32_t)a);
                item_channel.push_back((int32_t)c);
                item_weight.push_back((float)w);
                item_radius.push_back(r);
            }
        }
        ex_end[e] = (int32_t)item_atom.size();
    }
    std::vector<double> atom_radius(atom_radii, atom_radii + natoms);
    std::vector<int32_t> atom_type;
    gm_params p = host_params(npts, res, grm, rmult, binary, radius_type_indexed);
    return run_host_forward(out, nexamples, nch, npts, coords, natoms, atom_set, atom_type,
                            atom_radius, item_atom, item_channel, item_weight, item_radius, true,
                            sets, ex_start, ex_end, origins, p);
}

static gm_status run_host_backward(double *coord_grad, double *type_grad, const double *coords,
                                   const double *radii, const int64_t *tidx,
                                   const double *weights, int64_t n, int64_t nt,
                                   const float *grid_grad, int64_t npts, const double *type_radii,
                                   int32_t rti, const double *origin, double res, double grm,
                                   double rmult) {
    if (n == 0) return GM_OK;
    const bool vector_mode = weights != nullptr;
    std::vector<int32_t> atom_set(n, 0), atom_type;
    if (!vector_mode) {
        atom_type.resize(n);
        for (int64_t a = 0; a < n; a++) atom_type[a] = (int32_t)tidx[a];
    }
    std::vector<float> w32;
    if (vector_mode) w32.assign(weights, weights + n * nt);
    const int32_t set_start = 0, set_end = (int32_t)n, set_example = 0, set_choff = 0,
                  set_t = (int32_t)nt, set_ws = 0, set_tr = 0;
    const int32_t ex_s = 0, ex_e = (int32_t)n;
    const size_t D3 = (size_t)npts * npts * npts;
    HostPlan plan;
    const size_t o_coords = plan.add(coords, sizeof(double) * 3 * n);
    const size_t o_rad = plan.add(radii, sizeof(double) * n);
    const size_t o_aset = plan.add(atom_set.data(), 4 * n);
    const size_t o_atype = plan.add(atom_type.data(), 4 * atom_type.size());
    const size_t o_ss = plan.add(&set_start, 4), o_se = plan.add(&set_end, 4),
                 o_sx = plan.add(&set_example, 4), o_sc = plan.add(&set_choff, 4),
                 o_st = plan.add(&set_t, 4), o_sw = plan.add(&set_ws, 4),
                 o_str = plan.add(&set_tr, 4);
    const size_t o_w = plan.add(w32.data(), 4 * w32.size());
    const size_t o_tr = plan.add(type_radii, type_radii ? sizeof(double) * nt : 0);
    const size_t o_exs = plan.add(&ex_s, 4), o_exe = plan.add(&ex_e, 4);
    const size_t o_orig = plan.add(origin, sizeof(double) * 3);
    const size_t o_gg = plan.add(grid_grad, sizeof(float) * nt * D3);
    const size_t ws_bytes = gm_workspace_bytes((int32_t)n, (int32_t)n);
    const size_t o_ws = plan.add(nullptr, ws_bytes);
    const size_t o_cg = plan.add(nullptr, sizeof(float) * 3 * n);
    const size_t o_tg = plan.add(nullptr, sizeof(float) * (vector_mode ? n * nt : 1));
    Arena &ar = t_arena;
    CUDA_TRY(ar.buf.reserve(plan.used));
    char *d = (char *)ar.buf.ptr;
    for (auto &u : plan.uploads)
        CUDA_TRY(cudaMemcpy(d + u.first, u.second.first, u.second.second, cudaMemcpyHostToDevice));
    gm_batch b;
    memset(&b, 0, sizeof b);
    b.nexamples = 1;
    b.nsets = 1;
    b.natoms = (int32_t)n;
    b.nitems = (int32_t)n;
    b.nchannels = (int32_t)nt;
    b.vector_mode = vector_mode;
    b.coords64 = (const double *)(d + o_coords);
    b.atom_radius = (const double *)(d + o_rad);
    b.atom_set = (const int32_t *)(d + o_aset);
    b.atom_type = vector_mode ? nullptr : (const int32_t *)(d + o_atype);
    b.set_start = (const int32_t *)(d + o_ss);
    b.set_end = (const int32_t *)(d + o_se);
    b.set_example = (const int32_t *)(d + o_sx);
    b.set_choff = (const int32_t *)(d + o_sc);
    b.set_t = (const int32_t *)(d + o_st);
    b.set_wstart = (const int32_t *)(d + o_sw);
    b.set_trstart = (const int32_t *)(d + o_str);
    b.nweights = vector_mode ? (int32_t)(n * nt) : 0;
    b.weights = vector_mode ? (const float *)(d + o_w) : nullptr;
    b.type_radius = type_radii ? (const double *)(d + o_tr) : nullptr;
    b.item_channel = nullptr;
    b.ex_item_start = (const int32_t *)(d + o_exs);
    b.ex_item_end = (const int32_t *)(d + o_exe);
    b.origins = (const double *)(d + o_orig);
    gm_params p = host_params(npts, res, grm, rmult, 0, rti);
    // positions only (no transform); items are not needed by the backward
    PrepArgs A;
    A.p = p;
    A.b = b;
    carve(d + o_ws, b.natoms, b.nitems, &A.ws);
    k_prepare_atoms<<<(b.natoms + 255) / 256, 256>>>(A);
    LAUNCH_CHECK();
    gm_status st = gm_backward(&p, &b, d + o_ws, (const float *)(d + o_gg), (float *)(d + o_cg),
                               vector_mode ? (float *)(d + o_tg) : nullptr, nullptr);
    if (st) return st;
    std::vector<float> cg(3 * n), tg(vector_mode ? n * nt : 0);
    CUDA_TRY(cudaMemcpy(cg.data(), d + o_cg, sizeof(float) * 3 * n, cudaMemcpyDeviceToHost));
    for (int64_t i = 0; i < 3 * n; i++) coord_grad[i] = cg[i];
    if (vector_mode) {
        CUDA_TRY(cudaMemcpy(tg.data(), d + o_tg, sizeof(float) * n * nt, cudaMemcpyDeviceToHost));
        for (int64_t i = 0; i < n * nt; i++) type_grad[i] = tg[i];
    }
    return GM_OK;
}

extern "C" gm_status gm_backward_index_host(double *coord_grad, const double *coords,
                                            const double *radii, const int64_t *tidx, int64_t n,
                                            const float *grid_grad, int64_t ntypes, int64_t npts,
                                            const double *origin, double res, double grm,
                                            double rmult) {
    if (n && (!coord_grad || !coords || !radii || !tidx || !grid_grad || !origin))
        return fail(GM_ERR_INVALID, "NULL argument");
    return run_host_backward(coord_grad, nullptr, coords, radii, tidx, nullptr, n, ntypes,
                             grid_grad, npts, nullptr, 0, origin, res, grm, rmult);
}

extern "C" gm_status gm_backward_vector_host(double *coord_grad, double *type_grad,
                                             const double *coords, const double *atom_radii,
                                             const double *weights, int64_t n, int64_t nt,
                                             const float *grid_grad, int64_t npts,
                                             const double *type_radii, int32_t rti,
                                             const double *origin, double res, double grm,
                                             double rmult) {
    if (n && (!coord_grad || !type_grad || !coords || !atom_radii || !weights || !grid_grad ||
              !origin || (rti && !type_radii)))
        return fail(GM_ERR_INVALID, "NULL argument");
    return run_host_backward(coord_grad, type_grad, coords, atom_radii, nullptr, weights, n, nt,
                             grid_grad, npts, type_radii, rti, origin, res, grm, rmult);
}

extern "C" const char *gm_last_error(void) { return g_err.c_str(); }
extern "C" const char *gm_version(void) { return GM_VERSION; }
extern "C" int32_t gm_device_count(void) {
    int n = 0;
    if (cudaGetDeviceCount(&n) != cudaSuccess) return 0;
    return n;
}
extern "C" int32_t gm_struct_size(int32_t which) {
    return which == 0 ? (int32_t)sizeof(gm_params) : which == 1 ? (int32_t)sizeof(gm_batch) : -1;
}
extern "C" int64_t gm_launch_count(int32_t reset) {
    return reset ? g_launches.exchange(0) : g_launches.load();
}
