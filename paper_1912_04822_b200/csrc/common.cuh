// common.cuh -- records, workspace layout and device helpers shared by the
// gridding kernels (prepare.cu, forward.cu, backward.cu) and the C ABI (abi.cu).
#pragma once

#include <cuda_runtime.h>
#include <math_constants.h>
#include <stdarg.h>
#include <stdint.h>
#include <stdio.h>
#include <string.h>

#include <algorithm>
#include <atomic>
#include <utility>

#include "../../include/gridmaker_b200.h"

// ---------------------------------------------------------------------------
// error plumbing (abi.cu)
// ---------------------------------------------------------------------------
gm_status gm_fail(gm_status code, const char *fmt, ...);
void gm_count_launch();
// cudaFuncSetAttribute(MaxDynamicSharedMemorySize) once per (device, kernel, size).
cudaError_t gm_ensure_smem(const void *func, int bytes);

#define CUDA_TRY(expr)                                                                       \
    do {                                                                                     \
        cudaError_t _e = (expr);                                                             \
        if (_e != cudaSuccess)                                                               \
            return gm_fail(GM_ERR_CUDA, "%s failed: %s (%s:%d)", #expr,                      \
                           cudaGetErrorString(_e), __FILE__, __LINE__);                      \
    } while (0)

#define LAUNCH_CHECK()                                                                       \
    do {                                                                                     \
        gm_count_launch();                                                                   \
        cudaError_t _e = cudaGetLastError();                                                 \
        if (_e != cudaSuccess)                                                               \
            return gm_fail(GM_ERR_CUDA, "kernel launch failed: %s (%s:%d)",                  \
                           cudaGetErrorString(_e), __FILE__, __LINE__);                      \
    } while (0)

// ---------------------------------------------------------------------------
// device records
// ---------------------------------------------------------------------------
// One forward item: index mode -> an atom; vector mode -> an (atom, channel)
// pair with nonzero weight (_kernels.py:159-166).  64 B = 4 x LDS.128.
struct __align__(16) FwdItem {
    float cxh, cyh, czh, cexp;  // offset voxel(box corner) - atom per axis, hi part; -2 log2(e)/r^2
    float cxl, cyl, czl, d02;   // lo parts (offset = hi + lo to ~2^-48); (grm r)^2
    float dzr, qa, w;           // cutoff (rmult*r, or r in binary mode); quadratic coeff.; weight
    int ch;                  // absolute output channel
    int ibox, jbox, kbox;    // voxel box per axis: lo | hi << 16 (_kernels.py:22-30)
    int atom;                // packed atom index
};
static_assert(sizeof(FwdItem) == 64, "FwdItem must be 64 bytes");

// Exact binary-mode record: transformed f64 position and r^2 (_kernels.py:81,95-98).
struct __align__(16) BinItem {
    double x, y, z, r2;
};

// Index-mode backward record of one atom, written by the prepare pass so the
// backward starts from one independent 16-B-load level.
struct __align__(16) BwdAtom {
    double lx, ly, lz;       // transformed position minus the example's origin
    double dzr, dzr2, d02;   // cutoff rmult*r and its square, (grm r)^2
    double qa2, m4inv_r2;    // 2 qa (_kernels.py:224 tail slope), -4 / r^2
    double m2inv_r2;         // -2 / r^2 (per-axis Gaussian tables)
    int atom, pad;           // packed atom index (records may be permuted: gm_batch.bwd_slot)
    int slab;                // e * nchannels + channel: the atom's grid_grad block
    int ibox, jbox, kbox;    // voxel box (lo | hi << 16); ibox lo > hi if it misses
};
static_assert(sizeof(BwdAtom) == 96, "BwdAtom must be 96 bytes");

// Vector-mode backward record of one atom, at its launch slot: everything
// the walk needs in one load level (instead of atom -> set -> example chains).
struct __align__(16) VBwdAtom {
    double x, y, z;          // transformed position
    double ox, oy, oz;       // the example's origin
    double r;                // radius * radius_scale
    int atom;                // packed atom index
    int slab;                // e * nchannels + set_choff: the set's first grid_grad slab
    int row;                 // first entry of the atom's weight row
    int T;                   // the set's channel count
    int set;                 // packed set index
    int pad;
};
static_assert(sizeof(VBwdAtom) == 80, "VBwdAtom must be 80 bytes");

__host__ __device__ inline int box_lo(int b) { return b & 0xffff; }
__host__ __device__ inline int box_hi(int b) { return b >> 16; }

// Plane buckets of the per-channel item sort: plane i -> bucket i * kBuckets / D
// (one bucket per plane up to 64^3).  Per (example, channel) record: bucket
// start offsets [0, kBuckets + 1] (entry kBuckets: items whose box misses the
// grid; entry kBuckets + 1 = count) and the widest box in planes.
constexpr int kBuckets = 64;
constexpr int kPlaneRec = kBuckets + 3;
__host__ __device__ inline int plane_bucket(int i, int D) { return (int)(((long long)i * kBuckets) / D); }

#ifndef GM_PLANE_SORT
#define GM_PLANE_SORT 1
#endif
// Whether the prepare pass sorts each channel's items by first plane and the
// forward scans plane ranges.  Measured (B200): the extra pass (~11 us) pays
// on fine grids (96^3: forward -30 us) and vector typing (3.5 items per atom:
// -20 us per step), not on 48^3 index grids (the forward saves what the pass
// costs) -- there the items stay in item order.
#ifndef GM_PLANE_SORT_MIND
#define GM_PLANE_SORT_MIND 64  // index typing: plane-sort grids above this size
#endif
inline bool use_plane_sort(const gm_params *p, const gm_batch *b) {
    return GM_PLANE_SORT && (p->npts > GM_PLANE_SORT_MIND || b->vector_mode);
}

// ---------------------------------------------------------------------------
// workspace: one caller-provided device buffer
// ---------------------------------------------------------------------------
struct Workspace {
    double *pos;         // natoms * 3: transformed f64 coordinates
    FwdItem *items;      // nitems, packed order
    BinItem *bitems;     // nitems, packed order
    int32_t *item_ch;    // nitems: channel, or -1 when the box misses the grid
    FwdItem *sorted;     // nitems: per example, grouped by channel in item order
    BinItem *bsorted;    // nitems (binary mode)
    int2 *sbox;          // nitems: {ibox, jbox} of sorted items (forward culling)
    int32_t *chan_off;   // nexamples * (nchannels + 1): ranges into sorted
    BwdAtom *batoms;     // natoms (index mode): backward records
    FwdItem *psorted;    // nitems: each (example, channel) range sorted by first plane (stable)
    int2 *psbox;         // nitems: {ibox, jbox} of psorted
    BinItem *pbsorted;   // nitems (binary mode)
    int32_t *poff;       // nexamples * nchannels * kPlaneRec: plane-bucket offsets + max width
    int32_t *atom_order; // natoms (vector mode with gm_batch.bwd_slot): atom of each launch slot
    VBwdAtom *vbatoms;   // natoms (vector mode): backward records at launch slots
};

inline size_t align_up(size_t x, size_t a) { return (x + a - 1) / a * a; }

inline size_t carve_workspace(void *base, int32_t natoms, int32_t nitems, int32_t nex,
                              int32_t nch, Workspace *w) {
    char *p = (char *)base;
    size_t off = 0;
    auto take = [&](size_t bytes) {
        char *q = p ? p + off : nullptr;
        off = align_up(off + std::max<size_t>(bytes, 16), 256);
        return q;
    };
    const size_t na = (size_t)std::max(natoms, 1), ni = (size_t)std::max(nitems, 1);
    Workspace tmp;
    Workspace *ws = w ? w : &tmp;
    ws->pos = (double *)take(sizeof(double) * 3 * na);
    ws->items = (FwdItem *)take(sizeof(FwdItem) * ni);
    ws->bitems = (BinItem *)take(sizeof(BinItem) * ni);
    ws->item_ch = (int32_t *)take(sizeof(int32_t) * ni);
    ws->sorted = (FwdItem *)take(sizeof(FwdItem) * ni);
    ws->bsorted = (BinItem *)take(sizeof(BinItem) * ni);
    ws->sbox = (int2 *)take(sizeof(int2) * ni);
    ws->chan_off = (int32_t *)take(sizeof(int32_t) * (size_t)std::max(nex, 1) * (nch + 1));
    ws->batoms = (BwdAtom *)take(sizeof(BwdAtom) * na);
    ws->psorted = (FwdItem *)take(sizeof(FwdItem) * ni);
    ws->psbox = (int2 *)take(sizeof(int2) * ni);
    ws->pbsorted = (BinItem *)take(sizeof(BinItem) * ni);
    ws->poff = (int32_t *)take(sizeof(int32_t) * (size_t)std::max(nex, 1) * std::max(nch, 1) * kPlaneRec);
    ws->atom_order = (int32_t *)take(sizeof(int32_t) * na);
    ws->vbatoms = (VBwdAtom *)take(sizeof(VBwdAtom) * na);
    return off + 256;
}

// ---------------------------------------------------------------------------
// device helpers
// ---------------------------------------------------------------------------
// _kernels.py:22-30 in f64 with the reference's operation order:
//   lo = ceil(((x - cut) - origin) / res), hi = floor(((x + cut) - origin) / res),
// clamped to [0, D-1] (the clamp keeps lo > hi for boxes that miss the grid).
__device__ __forceinline__ void axis_bounds(double x, double cut, double origin, double res,
                                            int D, int &lo, int &hi) {
    const double nl = __dsub_rn(__dsub_rn(x, cut), origin);
    const double nh = __dsub_rn(__dadd_rn(x, cut), origin);
    double l, h;
    // a power-of-two spacing (0.5, 0.25, 1 A ...): dividing by it is an exact
    // scaling, so multiplying by its exact reciprocal gives the same bits
    // without the DDIV sequence (warp-uniform branch)
    const unsigned long long rb = (unsigned long long)__double_as_longlong(res);
    const unsigned ex = (unsigned)(rb >> 52) & 0x7ffu;
    if ((rb & 0x000fffffffffffffULL) == 0 && ex > 0 && ex < 2046 && !(rb >> 63)) {
        const double inv = __longlong_as_double((long long)((2046ull - ex) << 52));
        l = ceil(__dmul_rn(nl, inv));
        h = floor(__dmul_rn(nh, inv));
    } else {
        l = ceil(__ddiv_rn(nl, res));
        h = floor(__ddiv_rn(nh, res));
    }
    l = fmin(fmax(l, 0.0), (double)D);
    h = fmax(fmin(h, (double)(D - 1)), -1.0);
    lo = (int)l;
    hi = (int)h;
}

// Programmatic dependent launch (PDL): a kernel launched with
// gm_launch_pdl may start while the previous kernel of the stream drains;
// pdl_wait() blocks until that kernel has completed and its writes are
// visible.  pdl_trigger() lets the next PDL-launched kernel start; our kernels
// call it only after their own pdl_wait(), so everything before the previous
// kernel (e.g. the prepare pass) is complete when a dependent starts.
#ifndef GM_PDL
#define GM_PDL 1
#endif
__device__ __forceinline__ void pdl_wait() {
#if GM_PDL
    asm volatile("griddepcontrol.wait;" ::: "memory");
#endif
}
__device__ __forceinline__ void pdl_trigger() {
#if GM_PDL
    asm volatile("griddepcontrol.launch_dependents;" ::: "memory");
#endif
}

template <typename... KArgs, typename... Args>
cudaError_t gm_launch_pdl(void (*kern)(KArgs...), dim3 grid, dim3 block, size_t smem,
                          cudaStream_t s, Args &&...args) {
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = grid;
    cfg.blockDim = block;
    cfg.dynamicSmemBytes = smem;
    cfg.stream = s;
    cudaLaunchAttribute attr[1];
    attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    attr[0].val.programmaticStreamSerializationAllowed = GM_PDL ? 1 : 0;
    cfg.attrs = attr;
    cfg.numAttrs = 1;
    return cudaLaunchKernelEx(&cfg, kern, std::forward<Args>(args)...);
}

__device__ __forceinline__ double warp_sum(double v) {
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
    return v;
}

// Warp sums of N2 values at once (N2 a power of two <= 32): each butterfly
// level first halves the values a lane carries -- the lane keeps one half,
// sends the other to its partner -- so the whole reduction moves
// N2 - 1 + 5 - log2(N2) values instead of 5 N2.  Returns the full sum of
// value `idx`; every lane of the idx group holds the same bits.
template <int N2>
__device__ __forceinline__ double warp_sum_split(double (&v)[N2], int lane, int &idx) {
    static_assert(N2 >= 1 && N2 <= 32 && (N2 & (N2 - 1)) == 0, "N2: power of two <= 32");
    idx = 0;
    int o = 16;
#pragma unroll
    for (int h = N2 / 2; h >= 1; h >>= 1, o >>= 1) {
        const bool up = (lane & o) != 0;
#pragma unroll
        for (int k = 0; k < h; k++) {
            const double send = up ? v[k] : v[h + k];
            const double keep = up ? v[h + k] : v[k];
            v[k] = keep + __shfl_xor_sync(0xffffffffu, send, o);
        }
        if (up) idx += h;
    }
    double s = v[0];
#pragma unroll
    for (; o > 0; o >>= 1) s += __shfl_xor_sync(0xffffffffu, s, o);
    return s;
}

// floor(a / b) for 0 <= a < 64, 1 <= b <= 64 without an integer divide:
// (a + 0.5) / b is at least 1/128 away from an integer.
__device__ __forceinline__ int small_div(int a, float inv_b) {
    return (int)(((float)a + 0.5f) * inv_b);
}

// Resident CTAs per SM x SM count for a persistent launch (cached per device,
// kernel, block size and dynamic shared memory size); 0 on failure.
int gm_persistent_blocks(const void *func, int threads, size_t smem);

// ---------------------------------------------------------------------------
// host-side implementation entry points (used by abi.cu)
// ---------------------------------------------------------------------------
gm_status prepare_impl(const gm_params *p, const gm_batch *b, const Workspace &ws,
                       cudaStream_t s, bool items_too);
gm_status prepare_inline_impl(const gm_params *p, const gm_batch *b, const Workspace &ws,
                              const double *origins, const double *xforms, cudaStream_t s);
// *launched: whether a kernel was launched (an empty job table launches none)
gm_status forward_impl(const gm_params *p, const gm_batch *b, const Workspace &ws, float *out,
                       cudaStream_t s, bool *launched = nullptr);
int32_t forward_jobs_impl(const gm_params *p, int32_t nex, int32_t nch, const int32_t *chan_off,
                          int32_t *jobs, int32_t cap);
gm_status backward_impl(const gm_params *p, const gm_batch *b, const Workspace &ws,
                        const float *grid_grad, float *coord_grad, float *type_grad,
                        cudaStream_t s, bool early_prologue = false,
                        double *coord_grad64 = nullptr, double *type_grad64 = nullptr);
