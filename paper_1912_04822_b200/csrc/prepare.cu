// prepare.cu -- fused Transform, item records and per-channel binning.
//
//   k_prepare_example  one CTA per example: geom.py:99-112 in numpy's FMA order
//                      -> f64 positions; _kernels.py:22-30 boxes, grid-local
//                      hi/lo coordinates, density constants (_kernels.py:81-85);
//                      stable grouping of the items by output channel, so each
//                      forward CTA reads only its channel's items, in order
//   k_prepare_static   batches packed with a static grouping (gm_batch.item_perm):
//                      the same records in one fully parallel pass, per-call
//                      arrays inside the launch (gm_prepare_inline) or read
//                      from the batch's device buffers (gm_prepare, graphs)
//   k_prepare_atoms    positions only (backward without a forward)
#include <string.h>

#include "common.cuh"

#ifndef GM_PREP_STATIC_DEV
#define GM_PREP_STATIC_DEV 1  // gm_prepare on a statically grouped batch: k_prepare_static<DEV>
#endif
#ifndef GM_SORT_SIZED
#define GM_SORT_SIZED 1  // plane-sort CTA size from gm_batch.max_seg_items
#endif
#ifndef GM_PREP_THREADS
#define GM_PREP_THREADS 64  // small blocks: the ~50k item threads spread over every SM
#endif

struct PrepArgs;
gm_status sort_planes(const PrepArgs &A, cudaStream_t s);

// per-channel plane sort (k_sort_planes): CTA sizes 64 / 128 / 256 threads,
// each sorting up to kSortRounds items per thread in shared memory
constexpr int kSortThreads = 256;  // the largest variant
constexpr int kSortRounds = 4;

struct PrepArgs {
    gm_params p;
    gm_batch b;
    Workspace ws;
    double eg;  // exp(-2 grm^2), the tail's constant factor (host libm)
};

// One output coordinate of (x - c) @ R.T, the 3-term dot product evaluated in
// the FMA order numpy/BLAS uses on the host (codes: geom.matmul_order).
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

// geom.py:105: x' = ((x - c) @ R.T + c) + t in float64, X = the example's
// transform (R row-major, center, translation) or NULL.  Without a transform
// the float32 input is widened exactly (voxelizer.py:366).
__device__ __forceinline__ void transform_atom_x(const PrepArgs &A, int a, int s, const double *X,
                                                 double x[3]) {
    const gm_batch &b = A.b;
    if (b.coords64) {
        x[0] = b.coords64[3 * a + 0];
        x[1] = b.coords64[3 * a + 1];
        x[2] = b.coords64[3 * a + 2];
    } else {
        x[0] = (double)b.coords32[3 * a + 0];
        x[1] = (double)b.coords32[3 * a + 1];
        x[2] = (double)b.coords32[3 * a + 2];
    }
    if (X) {
        const int nset = b.set_end[s] - b.set_start[s];
        const int order = nset == 1 ? A.p.matmul_order_1 : A.p.matmul_order_n;
        const double d[3] = {__dsub_rn(x[0], X[9]), __dsub_rn(x[1], X[10]),
                             __dsub_rn(x[2], X[11])};
#pragma unroll
        for (int j = 0; j < 3; j++)
            x[j] = __dadd_rn(__dadd_rn(dot3(d, X + 3 * j, order), X[9 + j]), X[12 + j]);
    }
}

__device__ __forceinline__ void transform_atom(const PrepArgs &A, int a, double x[3]) {
    const gm_batch &b = A.b;
    const int s = b.atom_set[a];
    const double *X = b.xforms ? b.xforms + 15 * (size_t)b.set_example[s] : nullptr;
    transform_atom_x(A, a, s, X, x);
}

__device__ __forceinline__ void store_pos(const PrepArgs &A, int a, const double x[3]) {
    A.ws.pos[3 * a + 0] = x[0];
    A.ws.pos[3 * a + 1] = x[1];
    A.ws.pos[3 * a + 2] = x[2];
}

// Vector mode: the backward's per-atom record at its launch slot.
__device__ __forceinline__ void store_vbwd_atom(const PrepArgs &A, int a, int s, int e,
                                                const double *O, const double x[3], int slot) {
    const gm_batch &b = A.b;
    if (!b.set_wstart) return;  // no weight rows: the batch has no vector backward
    VBwdAtom v;
    v.x = x[0];
    v.y = x[1];
    v.z = x[2];
    v.ox = O[0];
    v.oy = O[1];
    v.oz = O[2];
    v.r = b.atom_radius[a];
    v.atom = a;
    v.slab = e * b.nchannels + b.set_choff[s];
    v.T = b.set_t[s];
    v.row = b.set_wstart[s] + (a - b.set_start[s]) * v.T;
    v.set = s;
    v.pad = 0;
    A.ws.vbatoms[slot] = v;
}

// Positions only (the vector-mode backward needs every atom, with or without
// items).
__global__ void __launch_bounds__(256) k_prepare_atoms(const PrepArgs A) {
    for (int a = blockIdx.x * blockDim.x + threadIdx.x; a < A.b.natoms;
         a += gridDim.x * blockDim.x) {
        double x[3];
        transform_atom(A, a, x);
        store_pos(A, a, x);
        if (A.b.vector_mode) {
            const int slot = A.b.bwd_slot ? A.b.bwd_slot[a] : a;
            if (A.b.bwd_slot) A.ws.atom_order[slot] = a;
            const int st = A.b.atom_set[a], ex = A.b.set_example[st];
            store_vbwd_atom(A, a, st, ex, A.b.origins + 3 * (size_t)ex, x, slot);
        }
    }
}

__device__ __forceinline__ void split_hilo(double v, float &hi, float &lo) {
    hi = (float)v;
    lo = (float)(v - (double)hi);
}

// The forward record of item `it` (atom a at transformed position x):
// _kernels.py:22-30 boxes, grid-local hi/lo corner offsets, density constants
// (_kernels.py:81-85).  Returns its channel, or -1 when the box misses the grid.
__device__ __forceinline__ int make_item_o(const PrepArgs &A, int it, int a, int s,
                                           const double *O, const double x3[3], FwdItem &f,
                                           BinItem &bi) {
    const gm_batch &b = A.b;
    const gm_params &p = A.p;
    const int D = p.npts;
    const double res = p.resolution, grm = p.gaussian_radius_multiple, rmult = p.radius_multiple;
    const int ch = b.set_choff[s] + (b.item_channel ? b.item_channel[it] : b.atom_type[a]);
    const double r = b.item_radius ? b.item_radius[it] : b.atom_radius[a];
    const float w = b.item_weight ? b.item_weight[it] : 1.0f;
    const double x = x3[0], y = x3[1], z = x3[2];
    const double ox = O[0], oy = O[1], oz = O[2];
    // _kernels.py:55/74 (index), 144/167 (vector): cut = r (binary) or r * rmult
    const double cut = p.binary ? r : __dmul_rn(r, rmult);
    int i0, i1, j0, j1, k0, k1;
    axis_bounds(x, cut, ox, res, D, i0, i1);
    axis_bounds(y, cut, oy, res, D, j0, j1);
    axis_bounds(z, cut, oz, res, D, k0, k1);
    const bool valid = i0 <= i1 && j0 <= j1 && k0 <= k1;
    // offsets (o + lo*res) - x of the box-corner voxel, as hi + lo floats
    split_hilo((double)i0 * res - (x - ox), f.cxh, f.cxl);
    split_hilo((double)j0 * res - (y - oy), f.cyh, f.cyl);
    split_hilo((double)k0 * res - (z - oz), f.czh, f.czl);
    const double r2 = r * r;
    f.cexp = (float)((-2.0 * CUDART_L2E) / r2);
    const double gr = grm * r;
    f.d02 = (float)(gr * gr);
    f.dzr = (float)cut;
    const double q0 = (2.0 * grm) / r;
    f.qa = (float)(A.eg * (q0 * q0));
    f.w = w;
    f.ch = ch;
    f.ibox = i0 | (i1 << 16);
    f.jbox = j0 | (j1 << 16);
    f.kbox = k0 | (k1 << 16);
    f.atom = a;
    bi = BinItem{x, y, z, __dmul_rn(r, r)};
    return valid ? ch : -1;
}

// Index mode: the backward's per-atom record (same box as the forward item,
// _kernels.py:225-227; constants of _kernels.py:224-251).
__device__ __forceinline__ void store_bwd_atom(const PrepArgs &A, int a, int e, int ch,
                                               const double *O, const double x[3],
                                               const FwdItem &f) {
    const double r = A.b.atom_radius[a];
    const double grm = A.p.gaussian_radius_multiple;
    BwdAtom w;
    w.lx = x[0] - O[0];
    w.ly = x[1] - O[1];
    w.lz = x[2] - O[2];
    w.dzr = A.p.radius_multiple * r;
    w.dzr2 = w.dzr * w.dzr;
    const double d0 = grm * r;
    w.d02 = d0 * d0;
    const double q0 = (2.0 * grm) / r;
    w.qa2 = 2.0 * (A.eg * (q0 * q0));
    w.m4inv_r2 = -4.0 / (r * r);
    w.m2inv_r2 = 0.5 * w.m4inv_r2;
    w.atom = a;
    w.pad = 0;
    w.slab = e * A.b.nchannels + ch;
    w.ibox = f.ibox;
    w.jbox = f.jbox;
    w.kbox = f.kbox;
    A.ws.batoms[A.b.bwd_slot ? A.b.bwd_slot[a] : a] = w;
}

__device__ __forceinline__ int make_item(const PrepArgs &A, int it, int a, const double x3[3],
                                         FwdItem &f, BinItem &bi) {
    const int s = A.b.atom_set[a];
    return make_item_o(A, it, a, s, A.b.origins + 3 * (size_t)A.b.set_example[s], x3, f, bi);
}

// ---------------------------------------------------------------------------
// Static grouping (gm_batch.item_perm / chan_off, computed when the batch is
// packed): one fully parallel pass, thread t <-> grouped slot t.  The per-call
// arrays (origins, transforms) travel inside the launch (kernel parameters,
// up to CAP examples): no separate host->device copy.  Items whose box misses
// the grid stay in their channel's range with an empty box (ibox lo > hi), so
// the forward's cull and the backward's box test skip them.
// ---------------------------------------------------------------------------
// Index mode, static grouping: everything the prepare pass needs about the
// item in slot t, gathered once at pack time (gm_batch.slot_rec), so the
// pass starts from ONE coalesced load instead of three dependent ones
// (item_perm -> atom arrays -> set arrays).
struct __align__(16) SlotRec {
    float x, y, z;    // input-frame coordinates (coords32)
    int atom;         // packed atom index
    int ch;           // absolute output channel (set_choff + type)
    int ex;           // example
    int single;       // 1: the atom's set has one atom (numpy's (1,3)@(3,3) FMA order)
    int bslot;        // backward launch slot (gm_batch.bwd_slot, else atom)
    double r;         // radius * radius_scale
    double pad;
};
static_assert(sizeof(SlotRec) == 48, "SlotRec must be 48 bytes");

template <int CAP>
struct CallArgs {
    int nex, has_xf;
    double v[18 * CAP];  // origins (nex,3), then transforms (nex,15)
};

// Everything the prepare pass does for grouped slot t (static grouping):
// transform (geom.py:105), forward record + binary record (returned), and in
// index mode the position and the backward record (stored).
// org: the call's origins (nex,3); xf: its transforms (nex,15) or null --
// launch parameters (inline path) or the batch's device buffers.
// Index mode with slot records: loads and arithmetic only (nothing is
// stored), so the pass can run this before its PDL wait -- while the previous
// kernel on the workspace drains -- and store afterwards (store_slot).
struct SlotOut {
    FwdItem f;
    BinItem bi;
    BwdAtom w;
    double x[3];
    int a, bslot;
};

__device__ __forceinline__ void compute_slot(const PrepArgs &A, const double *org,
                                             const double *xf, int t, SlotOut &o) {
    const gm_batch &b = A.b;
    FwdItem &f = o.f;
    {
        const SlotRec R = reinterpret_cast<const SlotRec *>(b.slot_rec)[t];
        const gm_params &p = A.p;
        const int D = p.npts, e = R.ex, a = R.atom;
        const double *X = xf ? xf + 15 * e : nullptr;
        const double *O = org + 3 * e;
        double x[3] = {(double)R.x, (double)R.y, (double)R.z};
        if (b.coords64) {  // positions given in f64 (host-transformed exact mode)
            x[0] = b.coords64[3 * a + 0];
            x[1] = b.coords64[3 * a + 1];
            x[2] = b.coords64[3 * a + 2];
        }
        if (X) {  // geom.py:105 in numpy's FMA order
            const double d[3] = {__dsub_rn(x[0], X[9]), __dsub_rn(x[1], X[10]),
                                 __dsub_rn(x[2], X[11])};
#pragma unroll
            for (int j = 0; j < 3; j++)
                x[j] = __dadd_rn(__dadd_rn(dot3(d, X + 3 * j, R.single ? p.matmul_order_1
                                                                            : p.matmul_order_n),
                                           X[9 + j]), X[12 + j]);
        }
        o.x[0] = x[0];
        o.x[1] = x[1];
        o.x[2] = x[2];
        o.a = a;
        o.bslot = R.bslot;
        const double res = p.resolution, grm = p.gaussian_radius_multiple, rmult = p.radius_multiple;
        const double r = R.r;
        const double cut = p.binary ? r : __dmul_rn(r, rmult);
        int i0, i1, j0, j1, k0, k1;
        axis_bounds(x[0], cut, O[0], res, D, i0, i1);
        axis_bounds(x[1], cut, O[1], res, D, j0, j1);
        axis_bounds(x[2], cut, O[2], res, D, k0, k1);
        const bool valid = i0 <= i1 && j0 <= j1 && k0 <= k1;
        split_hilo((double)i0 * res - (x[0] - O[0]), f.cxh, f.cxl);
        split_hilo((double)j0 * res - (x[1] - O[1]), f.cyh, f.cyl);
        split_hilo((double)k0 * res - (x[2] - O[2]), f.czh, f.czl);
        const double r2 = r * r;
        f.cexp = (float)((-2.0 * CUDART_L2E) / r2);
        const double gr = grm * r;
        f.d02 = (float)(gr * gr);
        f.dzr = (float)cut;
        const double q0 = (2.0 * grm) / r;
        const double qa = A.eg * (q0 * q0);
        f.qa = (float)qa;
        f.w = 1.0f;
        f.ch = R.ch;
        f.ibox = valid ? (i0 | (i1 << 16)) : 0x7fff;  // empty: the forward skips it
        f.jbox = j0 | (j1 << 16);
        f.kbox = k0 | (k1 << 16);
        f.atom = a;
        o.bi = BinItem{x[0], x[1], x[2], __dmul_rn(r, r)};
        // the backward's record (_kernels.py:224-251 constants, same box)
        BwdAtom &w = o.w;
        w.lx = x[0] - O[0];
        w.ly = x[1] - O[1];
        w.lz = x[2] - O[2];
        w.dzr = rmult * r;
        w.dzr2 = w.dzr * w.dzr;
        const double d0 = grm * r;
        w.d02 = d0 * d0;
        w.qa2 = 2.0 * qa;
        w.m4inv_r2 = -4.0 / (r * r);
        w.m2inv_r2 = 0.5 * w.m4inv_r2;
        w.atom = a;
        w.pad = 0;
        w.slab = e * b.nchannels + R.ch;
        w.ibox = f.ibox;
        w.jbox = f.jbox;
        w.kbox = f.kbox;
    }
}

__device__ __forceinline__ void store_slot(const PrepArgs &A, int t, const SlotOut &o) {
    store_pos(A, o.a, o.x);
    A.ws.batoms[o.bslot] = o.w;
    A.ws.sorted[t] = o.f;
    A.ws.sbox[t] = make_int2(o.f.ibox, o.f.jbox);
    if (A.p.binary) A.ws.bsorted[t] = o.bi;
}

// Everything the prepare pass does for grouped slot t without slot records
// (vector typing, or batches packed without them): loads, arithmetic and the
// position / backward-record stores; the forward records are returned.
__device__ __forceinline__ void build_slot(const PrepArgs &A, const double *org,
                                           const double *xf, int t, FwdItem &f, BinItem &bi) {
    const gm_batch &b = A.b;
    const bool vector = b.item_atom != nullptr;
    {
        const int it = b.item_perm[t];
        const int a = vector ? b.item_atom[it] : it;
        const int s = b.atom_set[a];
        const int e = b.set_example[s];
        double x[3];
        transform_atom_x(A, a, s, xf ? xf + 15 * e : nullptr, x);
        if (!vector) store_pos(A, a, x);
        if (make_item_o(A, it, a, s, org + 3 * e, x, f, bi) < 0) f.ibox = 0x7fff;  // empty
        if (!vector) store_bwd_atom(A, a, e, f.ch, org + 3 * e, x, f);
    }
}


// DEV: the call's origins / transforms are already in the batch's device
// buffers (b.origins / b.xforms: gm_prepare, CUDA-graph replays); otherwise
// they travel in K and the origins are copied out for forward / backward.
template <int CAP, bool DEV>
__global__ void __launch_bounds__(GM_PREP_THREADS) k_prepare_static(const PrepArgs A, const __grid_constant__ CallArgs<CAP> K) {
    const gm_batch &b = A.b;
    const int t = blockIdx.x * blockDim.x + threadIdx.x;
    const int nex = b.nexamples;
    const bool vector = b.item_atom != nullptr;
    const double *org = DEV ? b.origins : K.v;
    const double *xf = DEV ? b.xforms : (K.has_xf ? K.v + 3 * nex : nullptr);
    // Index mode with slot records: the slot's loads and arithmetic run before
    // the PDL wait (they read only the batch's inputs, which no kernel of ours
    // writes), overlapping the tail of the previous kernel on this workspace
    const bool early = !vector && b.slot_rec && t < b.nitems;
    SlotOut o;
    if (early) compute_slot(A, org, xf, t, o);
    // PDL: the previous kernel (a backward reading this workspace) must be
    // done before anything is written; then the forward may launch
    pdl_wait();
    pdl_trigger();
    if (early) store_slot(A, t, o);
    if (!DEV && t < 3 * nex) const_cast<double *>(b.origins)[t] = K.v[t];  // for forward / backward
    if (t < nex * (b.nchannels + 1)) A.ws.chan_off[t] = b.chan_off[t];
    if (vector && t < b.natoms) {  // positions of all atoms
        const int s = b.atom_set[t];
        const int e = b.set_example[s];
        double x[3];
        transform_atom_x(A, t, s, xf ? xf + 15 * e : nullptr, x);
        store_pos(A, t, x);
        const int slot = b.bwd_slot ? b.bwd_slot[t] : t;
        if (b.bwd_slot) A.ws.atom_order[slot] = t;  // vector backward launch order
        store_vbwd_atom(A, t, s, e, org + 3 * e, x, slot);
    }
    if (!early && t < b.nitems) {
        FwdItem f;
        BinItem bi;
        build_slot(A, org, xf, t, f, bi);
        A.ws.sorted[t] = f;
        A.ws.sbox[t] = make_int2(f.ibox, f.jbox);
        if (A.p.binary) A.ws.bsorted[t] = bi;
    }
}

template <int CAP>
gm_status launch_static(const PrepArgs &A, const double *origins, const double *xforms,
                        cudaStream_t s) {
    CallArgs<CAP> K;
    const int nex = A.b.nexamples;
    K.nex = nex;
    K.has_xf = xforms != nullptr;
    memcpy(K.v, origins, sizeof(double) * 3 * nex);
    if (xforms) memcpy(K.v + 3 * nex, xforms, sizeof(double) * 15 * nex);
    const int n = std::max(std::max(A.b.nitems, A.b.natoms),
                           std::max(3 * nex, nex * (A.b.nchannels + 1)));
    if (n > 0) {
        CUDA_TRY(gm_launch_pdl(k_prepare_static<CAP, false>,
                               dim3((n + GM_PREP_THREADS - 1) / GM_PREP_THREADS),
                               dim3(GM_PREP_THREADS), 0, s, A, K));
        LAUNCH_CHECK();
    }
    return use_plane_sort(&A.p, &A.b) ? sort_planes(A, s) : GM_OK;
}

// Static grouping, per-call arrays already on the device (b.origins / b.xforms).
static gm_status launch_static_dev(const PrepArgs &A, cudaStream_t s) {
    CallArgs<1> K;
    K.nex = A.b.nexamples;
    K.has_xf = A.b.xforms != nullptr;
    K.v[0] = 0.0;
    const int nex = A.b.nexamples;
    const int n = std::max(std::max(A.b.nitems, A.b.natoms), nex * (A.b.nchannels + 1));
    if (n > 0) {
        CUDA_TRY(gm_launch_pdl(k_prepare_static<1, true>,
                               dim3((n + GM_PREP_THREADS - 1) / GM_PREP_THREADS),
                               dim3(GM_PREP_THREADS), 0, s, A, K));
        LAUNCH_CHECK();
    }
    return use_plane_sort(&A.p, &A.b) ? sort_planes(A, s) : GM_OK;
}

// One CTA per example, in phases separated by CTA barriers:
//   1. one thread per item: transform its atom (geom.py:105), build its record
//      (staged in shared memory, or in the workspace when the example is too
//      big) and note its channel (-1: box misses the grid);
//   2. one warp per chunk of 32 items: rank each item among the chunk's items
//      of its channel (match.any), chunk x channel counts into a table;
//   3. per channel, exclusive scan of the table over chunks; channel offsets;
//   4. move every record to offset + chunk prefix + rank: a stable partition by
//      channel, so the forward keeps the reference's per-voxel accumulation
//      order while each forward CTA reads only its channel.
template <bool SMEM_STAGE>
__global__ void __launch_bounds__(1024) k_prepare_example(const PrepArgs A) {
    extern __shared__ __align__(16) unsigned char smraw[];
    const gm_batch &b = A.b;
    const int C = b.nchannels;
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5, nw = blockDim.x >> 5;
    const int e = blockIdx.x;
    const int is = b.ex_item_start[e];
    const int n = b.ex_item_end[e] - is;
    const int nchunk = (n + 31) >> 5;
    const bool binary = A.p.binary;
    const bool vector = b.item_atom != nullptr;
    unsigned char *p = smraw;
    FwdItem *stage = A.ws.items + is;
    BinItem *bstage = A.ws.bitems + is;
    if (SMEM_STAGE) {
        stage = reinterpret_cast<FwdItem *>(p);
        p += sizeof(FwdItem) * n;
        if (binary) {
            bstage = reinterpret_cast<BinItem *>(p);
            p += sizeof(BinItem) * n;
        }
    }
    int *chs = reinterpret_cast<int *>(p);
    int *rank = chs + n;
    int *tab = rank + n;  // [nchunk][C]
    int *off = tab + nchunk * C;
    for (int t = threadIdx.x; t < nchunk * C; t += blockDim.x) tab[t] = 0;
    if (vector) {  // positions of all atoms (items only see atoms that have weights)
        for (int a = blockIdx.x * blockDim.x + threadIdx.x; a < b.natoms;
             a += gridDim.x * blockDim.x) {
            double x[3];
            transform_atom(A, a, x);
            store_pos(A, a, x);
            const int slot = b.bwd_slot ? b.bwd_slot[a] : a;
            if (b.bwd_slot) A.ws.atom_order[slot] = a;
            const int st = b.atom_set[a], ex = b.set_example[st];
            store_vbwd_atom(A, a, st, ex, b.origins + 3 * (size_t)ex, x, slot);
        }
    }
    for (int q = threadIdx.x; q < n; q += blockDim.x) {
        const int it = is + q;
        const int a = vector ? b.item_atom[it] : it;
        double x[3];
        transform_atom(A, a, x);
        if (!vector) store_pos(A, a, x);
        FwdItem f;
        BinItem bi;
        chs[q] = make_item(A, it, a, x, f, bi);
        if (!vector) {
            FwdItem g = f;
            if (chs[q] < 0) g.ibox = 0x7fff;
            const int s = b.atom_set[a];
            const int ex = b.set_example[s];
            store_bwd_atom(A, a, ex, f.ch, b.origins + 3 * (size_t)ex, x, g);
        }
        A.ws.items[it] = f;  // packed order: the index-mode backward reads its boxes
        if (SMEM_STAGE) stage[q] = f;
        if (binary) bstage[q] = bi;
    }
    __syncthreads();
    const unsigned lt = (1u << lane) - 1u;
    for (int k = warp; k < nchunk; k += nw) {
        const int q = k * 32 + lane;
        const int c = q < n ? chs[q] : -1;
        const unsigned m = __match_any_sync(0xffffffffu, c);
        if (c >= 0) {
            rank[q] = __popc(m & lt);
            if ((m & lt) == 0) tab[k * C + c] = __popc(m);
        }
    }
    __syncthreads();
    for (int c = threadIdx.x; c < C; c += blockDim.x) {
        int s = 0;
        for (int k = 0; k < nchunk; k++) {
            const int v = tab[k * C + c];
            tab[k * C + c] = s;
            s += v;
        }
        off[c] = s;
    }
    __syncthreads();
    if (warp == 0) {
        // channel offsets: exclusive scan of the counts, 32 channels per pass
        int32_t *co = A.ws.chan_off + (size_t)e * (C + 1);
        int pos = is;
        for (int c0 = 0; c0 < C; c0 += 32) {
            const int c = c0 + lane;
            const int k = c < C ? off[c] : 0;
            int sc = k;
#pragma unroll
            for (int o = 1; o < 32; o <<= 1) {
                const int t = __shfl_up_sync(0xffffffffu, sc, o);
                if (lane >= o) sc += t;
            }
            __syncwarp();
            if (c < C) {
                off[c] = pos + sc - k;
                co[c] = pos + sc - k;
            }
            pos += __shfl_sync(0xffffffffu, sc, 31);
        }
        if (lane == 0) co[C] = pos;
    }
    __syncthreads();
    // 16-byte chunks, coalesced within a record
    for (int t = threadIdx.x; t < 4 * n; t += blockDim.x) {
        const int q = t >> 2, part = t & 3;
        const int c = chs[q];
        if (c < 0) continue;
        const int dst = off[c] + tab[(q >> 5) * C + c] + rank[q];
        const int4 v = reinterpret_cast<const int4 *>(stage + q)[part];
        reinterpret_cast<int4 *>(A.ws.sorted + dst)[part] = v;
        if (part == 3) A.ws.sbox[dst] = make_int2(v.x, v.y);  // ibox, jbox
        if (binary && part < 2)
            reinterpret_cast<int4 *>(A.ws.bsorted + dst)[part] =
                reinterpret_cast<const int4 *>(bstage + q)[part];
    }
}

// ---------------------------------------------------------------------------
// Per (example, channel) stable counting sort of the grouped items by the
// plane bucket of their box's first plane (k_forward then scans, for plane i,
// only the items whose first plane lies within the widest box of plane i --
// instead of every item of the channel).  One CTA per (example, channel);
// ranks within 32-item chunks from match.any, chunk x bucket prefix tables in
// shared memory; the order is (bucket, item order): deterministic.
// ---------------------------------------------------------------------------

template <bool SEGS, int NT>
__global__ void __launch_bounds__(NT) k_sort_planes(const PrepArgs A) {
    constexpr int kSortThreads = NT, kSortMax = NT * kSortRounds;  // this variant
    pdl_wait();
    pdl_trigger();
    __shared__ int tab[(kSortMax / 32) * (kBuckets + 1)];  // chunk x bucket prefix
    __shared__ int off[kBuckets + 2];
    __shared__ int wmax_s;
    const gm_batch &b = A.b;
    const int C = b.nchannels, D = A.p.npts;
    // one CTA per (example, channel) -- or per group with items when the
    // batch lists them (gm_batch.segs; the others are zero tiles)
    const int seg = SEGS ? b.segs[blockIdx.x] : blockIdx.x, e = seg / C, c = seg - e * C;
    const int cs = A.ws.chan_off[(size_t)e * (C + 1) + c], ce = A.ws.chan_off[(size_t)e * (C + 1) + c + 1];
    const int n = ce - cs;
    int32_t *rec = A.ws.poff + (size_t)seg * kPlaneRec;
    const int tid = threadIdx.x, lane = tid & 31;
    if (n <= 0) {
        for (int t = tid; t < kPlaneRec; t += kSortThreads) rec[t] = 0;
        return;
    }
    const bool binary = A.p.binary;
    const bool sortable = n <= kSortMax;
    if (tid == 0) wmax_s = 0;
    const int nchunk = (n + 31) >> 5;
    if (sortable)
        for (int t = tid; t < nchunk * (kBuckets + 1); t += kSortThreads) tab[t] = 0;
    __syncthreads();
    // item q = tid + round * kSortThreads: chunks of 32 consecutive items are
    // one warp's lanes in one round
    int key[kSortRounds], rank[kSortRounds];
    int2 bx[kSortRounds];
    int wloc = 0;
    // every round's boxes in flight at once
#pragma unroll
    for (int r = 0; r < kSortRounds; r++) {
        const int q = tid + r * kSortThreads;
        bx[r] = make_int2(0x7fff, 0);
        if (sortable && q < n) bx[r] = A.ws.sbox[cs + q];
    }
#pragma unroll
    for (int r = 0; r < kSortRounds; r++) {
        const int q = tid + r * kSortThreads;
        key[r] = kBuckets + 1;
        rank[r] = 0;
        if (!sortable || r * kSortThreads >= n) continue;  // warp-uniform
        if (q < n) {
            const int lo = box_lo(bx[r].x), hi = box_hi(bx[r].x);
            key[r] = lo <= hi && lo < D ? plane_bucket(lo, D) : kBuckets;
            if (key[r] < kBuckets) wloc = max(wloc, hi - lo + 1);
        }
        const unsigned m = __match_any_sync(0xffffffffu, key[r]);
        rank[r] = __popc(m & ((1u << lane) - 1u));
        if (q < n && rank[r] == 0) tab[(q >> 5) * (kBuckets + 1) + key[r]] = __popc(m);
    }
    if (!sortable)
        for (int q = tid; q < n; q += kSortThreads) {
            const int ib = A.ws.sbox[cs + q].x;
            if (box_lo(ib) <= box_hi(ib)) wloc = max(wloc, box_hi(ib) - box_lo(ib) + 1);
        }
    atomicMax(&wmax_s, wloc);
    __syncthreads();
    if (sortable) {
        // per bucket: exclusive prefix over the chunks
        for (int t = tid; t <= kBuckets; t += kSortThreads) {
            int run = 0;
            for (int k = 0; k < nchunk; k++) {
                const int v = tab[k * (kBuckets + 1) + t];
                tab[k * (kBuckets + 1) + t] = run;
                run += v;
            }
            off[t] = run;  // bucket count, scanned below
        }
        __syncthreads();
        if (tid < 32) {
            // exclusive scan of the kBuckets + 1 counts, 32 per pass
            int carry = 0;
            for (int b0 = 0; b0 <= kBuckets; b0 += 32) {
                const int bk = b0 + lane;
                const int v = bk <= kBuckets ? off[bk] : 0;
                int sc = v;
#pragma unroll
                for (int o = 1; o < 32; o <<= 1) {
                    const int t = __shfl_up_sync(0xffffffffu, sc, o);
                    if (lane >= o) sc += t;
                }
                if (bk <= kBuckets) off[bk] = carry + sc - v;
                carry += __shfl_sync(0xffffffffu, sc, 31);
            }
            if (lane == 0) off[kBuckets + 1] = carry;
        }
        __syncthreads();
        // all records of the thread loaded before any is stored
        int4 rv[kSortRounds][4];
#pragma unroll
        for (int r = 0; r < kSortRounds; r++) {
            const int q = tid + r * kSortThreads;
            if (q < n) {
                const int4 *src4 = reinterpret_cast<const int4 *>(A.ws.sorted + cs + q);
#pragma unroll
                for (int w4 = 0; w4 < 4; w4++) rv[r][w4] = src4[w4];
            }
        }
#pragma unroll
        for (int r = 0; r < kSortRounds; r++) {
            const int q = tid + r * kSortThreads;
            if (q >= n) continue;
            const int dst = cs + off[key[r]] + tab[(q >> 5) * (kBuckets + 1) + key[r]] + rank[r];
            int4 *dst4 = reinterpret_cast<int4 *>(A.ws.psorted + dst);
#pragma unroll
            for (int w4 = 0; w4 < 4; w4++) dst4[w4] = rv[r][w4];
            A.ws.psbox[dst] = bx[r];
            if (binary) A.ws.pbsorted[dst] = A.ws.bsorted[cs + q];
        }
    } else {
        for (int q = tid; q < n; q += kSortThreads) {  // unsorted: a plain copy
            const int4 *src4 = reinterpret_cast<const int4 *>(A.ws.sorted + cs + q);
            int4 *dst4 = reinterpret_cast<int4 *>(A.ws.psorted + cs + q);
#pragma unroll
            for (int w4 = 0; w4 < 4; w4++) dst4[w4] = src4[w4];
            A.ws.psbox[cs + q] = A.ws.sbox[cs + q];
            if (binary) A.ws.pbsorted[cs + q] = A.ws.bsorted[cs + q];
        }
    }
    for (int t = tid; t <= kBuckets + 1; t += kSortThreads)
        rec[t] = sortable ? off[t] : (t == 0 ? 0 : n);
    if (tid == 0) rec[kBuckets + 2] = sortable ? wmax_s : D;  // unsorted: scan everything
}

template <int NT>
static gm_status sort_planes_nt(const PrepArgs &A, cudaStream_t s) {
    const int nseg = A.b.nexamples * A.b.nchannels;
    if (A.b.segs) {
        if (A.b.nsegs > 0)
            CUDA_TRY(gm_launch_pdl(k_sort_planes<true, NT>, dim3(A.b.nsegs), dim3(NT), 0, s, A));
    } else if (nseg > 0) {
        CUDA_TRY(gm_launch_pdl(k_sort_planes<false, NT>, dim3(nseg), dim3(NT), 0, s, A));
    }
    LAUNCH_CHECK();
    return GM_OK;
}

// The smallest CTA that sorts the largest group in shared memory (all groups
// resident in about one wave); unknown sizes take the largest.
gm_status sort_planes(const PrepArgs &A, cudaStream_t s) {
    const int m = A.b.max_seg_items;
    if (GM_SORT_SIZED && m > 0 && m <= 64 * kSortRounds) return sort_planes_nt<64>(A, s);
    if (GM_SORT_SIZED && m > 0 && m <= 128 * kSortRounds) return sort_planes_nt<128>(A, s);
    return sort_planes_nt<kSortThreads>(A, s);
}

gm_status prepare_impl(const gm_params *p, const gm_batch *b, const Workspace &ws,
                       cudaStream_t s, bool items_too) {
    PrepArgs A;
    A.p = *p;
    A.b = *b;
    A.ws = ws;
    A.eg = exp((-2.0 * p->gaussian_radius_multiple) * p->gaussian_radius_multiple);
    if (!items_too || b->nexamples == 0) {
        if (b->natoms > 0) {
            const int blocks = std::min((b->natoms + 255) / 256, 148 * 16);
            k_prepare_atoms<<<blocks, 256, 0, s>>>(A);
            LAUNCH_CHECK();
        }
        return GM_OK;
    }
    if (b->item_perm && b->chan_off && GM_PREP_STATIC_DEV) return launch_static_dev(A, s);
    if (b->max_example_items < 0) return gm_fail(GM_ERR_INVALID, "max_example_items < 0");
    const size_t n = (size_t)b->max_example_items, nchunk = (n + 31) / 32;
    const size_t base = sizeof(int) * (2 * n + nchunk * b->nchannels + b->nchannels + 1);
    const size_t staged = base + n * (sizeof(FwdItem) + (p->binary ? sizeof(BinItem) : 0));
    const size_t limit = 200 * 1024;
    if (base > limit)
        return gm_fail(GM_ERR_INVALID, "too many items per example (%d)", b->max_example_items);
    if (staged <= limit) {
        if (staged > 48 * 1024) CUDA_TRY(gm_ensure_smem((const void *)k_prepare_example<true>, (int)staged));
        k_prepare_example<true><<<b->nexamples, 1024, staged, s>>>(A);
    } else {
        if (base > 48 * 1024) CUDA_TRY(gm_ensure_smem((const void *)k_prepare_example<false>, (int)base));
        k_prepare_example<false><<<b->nexamples, 1024, base, s>>>(A);
    }
    LAUNCH_CHECK();
    return use_plane_sort(&A.p, &A.b) ? sort_planes(A, s) : GM_OK;
}

// Per-call arrays from host memory (see gm_prepare_inline).
gm_status prepare_inline_impl(const gm_params *p, const gm_batch *b, const Workspace &ws,
                              const double *origins, const double *xforms, cudaStream_t s) {
    PrepArgs A;
    A.p = *p;
    A.b = *b;
    A.ws = ws;
    A.eg = exp((-2.0 * p->gaussian_radius_multiple) * p->gaussian_radius_multiple);
    const int nex = b->nexamples;
    if (nex <= 8) return launch_static<8>(A, origins, xforms, s);
    if (nex <= 64) return launch_static<64>(A, origins, xforms, s);
    return launch_static<GM_INLINE_MAX_EXAMPLES>(A, origins, xforms, s);
}
