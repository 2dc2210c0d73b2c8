// prepare.cu -- fused Transform, item records and per-channel binning.
//
//   k_prepare_atoms  geom.py:99-112 in numpy's FMA order -> f64 positions
//   k_prepare_items  _kernels.py:22-30 boxes, grid-local hi/lo coordinates,
//                    density constants (_kernels.py:81-85)
//   k_bin            per example: stable grouping of items by output channel, so
//                    each forward CTA reads only its channel's items, in order
#include "common.cuh"

struct PrepArgs {
    gm_params p;
    gm_batch b;
    Workspace ws;
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

// geom.py:105: x' = ((x - c) @ R.T + c) + t in float64.  Without a transform
// the float32 input is widened exactly (voxelizer.py:366).
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
            const double d[3] = {__dsub_rn(x[0], X[9]), __dsub_rn(x[1], X[10]),
                                 __dsub_rn(x[2], X[11])};
#pragma unroll
            for (int j = 0; j < 3; j++)
                x[j] = __dadd_rn(__dadd_rn(dot3(d, X + 3 * j, order), X[9 + j]), X[12 + j]);
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
        // _kernels.py:55/74 (index), 144/167 (vector): cut = r (binary) or r * rmult
        const double cut = p.binary ? r : __dmul_rn(r, rmult);
        int i0, i1, j0, j1, k0, k1;
        axis_bounds(x, cut, ox, res, D, i0, i1);
        axis_bounds(y, cut, oy, res, D, j0, j1);
        axis_bounds(z, cut, oz, res, D, k0, k1);
        const bool valid = i0 <= i1 && j0 <= j1 && k0 <= k1;
        FwdItem f;
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
        f.qa = (float)(exp((-2.0 * grm) * grm) * (q0 * q0));
        f.w = w;
        f.ch = ch;
        f.ibox = i0 | (i1 << 16);
        f.jbox = j0 | (j1 << 16);
        f.kbox = k0 | (k1 << 16);
        f.atom = a;
        A.ws.items[it] = f;
        if (p.binary) A.ws.bitems[it] = BinItem{x, y, z, __dmul_rn(r, r)};
        A.ws.item_ch[it] = valid ? ch : -1;
    }
}

// One CTA (32 warps) per example.  Warp w owns channels w, w+32, ...: it
// counts, then (after a CTA-wide scan) copies its channel's items in item
// order with a ballot compaction -- a stable partition by channel, so the
// forward keeps the reference's per-voxel accumulation order.
struct BinArgs {
    const FwdItem *items;
    const BinItem *bitems;
    const int32_t *item_ch;
    const int32_t *ex_item_start, *ex_item_end;
    FwdItem *sorted;
    BinItem *bsorted;
    int2 *sbox;
    int32_t *chan_off;
    int C;
    int binary;
};

__global__ void __launch_bounds__(1024) k_bin(const BinArgs A) {
    // smem: C+1 channel offsets, then per item its channel and its rank
    // among the example's earlier items of the same channel
    extern __shared__ int sh[];
    int *cnt = sh;
    int *chs = sh + A.C + 1;
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5, nw = blockDim.x >> 5;
    const int e = blockIdx.x;
    const int is = A.ex_item_start[e], ie = A.ex_item_end[e];
    const int n = ie - is;
    int *rank = chs + n;
    const unsigned lt = (1u << lane) - 1u;
    for (int q = threadIdx.x; q < n; q += blockDim.x) chs[q] = A.item_ch[is + q];
    __syncthreads();
    // warp w ranks the items of channels w, w+32, ... (ordered ballot scan)
    for (int c = warp; c < A.C; c += nw) {
        int k = 0;
        for (int base = 0; base < n; base += 32) {
            const int q = base + lane;
            const bool mine = q < n && chs[q] == c;
            const unsigned m = __ballot_sync(0xffffffffu, mine);
            if (mine) rank[q] = k + __popc(m & lt);
            k += __popc(m);
        }
        if (lane == 0) cnt[c] = k;
    }
    __syncthreads();
    if (threadIdx.x == 0) {
        int pos = is;
        int32_t *off = A.chan_off + (size_t)e * (A.C + 1);
        for (int c = 0; c < A.C; c++) {
            const int k = cnt[c];
            cnt[c] = pos;
            off[c] = pos;
            pos += k;
        }
        off[A.C] = pos;
    }
    __syncthreads();
    // all threads move records: 16-byte chunks, coalesced within a record
    for (int t = threadIdx.x; t < 4 * n; t += blockDim.x) {
        const int q = t >> 2, part = t & 3;
        const int c = chs[q];
        if (c < 0) continue;
        const int dst = cnt[c] + rank[q];
        const int4 v = reinterpret_cast<const int4 *>(A.items + is + q)[part];
        reinterpret_cast<int4 *>(A.sorted + dst)[part] = v;
        if (part == 3) A.sbox[dst] = make_int2(v.x, v.y);  // ibox, jbox
        if (A.binary && part < 2)
            reinterpret_cast<int4 *>(A.bsorted + dst)[part] =
                reinterpret_cast<const int4 *>(A.bitems + is + q)[part];
    }
}

gm_status prepare_impl(const gm_params *p, const gm_batch *b, const Workspace &ws,
                       cudaStream_t s, bool items_too) {
    PrepArgs A;
    A.p = *p;
    A.b = *b;
    A.ws = ws;
    if (b->natoms > 0) {
        const int blocks = std::min((b->natoms + 255) / 256, 148 * 16);
        k_prepare_atoms<<<blocks, 256, 0, s>>>(A);
        LAUNCH_CHECK();
    }
    if (!items_too) return GM_OK;
    if (b->nitems > 0) {
        const int blocks = std::min((b->nitems + 255) / 256, 148 * 16);
        k_prepare_items<<<blocks, 256, 0, s>>>(A);
        LAUNCH_CHECK();
    }
    if (b->nexamples > 0) {
        BinArgs B;
        B.items = ws.items;
        B.bitems = ws.bitems;
        B.item_ch = ws.item_ch;
        B.ex_item_start = b->ex_item_start;
        B.ex_item_end = b->ex_item_end;
        B.sorted = ws.sorted;
        B.bsorted = ws.bsorted;
        B.sbox = ws.sbox;
        B.chan_off = ws.chan_off;
        B.C = b->nchannels;
        B.binary = p->binary;
        if (b->max_example_items < 0) return gm_fail(GM_ERR_INVALID, "max_example_items < 0");
        const size_t smem = sizeof(int) * (size_t)(b->nchannels + 1 + 2 * b->max_example_items);
        if (smem > 200 * 1024)
            return gm_fail(GM_ERR_INVALID, "too many items per example (%d)", b->max_example_items);
        if (smem > 48 * 1024) CUDA_TRY(gm_ensure_smem((const void *)k_bin, (int)smem));
        k_bin<<<b->nexamples, 1024, smem, s>>>(B);
        LAUNCH_CHECK();
    }
    return GM_OK;
}
