// assemble.cu -- index-mode batches assembled on the device from a resident
// dataset (gm_assemble, include/gridmaker_b200.h).
//
// Reference: GridMaker._run_batch packs every call on the host
// (/root/reference/pkg/src/voxmol/voxelizer.py:372-435: CSR concatenation of
// the sets, radii * radius_scale in f64, per-set channel offsets) behind
// ExampleProvider.next_batch (sampling.py:364-380).  Here the examples live in
// HBM already grouped by channel (the grouping of a batch is the
// concatenation of its examples' groupings), so a batch is an index list:
// CTAs per (batch example, 256-atom chunk) copy its 32-B atom records into the packed
// arrays the prepare pass reads (slot records in channel order, atoms in set
// order), writes its set rows, channel offsets and nonzero-channel list.  The
// forward job table follows on the device (forward.cu: k_job_build).  Batch
// sizes come from the dataset's host mirrors: no sync.
#include <algorithm>
#include <cstring>
#include <type_traits>

#include "common.cuh"

namespace {

// gm_dataset.records entry
struct __align__(16) DsAtom {
    float x, y, z, r;  // input-frame coordinates, unscaled radius
    int atom;          // local atom index (set order)
    int ch;            // absolute channel within the example
    int brank;         // local backward launch rank
    int set_single;    // local set index | single-atom-set flag << 16
};
static_assert(sizeof(DsAtom) == 32, "DsAtom must be 32 bytes");

// gm_batch.slot_rec entry (packing.py _SLOT_DTYPE, prepare.cu SlotRec)
struct __align__(16) SlotOut {
    float x, y, z;
    int atom, ch, ex, single, bslot;
    double r, pad;
};
static_assert(sizeof(SlotOut) == 48, "SlotOut must be 48 bytes");

// CAP: examples the launch parameters hold (8, 64 or GM_INLINE_MAX_EXAMPLES):
// the smallest that fits, so small batches launch with small parameter blocks
template <int CAP>
struct AsmArgs {
    gm_dataset ds;
    gm_batch b;
    double scale;
    int n;
    int4 ex[CAP];  // per batch example: id, atom base, set base, seg base
};

// grid (batch example, atom chunk of kAsmChunk): chunk 0 also writes the
// example's set rows, channel offsets and nonzero-channel list
constexpr int kAsmChunk = 256;

template <int CAP>
__global__ void __launch_bounds__(256) k_assemble(const __grid_constant__ AsmArgs<CAP> A) {
    const int bi = blockIdx.x, tid = threadIdx.x;
    const int q0 = blockIdx.y * kAsmChunk;
    const int4 X = A.ex[bi];
    const int id = X.x, abase = X.y, sbase = X.z, gbase = X.w;
    const gm_dataset &ds = A.ds;
    const gm_batch &b = A.b;
    const int C = ds.nchannels;
    const int a0 = ds.ex_atom_off[id], na = ds.ex_atom_off[id + 1] - a0;
    const int s0 = ds.ex_set_off[id], ns = ds.ex_set_off[id + 1] - s0;
    if (q0 >= na && blockIdx.y > 0) return;
    if (blockIdx.y == 0) {
        // set rows (voxelizer.py:388-395 layout)
        for (int t = tid; t < ns; t += blockDim.x) {
            const int st = abase + ds.set_aoff[s0 + t];
            int32_t *w = const_cast<int32_t *>(b.set_start);
            w[sbase + t] = st;
            const_cast<int32_t *>(b.set_end)[sbase + t] = st + ds.set_natoms[s0 + t];
            const_cast<int32_t *>(b.set_example)[sbase + t] = bi;
            const_cast<int32_t *>(b.set_choff)[sbase + t] = ds.set_choff[s0 + t];
            const_cast<int32_t *>(b.set_t)[sbase + t] = ds.set_t[s0 + t];
        }
        if (tid == 0) {
            const_cast<int32_t *>(b.ex_item_start)[bi] = abase;
            const_cast<int32_t *>(b.ex_item_end)[bi] = abase + na;
        }
        // channel offsets and the groups with items (gm_batch.segs, ascending)
        const int32_t *lco = ds.ex_chan_off + (size_t)id * (C + 1);
        for (int c = tid; c <= C; c += blockDim.x)
            const_cast<int32_t *>(b.chan_off)[(size_t)bi * (C + 1) + c] = abase + lco[c];
        if (tid < 32) {
            int carry = 0;
            for (int c0 = 0; c0 < C; c0 += 32) {
                const int c = c0 + tid;
                const bool nz = c < C && lco[c + 1] > lco[c];
                const unsigned m = __ballot_sync(0xffffffffu, nz);
                if (nz)
                    const_cast<int32_t *>(b.segs)[gbase + carry + __popc(m & ((1u << tid) - 1u))] =
                        bi * C + c;
                carry += __popc(m);
            }
        }
    }  // chunk 0
    // atoms: slot records in channel order, per-atom arrays in set order
    const DsAtom *rec = reinterpret_cast<const DsAtom *>(ds.records) + a0;
    SlotOut *slot = reinterpret_cast<SlotOut *>(const_cast<void *>(b.slot_rec)) + abase;
    for (int q = q0 + tid; q < min(na, q0 + kAsmChunk); q += blockDim.x) {
        const DsAtom R = rec[q];
        const int a = abase + R.atom;
        const int sl = R.set_single & 0xffff;
        const double r = __dmul_rn((double)R.r, A.scale);  // voxelizer.py:430
        SlotOut o;
        o.x = R.x;
        o.y = R.y;
        o.z = R.z;
        o.atom = a;
        o.ch = R.ch;
        o.ex = bi;
        o.single = R.set_single >> 16;
        o.bslot = abase + R.brank;
        o.r = r;
        o.pad = 0.0;
        slot[q] = o;
        const_cast<int32_t *>(b.item_perm)[abase + q] = a;
        float *c32 = const_cast<float *>(b.coords32);
        c32[3 * a + 0] = R.x;
        c32[3 * a + 1] = R.y;
        c32[3 * a + 2] = R.z;
        const_cast<double *>(b.atom_radius)[a] = r;
        const_cast<int32_t *>(b.atom_set)[a] = sbase + sl;
        const_cast<int32_t *>(b.atom_type)[a] = R.ch - ds.set_choff[s0 + sl];
        const_cast<int32_t *>(b.bwd_slot)[a] = abase + R.brank;
    }
}

// Vector typing: grid (batch example, chunk); chunk y covers atoms and items
// [256 y, 256 (y+1)) and weights [4096 y, 4096 (y+1)) of the example.
struct __align__(16) DsItem {
    int atom;   // local atom (set order)
    int ch;     // channel within the set
    float w;    // weight
    int gpos;   // slot in the example's channel grouping
};
static_assert(sizeof(DsItem) == 16, "DsItem must be 16 bytes");

template <int CAP>
struct VAsmArgs {
    gm_dataset ds;
    gm_batch b;
    double scale;
    int rti;
    int n;
    int4 ex[CAP];   // id, atom base, set base, seg base
    int4 ex2[CAP];  // item base, weight base, type-radius base, -
};

template <int CAP>
__global__ void __launch_bounds__(256) k_assemble_vector(const __grid_constant__ VAsmArgs<CAP> A) {
    const int bi = blockIdx.x, tid = threadIdx.x, y = blockIdx.y;
    const int4 X = A.ex[bi], X2 = A.ex2[bi];
    const int id = X.x, abase = X.y, sbase = X.z, gbase = X.w;
    const int ibase = X2.x, wbase = X2.y, tbase = X2.z;
    const gm_dataset &ds = A.ds;
    const gm_batch &b = A.b;
    const int C = ds.nchannels;
    const int a0 = ds.ex_atom_off[id], na = ds.ex_atom_off[id + 1] - a0;
    const int s0 = ds.ex_set_off[id], ns = ds.ex_set_off[id + 1] - s0;
    const int i0 = ds.ex_item_off[id], ni = ds.ex_item_off[id + 1] - i0;
    const int w0 = ds.ex_w_off[id], nw = ds.ex_w_off[id + 1] - w0;
    const int t0 = ds.ex_tr_off[id], nt = ds.ex_tr_off[id + 1] - t0;
    if (y == 0) {
        for (int t = tid; t < ns; t += blockDim.x) {
            const int st = abase + ds.set_aoff[s0 + t];
            const_cast<int32_t *>(b.set_start)[sbase + t] = st;
            const_cast<int32_t *>(b.set_end)[sbase + t] = st + ds.set_natoms[s0 + t];
            const_cast<int32_t *>(b.set_example)[sbase + t] = bi;
            const_cast<int32_t *>(b.set_choff)[sbase + t] = ds.set_choff[s0 + t];
            const_cast<int32_t *>(b.set_t)[sbase + t] = ds.set_t[s0 + t];
            const_cast<int32_t *>(b.set_wstart)[sbase + t] = wbase + ds.set_woff[s0 + t];
            const_cast<int32_t *>(b.set_trstart)[sbase + t] = tbase + ds.set_troff[s0 + t];
        }
        if (tid == 0) {
            const_cast<int32_t *>(b.ex_item_start)[bi] = ibase;
            const_cast<int32_t *>(b.ex_item_end)[bi] = ibase + ni;
        }
        const int32_t *lco = ds.ex_chan_off + (size_t)id * (C + 1);
        for (int c = tid; c <= C; c += blockDim.x)
            const_cast<int32_t *>(b.chan_off)[(size_t)bi * (C + 1) + c] = ibase + lco[c];
        if (tid < 32) {
            int carry = 0;
            for (int c0 = 0; c0 < C; c0 += 32) {
                const int c = c0 + tid;
                const bool nz = c < C && lco[c + 1] > lco[c];
                const unsigned m = __ballot_sync(0xffffffffu, nz);
                if (nz)
                    const_cast<int32_t *>(b.segs)[gbase + carry + __popc(m & ((1u << tid) - 1u))] =
                        bi * C + c;
                carry += __popc(m);
            }
        }
        // type radii (voxelizer.py:318: f32 -> f64 times radius_scale; ones when
        // radii are per atom, as the reference's packing fills them)
        for (int t = tid; t < nt; t += blockDim.x) {
            int sl = 0;  // the entry's set (an example has a few sets)
            while (sl + 1 < ns && ds.set_troff[s0 + sl + 1] <= t) sl++;
            const bool own = A.rti && ds.set_natoms[s0 + sl] > 0;
            const_cast<double *>(b.type_radius)[tbase + t] =
                own ? __dmul_rn((double)ds.type_radii[t0 + t], A.scale) : 1.0;
        }
    }
    const DsAtom *rec = reinterpret_cast<const DsAtom *>(ds.records) + a0;
    for (int q = y * kAsmChunk + tid; q < min(na, (y + 1) * kAsmChunk); q += blockDim.x) {
        const DsAtom R = rec[q];
        const int a = abase + q;
        float *c32 = const_cast<float *>(b.coords32);
        c32[3 * a + 0] = R.x;
        c32[3 * a + 1] = R.y;
        c32[3 * a + 2] = R.z;
        const_cast<double *>(b.atom_radius)[a] = __dmul_rn((double)R.r, A.scale);
        const_cast<int32_t *>(b.atom_set)[a] = sbase + (R.set_single & 0xffff);
        const_cast<int32_t *>(b.bwd_slot)[a] = abase + R.brank;
    }
    const DsItem *it = reinterpret_cast<const DsItem *>(ds.items) + i0;
    for (int q = y * kAsmChunk + tid; q < min(ni, (y + 1) * kAsmChunk); q += blockDim.x) {
        const DsItem I = it[q];
        const int a = abase + I.atom;
        const_cast<int32_t *>(b.item_atom)[ibase + q] = a;
        const_cast<int32_t *>(b.item_channel)[ibase + q] = I.ch;
        const_cast<float *>(b.item_weight)[ibase + q] = I.w;
        const int sl = rec[I.atom].set_single & 0xffff;
        const double r = A.rti ? __dmul_rn((double)ds.type_radii[t0 + ds.set_troff[s0 + sl] + I.ch], A.scale)
                               : __dmul_rn((double)rec[I.atom].r, A.scale);
        const_cast<double *>(b.item_radius)[ibase + q] = r;
        const_cast<int32_t *>(b.item_perm)[ibase + I.gpos] = ibase + q;
    }
    const float *ws = ds.weights + w0;
    for (int q = y * (16 * kAsmChunk) + tid; q < min(nw, (y + 1) * (16 * kAsmChunk)); q += blockDim.x)
        const_cast<float *>(b.weights)[wbase + q] = ws[q];
}

}  // namespace

long long forward_job_count(int D, long long work_groups, long long zero_groups);
gm_status forward_jobs_device(const gm_params *p, int nex, int nch, const int32_t *chan_off,
                              int32_t *jobs, long long work_groups, long long zero_groups,
                              int4 *stats, cudaStream_t s);

gm_status assemble_impl(const gm_params *p, const gm_dataset *ds, const int32_t *ids, int32_t n,
                        gm_batch *b, const gm_capacity *cap, int32_t *jobs, cudaStream_t s) {
    if (n < 1 || n > GM_INLINE_MAX_EXAMPLES)
        return gm_fail(GM_ERR_INVALID, "batch of %d examples (1..%d)", n, GM_INLINE_MAX_EXAMPLES);
    const int C = ds->nchannels;
    const bool vec = ds->vector_mode != 0;
    long long natoms = 0, nsets = 0, nsegs = 0, nitems = 0, nw = 0, ntr = 0;
    int maxa = 0, maxi = 0, maxw = 0, maxseg = 0;
    int4 ex[GM_INLINE_MAX_EXAMPLES], ex2[GM_INLINE_MAX_EXAMPLES];
    for (int i = 0; i < n; i++) {
        const int id = ids[i];
        if (id < 0 || id >= ds->nexamples)
            return gm_fail(GM_ERR_INVALID, "example id %d out of range [0, %d)", id, ds->nexamples);
        const int na = ds->h_ex_atom_off[id + 1] - ds->h_ex_atom_off[id];
        const int ni = vec ? ds->h_ex_item_off[id + 1] - ds->h_ex_item_off[id] : na;
        const int nwt = vec ? ds->h_ex_w_off[id + 1] - ds->h_ex_w_off[id] : 0;
        ex[i] = make_int4(id, (int)natoms, (int)nsets, (int)nsegs);
        ex2[i] = make_int4((int)nitems, (int)nw, (int)ntr, 0);
        natoms += na;
        nitems += ni;
        nw += nwt;
        if (vec) ntr += ds->h_ex_tr_off[id + 1] - ds->h_ex_tr_off[id];
        nsets += ds->h_ex_set_off[id + 1] - ds->h_ex_set_off[id];
        nsegs += ds->h_ex_nzch[id];
        maxa = std::max(maxa, na);
        maxi = std::max(maxi, ni);
        maxw = std::max(maxw, nwt);
        maxseg = std::max(maxseg, ds->h_ex_maxch[id]);
    }
    if (natoms > cap->atoms || nsets > cap->sets || (vec && (nitems > cap->items ||
                                                             nw > cap->weights || ntr > cap->type_radii)))
        return gm_fail(GM_ERR_INVALID,
                       "batch needs %lld atoms / %lld sets / %lld items / %lld weights / %lld type "
                       "radii, capacity %d / %d / %d / %d / %d",
                       natoms, nsets, nitems, nw, ntr, cap->atoms, cap->sets, cap->items,
                       cap->weights, cap->type_radii);
    const long long G = (long long)n * C;
    const long long njobs = forward_job_count(p->npts, nsegs, G - nsegs);
    if (njobs + 2 * G > cap->jobs)
        return gm_fail(GM_ERR_INVALID, "job table needs %lld + %lld scratch entries, capacity %d",
                       njobs, 2 * G, cap->jobs);
    b->nexamples = n;
    b->nsets = (int32_t)nsets;
    b->natoms = (int32_t)natoms;
    b->nitems = (int32_t)nitems;
    b->nweights = (int32_t)nw;
    b->nchannels = C;
    b->vector_mode = vec ? 1 : 0;
    b->max_example_items = vec ? maxi : maxa;
    b->nsegs = (int32_t)nsegs;
    b->max_seg_items = maxseg;
    b->fwd_jobs = jobs;
    b->nfwd_jobs = (int32_t)njobs;
    b->fwd_jobs_npts = p->npts;
    const int chunks_idx = std::max(1, (maxa + kAsmChunk - 1) / kAsmChunk);
    const int chunks_vec = std::max(std::max((maxa + kAsmChunk - 1) / kAsmChunk,
                                             (maxi + kAsmChunk - 1) / kAsmChunk),
                                    std::max(1, (maxw + 16 * kAsmChunk - 1) / (16 * kAsmChunk)));
    auto launch = [&](auto capc) {
        constexpr int CAP = decltype(capc)::value;
        if (vec) {
            VAsmArgs<CAP> V;
            V.ds = *ds;
            V.b = *b;
            V.scale = p->radius_scale;
            V.rti = p->radius_type_indexed ? 1 : 0;
            V.n = n;
            memcpy(V.ex, ex, sizeof(int4) * n);
            memcpy(V.ex2, ex2, sizeof(int4) * n);
            k_assemble_vector<CAP><<<dim3(n, (unsigned)std::max(1, chunks_vec)), 256, 0, s>>>(V);
        } else {
            AsmArgs<CAP> A;
            A.ds = *ds;
            A.scale = p->radius_scale;
            A.n = n;
            memcpy(A.ex, ex, sizeof(int4) * n);
            A.b = *b;
            k_assemble<CAP><<<dim3(n, (unsigned)chunks_idx), 256, 0, s>>>(A);
        }
    };
    if (n <= 8) launch(std::integral_constant<int, 8>{});
    else if (n <= 64) launch(std::integral_constant<int, 64>{});
    else launch(std::integral_constant<int, GM_INLINE_MAX_EXAMPLES>{});
    LAUNCH_CHECK();
    return forward_jobs_device(p, n, C, b->chan_off, jobs, nsegs, G - nsegs,
                               reinterpret_cast<int4 *>(jobs + 4 * njobs), s);
}
