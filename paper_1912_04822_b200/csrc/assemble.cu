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
// forward job table follows on the device (forward.cu: k_job_stats /
// k_job_place).  Batch sizes come from the dataset's host mirrors: no sync.
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

struct AsmArgs {
    gm_dataset ds;
    gm_batch b;
    double scale;
    int n;
    int4 ex[GM_INLINE_MAX_EXAMPLES];  // per batch example: id, atom base, set base, seg base
};

// grid (batch example, atom chunk of kAsmChunk): chunk 0 also writes the
// example's set rows, channel offsets and nonzero-channel list
constexpr int kAsmChunk = 256;

__global__ void __launch_bounds__(256) k_assemble(const __grid_constant__ AsmArgs A) {
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

}  // namespace

long long forward_job_count(int D, long long work_groups, long long zero_groups);
gm_status forward_jobs_device(const gm_params *p, int nex, int nch, const int32_t *chan_off,
                              int32_t *jobs, long long work_groups, long long zero_groups,
                              int4 *stats, cudaStream_t s);

gm_status assemble_impl(const gm_params *p, const gm_dataset *ds, const int32_t *ids, int32_t n,
                        gm_batch *b, int32_t atom_capacity, int32_t set_capacity, int32_t *jobs,
                        int32_t jobs_capacity, cudaStream_t s) {
    if (n < 1 || n > GM_INLINE_MAX_EXAMPLES)
        return gm_fail(GM_ERR_INVALID, "batch of %d examples (1..%d)", n, GM_INLINE_MAX_EXAMPLES);
    const int C = ds->nchannels;
    AsmArgs A;
    A.ds = *ds;
    A.scale = p->radius_scale;
    A.n = n;
    long long natoms = 0, nsets = 0, nsegs = 0;
    int maxex = 0, maxseg = 0;
    for (int i = 0; i < n; i++) {
        const int id = ids[i];
        if (id < 0 || id >= ds->nexamples)
            return gm_fail(GM_ERR_INVALID, "example id %d out of range [0, %d)", id, ds->nexamples);
        const int na = ds->h_ex_atom_off[id + 1] - ds->h_ex_atom_off[id];
        A.ex[i] = make_int4(id, (int)natoms, (int)nsets, (int)nsegs);
        natoms += na;
        nsets += ds->h_ex_set_off[id + 1] - ds->h_ex_set_off[id];
        nsegs += ds->h_ex_nzch[id];
        maxex = std::max(maxex, na);
        maxseg = std::max(maxseg, ds->h_ex_maxch[id]);
    }
    if (natoms > atom_capacity || nsets > set_capacity)
        return gm_fail(GM_ERR_INVALID, "batch needs %lld atoms / %lld sets, capacity %d / %d",
                       natoms, nsets, atom_capacity, set_capacity);
    const long long G = (long long)n * C;
    const long long njobs = forward_job_count(p->npts, nsegs, G - nsegs);
    if (njobs + 2 * G > jobs_capacity)
        return gm_fail(GM_ERR_INVALID, "job table needs %lld + %lld scratch entries, capacity %d",
                       njobs, 2 * G, jobs_capacity);
    b->nexamples = n;
    b->nsets = (int32_t)nsets;
    b->natoms = (int32_t)natoms;
    b->nitems = (int32_t)natoms;
    b->nchannels = C;
    b->vector_mode = 0;
    b->max_example_items = maxex;
    b->nsegs = (int32_t)nsegs;
    b->max_seg_items = maxseg;
    b->fwd_jobs = jobs;
    b->nfwd_jobs = (int32_t)njobs;
    b->fwd_jobs_npts = p->npts;
    A.b = *b;
    k_assemble<<<dim3(n, (unsigned)std::max(1, (maxex + kAsmChunk - 1) / kAsmChunk)), 256, 0, s>>>(A);
    LAUNCH_CHECK();
    return forward_jobs_device(p, n, C, b->chan_off, jobs, nsegs, G - nsegs,
                               reinterpret_cast<int4 *>(jobs + 4 * njobs), s);
}
