// pack.cu -- host packing of an index-typed batch (gm_pack_index_host).
//
// The packing of GridMaker._run_batch
// (/root/reference/pkg/src/voxmol/voxelizer.py:372-435: sets concatenated in
// example / set order, radii widened to f64 and scaled, per-set channel
// offsets) plus what this library adds to a packed batch -- the static
// grouping (items of each example in (channel, atom) order and the channel
// offsets), the groups with items, the per-slot records the prepare pass
// starts from and the backward launch order -- in one native pass written
// straight into the caller's (pinned) image of the batch.  Same arrays as the
// numpy packing in packing.py, byte for byte except the launch order (a
// permutation that only affects speed).  Host code only.
#include <algorithm>
#include <cmath>
#include <cstring>
#include <vector>

#include "common.cuh"

namespace {

// gm_batch.slot_rec entry (prepare.cu SlotRec)
struct PackSlot {
    float x, y, z;
    int32_t atom, ch, ex, single, bslot;
    double r, pad;
};
static_assert(sizeof(PackSlot) == 48, "PackSlot must be 48 bytes");

template <typename T>
T *at(uint8_t *dst, int64_t off) {
    return off < 0 ? nullptr : reinterpret_cast<T *>(dst + off);
}

// Stable LSD radix sort of idx by 64-bit keys, 16 bits per pass (as many
// passes as the largest key needs).
void radix_sort(std::vector<uint64_t> &key, std::vector<int32_t> &idx) {
    const size_t n = idx.size();
    uint64_t kmax = 0;
    for (uint64_t k : key) kmax = k > kmax ? k : kmax;
    std::vector<uint64_t> k2(n);
    std::vector<int32_t> i2(n);
    std::vector<uint32_t> cnt(65537);
    for (int shift = 0; shift < 64 && (kmax >> shift) != 0; shift += 16) {
        std::fill(cnt.begin(), cnt.end(), 0u);
        for (size_t q = 0; q < n; q++) cnt[((key[q] >> shift) & 0xffff) + 1]++;
        for (int d = 0; d < 65536; d++) cnt[d + 1] += cnt[d];
        for (size_t q = 0; q < n; q++) {
            const uint32_t p = cnt[(key[q] >> shift) & 0xffff]++;
            k2[p] = key[q];
            i2[p] = idx[q];
        }
        key.swap(k2);
        idx.swap(i2);
    }
}

}  // namespace

extern "C" gm_status gm_pack_index_host(const gm_pack_set *sets, int32_t nsets, int32_t nexamples,
                                        int32_t nchannels, double radius_scale,
                                        const double *centers, int32_t bwd_order, uint8_t *dst,
                                        const gm_pack_layout *L, gm_pack_info *info) {
    if (nsets < 0 || nexamples < 0 || nchannels < 0)
        return gm_fail(GM_ERR_INVALID, "negative batch size");
    if ((nsets > 0 && !sets) || !dst || !L || !info || (nexamples > 0 && !centers))
        return gm_fail(GM_ERR_INVALID, "NULL argument");
    const int64_t C = nchannels > 0 ? nchannels : 1;
    // sets: example order, channel offsets, atom counts
    std::vector<int32_t> choff(nsets);
    int64_t natoms = 0;
    for (int32_t s = 0; s < nsets; s++) {
        const gm_pack_set &S = sets[s];
        if (S.example < 0 || S.example >= nexamples || (s > 0 && S.example < sets[s - 1].example))
            return gm_fail(GM_ERR_INVALID, "set %d: example %d out of order", s, S.example);
        if (S.n < 0 || S.num_types < 0 || (S.n > 0 && (!S.coords || !S.radii || !S.type_index)))
            return gm_fail(GM_ERR_INVALID, "set %d: bad arrays", s);
        choff[s] = (s > 0 && sets[s - 1].example == S.example)
                       ? choff[s - 1] + sets[s - 1].num_types : 0;
        if (choff[s] + S.num_types > nchannels)
            return gm_fail(GM_ERR_INVALID, "set %d: channels %d..%d beyond %d", s, choff[s],
                           choff[s] + S.num_types, nchannels);
        natoms += S.n;
    }
    if (natoms > 0x7fffffffLL) return gm_fail(GM_ERR_INVALID, "too many atoms (%lld)", natoms);
    const int32_t A = (int32_t)natoms;
    float *coords32 = at<float>(dst, L->coords32);
    double *radius = at<double>(dst, L->atom_radius);
    int32_t *atom_set = at<int32_t>(dst, L->atom_set), *atom_type = at<int32_t>(dst, L->atom_type);
    int32_t *set_start = at<int32_t>(dst, L->set_start), *set_end = at<int32_t>(dst, L->set_end);
    int32_t *set_ex = at<int32_t>(dst, L->set_example), *set_co = at<int32_t>(dst, L->set_choff);
    int32_t *set_t = at<int32_t>(dst, L->set_t);
    int32_t *ex_start = at<int32_t>(dst, L->ex_item_start), *ex_end = at<int32_t>(dst, L->ex_item_end);
    int32_t *perm = at<int32_t>(dst, L->item_perm), *chan_off = at<int32_t>(dst, L->chan_off);
    int32_t *segs = at<int32_t>(dst, L->segs), *bslot = at<int32_t>(dst, L->bwd_slot);
    PackSlot *rec = at<PackSlot>(dst, L->slot_rec);
    if (!coords32 || !radius || !atom_set || !atom_type || !set_start || !set_end || !set_ex ||
        !set_co || !set_t || !ex_start || !ex_end || !perm || !chan_off || !segs ||
        (A > 0 && !rec))
        return gm_fail(GM_ERR_INVALID, "layout is missing arrays");

    // atoms and sets (voxelizer.py:410-430)
    std::vector<int64_t> chan(A);
    std::vector<int32_t> aex(A);
    std::memset(ex_start, 0, sizeof(int32_t) * nexamples);
    std::memset(ex_end, 0, sizeof(int32_t) * nexamples);
    int32_t a = 0;
    for (int32_t s = 0; s < nsets; s++) {
        const gm_pack_set &S = sets[s];
        const int32_t n = (int32_t)S.n, e = S.example;
        set_start[s] = a;
        set_end[s] = a + n;
        set_ex[s] = e;
        set_co[s] = choff[s];
        set_t[s] = S.num_types;
        if (s == 0 || sets[s - 1].example != e) ex_start[e] = a;
        ex_end[e] = a + n;
        if (n) std::memcpy(coords32 + 3 * (size_t)a, S.coords, sizeof(float) * 3 * (size_t)n);
        for (int32_t k = 0; k < n; k++, a++) {
            const int64_t t = S.type_index[k];
            if (t < 0 || t >= S.num_types)
                return gm_fail(GM_ERR_INVALID, "set %d atom %d: type %lld outside [0, %d)", s, k,
                               (long long)t, S.num_types);
            radius[a] = (double)S.radii[k] * radius_scale;
            atom_set[a] = s;
            atom_type[a] = (int32_t)t;
            chan[a] = choff[s] + t;
            aex[a] = e;
        }
    }
    int32_t max_ex = 0;
    for (int32_t e = 0; e < nexamples; e++) max_ex = std::max(max_ex, ex_end[e] - ex_start[e]);

    // static grouping: stable counting sort by (example, channel)
    const int64_t G = (int64_t)nexamples * C;
    std::vector<int32_t> gcount(G + 1, 0);
    for (int32_t q = 0; q < A; q++) gcount[aex[q] * C + chan[q] + 1]++;
    for (int64_t g = 0; g < G; g++) gcount[g + 1] += gcount[g];
    {
        std::vector<int32_t> pos(gcount.begin(), gcount.end() - 1);
        for (int32_t q = 0; q < A; q++) perm[pos[aex[q] * C + chan[q]]++] = q;
    }
    int32_t nsegs = 0, max_seg = 0;
    for (int32_t e = 0; e < nexamples; e++)
        for (int32_t c = 0; c <= nchannels; c++) {
            const int64_t g = (int64_t)e * C + c;
            chan_off[(int64_t)e * (nchannels + 1) + c] = gcount[std::min(g, G)];
            if (c < nchannels) {
                const int32_t k = gcount[g + 1] - gcount[g];
                if (k > 0) segs[nsegs++] = (int32_t)g;
                max_seg = std::max(max_seg, k);
            }
        }

    // backward launch order (packing._bwd_slots "slab"): atoms of one
    // (example, channel) grid_grad slab together, nearest the example's
    // center first within it (1/16 A steps)
    std::vector<int32_t> slot;
    if (bwd_order && bslot && A > 0) {
        std::vector<uint64_t> key(A);
        std::vector<int32_t> idx(A);
        for (int32_t q = 0; q < A; q++) {
            const double *c = centers + 3 * aex[q];
            const float dx = coords32[3 * q + 0] - (float)c[0];
            const float dy = coords32[3 * q + 1] - (float)c[1];
            const float dz = coords32[3 * q + 2] - (float)c[2];
            const float d = std::sqrt(dx * dx + dy * dy + dz * dz) * 16.0f;
            const uint64_t k16 = (uint64_t)std::min(d, 32767.0f);
            key[q] = ((uint64_t)(aex[q] * C + chan[q]) << 16) | k16;
            idx[q] = q;
        }
        radix_sort(key, idx);
        slot.resize(A);
        for (int32_t k = 0; k < A; k++) slot[idx[k]] = k;
        std::memcpy(bslot, slot.data(), sizeof(int32_t) * (size_t)A);
    }

    // per-slot records of the static grouping (item_perm order)
    for (int32_t k = 0; k < A; k++) {
        const int32_t q = perm[k], s = atom_set[q];
        PackSlot &R = rec[k];
        R.x = coords32[3 * q + 0];
        R.y = coords32[3 * q + 1];
        R.z = coords32[3 * q + 2];
        R.atom = q;
        R.ch = (int32_t)chan[q];
        R.ex = aex[q];
        R.single = sets[s].n == 1 ? 1 : 0;
        R.bslot = slot.empty() ? q : slot[q];
        R.r = radius[q];
        R.pad = 0.0;
    }
    info->natoms = A;
    info->nsegs = nsegs;
    info->max_seg_items = (nexamples > 0 && nchannels > 0) ? max_seg : 0;
    info->max_example_items = max_ex;
    return GM_OK;
}

// Vector typing (packing.PackedBatch's vector branch): atoms and sets as
// above, plus each set's weight rows and type radii, and one forward item per
// nonzero weight, atom-major then channel (_kernels.py:159-166), with its
// weight-row entry (item_windex, host side: autograd weight refresh).
extern "C" gm_status gm_pack_vector_host(const gm_pack_vset *sets, int32_t nsets, int32_t nexamples,
                                         int32_t nchannels, double radius_scale,
                                         int32_t radius_type_indexed, const double *centers,
                                         int32_t bwd_order, uint8_t *dst, const gm_pack_vlayout *L,
                                         int64_t *item_windex, gm_pack_info *info) {
    if (nsets < 0 || nexamples < 0 || nchannels < 0)
        return gm_fail(GM_ERR_INVALID, "negative batch size");
    if ((nsets > 0 && !sets) || !dst || !L || !info || (nexamples > 0 && !centers))
        return gm_fail(GM_ERR_INVALID, "NULL argument");
    const int64_t C = nchannels > 0 ? nchannels : 1;
    std::vector<int32_t> choff(nsets);
    int64_t natoms = 0, nitems = 0, nweights = 0, ntr = 0;
    for (int32_t s = 0; s < nsets; s++) {
        const gm_pack_vset &S = sets[s];
        if (S.example < 0 || S.example >= nexamples || (s > 0 && S.example < sets[s - 1].example))
            return gm_fail(GM_ERR_INVALID, "set %d: example %d out of order", s, S.example);
        if (S.n < 0 || S.num_types < 0 || (S.n > 0 && (!S.coords || !S.radii || !S.type_vector)))
            return gm_fail(GM_ERR_INVALID, "set %d: bad arrays", s);
        if (radius_type_indexed && S.n > 0 && !S.type_radii)
            return gm_fail(GM_ERR_INVALID, "set %d: type radii missing", s);
        choff[s] = (s > 0 && sets[s - 1].example == S.example)
                       ? choff[s - 1] + sets[s - 1].num_types : 0;
        if (choff[s] + S.num_types > nchannels)
            return gm_fail(GM_ERR_INVALID, "set %d: channels %d..%d beyond %d", s, choff[s],
                           choff[s] + S.num_types, nchannels);
        natoms += S.n;
        nweights += S.n * S.num_types;
        ntr += S.num_types;
        for (int64_t q = 0; q < S.n * S.num_types; q++) nitems += S.type_vector[q] != 0.0f;
    }
    if (natoms > 0x7fffffffLL || nitems > 0x7fffffffLL || nweights > 0x7fffffffLL)
        return gm_fail(GM_ERR_INVALID, "batch too large");
    const int32_t A = (int32_t)natoms, I = (int32_t)nitems;
    float *coords32 = at<float>(dst, L->coords32);
    double *radius = at<double>(dst, L->atom_radius);
    int32_t *atom_set = at<int32_t>(dst, L->atom_set);
    int32_t *set_start = at<int32_t>(dst, L->set_start), *set_end = at<int32_t>(dst, L->set_end);
    int32_t *set_ex = at<int32_t>(dst, L->set_example), *set_co = at<int32_t>(dst, L->set_choff);
    int32_t *set_t = at<int32_t>(dst, L->set_t), *set_w = at<int32_t>(dst, L->set_wstart);
    int32_t *set_tr = at<int32_t>(dst, L->set_trstart);
    float *weights = at<float>(dst, L->weights);
    double *type_radius = at<double>(dst, L->type_radius);
    int32_t *it_atom = at<int32_t>(dst, L->item_atom), *it_ch = at<int32_t>(dst, L->item_channel);
    float *it_w = at<float>(dst, L->item_weight);
    double *it_r = at<double>(dst, L->item_radius);
    int32_t *ex_start = at<int32_t>(dst, L->ex_item_start), *ex_end = at<int32_t>(dst, L->ex_item_end);
    int32_t *perm = at<int32_t>(dst, L->item_perm), *chan_off = at<int32_t>(dst, L->chan_off);
    int32_t *segs = at<int32_t>(dst, L->segs), *bslot = at<int32_t>(dst, L->bwd_slot);
    if (!coords32 || !radius || !atom_set || !set_start || !set_end || !set_ex || !set_co ||
        !set_t || !set_w || !set_tr || !weights || !type_radius || !it_atom || !it_ch || !it_w ||
        !it_r || !ex_start || !ex_end || !perm || !chan_off || !segs || (I > 0 && !item_windex))
        return gm_fail(GM_ERR_INVALID, "layout is missing arrays");

    std::vector<int32_t> aex(A);
    std::vector<int64_t> ichan(I);  // absolute channel of each item
    std::vector<int32_t> iex(I);
    std::memset(ex_start, 0, sizeof(int32_t) * nexamples);
    std::memset(ex_end, 0, sizeof(int32_t) * nexamples);
    int32_t a = 0, ip = 0;
    int64_t wpos = 0, tpos = 0;
    for (int32_t s = 0; s < nsets; s++) {
        const gm_pack_vset &S = sets[s];
        const int32_t n = (int32_t)S.n, nt = S.num_types, e = S.example;
        set_start[s] = a;
        set_end[s] = a + n;
        set_ex[s] = e;
        set_co[s] = choff[s];
        set_t[s] = nt;
        set_w[s] = (int32_t)wpos;
        set_tr[s] = (int32_t)tpos;
        if (s == 0 || sets[s - 1].example != e) ex_start[e] = ip;
        // type radii (scaled) when type-indexed and the set has atoms, else ones
        const bool rti = radius_type_indexed && n > 0;
        for (int32_t c = 0; c < nt; c++)
            type_radius[tpos + c] = rti ? (double)S.type_radii[c] * radius_scale : 1.0;
        if (n) {
            std::memcpy(coords32 + 3 * (size_t)a, S.coords, sizeof(float) * 3 * (size_t)n);
            std::memcpy(weights + wpos, S.type_vector, sizeof(float) * (size_t)n * nt);
        }
        for (int32_t k = 0; k < n; k++) {
            const int32_t q = a + k;
            radius[q] = (double)S.radii[k] * radius_scale;
            atom_set[q] = s;
            aex[q] = e;
            for (int32_t c = 0; c < nt; c++) {
                const float w = S.type_vector[(int64_t)k * nt + c];
                if (w == 0.0f) continue;
                it_atom[ip] = q;
                it_ch[ip] = c;
                it_w[ip] = w;
                it_r[ip] = rti ? type_radius[tpos + c] : radius[q];
                item_windex[ip] = wpos + (int64_t)k * nt + c;
                ichan[ip] = choff[s] + c;
                iex[ip] = e;
                ip++;
            }
        }
        ex_end[e] = ip;
        a += n;
        wpos += (int64_t)n * nt;
        tpos += nt;
    }
    int32_t max_ex = 0;
    for (int32_t e = 0; e < nexamples; e++) max_ex = std::max(max_ex, ex_end[e] - ex_start[e]);

    // static grouping of the items by (example, channel)
    const int64_t G = (int64_t)nexamples * C;
    std::vector<int32_t> gcount(G + 1, 0);
    for (int32_t q = 0; q < I; q++) gcount[iex[q] * C + ichan[q] + 1]++;
    for (int64_t g = 0; g < G; g++) gcount[g + 1] += gcount[g];
    {
        std::vector<int32_t> pos(gcount.begin(), gcount.end() - 1);
        for (int32_t q = 0; q < I; q++) perm[pos[iex[q] * C + ichan[q]]++] = q;
    }
    int32_t nsegs = 0, max_seg = 0;
    for (int32_t e = 0; e < nexamples; e++)
        for (int32_t c = 0; c <= nchannels; c++) {
            const int64_t g = (int64_t)e * C + c;
            chan_off[(int64_t)e * (nchannels + 1) + c] = gcount[std::min(g, G)];
            if (c < nchannels) {
                const int32_t k = gcount[g + 1] - gcount[g];
                if (k > 0) segs[nsegs++] = (int32_t)g;
                max_seg = std::max(max_seg, k);
            }
        }

    // backward launch order: within each example, nearest its center first
    // (packing._bwd_slots per_example: every channel of the example is read)
    if (bwd_order && bslot && A > 0) {
        std::vector<uint64_t> key(A);
        std::vector<int32_t> idx(A);
        for (int32_t q = 0; q < A; q++) {
            const double *c = centers + 3 * aex[q];
            const float dx = coords32[3 * q + 0] - (float)c[0];
            const float dy = coords32[3 * q + 1] - (float)c[1];
            const float dz = coords32[3 * q + 2] - (float)c[2];
            const float d = std::sqrt(dx * dx + dy * dy + dz * dz) * 16.0f;
            key[q] = ((uint64_t)aex[q] << 16) | (uint64_t)std::min(d, 32767.0f);
            idx[q] = q;
        }
        radix_sort(key, idx);
        for (int32_t k = 0; k < A; k++) bslot[idx[k]] = k;
    }
    info->natoms = A;
    info->nsegs = nsegs;
    info->max_seg_items = (nexamples > 0 && nchannels > 0) ? max_seg : 0;
    info->max_example_items = max_ex;
    return GM_OK;
}
