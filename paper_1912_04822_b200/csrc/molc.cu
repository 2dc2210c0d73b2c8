// molc.cu -- MOLC cache records -> typed device atoms (gm_molc_decode,
// include/gridmaker_b200.h).
//
// Reference: the cache reader builds one RawAtom per record
// (/root/reference/pkg/src/voxmol/chemio.py:353-356) and type_molecule
// (atomtypes.py:272-291) types them one by one with the default element
// typer, dropping atoms it maps to no type (hydrogens, noble gases,
// unmapped elements, atomtypes.py:125-135).  Here the raw 13-byte records of
// many entries arrive in one buffer and three small kernels decode them:
//   k_molc_count  CTA per entry: atoms the typing table keeps;
//   k_molc_scan   one CTA: per-entry output offsets (exclusive scan);
//   k_molc_write  CTA per entry: in-order compaction (warp ballots + a block
//                 scan) of coordinates, type index and type radius.
// Record layout (little-endian, unaligned): u8 element, f32 x, y, z.
#include "common.cuh"

namespace {

constexpr int kMolcThreads = 256;

__device__ __forceinline__ float load_f32_le(const uint8_t *p) {
    const uint32_t u = (uint32_t)p[0] | ((uint32_t)p[1] << 8) | ((uint32_t)p[2] << 16) |
                       ((uint32_t)p[3] << 24);
    return __uint_as_float(u);
}

__global__ void __launch_bounds__(kMolcThreads) k_molc_count(const uint8_t *raw, const int64_t *start,
                                                             const int16_t *table, int64_t *offsets) {
    __shared__ int warp_cnt[kMolcThreads / 32];
    const int e = blockIdx.x, tid = threadIdx.x;
    const int64_t a0 = start[e], a1 = start[e + 1];
    int cnt = 0;
    for (int64_t a = a0 + tid; a < a1; a += kMolcThreads) cnt += table[raw[13 * a]] >= 0;
    for (int o = 16; o > 0; o >>= 1) cnt += __shfl_xor_sync(0xffffffffu, cnt, o);
    if ((tid & 31) == 0) warp_cnt[tid >> 5] = cnt;
    __syncthreads();
    if (tid == 0) {
        int s = 0;
        for (int w = 0; w < kMolcThreads / 32; w++) s += warp_cnt[w];
        offsets[e + 1] = s;
    }
}

// offsets[0] = 0, offsets[e + 1] = kept atoms of entries 0..e (in place over
// the counts k_molc_count left in offsets[1..n]).
__global__ void __launch_bounds__(1024) k_molc_scan(int64_t *offsets, int n) {
    __shared__ int64_t warp_sum[32];
    __shared__ int64_t carry;
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    if (tid == 0) {
        carry = 0;
        offsets[0] = 0;
    }
    __syncthreads();
    for (int base = 0; base < n; base += 1024) {
        const int i = base + tid;
        int64_t v = i < n ? offsets[i + 1] : 0;
        for (int o = 1; o < 32; o <<= 1) {
            const int64_t t = __shfl_up_sync(0xffffffffu, v, o);
            if (lane >= o) v += t;
        }
        if (lane == 31) warp_sum[warp] = v;
        __syncthreads();
        if (warp == 0) {
            int64_t w = warp_sum[lane];
            for (int o = 1; o < 32; o <<= 1) {
                const int64_t t = __shfl_up_sync(0xffffffffu, w, o);
                if (lane >= o) w += t;
            }
            warp_sum[lane] = w;
        }
        __syncthreads();
        const int64_t incl = carry + v + (warp > 0 ? warp_sum[warp - 1] : 0);
        if (i < n) offsets[i + 1] = incl;
        __syncthreads();
        if (tid == 1023) carry = incl;
        __syncthreads();
    }
}

__global__ void __launch_bounds__(kMolcThreads) k_molc_write(const uint8_t *raw, const int64_t *start,
                                                             const int16_t *table, const float *radii,
                                                             const int64_t *offsets, float *coords,
                                                             int32_t *type_index, float *radius) {
    __shared__ int warp_cnt[kMolcThreads / 32];
    const int e = blockIdx.x, tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    const int64_t a0 = start[e], a1 = start[e + 1];
    int64_t out = offsets[e];
    for (int64_t base = a0; base < a1; base += kMolcThreads) {
        const int64_t a = base + tid;
        int t = -1;
        const uint8_t *r = raw + 13 * a;
        if (a < a1) t = table[r[0]];
        const bool keep = t >= 0;
        const unsigned m = __ballot_sync(0xffffffffu, keep);
        if (lane == 0) warp_cnt[warp] = __popc(m);
        __syncthreads();
        int before = 0, total = 0;
        for (int w = 0; w < kMolcThreads / 32; w++) {
            const int c = warp_cnt[w];
            before += w < warp ? c : 0;
            total += c;
        }
        if (keep) {
            const int64_t o = out + before + __popc(m & ((1u << lane) - 1u));
            coords[3 * o + 0] = load_f32_le(r + 1);
            coords[3 * o + 1] = load_f32_le(r + 5);
            coords[3 * o + 2] = load_f32_le(r + 9);
            type_index[o] = t;
            radius[o] = radii[t];
        }
        out += total;
        __syncthreads();  // warp_cnt is rewritten by the next chunk
    }
}

}  // namespace

gm_status molc_decode_impl(const uint8_t *raw, const int64_t *entry_start, int32_t nentries,
                           const int16_t *type_table, const float *type_radii, float *coords,
                           int32_t *type_index, float *radius, int64_t *offsets, cudaStream_t s) {
    if (nentries <= 0) {
        CUDA_TRY(cudaMemsetAsync(offsets, 0, sizeof(int64_t), s));
        return GM_OK;
    }
    k_molc_count<<<nentries, kMolcThreads, 0, s>>>(raw, entry_start, type_table, offsets);
    LAUNCH_CHECK();
    k_molc_scan<<<1, 1024, 0, s>>>(offsets, nentries);
    LAUNCH_CHECK();
    k_molc_write<<<nentries, kMolcThreads, 0, s>>>(raw, entry_start, type_table, type_radii, offsets,
                                                   coords, type_index, radius);
    LAUNCH_CHECK();
    return GM_OK;
}
