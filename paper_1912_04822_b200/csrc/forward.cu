// forward.cu -- k_forward: typed items -> dense density grids.
//
// Reference: _kernels.py:33-113 (index), 116-206 (vector); each (example,
// channel) block of the output is the sum, in item order, of every item's
// density over its integer voxel box, rounded once to f32.
//
// Work decomposition (B200): one CTA per (example, channel, tile of TI planes
// x TJ rows x all D columns); the tile accumulates in shared memory (dense
// [TI][TJ][D]).  Default: one-warp CTAs owning one plane (48^3: 9 KB, 16
// CTAs per SM; 96^3: a band of rows) -- no warp waits for another.  Each warp
// owns a disjoint region of the tile and walks the channel's items
// (k_prepare_example grouped them by channel, in item order) 32 at a time:
//   phase A (lane t <-> item t): box test against the region, the sphere's
//           cross-section with the plane (row / column spans, ~2/3 of the box
//           face), per-visit constants -> a per-warp shared-memory slot;
//   phase B (items in order): every lane reads the slot (broadcast) and
//           scatters its (row, column) voxels: one FMA per row coordinate,
//           d^2, ex2 (Gaussian core), sqrt (tail), a shared-memory accumulate.
// Regions are disjoint and each warp adds its items in order, without
// atomics.  With the items in channel order (index typing on grids up to
// 64^3) that is the reference's item order; where the prepare pass sorts each
// channel's items by first plane (vector typing, grids above 64^3) a voxel's
// sum runs bucket by bucket, item order within a bucket -- a fixed order (run
// to run and batch-size independent), within the f32 tolerance of the
// reference's.  The finished tile
// (zeros included) leaves through TMA bulk stores (cp.async.bulk) when
// D % 4 == 0: the planes of a tile are contiguous in global memory.  A
// channel without items is written by one CTA (its tile 0) re-sending one
// zeroed buffer over the whole slab; the slab's other CTAs exit at once.
// Consecutive CTAs are the channels of one tile, so scatter work and the
// stores of empty channels interleave finely (HBM keeps writing while SMs
// compute).
#include <vector>

#include "common.cuh"

namespace {

#ifndef GM_FWD_EVICT
#define GM_FWD_EVICT 1  // L2 evict-first hint on the grid bulk stores (C2 112.6 -> 106.7 us)
#endif
#ifndef GM_FWD_WARPS
#define GM_FWD_WARPS 1
#endif
#ifndef GM_FWD_MINB
#define GM_FWD_MINB 16
#endif
#ifndef GM_FWD_ZGROUP
#define GM_FWD_ZGROUP 16  // tiles of a zero slab written by one CTA (C2 step: 8 203.0 us,
                           // 12 202.5, 16 201.1, 24 203.2, 32 205.0)
#endif
#ifndef GM_FWD_LPT
#define GM_FWD_LPT 2  // job table: 0 dense order, 1 heaviest first, 2 heavy/light alternating
#endif
#ifndef GM_FWD_LPT_GROUP
#define GM_FWD_LPT_GROUP 0  // examples per reordering group (0: the whole batch)
#endif
#ifndef GM_FWD_LPT_MAXD
#define GM_FWD_LPT_MAXD 128  // reorder only up to this grid size (48^3 gains 14%; 96^3 lost
                             // 8% before the evict-first stores, gains 1.8% with them)
#endif
// job order: GM_FWD_ALT_H jobs from the heavy end of the sorted list, then
// GM_FWD_ALT_L from the light end (measured on C2 before the evict-first
// stores: 1:1 116.6 us, 1:3 112.8, 2:3 112.4, 1:6 127.5; with them: 1:1 110.8,
// 1:2 106.8, 1:3 105.6, 1:4 109.9, 2:3 106.8, 2:5 105.6, 2:7 107.6; and with
// zero groups of 16: 1:2 106.5, 1:3 103.3, 1:4 107.6, 2:3 109.9, 2:5 104.1)
#ifndef GM_FWD_ALT_H
#define GM_FWD_ALT_H 1
#endif
#ifndef GM_FWD_ALT_L
#define GM_FWD_ALT_L 3
#endif
#ifndef GM_FWD_ZPLACE
#define GM_FWD_ZPLACE 0  // zero groups in the job table: 0 spread evenly, 1 first, 2 last
#endif
#ifndef GM_FWD_TMA_ITEMS
// 1: the cull's item records staged in shared memory by TMA bulk copies (one
// lane, mbarrier-completed, next chunk in flight) instead of register
// prefetch.  Bit-identical; measured 10 % slower (C2 forward 108.6 -> 119.5
// us): the 2 KB stage per warp costs two resident CTAs per SM.
#define GM_FWD_TMA_ITEMS 0
#endif
#ifndef GM_FWD_BUDGET_KB
#define GM_FWD_BUDGET_KB 10
#endif
constexpr int kThreads = 32 * GM_FWD_WARPS;
constexpr int kWarps = kThreads / 32;

struct FwdArgs {
    const FwdItem *sorted;
    const BinItem *bsorted;
    const int2 *sbox;
    const int32_t *chan_off;
    const double *origins;
    float *out;
    double res;
    float resf, resl, inv_res;  // res = resf + resl
    const int4 *jobs;  // optional job table (gm_batch.fwd_jobs) or NULL
    const int32_t *poff;  // per (example, channel) plane-bucket item offsets, or NULL
    int D, C, TI, TJ, ntj, wpp, rpw;
    int ntiles;        // tiles per (example, channel) slab
    int bulk;
    size_t acc_floats;
};

// Per-visit constants of one item for one warp region (phase A -> phase B).
struct __align__(16) Slot {
    float yh, yl, zh, zl;      // row / column offsets at the box corner (hi, lo)
    float dx2, cexp, d02, cut; // plane offset^2, -2 log2(e)/r^2, (grm r)^2, cutoff
    float qa, w;               // quadratic coefficient, weight
    int jspan, kspan;          // first row / column relative to the box corner | count << 16
    int arow;                  // accumulator offset of (first row, box column 0)
    int rpi;                   // columns per pass = min(32, columns)
    int src;                   // item index (binary mode re-reads the f64 record)
    int pad;                   // bits of 1 / (columns per pass)
};
static_assert(sizeof(Slot) == 64, "Slot must be 64 bytes");

__device__ __forceinline__ void bulk_store(float *gdst, const float *ssrc, uint32_t bytes) {
    const uint32_t s = (uint32_t)__cvta_generic_to_shared(ssrc);
#if GM_FWD_EVICT
    // the grids stream out: an L2 evict-first policy for their lines
    uint64_t pol;
    asm volatile("createpolicy.fractional.L2::evict_first.b64 %0, 1.0;" : "=l"(pol));
    asm volatile("cp.async.bulk.global.shared::cta.bulk_group.L2::cache_hint [%0], [%1], %2, %3;"
                 ::"l"(gdst), "r"(s), "r"(bytes), "l"(pol)
                 : "memory");
#else
    asm volatile("cp.async.bulk.global.shared::cta.bulk_group [%0], [%1], %2;" ::"l"(gdst), "r"(s),
                 "r"(bytes)
                 : "memory");
#endif
}

// Ex2 / sqrt on the MUFU unit (no denormal / special-case paths: arguments
// are finite, d^2 >= 0, densities >= 2^-126 where they matter).
__device__ __forceinline__ float fast_ex2(float x) {
    float y;
    asm("ex2.approx.ftz.f32 %0, %1;" : "=f"(y) : "f"(x));
    return y;
}
__device__ __forceinline__ float fast_sqrt(float x) {
    float y;
    asm("sqrt.approx.ftz.f32 %0, %1;" : "=f"(y) : "f"(x));
    return y;
}

// Conservative index range [lo, hi] (relative to the box corner) of voxels
// whose axis offset c + idx*res lies in [-rho, rho].
__device__ __forceinline__ void sphere_span(float c, float rho, float inv_res, int n, int &lo,
                                            int &hi) {
    const float a = (-rho - c) * inv_res, b = (rho - c) * inv_res;
    lo = max(0, (int)ceilf(fmaxf(a, -1.0f)));
    hi = min(n - 1, (int)floorf(fminf(b, (float)n)));
}

// Phase A for one item: does it touch plane i, rows [jg0, jg1] inside its
// cutoff sphere?  If so fill the slot.
__device__ __forceinline__ bool plan_visit(const FwdItem &it, int i, int jg0, int jg1, int j0,
                                           int D, float resf, float resl, float inv_res,
                                           Slot &S) {
    const int4 bx = *reinterpret_cast<const int4 *>(&it.ibox);
    const int ilo = box_lo(bx.x);
    if (i < ilo || i > box_hi(bx.x)) return false;
    const int jlo_b = box_lo(bx.y), klo_b = box_lo(bx.z);
    const int jlo = max(jlo_b, jg0), jhi = min(box_hi(bx.y), jg1);
    if (jlo > jhi) return false;
    const float4 P = *reinterpret_cast<const float4 *>(&it.cxh);
    const float4 Q = *reinterpret_cast<const float4 *>(&it.cxl);
    const float4 R = *reinterpret_cast<const float4 *>(&it.dzr);
    const float cut = R.x;
    const float fi = (float)(i - ilo);
    const float dx = fmaf(fi, resf, P.x) + fmaf(fi, resl, Q.x);
    const float rho2 = fmaf(-dx, dx, cut * cut);
    if (rho2 < -1e-5f * cut * cut) return false;
    const float rho = fmaf(fast_sqrt(fmaxf(rho2, 0.0f)), 1.00002f, 1e-4f * cut);
    int jr0, jr1, kr0, kr1;
    sphere_span(P.y + Q.y, rho, inv_res, box_hi(bx.y) - jlo_b + 1, jr0, jr1);
    sphere_span(P.z + Q.z, rho, inv_res, box_hi(bx.z) - klo_b + 1, kr0, kr1);
    jr0 = max(jr0, jlo - jlo_b);
    jr1 = min(jr1, jhi - jlo_b);
    if (jr0 > jr1 || kr0 > kr1) return false;
    const int nk = kr1 - kr0 + 1;
    S.yh = P.y;
    S.yl = Q.y;
    S.zh = P.z;
    S.zl = Q.z;
    S.dx2 = dx * dx;
    S.cexp = P.w;
    S.d02 = Q.w;
    S.cut = cut;
    S.qa = R.y;
    S.w = R.z;
    S.jspan = jr0 | ((jr1 - jr0 + 1) << 16);
    S.kspan = kr0 | (nk << 16);
    S.arow = (jlo_b + jr0 - j0) * D + klo_b;
    S.rpi = min(32, nk);  // columns per pass
    S.pad = __float_as_int(__frcp_rn((float)S.rpi));
    return true;
}

// Phases A/B of one warp region: the channel's items [cs, ce) scattered, in
// order, into plane i, rows [jg0, jg1] of the accumulator (accp: plane i of
// the tile, row j at (j - j0) * D).
__device__ __forceinline__ void mbar_wait(uint32_t bar, uint32_t phase) {
    uint32_t done = 0;
    while (!done)
        asm volatile(
            "{ .reg .pred p; mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2; selp.u32 %0, 1, 0, p; }"
            : "=r"(done)
            : "r"(bar), "r"(phase)
            : "memory");
}

// One lane stages items [from, from + n) (64 B each, contiguous) into shared
// memory with a TMA bulk copy completing on mbarrier `bar`.
__device__ __forceinline__ void stage_items(const FwdItem *src, FwdItem *dst, int n, uint32_t bar) {
    const uint32_t bytes = (uint32_t)n * (uint32_t)sizeof(FwdItem);
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(bar), "r"(bytes)
                 : "memory");
    asm volatile(
        "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
            (uint32_t)__cvta_generic_to_shared(dst)),
        "l"(src), "r"(bytes), "r"(bar)
        : "memory");
}

// Phase B of one visit: every lane scatters its (row, column) voxels of the
// item planned in slot *sp into plane i of the accumulator (accp).
template <bool BINARY, bool VECTOR, bool RESL>
__device__ __forceinline__ void scatter_visit(const FwdArgs &A, float *accp, const Slot *sp, int lane,
                                              int i, double ox, double oy, double oz) {
    const int D = A.D;
    const double res = A.res;
    const float resf = A.resf, resl = A.resl;
    const float4 S0 = *reinterpret_cast<const float4 *>(&sp->yh);
    const float4 S1 = *reinterpret_cast<const float4 *>(&sp->dx2);
    const float4 S2 = *reinterpret_cast<const float4 *>(&sp->qa);
    const int4 S3 = *reinterpret_cast<const int4 *>(&sp->arow);
    const int jr0 = box_lo(__float_as_int(S2.z)), nj = box_hi(__float_as_int(S2.z));
    const int kr0 = box_lo(__float_as_int(S2.w)), nk = box_hi(__float_as_int(S2.w));
    const int nks = S3.y;
    const float inv = __int_as_float(S3.w);  // 1/nks (approximate, exact enough)
    const int r = small_div(lane, inv), rpi = small_div(32, inv);
    if (BINARY) {
        // _kernels.py:87-98 (index) / 180-192 (vector): the occupancy test
        // d^2 <= r^2 decided like the reference's f64 expression.  The f32
        // distance from the hi/lo offsets is within ~1e-5 A^2 of it, so
        // outside a band of 1e-4 (r^2 + 1 A^2) around r^2 its answer is
        // the reference's; inside the band (rare) the exact f64
        // expression, same association, no contraction, decides.
        const float w = S2.y;
        const float r2f = S1.w * S1.w;  // cut = r in binary mode
        const float band = 1e-4f * (r2f + 1.0f);
        const float lo2 = r2f - band, hi2 = r2f + band;
        for (int kb = 0; kb < nk; kb += 32) {
            const int nkb = min(32, nk - kb);
            const float invb = __frcp_rn((float)nkb);
            const int rpb = small_div(32, invb);
            const int rr = small_div(lane, invb), kk = kb + lane - rr * nkb;
            if (rr >= rpb) continue;
            const float fk = (float)(kr0 + kk);
            const float dzf = fmaf(fk, resf, S0.z) + fmaf(fk, resl, S0.w);
            const float b2f = fmaf(dzf, dzf, S1.x);
            float *ap = accp + S3.x + kr0 + kk + (size_t)rr * D;
            for (int jj = rr; jj < nj; jj += rpb, ap += (size_t)rpb * D) {
                const float jf = (float)(jr0 + jj);
                const float dyf = fmaf(jf, resf, S0.x) + fmaf(jf, resl, S0.y);
                const float d2f = fmaf(dyf, dyf, b2f);
                bool in = d2f <= lo2;
                if (!in && d2f <= hi2) {
                    const BinItem bi = A.bsorted[S3.z];
                    const int4 bx = *reinterpret_cast<const int4 *>(&A.sorted[S3.z].ibox);
                    const double dxd =
                        __dsub_rn(__dadd_rn(ox, __dmul_rn((double)i, res)), bi.x);
                    const double dz = __dsub_rn(
                        __dadd_rn(oz, __dmul_rn((double)(box_lo(bx.z) + kr0 + kk), res)), bi.z);
                    const double dy = __dsub_rn(
                        __dadd_rn(oy, __dmul_rn((double)(box_lo(bx.y) + jr0 + jj), res)), bi.y);
                    const double d2 = __dadd_rn(__dadd_rn(__dmul_rn(dxd, dxd), __dmul_rn(dy, dy)),
                                                __dmul_rn(dz, dz));
                    in = d2 <= bi.r2;
                }
                if (in) {
                    if (VECTOR) *ap = fmaxf(*ap, w);
                    else *ap = 1.0f;
                }
            }
        }
    } else if (nk <= 32) {
        // _kernels.py:99-106: Gaussian core to d0, quadratic tail to the cutoff
        if (r < rpi) {
            const int kk = kr0 + lane - r * nks;
            const float fk = (float)kk;
            const float dz = fmaf(fk, resf, S0.z) + fmaf(fk, resl, S0.w);
            const float b2 = fmaf(dz, dz, S1.x);
            const float cexp = S1.y, d02 = S1.z, cut = S1.w, qa = S2.x, w = S2.y;
            const float rpif = (float)rpi;
            float *ap = accp + S3.x + kk + r * D;
            const int step = rpi * D;
            float jf = (float)(jr0 + r);
            auto val = [&](float y) {
                const float dy = RESL ? fmaf(y, resf, S0.x) + fmaf(y, resl, S0.y)
                                      : fmaf(y, resf, S0.x) + S0.y;
                const float d2 = fmaf(dy, dy, b2);
                const float g = fast_ex2(d2 * cexp);
                const float t2 = fmaxf(cut - fast_sqrt(d2), 0.0f);
                return d2 <= d02 ? g : qa * t2 * t2;
            };
            int jj = r;
            // two rows per iteration: both accumulator reads are
            // issued before either write (different rows)
            for (; jj + rpi < nj; jj += 2 * rpi, jf += 2.0f * rpif, ap += 2 * step) {
                const float v0 = val(jf), v1 = val(jf + rpif);
                const float a0 = ap[0], a1 = ap[step];
                ap[0] = fmaf(w, v0, a0);
                ap[step] = fmaf(w, v1, a1);
            }
            if (jj < nj) *ap = fmaf(w, val(jf), *ap);
        }
    } else {
        // > 32 columns (very fine grids): one row pass per 32 columns
        const float cexp = S1.y, d02 = S1.z, cut = S1.w, qa = S2.x, w = S2.y;
        for (int kb = lane; kb < nk; kb += 32) {
            const int kk = kr0 + kb;
            const float fk = (float)kk;
            const float dz = fmaf(fk, resf, S0.z) + fmaf(fk, resl, S0.w);
            const float b2 = fmaf(dz, dz, S1.x);
            float *ap = accp + S3.x + kk;
            for (int jj = 0; jj < nj; jj++, ap += D) {
                const float jf = (float)(jr0 + jj);
                const float dy = fmaf(jf, resf, S0.x) + fmaf(jf, resl, S0.y);
                const float d2 = fmaf(dy, dy, b2);
                const float g = fast_ex2(d2 * cexp);
                const float t2 = fmaxf(cut - fast_sqrt(d2), 0.0f);
                const float v = d2 <= d02 ? g : qa * t2 * t2;
                *ap = fmaf(w, v, *ap);
            }
        }
    }
}

template <bool BINARY, bool VECTOR, bool RESL>
__device__ __forceinline__ void scatter_items(const FwdArgs &A, float *accp, Slot *slots, int lane,
                                              int e, int i, int jg0, int jg1, int j0, int cs,
                                              int ce, FwdItem *stage, uint64_t *barp) {
    const int D = A.D;
    const double res = A.res;
    const float resf = A.resf, resl = A.resl, inv_res = A.inv_res;
    const double ox = A.origins[3 * e + 0], oy = A.origins[3 * e + 1],
                 oz = A.origins[3 * e + 2];
#if GM_FWD_TMA_ITEMS
    // the channel's item records arrive 32 at a time in shared memory by TMA
    // bulk copies (one lane issues; the next chunk's copy is in flight while
    // the current chunk scatters)
    const uint32_t bar = (uint32_t)__cvta_generic_to_shared(barp);
    uint32_t phase = 0;
    if (lane == 0 && cs < ce) {
        asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(bar));
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
        stage_items(A.sorted + cs, stage, min(32, ce - cs), bar);
    }
    __syncwarp();
#else
    // the next chunk's records are prefetched into registers while the
    // current chunk scatters (hides the L2 latency of phase A)
    FwdItem nxt;
    int2 nbox = make_int2(1, 0);  // empty box
    if (cs + lane < ce) {
        nbox = A.sbox[cs + lane];
        nxt = A.sorted[cs + lane];
    }
#endif
    for (int base = cs; base < ce; base += 32) {
        // ---- phase A: lane t plans item base + t ----
        const int it = base + lane;
#if GM_FWD_TMA_ITEMS
        mbar_wait(bar, phase);
        phase ^= 1u;
        FwdItem cur_item;
        int2 bx = make_int2(1, 0);
        if (it < ce) {
            cur_item = stage[lane];
            bx = make_int2(cur_item.ibox, cur_item.jbox);
        }
        __syncwarp();
        if (lane == 0 && base + 32 < ce) {
            // every lane has read the stage: reuse it for the next chunk
            asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
            stage_items(A.sorted + base + 32, stage, min(32, ce - base - 32), bar);
        }
#else
        const FwdItem cur_item = nxt;
        const int2 bx = nbox;
        nbox = make_int2(1, 0);
        if (it + 32 < ce) {
            nbox = A.sbox[it + 32];
            nxt = A.sorted[it + 32];
        }
#endif
        bool hit = false;
        if (it < ce && box_lo(bx.x) <= i && box_hi(bx.x) >= i && box_lo(bx.y) <= jg1 &&
            box_hi(bx.y) >= jg0) {
            Slot S;
            hit = plan_visit(cur_item, i, jg0, jg1, j0, D, resf, resl, inv_res, S);
            if (hit) {
                S.src = it;
                slots[lane] = S;
            }
        }
        unsigned m = __ballot_sync(0xffffffffu, hit);
        __syncwarp();
        // ---- phase B: items in order, all lanes scatter ----
        while (m) {
            const int t = __ffs(m) - 1;
            m &= m - 1;
            scatter_visit<BINARY, VECTOR, RESL>(A, accp, slots + t, lane, i, ox, oy, oz);
            __syncwarp();
        }
    }
}

template <bool BINARY, bool VECTOR, bool RESL>
__global__ void __launch_bounds__(kThreads, GM_FWD_MINB) k_forward(const FwdArgs A) {
    extern __shared__ __align__(128) unsigned char smem[];
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    // the job (built before the prepare pass, complete when it started) is
    // read before the wait; the prepare pass's records must be complete
    // before anything else, then the backward (next in the stream) may begin
    // its prologue while this grid drains
    const int4 job = A.jobs ? A.jobs[blockIdx.x] : make_int4(0, 0, 0, 0);
    pdl_wait();
    pdl_trigger();
    // grid (channel, tile, example): consecutive CTAs are the channels of one
    // tile, so scatter work and zero-tile stores interleave finely, which
    // keeps HBM writing while SMs compute
    int tile, e, c, cs, ce, i0, j0;
    const int D = A.D, TI = A.TI, TJ = A.TJ;
    if (A.jobs) {
        // job table: only tiles with items, one job per group of zero tiles;
        // {example | channel << 16, first item, end item, first plane | first
        // row << 16}: the channel's item range of the static grouping travels
        // in the job (the prepare pass keeps every item of the grouping in
        // place), so the first load is the items themselves -- no dependent
        // chan_off load and no integer division before it
        const int4 j = job;
        e = j.x & 0xffff;
        c = (int)((unsigned)j.x >> 16);
        cs = j.y;
        ce = j.z;
        i0 = j.w & 0xffff;
        j0 = j.w >> 16;
        tile = -1;  // derived below where needed (zero groups)
    } else {
        tile = blockIdx.y;
        e = blockIdx.z;
        c = blockIdx.x;
        i0 = (tile / A.ntj) * TI;
        j0 = (tile % A.ntj) * TJ;
        cs = A.chan_off[(size_t)e * (A.C + 1) + c];
        ce = A.chan_off[(size_t)e * (A.C + 1) + c + 1];
    }
    const int TIv = min(TI, D - i0), TJv = min(TJ, D - j0);
    const size_t plane = (size_t)D * D;
    float *obase = A.out + ((size_t)e * A.C + c) * D * plane + (size_t)i0 * plane + (size_t)j0 * D;
    const int chunk = TJv * D;  // contiguous floats per plane of the tile (global and smem)

    if (cs == ce) {
        // no item of this channel: the whole (example, channel) slab is zero.
        // Every GM_FWD_ZGROUP-th CTA of the slab writes its group of tiles
        // (contiguous in memory); the other CTAs of the group leave at once
        // (the job table does not even launch them).
        if (tile < 0) tile = (i0 / TI) * A.ntj + j0 / TJ;
        if (tile % GM_FWD_ZGROUP) return;
        const int t1 = min(tile + GM_FWD_ZGROUP, A.ntiles);
        const int i1 = (t1 - 1) / A.ntj * TI, jl = ((t1 - 1) % A.ntj) * TJ;
        // end of the last tile of the group: plane min(i1+TI, D), row band jl
        const size_t end = min(TJ + jl, D) == D ? (size_t)min(i1 + TI, D) * plane
                                                : (size_t)i1 * plane + (size_t)(jl + TJ) * D;
        float *slab = A.out + ((size_t)e * A.C + c) * D * plane;
        const size_t begin = (size_t)i0 * plane + (size_t)j0 * D;
        const size_t total = end - begin;
        if (A.bulk) {
            // one zeroed shared buffer re-sent through TMA bulk stores
            float4 *z4 = reinterpret_cast<float4 *>(smem);
            const float4 z = make_float4(0.f, 0.f, 0.f, 0.f);
            const int nz4 = (int)(A.acc_floats >> 2);
            for (int q = tid; q < nz4; q += kThreads) z4[q] = z;
            asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
            __syncthreads();
            const size_t per = (size_t)nz4 * 4;
            const size_t nst = (total + per - 1) / per;
            for (size_t q = tid; q < nst; q += kThreads) {
                const size_t o = q * per;
                bulk_store(slab + begin + o, reinterpret_cast<const float *>(smem),
                           (uint32_t)(std::min(per, total - o) * 4u));
            }
            asm volatile("cp.async.bulk.commit_group;" ::: "memory");
            asm volatile("cp.async.bulk.wait_group.read 0;" ::: "memory");
        } else {
            for (size_t q = tid; q < total; q += kThreads) __stcs(slab + begin + q, 0.f);
        }
        return;
    }

    float *acc = reinterpret_cast<float *>(smem);
    Slot *slots = reinterpret_cast<Slot *>(smem + A.acc_floats * 4) + warp * 32;
    // this warp's region: plane p, global rows [jg0, jg1]; warps are
    // independent until the final store
    const int p = warp / A.wpp, part = warp - p * A.wpp;
    const int i = i0 + p;
    const int jg0 = j0 + part * A.rpw, jg1 = j0 + min((part + 1) * A.rpw, TJv) - 1;
    const bool region_ok = p < TIv && jg0 <= jg1;
    float *accp = acc + (size_t)p * TJ * D;  // plane p of the tile, row j at (j - j0) * D
    if (A.poff) {
        // items sorted by first plane (k_sort_planes): only those whose first
        // plane lies within the channel's widest box of plane i can reach it
        // the channel's bucket record read by the warp in one load level
        // (lanes hold entries lane, lane + 32, lane + 64), picked by shuffles
        static_assert(kPlaneRec <= 96 && kBuckets == 64, "bucket record layout");
        const int32_t *rec = A.poff + ((size_t)e * A.C + c) * kPlaneRec;
        const int v0 = rec[lane], v1 = rec[32 + lane];
        const int v2 = lane < kPlaneRec - 64 ? rec[64 + lane] : 0;
        auto pick = [&](int k) {
            const int a0 = __shfl_sync(0xffffffffu, v0, k & 31), a1 = __shfl_sync(0xffffffffu, v1, k & 31),
                      a2 = __shfl_sync(0xffffffffu, v2, k & 31);
            return k < 32 ? a0 : (k < 64 ? a1 : a2);
        };
        const int wmax = pick(kBuckets + 2);
        const int b0 = plane_bucket(max(0, i - wmax + 1), D), b1 = plane_bucket(min(i, D - 1), D);
        const int rs = pick(b0), re = pick(b1 + 1);
        ce = cs + re;
        cs = cs + rs;
    }
    if (region_ok) {
        {
            const int nf = (jg1 - jg0 + 1) * D;
            if ((D & 3) == 0) {
                float4 *r0 = reinterpret_cast<float4 *>(accp + (size_t)(jg0 - j0) * D);
                const float4 z = make_float4(0.f, 0.f, 0.f, 0.f);
                for (int q = lane; q < (nf >> 2); q += 32) r0[q] = z;
            } else {
                float *rs = accp + (size_t)(jg0 - j0) * D;
                for (int q = lane; q < nf; q += 32) rs[q] = 0.0f;
            }
        }
        FwdItem *stage = reinterpret_cast<FwdItem *>(smem + A.acc_floats * 4 +
                                                     (size_t)kWarps * 32 * sizeof(Slot)) + warp * 32;
        uint64_t *barp = reinterpret_cast<uint64_t *>(smem + A.acc_floats * 4 +
                                                      (size_t)kWarps * 32 * (sizeof(Slot) + sizeof(FwdItem))) + warp;
        scatter_items<BINARY, VECTOR, RESL>(A, accp, slots, lane, e, i, jg0, jg1, j0, cs, ce,
                                            stage, barp);
    }

    // ---- the finished tile, zeros included ----
    if (A.bulk) {
        asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
        __syncthreads();
        if (tid == 0) {
            if (TJv == D) {
                bulk_store(obase, acc, (uint32_t)(TIv * chunk) * 4u);
            } else {
                for (int pp = 0; pp < TIv; pp++)
                    bulk_store(obase + pp * plane, acc + (size_t)pp * TJ * D, (uint32_t)chunk * 4u);
            }
            asm volatile("cp.async.bulk.commit_group;" ::: "memory");
            asm volatile("cp.async.bulk.wait_group.read 0;" ::: "memory");
        }
    } else {
        __syncthreads();
        for (int pp = 0; pp < TIv; pp++)
            for (int q = tid; q < chunk; q += kThreads)
                __stcs(obase + pp * plane + q, acc[(size_t)pp * TJ * D + q]);
    }
}


struct FwdConfig {
    int TI, TJ, wpp, rpw;
    size_t acc_floats, smem;
};

FwdConfig choose_config(int D) {
    const size_t budget = GM_FWD_BUDGET_KB * 1024;  // acc; + 2 KB of slots per warp
    const size_t plane = (size_t)D * D * 4;
    FwdConfig cfg{};
    int TI = kWarps;
    while (TI > 1 && (TI * plane > budget || TI > D)) TI >>= 1;
    cfg.TI = TI;
    cfg.wpp = kWarps / TI;
    int TJ = D;
    if (plane > budget) TJ = std::max(cfg.wpp, (int)(budget / ((size_t)D * 4)) / cfg.wpp * cfg.wpp);
    cfg.TJ = std::min(TJ, D);
    cfg.rpw = (cfg.TJ + cfg.wpp - 1) / cfg.wpp;
    cfg.acc_floats = align_up((size_t)cfg.TI * cfg.TJ * D, 32);
    cfg.smem = cfg.acc_floats * 4 + (size_t)kWarps * 32 * sizeof(Slot) +
               (GM_FWD_TMA_ITEMS ? (size_t)kWarps * (32 * sizeof(FwdItem) + 8) : 0);
    return cfg;
}

template <bool BIN, bool VEC, bool RESL>
gm_status launch(const FwdArgs &A, const FwdConfig &cfg, int nex, int njobs, cudaStream_t s,
                 bool *launched) {
    auto kern = k_forward<BIN, VEC, RESL>;
    CUDA_TRY(gm_ensure_smem((const void *)kern, (int)cfg.smem));
    if (A.jobs) {
        if (njobs > 0) {
            CUDA_TRY(gm_launch_pdl(kern, dim3(njobs), dim3(kThreads), cfg.smem, s, A));
            LAUNCH_CHECK();
            if (launched) *launched = true;
        }
        return GM_OK;
    }
    if (A.ntiles > 65535 || nex > 65535) return gm_fail(GM_ERR_INVALID, "too many examples or tiles");
    dim3 grid(A.C, A.ntiles, nex);
    CUDA_TRY(gm_launch_pdl(kern, grid, dim3(kThreads), cfg.smem, s, A));
    LAUNCH_CHECK();
    if (launched) *launched = true;
    return GM_OK;
}

// ---------------------------------------------------------------------------
// The forward job table built on the device (batches assembled on the device
// change composition every call; the host builder, forward_jobs_impl below,
// costs milliseconds).  Same table, entry for entry: work jobs ordered by
// (channel item count descending, example, tile, channel) and dealt GM_FWD_ALT_H
// heavy : GM_FWD_ALT_L light, zero groups spread evenly -- each job's final
// slot is computed in closed form from per-group ranks, so the table needs
// no sort.
// ---------------------------------------------------------------------------
struct JobGeom {
    int ntiles, ntj, TI, TJ;
    int reorder;               // D <= GM_FWD_LPT_MAXD: GM_FWD_LPT (1 sorted, 2 dealt), else 0
    long long W, Z, n;         // work jobs, zero jobs, total
    long long H;               // heavy slots of the dealing
};

// zeros before table slot k: floor(k Z / n) (the host rule places zero job
// zi at the first slot k with (zi + 1) n <= (k + 1) Z)
__device__ __forceinline__ long long zeros_before(long long k, const JobGeom &J) {
    return J.Z ? (k * J.Z) / J.n : 0;
}

// The final slot of group g's tile t.
__device__ __forceinline__ void place_job(const int32_t *co, int nch, int g, int t, int4 s0,
                                          int4 s1, int4 *jobs, const JobGeom &J) {
    const int e = g / nch, c = g - e * nch;
    long long k;
    if (s1.w > 0) {
        // rank in the sorted work list, then its slot in the heavy/light deal
        long long srt, m;
        if (J.reorder) {
            srt = (long long)J.ntiles * (s0.x + s0.y) + (long long)t * s0.z + s0.w;
            if (J.reorder == 1) {
                m = srt;  // heaviest first, no dealing
            } else if (srt < J.H) {
                m = (long long)(GM_FWD_ALT_H + GM_FWD_ALT_L) * (srt / GM_FWD_ALT_H) + srt % GM_FWD_ALT_H;
            } else {
                const long long i = J.W - 1 - srt;  // i-th light job from the end
                m = (long long)(GM_FWD_ALT_H + GM_FWD_ALT_L) * (i / GM_FWD_ALT_L) + GM_FWD_ALT_H +
                    i % GM_FWD_ALT_L;
            }
        } else {
            m = (long long)J.ntiles * s1.x + (long long)t * s1.y + s1.z;
        }
        // work job m sits at the last slot k with k - zeros_before(k) == m
        long long lo = m, hi = J.n - 1;
        while (lo < hi) {  // smallest k with (k + 1) - zeros_before(k + 1) > m
            const long long mid = (lo + hi) >> 1;
            if ((mid + 1) - zeros_before(mid + 1, J) > m) hi = mid;
            else lo = mid + 1;
        }
        k = lo;
    } else {
        if (t % GM_FWD_ZGROUP) return;
        const long long nzt = (J.ntiles + GM_FWD_ZGROUP - 1) / GM_FWD_ZGROUP;
        const long long zi = nzt * s0.y + (long long)(t / GM_FWD_ZGROUP) * s0.z + s0.w;
        k = ((zi + 1) * J.n + J.Z - 1) / J.Z - 1;  // ceil((zi + 1) n / Z) - 1
    }
    jobs[k] = make_int4(e | (c << 16), co[e * (nch + 1) + c], co[e * (nch + 1) + c + 1],
                        ((t / J.ntj) * J.TI) | (((t % J.ntj) * J.TJ) << 16));
}

// One warp per (example, channel) group: ranks of the group among all groups.
// The group item counts are staged in shared memory first (the rank loop
// then runs on shared-memory reads instead of serial L2 round trips).
constexpr int kJobStatsMaxG = 12032;  // groups staged in shared memory (static 48 KB with the stats)
// CTA of 8 warps <-> 8 groups: each warp ranks its group, then the CTA places
// the groups' jobs (one launch for the whole table)
__global__ void __launch_bounds__(256) k_job_build(const int32_t *co, int nex, int nch,
                                                   int4 *jobs, const JobGeom J) {
    __shared__ int cnt[kJobStatsMaxG];
    __shared__ int4 st[8][2];
    const int G = nex * nch;
    const bool staged = G <= kJobStatsMaxG;
    if (staged)
        for (int q = threadIdx.x; q < G; q += blockDim.x) {
            const int e = q / nch, c = q - e * nch;
            cnt[q] = co[e * (nch + 1) + c + 1] - co[e * (nch + 1) + c];
        }
    __syncthreads();
    const int lane = threadIdx.x & 31;
    const int g = blockIdx.x * 8 + (threadIdx.x >> 5);
    const int e = g / nch, c = g - e * nch;
    auto count_of = [&](int q) {
        if (staged) return cnt[q];
        const int e2 = q / nch, c2 = q - e2 * nch;
        return co[e2 * (nch + 1) + c2 + 1] - co[e2 * (nch + 1) + c2];
    };
    const int k0 = g < G ? count_of(g) : 0;
    int gt = 0, eqb = 0, eqe = 0, eqc = 0, nwb = 0, nwe = 0, nwc = 0;
    const int gfirst = e * nch;  // first group of this example
    for (int q = lane; q < (g < G ? G : 0); q += 32) {
        const int k = count_of(q);
        const bool before = q < gfirst, same = q >= gfirst && q < gfirst + nch, cb = same && q < g;
        if (k0 > 0) {
            gt += k > k0;
            eqb += k == k0 && before;
            eqe += k == k0 && same;
            eqc += k == k0 && cb;
            nwb += k > 0 && before;
            nwe += k > 0 && same;
            nwc += k > 0 && cb;
        } else {  // zero groups: rank among zero groups
            eqb += k == 0 && before;
            eqe += k == 0 && same;
            eqc += k == 0 && cb;
        }
    }
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) {
        gt += __shfl_xor_sync(0xffffffffu, gt, o);
        eqb += __shfl_xor_sync(0xffffffffu, eqb, o);
        eqe += __shfl_xor_sync(0xffffffffu, eqe, o);
        eqc += __shfl_xor_sync(0xffffffffu, eqc, o);
        nwb += __shfl_xor_sync(0xffffffffu, nwb, o);
        nwe += __shfl_xor_sync(0xffffffffu, nwe, o);
        nwc += __shfl_xor_sync(0xffffffffu, nwc, o);
    }
    if (lane == 0) {
        st[threadIdx.x >> 5][0] = make_int4(gt, eqb, eqe, eqc);
        st[threadIdx.x >> 5][1] = make_int4(nwb, nwe, nwc, k0);
    }
    __syncthreads();
    // the CTA's groups' jobs: (group, tile) pairs, 256 threads at a time
    const int g0 = blockIdx.x * 8, ng = min(8, G - g0);
    for (int q = threadIdx.x; q < ng * J.ntiles; q += blockDim.x) {
        const int gl = q / J.ntiles, t = q - gl * J.ntiles;
        place_job(co, nch, g0 + gl, t, st[gl][0], st[gl][1], reinterpret_cast<int4 *>(jobs), J);
    }
}


}  // namespace

// Job count of a grid size for the given numbers of (example, channel) groups
// with and without items (gm_forward_jobs' table length).
long long forward_job_count(int D, long long work_groups, long long zero_groups) {
    const FwdConfig cfg = choose_config(D);
    const long long ntiles = (long long)((D + cfg.TI - 1) / cfg.TI) * ((D + cfg.TJ - 1) / cfg.TJ);
    return ntiles * work_groups + (ntiles + GM_FWD_ZGROUP - 1) / GM_FWD_ZGROUP * zero_groups;
}

gm_status forward_jobs_device(const gm_params *p, int nex, int nch, const int32_t *chan_off,
                              int32_t *jobs, long long work_groups, long long zero_groups,
                              int4 *stats, cudaStream_t s) {
    const int D = p->npts;
    const FwdConfig cfg = choose_config(D);
    JobGeom J;
    J.ntj = (D + cfg.TJ - 1) / cfg.TJ;
    J.ntiles = ((D + cfg.TI - 1) / cfg.TI) * J.ntj;
    J.TI = cfg.TI;
    J.TJ = cfg.TJ;
    J.reorder = D <= GM_FWD_LPT_MAXD ? GM_FWD_LPT : 0;
    J.W = (long long)J.ntiles * work_groups;
    J.Z = (J.ntiles + GM_FWD_ZGROUP - 1) / GM_FWD_ZGROUP * zero_groups;
    J.n = J.W + J.Z;
    // heavy slots of the deal: one per GM_FWD_ALT_H + GM_FWD_ALT_L, partial blocks included
    {
        const long long blk = GM_FWD_ALT_H + GM_FWD_ALT_L;
        J.H = J.W / blk * GM_FWD_ALT_H + std::min<long long>(J.W % blk, GM_FWD_ALT_H);
    }
    const int G = nex * nch;
    if (G == 0 || J.n == 0) return GM_OK;
    (void)stats;
    k_job_build<<<(G + 7) / 8, 256, 0, s>>>(chan_off, nex, nch, reinterpret_cast<int4 *>(jobs), J);
    LAUNCH_CHECK();
    return GM_OK;
}

gm_status forward_impl(const gm_params *p, const gm_batch *b, const Workspace &ws, float *out,
                       cudaStream_t s, bool *launched) {
    if (launched) *launched = false;
    const int D = p->npts;
    const FwdConfig cfg = choose_config(D);
    if (cfg.smem > 227 * 1024) return gm_fail(GM_ERR_INVALID, "grid too large for one tile row");
    FwdArgs A;
    // items sorted by first plane within each channel (k_sort_planes)
    const bool psort = use_plane_sort(p, b);
    A.sorted = psort ? ws.psorted : ws.sorted;
    A.bsorted = psort ? ws.pbsorted : ws.bsorted;
    A.sbox = psort ? ws.psbox : ws.sbox;
    A.poff = psort && kWarps == 1 ? ws.poff : nullptr;
    A.chan_off = ws.chan_off;
    A.origins = b->origins;
    A.out = out;
    A.res = p->resolution;
    A.resf = (float)p->resolution;
    A.resl = (float)(p->resolution - (double)A.resf);
    A.inv_res = (float)(1.0 / p->resolution);
    A.D = D;
    A.C = b->nchannels;
    A.TI = cfg.TI;
    A.TJ = cfg.TJ;
    A.ntj = (D + cfg.TJ - 1) / cfg.TJ;
    A.wpp = cfg.wpp;
    A.rpw = cfg.rpw;
    A.bulk = (D % 4) == 0 && ((uintptr_t)out % 16) == 0;
    A.acc_floats = cfg.acc_floats;
    A.ntiles = ((D + cfg.TI - 1) / cfg.TI) * A.ntj;
    // the job table carries the static grouping's item ranges: only with one
    const bool jobs = b->fwd_jobs && b->fwd_jobs_npts == D && b->nfwd_jobs >= 0 &&
                      b->item_perm && b->chan_off;
    A.jobs = jobs ? reinterpret_cast<const int4 *>(b->fwd_jobs) : nullptr;
    const int nj = jobs ? b->nfwd_jobs : 0;
    if (p->binary)
        return b->vector_mode ? launch<true, true, false>(A, cfg, b->nexamples, nj, s, launched)
                              : launch<true, false, false>(A, cfg, b->nexamples, nj, s, launched);
    // resolutions exactly representable in f32 (0.5, 0.25, 0.375 ...) drop the lo term
    return A.resl != 0.0f ? launch<false, false, true>(A, cfg, b->nexamples, nj, s, launched)
                          : launch<false, false, false>(A, cfg, b->nexamples, nj, s, launched);
}

// Job table of a static grouping: every tile of a channel with items, and the
// first tile of each GM_FWD_ZGROUP group of a zero slab -- none of the dense
// launch's CTAs that would only exit.  On small grids the scatter jobs are
// reordered by their channel's item count, alternating the heaviest and the
// lightest remaining job, so every wave mixes long scatter tiles with short
// store-bound ones and no many-item tile is left to close the launch; the zero
// groups are spread evenly between them so HBM keeps writing while SMs scatter.
int32_t forward_jobs_impl(const gm_params *p, int32_t nex, int32_t nch, const int32_t *co,
                          int32_t *jobs, int32_t cap) {
    const int D = p->npts;
    const FwdConfig cfg = choose_config(D);
    const int ntj = (D + cfg.TJ - 1) / cfg.TJ;
    const int ntiles = ((D + cfg.TI - 1) / cfg.TI) * ntj;
    struct Job { int32_t slab, tile, cs, ce; };
    std::vector<Job> work, zero;
    for (int e = 0; e < nex; e++)
        for (int t = 0; t < ntiles; t++)
            for (int c = 0; c < nch; c++) {
                const int cs = co[(size_t)e * (nch + 1) + c], ce = co[(size_t)e * (nch + 1) + c + 1];
                if (cs == ce) {
                    if (t % GM_FWD_ZGROUP == 0) zero.push_back({e * nch + c, t, cs, ce});
                } else {
                    work.push_back({e * nch + c, t, cs, ce});
                }
            }
    const long long n = (long long)work.size() + (long long)zero.size();
    if (n > 0x7fffffffLL || D > 0x7fff || nex > 0xffff || nch > 0x7fff)
        return -1;  // example | channel << 16 and plane | row << 16 must fit
    if (jobs && D <= GM_FWD_LPT_MAXD) {
#if GM_FWD_LPT
        // heaviest first within groups of GM_FWD_LPT_GROUP examples (0: globally)
        const int G = GM_FWD_LPT_GROUP > 0 ? GM_FWD_LPT_GROUP : std::max(nex, 1);
        std::stable_sort(work.begin(), work.end(), [=](const Job &a, const Job &b) {
            const int ga = a.slab / nch / G, gb = b.slab / nch / G;
            if (ga != gb) return ga < gb;
            return a.ce - a.cs > b.ce - b.cs;
        });
#if GM_FWD_LPT == 2
        // alternate the heavy and light ends of each group: every wave mixes
        // scatter-bound and store-bound tiles
        std::vector<Job> mixed;
        mixed.reserve(work.size());
        for (size_t g0 = 0; g0 < work.size();) {
            size_t g1 = g0;
            const int grp = work[g0].slab / nch / G;
            while (g1 < work.size() && work[g1].slab / nch / G == grp) g1++;
            size_t lo = g0, hi = g1;
            int phase = 0;  // GM_FWD_ALT_H heavy jobs, then GM_FWD_ALT_L light ones
            while (lo < hi) {
                const bool heavy = phase < GM_FWD_ALT_H;
                mixed.push_back(heavy ? work[lo++] : work[--hi]);
                phase = (phase + 1) % (GM_FWD_ALT_H + GM_FWD_ALT_L);
            }
            g0 = g1;
        }
        work.swap(mixed);
#endif
#endif
    }
    if (jobs) {
        size_t wi = 0, zi = 0;
        for (long long k = 0; k < n && k < cap; k++) {
            // zero job k' goes where the running share of zero jobs falls behind
#if GM_FWD_ZPLACE == 1  // zero groups first
            const bool z = zi < zero.size();
#elif GM_FWD_ZPLACE == 2  // zero groups last
            const bool z = wi >= work.size();
#else
            const bool z = zi < zero.size() &&
                           (wi >= work.size() || (zi + 1) * (double)n <= (k + 1) * (double)zero.size() + 1e-9);
#endif
            const Job &j = z ? zero[zi++] : work[wi++];
            int32_t *o = jobs + 4 * k;
            o[0] = (j.slab / nch) | ((j.slab % nch) << 16);  // example | channel << 16
            o[1] = j.cs;                                     // the channel's item range
            o[2] = j.ce;
            o[3] = ((j.tile / ntj) * cfg.TI) | (((j.tile % ntj) * cfg.TJ) << 16);
        }
    }
    return (int32_t)n;
}
