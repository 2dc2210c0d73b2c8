// forward.cu -- k_forward: typed items -> dense density grids.
//
// Reference: _kernels.py:33-113 (index), 116-206 (vector); each (example,
// channel) block of the output is the sum, in item order, of every item's
// density over its integer voxel box, rounded once to f32.
//
// Work decomposition (B200): one CTA per (example, channel, tile of TI planes
// x TJ rows x all D columns).  The tile accumulates in shared memory (dense
// [TI][TJ][D], <= 80 KB, 2 CTAs/SM).  The CTA reads only its channel's items
// (k_bin grouped them), keeps those whose box meets the tile (ordered ballot
// compaction into a shared list) and hands every warp a disjoint region of the
// tile (one plane, or a band of rows of one plane).  A warp walks the list in
// order and scatters each item's box cross-section into its region: lane ->
// (row offset, column) with the column fixed per item, so per voxel the work is
// one FMA for the row coordinate, d^2, exp2, rsqrt for the tail and a
// shared-memory accumulate.  Regions are disjoint and each warp adds items in
// order, so every voxel is summed in the reference's item order without
// atomics.  The finished tile (zeros included) is written with TMA bulk
// stores (cp.async.bulk) when D % 4 == 0: planes of the tile are contiguous in
// global memory.  CTAs whose channel has no items only stream zeros.
#include "common.cuh"

namespace {

constexpr int kThreads = 256;
constexpr int kWarps = kThreads / 32;
constexpr int kCap = 384;  // shared item-list capacity per round

struct FwdArgs {
    const FwdItem *sorted;
    const BinItem *bsorted;
    const int32_t *chan_off;
    const double *origins;
    float *out;
    double res;
    float resf, resl, inv_res;  // res = resf + resl
    int D, C, TI, TJ, ntj, wpp, rpw;
    int bulk;
    size_t acc_floats;
};

__device__ __forceinline__ void bulk_store(float *gdst, const float *ssrc, uint32_t bytes) {
    const uint32_t s = (uint32_t)__cvta_generic_to_shared(ssrc);
    asm volatile("cp.async.bulk.global.shared::cta.bulk_group [%0], [%1], %2;" ::"l"(gdst), "r"(s),
                 "r"(bytes)
                 : "memory");
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

// One item's contribution to a warp's region (plane i, rows [jg0, jg1]):
// the voxels of its box cross-section that can lie inside its cutoff sphere.
// Lane -> (row offset r, column kk), column fixed per item.
template <bool BINARY, bool VECTOR>
__device__ __forceinline__ void visit_item(const FwdItem &it, const BinItem &bi, int i, int jg0,
                                           int jg1, float *accw, int D, double res, float resf,
                                           float resl, float inv_res, double ox, double oy,
                                           double oz, int lane) {
    const int4 bx = *reinterpret_cast<const int4 *>(&it.ibox);
    const int ilo = box_lo(bx.x);
    if (i < ilo || i > box_hi(bx.x)) return;
    const int jlo_b = box_lo(bx.y), klo_b = box_lo(bx.z);
    const int jlo = max(jlo_b, jg0), jhi = min(box_hi(bx.y), jg1);
    if (jlo > jhi) return;
    const float4 P = *reinterpret_cast<const float4 *>(&it.cxh);
    const float4 Q = *reinterpret_cast<const float4 *>(&it.cxl);
    const float4 R = *reinterpret_cast<const float4 *>(&it.dzr);
    const float cut = R.x;
    // plane offset dx (f32, ~1 ulp) and the sphere cross-section radius
    const float fi = (float)(i - ilo);
    const float dx = fmaf(fi, resf, P.x) + fmaf(fi, resl, Q.x);
    const float rho2 = fmaf(-dx, dx, cut * cut);
    if (rho2 < -1e-5f * cut * cut) return;
    const float rho = fmaf(fast_sqrt(fmaxf(rho2, 0.0f)), 1.00002f, 1e-4f * cut);
    int jr0, jr1, kr0, kr1;
    sphere_span(P.y + Q.y, rho, inv_res, box_hi(bx.y) - jlo_b + 1, jr0, jr1);
    sphere_span(P.z + Q.z, rho, inv_res, box_hi(bx.z) - klo_b + 1, kr0, kr1);
    jr0 = max(jr0, jlo - jlo_b);
    jr1 = min(jr1, jhi - jlo_b);
    if (jr0 > jr1 || kr0 > kr1) return;
    const int nj = jr1 - jr0 + 1, nk = kr1 - kr0 + 1;
    float *arow = accw + (size_t)(jlo_b + jr0) * D + klo_b;
    if (BINARY) {
        // _kernels.py:87-98 (index) / 180-192 (vector): exact f64, no contraction
        const float w = R.z;
        const double dxd = __dsub_rn(__dadd_rn(ox, __dmul_rn((double)i, res)), bi.x);
        const double dx2 = __dmul_rn(dxd, dxd);
        for (int kb = 0; kb < nk; kb += 32) {
            const int nks = min(32, nk - kb);
            const float inv = __frcp_rn((float)nks);
            const int rpi = small_div(32, inv);
            const int r = small_div(lane, inv), kk = kr0 + kb + lane - r * nks;
            if (r >= rpi) continue;
            const double dz = __dsub_rn(__dadd_rn(oz, __dmul_rn((double)(klo_b + kk), res)), bi.z);
            const double dz2 = __dmul_rn(dz, dz);
            float *ap = arow + kk + (size_t)r * D;
            for (int jj = r; jj < nj; jj += rpi, ap += (size_t)rpi * D) {
                const double dy = __dsub_rn(
                    __dadd_rn(oy, __dmul_rn((double)(jlo_b + jr0 + jj), res)), bi.y);
                const double d2 = __dadd_rn(__dadd_rn(dx2, __dmul_rn(dy, dy)), dz2);
                if (d2 <= bi.r2) {
                    if (VECTOR) *ap = fmaxf(*ap, w);
                    else *ap = 1.0f;
                }
            }
        }
    } else {
        // _kernels.py:99-106: Gaussian core to d0, quadratic tail to the cutoff
        const float cexp = P.w, d02 = Q.w, qa = R.y, w = R.z;
        const float dx2 = dx * dx;
        for (int kb = 0; kb < nk; kb += 32) {
            const int nks = min(32, nk - kb);
            const float inv = __frcp_rn((float)nks);
            const int rpi = small_div(32, inv);
            const int r = small_div(lane, inv), kk = kr0 + kb + lane - r * nks;
            if (r >= rpi) continue;
            const float fk = (float)kk;
            const float dz = fmaf(fk, resf, P.z) + fmaf(fk, resl, Q.z);
            const float b2 = fmaf(dz, dz, dx2);
            const float rpif = (float)rpi;
            float *ap = arow + kk + (size_t)r * D;
            float jf = (float)(jr0 + r);
            for (int jj = r; jj < nj; jj += rpi, jf += rpif, ap += (size_t)rpi * D) {
                const float dy = fmaf(jf, resf, P.y) + fmaf(jf, resl, Q.y);
                const float d2 = fmaf(dy, dy, b2);
                const float g = fast_ex2(d2 * cexp);
                const float t = fmaxf(cut - fast_sqrt(d2), 0.0f);
                const float v = d2 <= d02 ? g : qa * t * t;
                *ap = fmaf(w, v, *ap);
            }
        }
    }
    __syncwarp();
}

template <bool BINARY, bool VECTOR>
__global__ void __launch_bounds__(kThreads, 2) k_forward(const FwdArgs A) {
    extern __shared__ __align__(128) unsigned char smem[];
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    const int c = blockIdx.x % A.C, tile = blockIdx.x / A.C, e = blockIdx.y;
    const int D = A.D, TI = A.TI, TJ = A.TJ;
    const int i0 = (tile / A.ntj) * TI, j0 = (tile % A.ntj) * TJ;
    const int TIv = min(TI, D - i0), TJv = min(TJ, D - j0);
    const size_t plane = (size_t)D * D;
    float *obase = A.out + ((size_t)e * A.C + c) * D * plane + (size_t)i0 * plane + (size_t)j0 * D;
    const int chunk = TJv * D;  // contiguous floats per plane of the tile (global and smem)
    const int32_t *co = A.chan_off + (size_t)e * (A.C + 1) + c;
    const int cs = co[0], ce = co[1];

    if (cs == ce) {  // no item of this channel: zeros
        if (A.bulk) {
            const float4 z = make_float4(0.f, 0.f, 0.f, 0.f);
            for (int p = 0; p < TIv; p++) {
                float4 *o = reinterpret_cast<float4 *>(obase + p * plane);
                for (int q = tid; q < (chunk >> 2); q += kThreads) __stcs(o + q, z);
            }
        } else {
            for (int p = 0; p < TIv; p++)
                for (int q = tid; q < chunk; q += kThreads) __stcs(obase + p * plane + q, 0.f);
        }
        return;
    }

    float *acc = reinterpret_cast<float *>(smem);
    FwdItem *list = reinterpret_cast<FwdItem *>(smem + A.acc_floats * 4);
    BinItem *blist = reinterpret_cast<BinItem *>(list + kCap);
    int *wcount = reinterpret_cast<int *>(BINARY ? (unsigned char *)(blist + kCap)
                                                 : (unsigned char *)blist);
    {
        const float4 z = make_float4(0.f, 0.f, 0.f, 0.f);
        float4 *a4 = reinterpret_cast<float4 *>(acc);
        for (int q = tid; q < (int)(A.acc_floats >> 2); q += kThreads) a4[q] = z;
    }

    // this warp's region: plane p, global rows [jg0, jg1]
    const int p = warp / A.wpp, part = warp - (warp / A.wpp) * A.wpp;
    const int i = i0 + p;
    const int jg0 = j0 + part * A.rpw, jg1 = j0 + min((part + 1) * A.rpw, TJv) - 1;
    const bool region_ok = p < TIv && jg0 <= jg1;
    float *accw = acc + (size_t)p * TJ * D - (size_t)j0 * D;  // accw[j * D + k]
    const double res = A.res;
    const float resf = A.resf, resl = A.resl, inv_res = A.inv_res;
    const double ox = A.origins[3 * e + 0], oy = A.origins[3 * e + 1], oz = A.origins[3 * e + 2];
    const int ti_hi = i0 + TIv - 1, tj_hi = j0 + TJv - 1;
    const unsigned lt = (1u << lane) - 1u;

    int count = 0;
    __syncthreads();
    for (int base = cs; base < ce; base += kThreads) {
        const int it = base + tid;
        bool keep = false;
        if (it < ce) {
            const int2 bx = *reinterpret_cast<const int2 *>(&A.sorted[it].ibox);
            keep = box_lo(bx.x) <= ti_hi && box_hi(bx.x) >= i0 && box_lo(bx.y) <= tj_hi &&
                   box_hi(bx.y) >= j0;
        }
        const unsigned m = __ballot_sync(0xffffffffu, keep);
        if (lane == 0) wcount[warp] = __popc(m);
        __syncthreads();
        int before = 0, total = 0;
#pragma unroll
        for (int w = 0; w < kWarps; w++) {
            const int n = wcount[w];
            before += (w < warp) ? n : 0;
            total += n;
        }
        if (keep) {
            const int pos = count + before + __popc(m & lt);
            list[pos] = A.sorted[it];
            if (BINARY) blist[pos] = A.bsorted[it];
        }
        count += total;
        __syncthreads();
        if (count > kCap - kThreads || base + kThreads >= ce) {
            if (region_ok) {
                for (int idx = 0; idx < count; idx++)
                    visit_item<BINARY, VECTOR>(list[idx], blist[idx], i, jg0, jg1, accw, D, res,
                                               resf, resl, inv_res, ox, oy, oz, lane);
            }
            __syncthreads();
            count = 0;
        }
    }

    // ---- the finished tile, zeros included ----
    if (A.bulk) {
        asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
        __syncthreads();
        if (tid == 0) {
            for (int pp = 0; pp < TIv; pp++)
                bulk_store(obase + pp * plane, acc + (size_t)pp * TJ * D, (uint32_t)chunk * 4u);
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

FwdConfig choose_config(int D, bool binary) {
    const size_t budget = 80 * 1024;
    const size_t plane = (size_t)D * D * 4;
    FwdConfig cfg{};
    int TI = 8;
    while (TI > 1 && (TI * plane > budget || TI > D)) TI >>= 1;
    cfg.TI = TI;
    cfg.wpp = kWarps / TI;
    int TJ = D;
    if (plane > budget) TJ = std::max(cfg.wpp, (int)(budget / ((size_t)D * 4)) / cfg.wpp * cfg.wpp);
    cfg.TJ = std::min(TJ, D);
    cfg.rpw = (cfg.TJ + cfg.wpp - 1) / cfg.wpp;
    cfg.acc_floats = align_up((size_t)cfg.TI * cfg.TJ * D, 32);
    cfg.smem = cfg.acc_floats * 4 + (size_t)kCap * (sizeof(FwdItem) + (binary ? sizeof(BinItem) : 0)) +
               64;
    return cfg;
}

template <bool BIN, bool VEC>
gm_status launch(const FwdArgs &A, const FwdConfig &cfg, int nex, cudaStream_t s) {
    auto kern = k_forward<BIN, VEC>;
    CUDA_TRY(gm_ensure_smem((const void *)kern, (int)cfg.smem));
    const int ntiles = ((A.D + cfg.TI - 1) / cfg.TI) * A.ntj;
    dim3 grid(ntiles * A.C, nex);
    kern<<<grid, kThreads, cfg.smem, s>>>(A);
    LAUNCH_CHECK();
    return GM_OK;
}

}  // namespace

gm_status forward_impl(const gm_params *p, const gm_batch *b, const Workspace &ws, float *out,
                       cudaStream_t s) {
    const int D = p->npts;
    const FwdConfig cfg = choose_config(D, p->binary != 0);
    if (cfg.smem > 227 * 1024) return gm_fail(GM_ERR_INVALID, "grid too large for one tile row");
    FwdArgs A;
    A.sorted = ws.sorted;
    A.bsorted = ws.bsorted;
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
    if (p->binary)
        return b->vector_mode ? launch<true, true>(A, cfg, b->nexamples, s)
                              : launch<true, false>(A, cfg, b->nexamples, s);
    return launch<false, false>(A, cfg, b->nexamples, s);
}
