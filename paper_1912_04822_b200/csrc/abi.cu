// abi.cu -- the C ABI (include/gridmaker_b200.h): argument checks, workspace
// carving and the reference-shaped host-buffer entry points.  Nothing here
// throws; every entry point returns a gm_status and records a message for
// gm_last_error().
#include <math.h>
#include <mutex>
#include <string>
#include <unordered_map>
#include <vector>

#include "common.cuh"

#define GM_VERSION "gridmaker_b200 0.3.0 (sm_100a)"

static thread_local std::string g_err;
static std::atomic<int64_t> g_launches{0};

gm_status gm_fail(gm_status code, const char *fmt, ...) {
    char buf[512];
    va_list ap;
    va_start(ap, fmt);
    vsnprintf(buf, sizeof buf, fmt, ap);
    va_end(ap);
    g_err = buf;
    return code;
}

void gm_count_launch() { g_launches.fetch_add(1, std::memory_order_relaxed); }

cudaError_t gm_ensure_smem(const void *func, int bytes) {
    static std::mutex mu;
    static std::vector<std::pair<std::pair<int, const void *>, int>> done;
    int dev = 0;
    cudaError_t e = cudaGetDevice(&dev);
    if (e != cudaSuccess) return e;
    std::lock_guard<std::mutex> lock(mu);
    for (auto &d : done)
        if (d.first.first == dev && d.first.second == func && d.second >= bytes) return cudaSuccess;
    e = cudaFuncSetAttribute(func, cudaFuncAttributeMaxDynamicSharedMemorySize, bytes);
    if (e == cudaSuccess) done.push_back({{dev, func}, bytes});
    return e;
}

int gm_persistent_blocks(const void *func, int threads, size_t smem) {
    static std::mutex mu;
    struct Entry { int dev; const void *f; int threads; size_t smem; int blocks; };
    static std::vector<Entry> done;
    int dev = 0;
    if (cudaGetDevice(&dev) != cudaSuccess) return 0;
    std::lock_guard<std::mutex> lock(mu);
    for (auto &d : done)
        if (d.dev == dev && d.f == func && d.threads == threads && d.smem == smem) return d.blocks;
    int sms = 0, per = 0;
    if (cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev) != cudaSuccess) return 0;
    if (cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per, func, threads, smem) != cudaSuccess)
        return 0;
    const int blocks = std::max(1, per) * sms;
    done.push_back({dev, func, threads, smem, blocks});
    return blocks;
}

static gm_status check_params(const gm_params *p) {
    if (!p) return gm_fail(GM_ERR_INVALID, "params is NULL");
    if (!(p->resolution > 0)) return gm_fail(GM_ERR_INVALID, "resolution must be > 0");
    if (p->npts < 1 || p->npts > 4096) return gm_fail(GM_ERR_INVALID, "npts %d out of range", p->npts);
    if (!(p->radius_multiple > 0)) return gm_fail(GM_ERR_INVALID, "radius_multiple must be > 0");
    return GM_OK;
}

static gm_status check_batch(const gm_batch *b) {
    if (!b) return gm_fail(GM_ERR_INVALID, "batch is NULL");
    if (b->nexamples < 0 || b->nsets < 0 || b->natoms < 0 || b->nitems < 0 || b->nchannels < 0)
        return gm_fail(GM_ERR_INVALID, "negative batch size");
    if (b->natoms > 0 && !b->coords32 && !b->coords64)
        return gm_fail(GM_ERR_INVALID, "batch has atoms but no coordinates");
    if (b->natoms > 0 && (!b->atom_set || !b->atom_radius || !b->set_example || !b->set_choff ||
                          !b->set_start || !b->set_end || !b->set_t))
        return gm_fail(GM_ERR_INVALID, "batch is missing atom/set arrays");
    if (b->nexamples > 0 && (!b->origins || !b->ex_item_start || !b->ex_item_end))
        return gm_fail(GM_ERR_INVALID, "batch is missing per-example arrays");
    if (b->nexamples > 65535) return gm_fail(GM_ERR_INVALID, "too many examples per launch");
    if (b->nchannels > 8192) return gm_fail(GM_ERR_INVALID, "too many channels");
    return GM_OK;
}

extern "C" size_t gm_workspace_bytes(int32_t natoms, int32_t nitems, int32_t nexamples,
                                     int32_t nchannels) {
    return carve_workspace(nullptr, natoms, nitems, nexamples, nchannels, nullptr);
}

// Which of our kernels last wrote / read a workspace (host-side launch order).
// k_backward_index reads its per-atom records before its PDL wait (the
// prologue overlaps the forward's tail).  That is only safe when the launch it
// follows cannot still be writing those records: the forward waits for the
// prepare pass before it triggers its dependents, the prepare pass triggers
// before its stores.  So the early prologue is allowed only when the last of
// our launches on this workspace was a forward.
enum WsState { WS_UNKNOWN = 0, WS_PREPARED = 1, WS_FORWARDED = 2 };
static std::mutex g_ws_mu;
static std::unordered_map<const void *, int> g_ws_state;

static void ws_mark(const void *workspace, int state) {
    std::lock_guard<std::mutex> lock(g_ws_mu);
    if (g_ws_state.size() > 4096 && !g_ws_state.count(workspace)) g_ws_state.clear();
    g_ws_state[workspace] = state;
}

static int ws_state(const void *workspace) {
    std::lock_guard<std::mutex> lock(g_ws_mu);
    auto it = g_ws_state.find(workspace);
    return it == g_ws_state.end() ? WS_UNKNOWN : it->second;
}

static Workspace ws_of(const void *workspace, const gm_batch *b) {
    Workspace w;
    carve_workspace(const_cast<void *>(workspace), b->natoms, b->nitems, b->nexamples,
                    b->nchannels, &w);
    return w;
}

extern "C" const double *gm_workspace_positions(const void *workspace) {
    return (const double *)workspace;  // positions are carved first
}

extern "C" gm_status gm_prepare(const gm_params *p, const gm_batch *b, void *workspace,
                                size_t workspace_bytes, void *stream) {
    gm_status st = check_params(p);
    if (st) return st;
    if ((st = check_batch(b))) return st;
    const size_t need = gm_workspace_bytes(b->natoms, b->nitems, b->nexamples, b->nchannels);
    if (!workspace || workspace_bytes < need)
        return gm_fail(GM_ERR_INVALID, "workspace too small (%zu < %zu)", workspace_bytes, need);
    if (!b->vector_mode && b->nitems != b->natoms)
        return gm_fail(GM_ERR_INVALID, "index mode needs one item per atom");
    if (b->nitems > 0 && !b->item_channel && !b->atom_type)
        return gm_fail(GM_ERR_INVALID, "items need item_channel or atom_type");
    ws_mark(workspace, WS_PREPARED);
    return prepare_impl(p, b, ws_of(workspace, b), (cudaStream_t)stream, true);
}

extern "C" gm_status gm_prepare_inline(const gm_params *p, const gm_batch *b, void *workspace,
                                       size_t workspace_bytes, const double *origins_host,
                                       const double *xforms_host, void *stream) {
    gm_status st = check_params(p);
    if (st) return st;
    if ((st = check_batch(b))) return st;
    if (!origins_host && b->nexamples > 0) return gm_fail(GM_ERR_INVALID, "origins_host is NULL");
    if (!b->origins && b->nexamples > 0) return gm_fail(GM_ERR_INVALID, "b->origins is NULL");
    const size_t need = gm_workspace_bytes(b->natoms, b->nitems, b->nexamples, b->nchannels);
    if (!workspace || workspace_bytes < need)
        return gm_fail(GM_ERR_INVALID, "workspace too small (%zu < %zu)", workspace_bytes, need);
    if (!b->vector_mode && b->nitems != b->natoms)
        return gm_fail(GM_ERR_INVALID, "index mode needs one item per atom");
    if (b->nitems > 0 && !b->item_channel && !b->atom_type)
        return gm_fail(GM_ERR_INVALID, "items need item_channel or atom_type");
    cudaStream_t s = (cudaStream_t)stream;
    ws_mark(workspace, WS_PREPARED);
    if (b->item_perm && b->chan_off && b->nexamples <= GM_INLINE_MAX_EXAMPLES)
        return prepare_inline_impl(p, b, ws_of(workspace, b), origins_host, xforms_host, s);
    // general path: stage the per-call arrays, then the per-example grouping pass
    if (xforms_host && !b->xforms) return gm_fail(GM_ERR_INVALID, "b->xforms is NULL");
    if (b->nexamples > 0) {
        CUDA_TRY(cudaMemcpyAsync(const_cast<double *>(b->origins), origins_host,
                                 sizeof(double) * 3 * b->nexamples, cudaMemcpyHostToDevice, s));
        if (xforms_host)
            CUDA_TRY(cudaMemcpyAsync(const_cast<double *>(b->xforms), xforms_host,
                                     sizeof(double) * 15 * b->nexamples, cudaMemcpyHostToDevice,
                                     s));
    }
    gm_batch bb = *b;
    if (!xforms_host) bb.xforms = nullptr;
    return prepare_impl(p, &bb, ws_of(workspace, b), s, true);
}

extern "C" int32_t gm_forward_jobs(const gm_params *p, int32_t nexamples, int32_t nchannels,
                                   const int32_t *chan_off_host, int32_t *jobs_out,
                                   int32_t capacity) {
    if (check_params(p) != GM_OK || nexamples < 0 || nchannels < 0 || capacity < 0 ||
        (nexamples > 0 && !chan_off_host))
        return -1;
    return forward_jobs_impl(p, nexamples, nchannels, chan_off_host, jobs_out, capacity);
}

extern "C" gm_status gm_forward(const gm_params *p, const gm_batch *b, const void *workspace,
                                float *out, void *stream) {
    gm_status st = check_params(p);
    if (st) return st;
    if ((st = check_batch(b))) return st;
    if (b->nexamples == 0 || b->nchannels == 0) return GM_OK;
    if (!out) return gm_fail(GM_ERR_INVALID, "out is NULL");
    if (!workspace) return gm_fail(GM_ERR_INVALID, "workspace is NULL");
    bool launched = false;
    st = forward_impl(p, b, ws_of(workspace, b), out, (cudaStream_t)stream, &launched);
    // an empty job table launches nothing: the prepare pass may still be running
    if (st == GM_OK && launched) ws_mark(workspace, WS_FORWARDED);
    return st;
}

gm_status assemble_impl(const gm_params *p, const gm_dataset *ds, const int32_t *ids, int32_t n,
                        gm_batch *b, const gm_capacity *cap, int32_t *jobs, cudaStream_t s);

extern "C" gm_status gm_assemble(const gm_params *p, const gm_dataset *ds, const int32_t *ids,
                                 int32_t n, gm_batch *b, const gm_capacity *cap, int32_t *jobs,
                                 void *stream) {
    gm_status st = check_params(p);
    if (st) return st;
    if (!ds || !b || !ids || !jobs || !cap) return gm_fail(GM_ERR_INVALID, "NULL argument");
    if (!ds->records || !ds->ex_atom_off || !ds->ex_set_off || !ds->ex_chan_off || !ds->set_aoff ||
        !ds->set_natoms || !ds->set_choff || !ds->set_t || !ds->h_ex_atom_off ||
        !ds->h_ex_set_off || !ds->h_ex_nzch || !ds->h_ex_maxch)
        return gm_fail(GM_ERR_INVALID, "dataset is missing arrays");
    if (ds->nchannels < 1 || ds->nchannels > 8192)
        return gm_fail(GM_ERR_INVALID, "dataset channel count %d", ds->nchannels);
    if (!b->coords32 || !b->atom_radius || !b->atom_set || !b->set_start || !b->set_end ||
        !b->set_example || !b->set_choff || !b->set_t || !b->ex_item_start || !b->ex_item_end ||
        !b->item_perm || !b->chan_off || !b->bwd_slot || !b->segs)
        return gm_fail(GM_ERR_INVALID, "batch is missing device arrays");
    if (!ds->vector_mode && (!b->atom_type || !b->slot_rec))
        return gm_fail(GM_ERR_INVALID, "index-mode batch needs atom_type and slot_rec");
    if (ds->vector_mode &&
        (!ds->items || !ds->weights || !ds->type_radii || !ds->ex_item_off || !ds->ex_w_off ||
         !ds->ex_tr_off || !ds->set_woff || !ds->set_troff || !ds->h_ex_item_off ||
         !ds->h_ex_w_off || !ds->h_ex_tr_off || !b->set_wstart || !b->set_trstart ||
         !b->weights || !b->type_radius || !b->item_atom || !b->item_channel ||
         !b->item_weight || !b->item_radius))
        return gm_fail(GM_ERR_INVALID, "vector-mode dataset / batch is missing arrays");
    return assemble_impl(p, ds, ids, n, b, cap, jobs, (cudaStream_t)stream);
}

gm_status molc_decode_impl(const uint8_t *raw, const int64_t *entry_start, int32_t nentries,
                           const int16_t *type_table, const float *type_radii, float *coords,
                           int32_t *type_index, float *radius, int64_t *offsets, cudaStream_t s);

extern "C" gm_status gm_molc_decode(const uint8_t *raw, const int64_t *entry_start, int32_t nentries,
                                    const int16_t *type_table, const float *type_radii,
                                    float *coords, int32_t *type_index, float *radius,
                                    int64_t *offsets, void *stream) {
    if (nentries < 0) return gm_fail(GM_ERR_INVALID, "nentries %d < 0", nentries);
    if (!offsets || (nentries > 0 && (!raw || !entry_start || !type_table || !type_radii ||
                                      !coords || !type_index || !radius)))
        return gm_fail(GM_ERR_INVALID, "NULL argument");
    return molc_decode_impl(raw, entry_start, nentries, type_table, type_radii, coords, type_index,
                            radius, offsets, (cudaStream_t)stream);
}

extern "C" gm_status gm_backward(const gm_params *p, const gm_batch *b, const void *workspace,
                                 const float *grid_grad, float *coord_grad, float *type_grad,
                                 void *stream) {
    gm_status st = check_params(p);
    if (st) return st;
    if ((st = check_batch(b))) return st;
    if (b->natoms == 0) return GM_OK;
    if (!coord_grad) return gm_fail(GM_ERR_INVALID, "coord_grad is NULL");
    cudaStream_t s = (cudaStream_t)stream;
    if (p->binary) {
        // voxelizer.py:284-289: binary grids are flat almost everywhere
        CUDA_TRY(cudaMemsetAsync(coord_grad, 0, sizeof(float) * 3 * (size_t)b->natoms, s));
        if (b->vector_mode && type_grad && b->nweights > 0)
            CUDA_TRY(cudaMemsetAsync(type_grad, 0, sizeof(float) * (size_t)b->nweights, s));
        return GM_OK;
    }
    if (!grid_grad || !workspace) return gm_fail(GM_ERR_INVALID, "grid_grad/workspace is NULL");
    if (!b->vector_mode && !b->atom_type) return gm_fail(GM_ERR_INVALID, "atom_type is NULL");
    if (b->vector_mode && (!b->weights || !b->set_wstart))
        return gm_fail(GM_ERR_INVALID, "vector backward needs weights and set_wstart");
    if (b->vector_mode && p->radius_type_indexed && (!b->type_radius || !b->set_trstart))
        return gm_fail(GM_ERR_INVALID, "radius_type_indexed needs type_radius and set_trstart");
    const bool early = ws_state(workspace) == WS_FORWARDED;
    return backward_impl(p, b, ws_of(workspace, b), grid_grad, coord_grad, type_grad, s, early);
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
    const size_t ws_bytes = gm_workspace_bytes((int32_t)natoms, nitems, (int32_t)nexamples, (int32_t)nch);
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
    b.max_example_items = 0;
    for (size_t e = 0; e < ex_start.size(); e++)
        b.max_example_items = std::max(b.max_example_items, ex_end[e] - ex_start[e]);
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
            return gm_fail(GM_ERR_INVALID, "set %lld has a bad atom range", (long long)s);
        if (set_example[s] < prev_e || set_example[s] >= nexamples)
            return gm_fail(GM_ERR_INVALID, "sets must be grouped by example in order");
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
        return gm_fail(GM_ERR_INVALID, "NULL argument");
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
        return gm_fail(GM_ERR_INVALID, "NULL argument");
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
                if (wi < 0 || wi >= nweights) return gm_fail(GM_ERR_INVALID, "weight index out of range");
                const double w = weights_flat[wi];
                if (w == 0.0) continue;  // _kernels.py:164
                double r = atom_radii[a];
                if (radius_type_indexed) {
                    const int64_t ti = tr_start[s] + c;
                    if (!type_radii_flat || ti < 0 || ti >= ntype_radii)
                        return gm_fail(GM_ERR_INVALID, "type radius index out of range");
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
    const size_t ws_bytes = gm_workspace_bytes((int32_t)n, (int32_t)n, 1, (int32_t)nt);
    const size_t o_ws = plan.add(nullptr, ws_bytes);
    // f64 outputs: the numba kernels return their f64 sums (_kernels.py:214,265-266)
    const size_t o_cg = plan.add(nullptr, sizeof(double) * 3 * n);
    const size_t o_tg = plan.add(nullptr, sizeof(double) * (vector_mode ? n * nt : 1));
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
    b.max_example_items = (int32_t)n;
    b.origins = (const double *)(d + o_orig);
    gm_params p = host_params(npts, res, grm, rmult, 0, rti);
    // positions only (no transform); items are not needed by the backward
    // index mode: the backward reuses the forward items' boxes
    gm_status st = prepare_impl(&p, &b, ws_of(d + o_ws, &b), nullptr, !vector_mode);
    if (st) return st;
    st = backward_impl(&p, &b, ws_of(d + o_ws, &b), (const float *)(d + o_gg), nullptr, nullptr,
                       nullptr, false, (double *)(d + o_cg),
                       vector_mode ? (double *)(d + o_tg) : nullptr);
    if (st) return st;
    CUDA_TRY(cudaMemcpy(coord_grad, d + o_cg, sizeof(double) * 3 * n, cudaMemcpyDeviceToHost));
    if (vector_mode)
        CUDA_TRY(cudaMemcpy(type_grad, d + o_tg, sizeof(double) * n * nt, cudaMemcpyDeviceToHost));
    return GM_OK;
}

extern "C" gm_status gm_backward_index_host(double *coord_grad, const double *coords,
                                            const double *radii, const int64_t *tidx, int64_t n,
                                            const float *grid_grad, int64_t ntypes, int64_t npts,
                                            const double *origin, double res, double grm,
                                            double rmult) {
    if (n && (!coord_grad || !coords || !radii || !tidx || !grid_grad || !origin))
        return gm_fail(GM_ERR_INVALID, "NULL argument");
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
        return gm_fail(GM_ERR_INVALID, "NULL argument");
    return run_host_backward(coord_grad, type_grad, coords, atom_radii, nullptr, weights, n, nt,
                             grid_grad, npts, type_radii, rti, origin, res, grm, rmult);
}

extern "C" gm_status gm_draw_transforms(const double *u, int64_t n, int32_t rotation,
                                        double translation, const double *centers,
                                        double *out) {
    if (n < 0 || (n > 0 && (!out || !centers))) return gm_fail(GM_ERR_INVALID, "NULL argument");
    const int k = (rotation ? 3 : 0) + (translation > 0 ? 3 : 0);
    if (n > 0 && k > 0 && !u) return gm_fail(GM_ERR_INVALID, "uniforms are NULL");
    const double tau = 2.0 * M_PI;
    for (int64_t e = 0; e < n; e++) {
        const double *ue = u + e * k;
        double *o = out + e * 15;
        if (rotation) {
            // geom.py:73-76 (Shoemake) and 28-36 (renormalise if |n-1| > 1e-6)
            const double a = sqrt(1.0 - ue[0]), b = sqrt(ue[0]);
            const double t2 = tau * ue[1], t3 = tau * ue[2];
            double w = b * cos(t3), x = a * sin(t2), y = a * cos(t2), z = b * sin(t3);
            const double nrm = sqrt(((pow(w, 2.0) + pow(x, 2.0)) + pow(y, 2.0)) + pow(z, 2.0));
            if (fabs(nrm - 1.0) > 1e-6) {
                w /= nrm;
                x /= nrm;
                y /= nrm;
                z /= nrm;
            }
            // geom.py:53-57
            o[0] = 1.0 - 2.0 * (y * y + z * z);
            o[1] = 2.0 * (x * y - z * w);
            o[2] = 2.0 * (x * z + y * w);
            o[3] = 2.0 * (x * y + z * w);
            o[4] = 1.0 - 2.0 * (x * x + z * z);
            o[5] = 2.0 * (y * z - x * w);
            o[6] = 2.0 * (x * z - y * w);
            o[7] = 2.0 * (y * z + x * w);
            o[8] = 1.0 - 2.0 * (x * x + y * y);
        } else {
            for (int q = 0; q < 9; q++) o[q] = (q % 4 == 0) ? 1.0 : 0.0;
        }
        o[9] = centers[3 * e];
        o[10] = centers[3 * e + 1];
        o[11] = centers[3 * e + 2];
        const int c = rotation ? 3 : 0;
        for (int q = 0; q < 3; q++)
            o[12 + q] = translation > 0 ? -translation + (2.0 * translation) * ue[c + q] : 0.0;
    }
    return GM_OK;
}

extern "C" const char *gm_last_error(void) { return g_err.c_str(); }
extern "C" const char *gm_version(void) { return GM_VERSION; }
extern "C" int32_t gm_device_count(void) {
    int n = 0;
    if (cudaGetDeviceCount(&n) != cudaSuccess) return 0;
    return n;
}
extern "C" int32_t gm_struct_size(int32_t which) {
    return which == 0   ? (int32_t)sizeof(gm_params)
           : which == 1 ? (int32_t)sizeof(gm_batch)
           : which == 2 ? (int32_t)sizeof(gm_dataset)
           : which == 3 ? (int32_t)sizeof(gm_capacity)
           : which == 4 ? (int32_t)sizeof(gm_pack_set)
           : which == 5 ? (int32_t)sizeof(gm_pack_layout)
           : which == 6 ? (int32_t)sizeof(gm_pack_info)
           : which == 7 ? (int32_t)sizeof(gm_pack_vset)
           : which == 8 ? (int32_t)sizeof(gm_pack_vlayout)
                        : -1;
}
extern "C" int64_t gm_launch_count(int32_t reset) {
    return reset ? g_launches.exchange(0) : g_launches.load();
}
