/*
 * gridmaker_b200.h -- C ABI of the B200 GridMaker hot path.
 *
 * Drop-in boundary for the reference's kernel layer
 * (/root/reference/pkg/src/voxmol/_kernels.py), which voxelizer.py calls with
 * packed CSR arrays (voxelizer.py:372-435 forward, 293-300 backward).  Every
 * entry point uses plain pointers and sizes; no C++ or torch types cross the
 * boundary, nothing throws, and every function returns a gm_status (0 = OK,
 * details from gm_last_error()).
 *
 * Two groups of entry points:
 *
 * 1. Reference-shaped kernels, same argument meaning as _kernels.py:
 *      gm_forward_index_sets   <- _kernels.forward_index_sets  (_kernels.py:33-36)
 *      gm_forward_vector_sets  <- _kernels.forward_vector_sets (_kernels.py:116-120)
 *      gm_backward_index       <- _kernels.backward_index      (_kernels.py:209-210)
 *      gm_backward_vector      <- _kernels.backward_vector     (_kernels.py:258-260)
 *    The *_host variants take HOST (numpy) buffers exactly like the numba
 *    kernels and do the host<->device copies internally (what a ctypes shim in
 *    voxelizer.py binds).  The *_dev variants take device
 *    pointers and a cudaStream_t (as void*).
 *
 * 2. The fused batch path used by the Python GridMaker (device pointers):
 *      gm_workspace_bytes, gm_prepare (transform + localise + boxes),
 *      gm_forward, gm_backward (batched over every set of every example).
 *
 * Layouts (C order): out / grid_grad (nexamples, nchannels, D, D, D) float32
 * with k (z) contiguous, i.e. out[e][c][i][j][k] at voxel
 * origin + res*(i, j, k) (_kernels.py:86-113).
 */
#ifndef GRIDMAKER_B200_H
#define GRIDMAKER_B200_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

typedef int gm_status;
#define GM_OK 0
#define GM_ERR_INVALID 1   /* bad argument (null pointer, size, mode) */
#define GM_ERR_CUDA 2      /* CUDA launch / copy / allocation failure */

/* Gridding parameters (GridMaker fields, voxelizer.py:97-105, plus derived). */
typedef struct {
    double resolution;               /* grid spacing (A) */
    double dimension;                /* cube side (A) */
    double radius_scale;             /* multiplies atom / type radii */
    double gaussian_radius_multiple; /* grm */
    double radius_multiple;          /* (1 + 2 grm^2) / (2 grm), voxelizer.py:148-152 */
    int32_t npts;                    /* D = floor(dimension/resolution + 0.5) + 1 */
    int32_t binary;                  /* 0/1 */
    int32_t radius_type_indexed;     /* 0/1 (vector mode only) */
    int32_t matmul_order_1;          /* FMA order of numpy (1,3)@(3,3), -1 = default */
    int32_t matmul_order_n;          /* FMA order of numpy (N,3)@(3,3), N >= 2 */
} gm_params;

/* A packed batch in device memory (CSR over sets, like voxelizer._run_batch).
 * Sets of one example are consecutive; atoms of one set are consecutive;
 * items (see below) of one example are consecutive. */
typedef struct {
    int32_t nexamples, nsets, natoms, nitems, nchannels;
    int32_t vector_mode;             /* 0: index types, 1: type_vector weights */
    /* atoms */
    const float *coords32;           /* (natoms,3) input frame, or NULL */
    const double *coords64;          /* (natoms,3) input frame, or NULL */
    const double *atom_radius;       /* (natoms) radius * radius_scale (f64) */
    const int32_t *atom_set;         /* (natoms) packed set index */
    const int32_t *atom_type;        /* (natoms) type index (index mode) */
    /* sets */
    const int32_t *set_start, *set_end, *set_example, *set_choff, *set_t; /* (nsets) */
    const int32_t *set_wstart;       /* (nsets) offset of the set's weight rows (vector) */
    const float *weights;            /* packed (atoms x T) rows per set (vector) */
    int32_t nweights;                /* total packed weight / type-gradient entries */
    const double *type_radius;       /* packed per set at set_trstart, scaled (vector) */
    const int32_t *set_trstart;      /* (nsets) */
    /* forward items: index mode -> one per atom (item_atom may be NULL = identity);
     * vector mode -> one per nonzero weight, atom-major then channel. */
    const int32_t *item_atom;        /* (nitems) or NULL */
    const int32_t *item_channel;     /* (nitems) channel within the set, or NULL = atom_type */
    const float *item_weight;        /* (nitems) or NULL = 1 */
    const double *item_radius;       /* (nitems) scaled radius, or NULL = atom_radius */
    const int32_t *ex_item_start, *ex_item_end; /* (nexamples) */
    int32_t max_example_items;       /* max over examples of (ex_item_end - ex_item_start) */
    /* per example */
    const double *origins;           /* (nexamples,3) center - dimension/2 */
    const double *xforms;            /* (nexamples,15) R row-major, center, translation; NULL = none */
    /* optional static grouping, computed once when the batch is packed (or NULL):
     * item_perm (nitems) lists example e's items in (channel, item) order in
     * slots [ex_item_start[e], ex_item_end[e]); chan_off (nexamples, nchannels+1)
     * holds each channel's absolute slot range.  With both, gm_prepare_inline is
     * one fully parallel pass. */
    const int32_t *item_perm;
    const int32_t *chan_off;
    /* optional forward job table (device, 4 int32 per job: example | channel
     * << 16, the channel's first and end item of the static grouping, first
     * plane | first row << 16), built by gm_forward_jobs
     * from the static chan_off for grids of fwd_jobs_npts points per side: only
     * tiles of channels with items plus one job per group of zero tiles are
     * launched.  Used only with a static grouping (item_perm, chan_off), whose
     * ranges the table carries.  NULL / 0 = one CTA per (channel, tile, example). */
    const int32_t *fwd_jobs;
    int32_t nfwd_jobs;
    int32_t fwd_jobs_npts;
    /* optional (natoms) index-mode backward launch slot of each atom (a
     * permutation), or NULL = atom order.  Cost-balanced orders shorten the
     * backward's tail; results do not depend on it. */
    const int32_t *bwd_slot;
    /* optional (nitems) index-mode slot records of the static grouping, 48 B each
     * in item_perm order: f32 x, y, z; int32 atom, absolute channel, example,
     * single-atom-set flag, backward slot; f64 radius * scale; 8 B pad.
     * Lets gm_prepare_inline start from one coalesced load per item. */
    const void *slot_rec;
    /* optional static list of the (example * nchannels + channel) groups that
     * have items (nsegs entries): the per-channel plane sort of the prepare
     * pass (fine grids, vector typing) then launches one CTA per listed group
     * instead of one per (example, channel). */
    const int32_t *segs;
    int32_t nsegs;
    /* optional: the largest item count of any (example, channel) group, or 0 =
     * unknown.  Sizes the plane sort's CTAs (small groups: small CTAs, one wave). */
    int32_t max_seg_items;
} gm_batch;

/* Device scratch needed by gm_prepare / gm_forward / gm_backward. */
size_t gm_workspace_bytes(int32_t natoms, int32_t nitems, int32_t nexamples, int32_t nchannels);

gm_status gm_prepare(const gm_params *p, const gm_batch *b, void *workspace,
                     size_t workspace_bytes, void *stream);
/* gm_prepare with the per-call arrays in HOST memory: origins_host (nexamples,3)
 * and xforms_host (nexamples,15) or NULL.  With a static grouping (item_perm,
 * chan_off) and nexamples <= GM_INLINE_MAX_EXAMPLES they travel inside the
 * kernel launch (no separate copy; the host arrays may be reused as soon as the
 * call returns); otherwise they are copied to b->origins / b->xforms first.
 * b->origins must be a device buffer of (nexamples,3) either way: the prepare
 * pass stores the origins there for gm_forward / gm_backward. */
#define GM_INLINE_MAX_EXAMPLES 200
gm_status gm_prepare_inline(const gm_params *p, const gm_batch *b, void *workspace,
                            size_t workspace_bytes, const double *origins_host,
                            const double *xforms_host, void *stream);
/* Forward job table for a static grouping (host memory): chan_off_host is the
 * (nexamples, nchannels+1) item ranges of gm_batch.chan_off.  Writes up to
 * capacity jobs (4 int32 each) to jobs_out (may be NULL) and returns the job
 * count, or -1 on invalid arguments.  Replaces the reference's dense launch over
 * every (set, channel) (_kernels.py:40-47) by the tiles that have items. */
int32_t gm_forward_jobs(const gm_params *p, int32_t nexamples, int32_t nchannels,
                        const int32_t *chan_off_host, int32_t *jobs_out, int32_t capacity);
/* out: (nexamples, nchannels, D, D, D) f32 device; every voxel is written. */
gm_status gm_forward(const gm_params *p, const gm_batch *b, const void *workspace,
                     float *out, void *stream);
/* grid_grad: (nexamples, nchannels, D, D, D) f32 device.
 * coord_grad: (natoms,3) f32 device, in the frame of the prepared coordinates.
 * type_grad: (sum over sets of atoms*T) f32 device packed like weights (vector), or NULL. */
gm_status gm_backward(const gm_params *p, const gm_batch *b, const void *workspace,
                      const float *grid_grad, float *coord_grad, float *type_grad,
                      void *stream);
/* Transformed coordinates computed by gm_prepare: (natoms,3) f64 device view. */
const double *gm_workspace_positions(const void *workspace);

/* ---- device-resident datasets: batch assembly on the device ----
 *
 * Replaces the per-call host packing of the reference's GridMaker._run_batch
 * (voxelizer.py:372-435, fed by ExampleProvider.next_batch, sampling.py:364-380)
 * for examples already resident in HBM: a batch is an index list, and
 * gm_assemble builds the index-mode gm_batch arrays (sets, channel grouping,
 * slot records, launch order) and the forward job table on the device.
 *
 * Dataset atom record (32 B, gm_dataset.records), per example in channel order
 * (stable: atom order within a channel): f32 x, y, z, radius (unscaled);
 * int32 local atom index (set order), absolute channel within the example,
 * local backward launch rank, local set index | single-atom-set flag << 16. */
typedef struct {
    int32_t nexamples;               /* examples in the dataset */
    int32_t nchannels;               /* channels of every example */
    int32_t natoms, nsets;           /* totals */
    const void *records;             /* device (natoms) 32-B atom records */
    const int32_t *ex_atom_off;      /* device (nexamples+1) record offsets */
    const int32_t *ex_set_off;       /* device (nexamples+1) set-table offsets */
    const int32_t *ex_chan_off;      /* device (nexamples*(nchannels+1)), local to the example */
    const int32_t *set_aoff;         /* device (nsets) first atom of the set, local */
    const int32_t *set_natoms, *set_choff, *set_t; /* device (nsets) */
    /* host mirrors (batch sizes are computed on the host without a sync) */
    const int32_t *h_ex_atom_off;    /* (nexamples+1) */
    const int32_t *h_ex_set_off;     /* (nexamples+1) */
    const int32_t *h_ex_nzch;        /* (nexamples) channels with atoms */
    const int32_t *h_ex_maxch;       /* (nexamples) largest channel (items in vector mode) */
    /* vector typing (vector_mode = 1): records are in SET order (their channel
     * field is unused); items are the nonzero weights, per example in item
     * order (atom-major, channel-minor per set, _kernels.py:159-166), 16 B each:
     * int32 local atom, channel within the set, f32 weight, the item's slot in
     * the example's channel grouping; ex_chan_off counts ITEMS; weight rows and
     * type radii per set as the CoordinateSets hold them (f32, unscaled). */
    int32_t vector_mode;
    int32_t nitems, nweights, ntype_radii; /* totals */
    const void *items;               /* device (nitems) */
    const float *weights;            /* device (nweights) */
    const float *type_radii;         /* device (ntype_radii) */
    const int32_t *ex_item_off, *ex_w_off, *ex_tr_off; /* device (nexamples+1) */
    const int32_t *set_woff, *set_troff; /* device (nsets), local to the example */
    const int32_t *h_ex_item_off, *h_ex_w_off, *h_ex_tr_off; /* host mirrors (nexamples+1) */
} gm_dataset;

/* Capacities of the caller's batch arrays for gm_assemble. */
typedef struct {
    int32_t atoms, sets, items, weights, type_radii; /* items: vector mode (index: = atoms) */
    int32_t jobs;                    /* forward job table entries (4 int32 each) + 2 per group */
} gm_capacity;

/* Assemble dataset examples ids[0..n) (host array) into the batch b: the
 * caller fills b's device array pointers with room for cap's counts --
 * index mode: coords32, atom_radius, atom_set, atom_type, set_start/end/
 * example/choff/t, ex_item_start/end, item_perm, chan_off, bwd_slot,
 * slot_rec, segs (n*nchannels), origins; vector mode: coords32, atom_radius,
 * atom_set, set_*, set_wstart, set_trstart, weights, type_radius, item_atom,
 * item_channel, item_weight, item_radius, ex_item_start/end, item_perm,
 * chan_off, bwd_slot, segs, origins.  gm_assemble writes the arrays on
 * `stream`, sets b's counts (nexamples, nsets, natoms, nitems, nweights,
 * nchannels, vector_mode, max_example_items, nsegs, max_seg_items) and its
 * forward job table (jobs: device, cap->jobs entries of 4 int32 -- the same
 * table gm_forward_jobs builds on the host).  Radii (and type radii) are
 * scaled by p->radius_scale in f64 like voxelizer.py:416,430; item radii
 * follow p->radius_type_indexed.  The batch equals the host packing of the
 * same examples (index mode: up to the backward launch order, per example
 * here, which never changes results). */
gm_status gm_assemble(const gm_params *p, const gm_dataset *ds, const int32_t *ids, int32_t n,
                      gm_batch *b, const gm_capacity *cap, int32_t *jobs, void *stream);

/* ---- reference-shaped kernels (argument meaning as _kernels.py) ---- */

/* _kernels.forward_index_sets(out, coords, radii, tidx, set_start, set_end,
 *   set_example, set_choff, set_t, origins, res, grm, rmult, binary)
 * out (nexamples, nch, npts^3) f32 (pre-zeroing not required: every voxel is
 * written); coords (natoms,3) f64; radii (natoms) f64 scaled; tidx/set_* int64. */
gm_status gm_forward_index_sets_host(float *out, int64_t nexamples, int64_t nch, int64_t npts,
                                     const double *coords, const double *radii,
                                     const int64_t *tidx, int64_t natoms,
                                     const int64_t *set_start, const int64_t *set_end,
                                     const int64_t *set_example, const int64_t *set_choff,
                                     const int64_t *set_t, int64_t nsets,
                                     const double *origins, double res, double grm,
                                     double rmult, int32_t binary);

/* _kernels.forward_vector_sets(out, coords, weights_flat, w_start, atom_radii,
 *   type_radii_flat, tr_start, radius_type_indexed, set_start, set_end,
 *   set_example, set_choff, set_t, origins, res, grm, rmult, binary) */
gm_status gm_forward_vector_sets_host(float *out, int64_t nexamples, int64_t nch, int64_t npts,
                                      const double *coords, int64_t natoms,
                                      const double *weights_flat, int64_t nweights,
                                      const int64_t *w_start, const double *atom_radii,
                                      const double *type_radii_flat, int64_t ntype_radii,
                                      const int64_t *tr_start, int32_t radius_type_indexed,
                                      const int64_t *set_start, const int64_t *set_end,
                                      const int64_t *set_example, const int64_t *set_choff,
                                      const int64_t *set_t, int64_t nsets,
                                      const double *origins, double res, double grm,
                                      double rmult, int32_t binary);

/* _kernels.backward_index(coords, radii, tidx, grid_grad, origin, res, grm, rmult)
 * -> coord_grad (n,3) f64 (written to the caller's buffer). grid_grad (ntypes, npts^3) f32. */
gm_status gm_backward_index_host(double *coord_grad, const double *coords, const double *radii,
                                 const int64_t *tidx, int64_t n, const float *grid_grad,
                                 int64_t ntypes, int64_t npts, const double *origin,
                                 double res, double grm, double rmult);

/* _kernels.backward_vector(coords, atom_radii, weights, grid_grad, type_radii,
 *   radius_type_indexed, origin, res, grm, rmult) -> (coord_grad (n,3), type_grad (n,nt)) f64 */
gm_status gm_backward_vector_host(double *coord_grad, double *type_grad, const double *coords,
                                  const double *atom_radii, const double *weights, int64_t n,
                                  int64_t nt, const float *grid_grad, int64_t npts,
                                  const double *type_radii, int32_t radius_type_indexed,
                                  const double *origin, double res, double grm, double rmult);

/* ---- host packing of an index-typed batch ----
 *
 * GridMaker._run_batch's CSR packing (voxelizer.py:372-435) plus this
 * library's static grouping, slot records and backward launch order, written
 * by one native pass into the caller's image of a gm_batch (e.g. the pinned
 * buffer it then copies to the device once).  sets: in example order; each
 * set's coords (n,3) f32, radii (n) f32 (unscaled), type_index (n) int64 in
 * [0, num_types).  centers: (nexamples,3) f64 default centers (launch-order
 * key only).  layout: byte offsets into dst of each array (sizes: atoms,
 * sets, nexamples, nexamples*(nchannels+1), segs nexamples*nchannels at most;
 * bwd_slot -1 = no launch order).  bwd_order: 0 atom order, 1 slab order.
 * Writes info (natoms, groups with items, largest group, largest example). */
typedef struct {
    const float *coords;
    const float *radii;
    const int64_t *type_index;
    int64_t n;
    int32_t example, num_types;
} gm_pack_set;

typedef struct {
    int64_t coords32, atom_radius, atom_set, atom_type, set_start, set_end, set_example,
        set_choff, set_t, bwd_slot, ex_item_start, ex_item_end, item_perm, chan_off, segs,
        slot_rec;
} gm_pack_layout;

typedef struct {
    int32_t natoms, nsegs, max_seg_items, max_example_items;
} gm_pack_info;

gm_status gm_pack_index_host(const gm_pack_set *sets, int32_t nsets, int32_t nexamples,
                             int32_t nchannels, double radius_scale, const double *centers,
                             int32_t bwd_order, uint8_t *dst, const gm_pack_layout *layout,
                             gm_pack_info *info);

/* The same for vector typing: each set's type_vector (n, num_types) f32 weight
 * rows and, when radius_type_indexed, its type_radii (num_types) f32 (may be
 * NULL otherwise).  Items = nonzero weights, atom-major then channel
 * (_kernels.py:159-166); item_windex (nitems, host) receives each item's entry
 * of the packed weight rows.  layout: as gm_pack_vlayout (weights nweights =
 * sum n*num_types, type_radius sum num_types, items nitems = nonzero weights). */
typedef struct {
    const float *coords;
    const float *radii;
    const float *type_vector;
    const float *type_radii;
    int64_t n;
    int32_t example, num_types;
} gm_pack_vset;

typedef struct {
    int64_t coords32, atom_radius, atom_set, set_start, set_end, set_example, set_choff, set_t,
        set_wstart, set_trstart, weights, type_radius, item_atom, item_channel, item_weight,
        item_radius, bwd_slot, ex_item_start, ex_item_end, item_perm, chan_off, segs;
} gm_pack_vlayout;

gm_status gm_pack_vector_host(const gm_pack_vset *sets, int32_t nsets, int32_t nexamples,
                              int32_t nchannels, double radius_scale, int32_t radius_type_indexed,
                              const double *centers, int32_t bwd_order, uint8_t *dst,
                              const gm_pack_vlayout *layout, int64_t *item_windex,
                              gm_pack_info *info);

/* ---- MOLC cache records -> typed atoms ----
 *
 * Replaces the reference's per-atom decode and typing of a cache entry
 * (chemio.py:353-356 RawAtom objects, atomtypes.py:272-291 type_molecule with
 * the default element typer).  raw: device, the 13-byte records (u8 element,
 * f32 x, y, z little-endian) of nentries entries back to back; entry_start:
 * device (nentries+1) int64 atom offsets of the entries in raw; type_table:
 * device (256) int16, element number -> type index or -1 (atom dropped);
 * type_radii: device, radius per type.  Writes, in record order with dropped
 * atoms removed: coords (kept,3) f32, type_index (kept) int32, radius (kept)
 * f32, and offsets (nentries+1) int64 (entry e owns [offsets[e],
 * offsets[e+1])).  Output arrays must hold entry_start[nentries] atoms. */
gm_status gm_molc_decode(const uint8_t *raw, const int64_t *entry_start, int32_t nentries,
                         const int16_t *type_table, const float *type_radii, float *coords,
                         int32_t *type_index, float *radius, int64_t *offsets, void *stream);

/* ---- host helpers ---- */

/* geom.make_transform for n examples from pre-drawn uniforms (geom.py:66-76,
 * 121-136): u is (n, k) row-major with k = 3*(rotation) + 3*(translation>0),
 * exactly rng.random((n, k)).  Writes out (n, 15): R row-major (the
 * quaternion's rotation_matrix, geom.py:50-57), center, translation
 * (-t + 2t*u).  Same IEEE expressions and libm calls as the Python reference,
 * so rows are bit-identical to the reference's draws. */
gm_status gm_draw_transforms(const double *u, int64_t n, int32_t rotation, double translation,
                             const double *centers, double *out);

/* ---- misc ---- */
const char *gm_last_error(void);
const char *gm_version(void);
int32_t gm_device_count(void);
/* sizeof(gm_params) (which = 0), gm_batch (1), gm_dataset (2), gm_capacity (3),
 * gm_pack_set (4), gm_pack_layout (5), gm_pack_info (6), gm_pack_vset (7) or
 * gm_pack_vlayout (8): ABI check. */
int32_t gm_struct_size(int32_t which);
/* Kernel launches issued by this process since the last reset (bench evidence). */
int64_t gm_launch_count(int32_t reset);

#ifdef __cplusplus
}
#endif
#endif /* GRIDMAKER_B200_H */
