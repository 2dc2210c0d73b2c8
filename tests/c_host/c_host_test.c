/* A non-Python host of the C ABI (include/gridmaker_b200.h): packs a small
 * index-typed batch by hand, runs gm_prepare_inline -> gm_forward ->
 * gm_backward on the GPU with device buffers of its own, and checks grids and
 * coordinate gradients against the CPU oracle (oracle/oracle.c, test
 * infrastructure) -- 1e-6 absolute + 1e-5 relative, as the north star asks.
 * Built and run by tests/test_gpu_c_host.py.  Exit status 0 = parity. */
#include <math.h>
#include <stdio.h>
#include <stdlib.h>
#include <string.h>

#include <cuda_runtime.h>

#include "gridmaker_b200.h"

void oracle_forward_index_sets(float *out, int64_t nch, int64_t npts, const double *coords,
                               const double *radii, const int64_t *tidx, const int64_t *set_start,
                               const int64_t *set_end, const int64_t *set_example,
                               const int64_t *set_choff, const int64_t *set_t, int64_t nsets,
                               const double *origins, double res, double grm, double rmult,
                               int binary);
void oracle_backward_index(double *coord_grad, const double *coords, const double *radii,
                           const int64_t *tidx, int64_t n, const float *grid_grad, int64_t npts,
                           const double *origin, double res, double grm, double rmult);

#define CK(x)                                                                  \
    do {                                                                       \
        cudaError_t e_ = (x);                                                  \
        if (e_ != cudaSuccess) {                                               \
            fprintf(stderr, "%s: %s\n", #x, cudaGetErrorString(e_));          \
            return 2;                                                          \
        }                                                                      \
    } while (0)
#define GK(x)                                                                  \
    do {                                                                       \
        if ((x) != GM_OK) {                                                    \
            fprintf(stderr, "%s: %s\n", #x, gm_last_error());                  \
            return 2;                                                          \
        }                                                                      \
    } while (0)

static uint64_t rng_state = 88172645463325252ull;
static double urand(void) { /* xorshift64 */
    rng_state ^= rng_state << 13;
    rng_state ^= rng_state >> 7;
    rng_state ^= rng_state << 17;
    return (double)(rng_state >> 11) / 9007199254740992.0;
}

static void *dev_copy(const void *h, size_t n) {
    void *d = NULL;
    if (cudaMalloc(&d, n ? n : 1) != cudaSuccess) return NULL;
    if (n) cudaMemcpy(d, h, n, cudaMemcpyHostToDevice);
    return d;
}

int main(void) {
    enum { NEX = 2, NSET = 4, C = 5 };
    const int set_t[NSET] = {3, 2, 3, 2}, set_choff[NSET] = {0, 3, 0, 3};
    const int set_ex[NSET] = {0, 0, 1, 1}, set_n[NSET] = {17, 1, 0, 40};
    int natoms = 0;
    for (int s = 0; s < NSET; s++) natoms += set_n[s];

    gm_params p;
    memset(&p, 0, sizeof p);
    p.resolution = 0.5;
    p.dimension = 8.0;
    p.radius_scale = 1.0;
    p.gaussian_radius_multiple = 1.0;
    p.radius_multiple = 1.5;
    p.npts = (int)floor(p.dimension / p.resolution + 0.5) + 1;
    p.matmul_order_1 = p.matmul_order_n = -1;
    const int D = p.npts;
    const size_t D3 = (size_t)D * D * D;

    float *xyz = malloc(sizeof(float) * 3 * natoms);
    double *xyz64 = malloc(sizeof(double) * 3 * natoms), *rad = malloc(sizeof(double) * natoms);
    int32_t *aset = malloc(sizeof(int32_t) * natoms), *atype = malloc(sizeof(int32_t) * natoms);
    int64_t *tidx = malloc(sizeof(int64_t) * natoms);
    int32_t sst[NSET], sen[NSET];
    int64_t sst64[NSET], sen64[NSET], sex64[NSET], sco64[NSET], st64[NSET];
    int32_t exs[NEX], exe[NEX];
    int a = 0;
    for (int s = 0; s < NSET; s++) {
        sst[s] = a;
        for (int k = 0; k < set_n[s]; k++, a++) {
            for (int q = 0; q < 3; q++) {
                xyz[3 * a + q] = (float)(urand() * 11.0 - 5.5);
                xyz64[3 * a + q] = (double)xyz[3 * a + q];
            }
            rad[a] = (double)(float)(1.0 + 1.2 * urand());
            aset[a] = s;
            atype[a] = (int32_t)(urand() * set_t[s]);
            tidx[a] = atype[a];
        }
        sen[s] = a;
        sst64[s] = sst[s];
        sen64[s] = sen[s];
        sex64[s] = set_ex[s];
        sco64[s] = set_choff[s];
        st64[s] = set_t[s];
    }
    exs[0] = 0;
    exe[0] = sen[1];
    exs[1] = sen[1];
    exe[1] = natoms;
    double origins[3 * NEX] = {-4.0, -4.0, -4.0, -3.75, -4.25, -4.0};

    gm_batch b;
    memset(&b, 0, sizeof b);
    b.nexamples = NEX;
    b.nsets = NSET;
    b.natoms = natoms;
    b.nitems = natoms;
    b.nchannels = C;
    b.coords32 = dev_copy(xyz, sizeof(float) * 3 * natoms);
    b.atom_radius = dev_copy(rad, sizeof(double) * natoms);
    b.atom_set = dev_copy(aset, sizeof(int32_t) * natoms);
    b.atom_type = dev_copy(atype, sizeof(int32_t) * natoms);
    b.set_start = dev_copy(sst, sizeof sst);
    b.set_end = dev_copy(sen, sizeof sen);
    b.set_example = dev_copy(set_ex, sizeof set_ex);
    b.set_choff = dev_copy(set_choff, sizeof set_choff);
    b.set_t = dev_copy(set_t, sizeof set_t);
    b.ex_item_start = dev_copy(exs, sizeof exs);
    b.ex_item_end = dev_copy(exe, sizeof exe);
    b.origins = dev_copy(origins, sizeof origins);
    int mx = 0;
    for (int e = 0; e < NEX; e++) mx = exe[e] - exs[e] > mx ? exe[e] - exs[e] : mx;
    b.max_example_items = mx;

    const size_t wsb = gm_workspace_bytes(natoms, natoms, NEX, C);
    void *ws = NULL, *out = NULL, *cg = NULL;
    CK(cudaMalloc(&ws, wsb));
    CK(cudaMalloc(&out, sizeof(float) * NEX * C * D3));
    CK(cudaMalloc(&cg, sizeof(float) * 3 * natoms));
    GK(gm_prepare_inline(&p, &b, ws, wsb, origins, NULL, NULL));
    GK(gm_forward(&p, &b, ws, out, NULL));
    GK(gm_backward(&p, &b, ws, out, cg, NULL, NULL));  /* grid_grad = the grid itself */
    CK(cudaDeviceSynchronize());

    float *grid = malloc(sizeof(float) * NEX * C * D3), *ref = calloc(NEX * C * D3, sizeof(float));
    float *cgh = malloc(sizeof(float) * 3 * natoms);
    CK(cudaMemcpy(grid, out, sizeof(float) * NEX * C * D3, cudaMemcpyDeviceToHost));
    CK(cudaMemcpy(cgh, cg, sizeof(float) * 3 * natoms, cudaMemcpyDeviceToHost));
    oracle_forward_index_sets(ref, C, D, xyz64, rad, tidx, sst64, sen64, sex64, sco64, st64, NSET,
                              origins, p.resolution, 1.0, 1.5, 0);
    double worst = 0.0;
    size_t bad = 0;
    for (size_t v = 0; v < (size_t)NEX * C * D3; v++) {
        const double d = fabs((double)grid[v] - ref[v]);
        if (d > 1e-6 + 1e-5 * fabs(ref[v])) bad++;
        worst = d > worst ? d : worst;
    }
    double gworst = 0.0;
    size_t gbad = 0;
    for (int s = 0; s < NSET; s++) {
        const int n = sen[s] - sst[s];
        if (!n) continue;
        double *g = malloc(sizeof(double) * 3 * n);
        oracle_backward_index(g, xyz64 + 3 * sst[s], rad + sst[s], tidx + sst[s], n,
                              grid + ((size_t)set_ex[s] * C + set_choff[s]) * D3, D,
                              origins + 3 * set_ex[s], p.resolution, 1.0, 1.5);
        for (int q = 0; q < 3 * n; q++) {
            const double d = fabs((double)cgh[3 * sst[s] + q] - g[q]);
            if (d > 1e-6 + 1e-5 * fabs(g[q])) gbad++;
            gworst = d > gworst ? d : gworst;
        }
        free(g);
    }
    printf("c host: %d atoms, %d^3 x %d ch x %d ex; forward max|d| %.3g (%zu bad), "
           "backward max|d| %.3g (%zu bad), %s\n",
           natoms, D, C, NEX, worst, bad, gworst, gbad, gm_version());
    return (bad || gbad) ? 1 : 0;
}
