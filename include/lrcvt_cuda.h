/*
 * lrcvt_cuda.h -- C ABI of the B200 (sm_100a) LSRCVT hot path.
 *
 * Plain pointers and sizes only. Every pointer argument named d_* is a
 * DEVICE pointer (cudaMalloc / torch CUDA tensor storage) on the current
 * device; `stream` is a cudaStream_t (NULL = legacy default stream). Calls are
 * stream-ordered; the entry points that return statistics synchronise the
 * stream once at the end (the reference returns Python ints there).
 *
 * Each entry point replaces one call site of the reference's kernel seam,
 * `lrcvt._kernels` imported as `K` in /root/reference/pkg/src/lrcvt/
 * tessellation.py (cited per function below). INTEGRATION.md shows the
 * ctypes binding a maintainer adds to the reference.
 *
 * Per-voxel state layout (HBM, flat x-fastest index v = x + nx*(y + ny*z),
 * grid.py:3-5):
 *   d_site_src : int32[N][2]  (site_of[v], src[v]) packed; -1 = none
 *   d_dist     : float64[N]   geodesic distance, +inf = unassigned
 *   d_state    : uint8[N]     LOS=1 | ACTIVE=2 | NODE=4 (tessellation.py:28-30)
 * lrcvt_unpack_site_src() splits the pair into the reference's separate
 * site_of / src arrays (tessellation.py:52-54).
 *
 * Return codes: 0 = success; > 0 = number of sites outside their recorded
 * component (the caller raises ValueError, tessellation.py:139-140);
 * < 0 = error (LRCVT_E_*), message via lrcvt_last_error().
 */
#ifndef LRCVT_CUDA_H
#define LRCVT_CUDA_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define LRCVT_E_CUDA (-1)
#define LRCVT_E_ARG (-2)
#define LRCVT_E_NOMEM (-3)

/* weight modes for lrcvt_centroidal_update (seeding.py:59-68 voxel_weights) */
#define LRCVT_W_ONES 0    /* weight_field None: m_v = 1                      */
#define LRCVT_W_F64 1     /* explicit float64[N] weights (m_v ** gamma)       */
#define LRCVT_W_F32_G1 2  /* float32[N] weight field, gamma == 1 (exact)      */
#define LRCVT_W_F32_G2 3  /* float32[N] weight field, gamma == 2 (exact m*m)  */

typedef struct lrcvt_plan lrcvt_plan;

typedef struct {
  int64_t rounds;        /* report["rounds"], tessellation.py:199-200     */
  int64_t sweeps;        /* report["sweeps"]                               */
  int64_t assigned;      /* report["assigned"], tessellation.py:203        */
  int64_t evaluations;   /* E: voxels evaluated over all rounds + sweeps   */
  int64_t commits;       /* C: committed improvements                      */
  int64_t bad_sites;     /* sites outside their component                  */
  int64_t phase1_rounds; /* rounds of phase 1 (subset of `rounds`)         */
  int64_t eligible;      /* in-band voxels of components that have sites   */
} lrcvt_classify_stats;

/* Plan: geometry + the static component volume (borrowed, must outlive the
 * plan) + scratch sized for up to max_sites sites. Replaces the per-call
 * scratch allocation of tessellation.py:142-149. */
int lrcvt_plan_create(lrcvt_plan **plan, int64_t nx, int64_t ny, int64_t nz, double sx,
                      double sy, double sz, const int32_t *d_comp, int32_t n_components,
                      int64_t max_sites, void *stream);
int lrcvt_plan_destroy(lrcvt_plan *plan);
/* in-band voxel count of the plan's component volume */
int64_t lrcvt_plan_inband(const lrcvt_plan *plan);

/* voronoi_classify core: replaces K._place_seeds (tessellation.py:136),
 * K._seed_worklist + K._run_phase (:151-156), the phase-2 loop with
 * K._run_phase / K._eval_list / K._apply_and_enqueue (:161-189) and the state
 * bits (:191-194). d_site_pos is float64[n_sites][3], d_site_comp int32.
 * d_state may be NULL. */
int lrcvt_classify(lrcvt_plan *plan, int64_t n_sites, const double *d_site_pos,
                   const int32_t *d_site_comp, int32_t *d_site_src, double *d_dist,
                   uint8_t *d_state, lrcvt_classify_stats *stats, void *stream);

/* centroidal_update core: replaces K._phi_chains + K._centroid_targets +
 * K._move_sites (tessellation.py:233-241). d_weights is NULL (LRCVT_W_ONES),
 * float64[N] (LRCVT_W_F64) or float32[N] (LRCVT_W_F32_*). backoff = 0.5 *
 * voxel_length (tessellation.py:237-240). Outputs: d_new_pos float64[S][3],
 * d_disp float64[S], optional d_sums float64[4][S] (wsum, tx, ty, tz), and
 * *empty_regions (report["empty_regions"]). */
int lrcvt_centroidal_update(lrcvt_plan *plan, int64_t n_sites, const double *d_site_pos,
                            const int32_t *d_site_comp, const int32_t *d_site_src,
                            int32_t weight_mode, const void *d_weights, double backoff,
                            double *d_new_pos, double *d_disp, double *d_sums,
                            int64_t *empty_regions, void *stream);

/* Sticky plan flag: the caller guarantees that centroidal_update is called
 * with the same site-component set as the preceding lrcvt_classify (true
 * inside a Lloyd loop, where components never change), so the eligible-voxel
 * list (tessellation.py:161-164) built by the classify is reused.
 * enable = 1 keeps the list the plan holds now; enable = 2 starts a new run:
 * the list is dropped, the next classify builds it for its sites and later
 * calls reuse that one (a loop whose sites may differ from the plan's last
 * classify with the same site count). */
int lrcvt_plan_reuse_eligible(lrcvt_plan *plan, int enable);

/* split packed (site_of, src) into two int32[N] arrays */
int lrcvt_unpack_site_src(const int32_t *d_site_src, int64_t n, int32_t *d_site_of,
                          int32_t *d_src, void *stream);

/* batch of K._segment_hit_t (_kernels.py:45-125): d_segs float64[n][6]
 * (ax, ay, az, bx, by, bz), d_want int32[n] -> d_t float64[n]. Backs
 * raycast_same_component (tessellation.py:82-99). */
int lrcvt_segment_hit_t(int64_t nx, int64_t ny, int64_t nz, double sx, double sy, double sz,
                        const int32_t *d_comp, const double *d_segs, const int32_t *d_want,
                        int64_t n, double *d_t, void *stream);

/* _segment_clear (_kernels.py:128-133) as the eval kernels compute it (the
 * DDA with the plan's static clearance shortcuts): d_clear[i] = 1 iff
 * segment i (d_segs float64[n][6]) stays in component d_want[i]. */
int lrcvt_segment_clear_batch(lrcvt_plan *plan, const double *d_segs, const int32_t *d_want, int64_t n,
                              uint8_t *d_clear, void *stream);

/* classify_isobands (grid.py:140-163): d_field float32[n], d_iso float64
 * [n_iso] strictly increasing -> d_layer int32[n] (band index or -1). */
int lrcvt_isobands(int64_t n, const float *d_field, const double *d_iso, int32_t n_iso,
                   int32_t *d_layer, void *stream);

/* label_components (grid.py:166-220): face-connected components of each
 * layer 0..n_layers-1 -> d_component int32[N] with dense ids ordered by
 * (layer, first voxel in row-major order); *n_components receives the count
 * (the call synchronises the stream). */
int lrcvt_label_components(int64_t nx, int64_t ny, int64_t nz, const int32_t *d_layer,
                           int32_t n_layers, int32_t *d_component, int32_t *n_components,
                           void *stream);

/* ComponentInfo table (grid.py:199-211) for ids 0..n_components-1:
 * d_count uint64[nc] voxel counts, d_bbox int32[nc][6] inclusive
 * (x0, y0, z0, x1, y1, z1), d_layer_of int32[nc]. */
int lrcvt_component_table(int64_t nx, int64_t ny, int64_t nz, const int32_t *d_component,
                          const int32_t *d_layer, int32_t n_components, uint64_t *d_count,
                          int32_t *d_bbox, int32_t *d_layer_of, void *stream);

/* aggregate_moments core (pipeline.py:187-238) + per-cell histograms
 * (stats.py:194-203 rule on fixed global axes). Cells: regions 0..n_sites-1
 * (site_of == r) and stray cells n_sites + c (unassigned in-band voxels of
 * component c); n_cells = n_sites + n_components. field_ptrs is a HOST array
 * of n_fields DEVICE float32[n] pointers; pairs a HOST int32[n_pairs][2] of
 * field indices. Outputs (device): d_count int64[n_cells]; d_sums
 * float64[n_cells][n_pairs][15] raw power sums in ORDERS order (stats.py:19);
 * d_minmax float64[n_cells][n_pairs][4] = (min_x, max_x, min_y, max_y).
 * n_bins > 0 also fills d_hist int64[n_cells][n_fields][n_bins + 2] (bins,
 * underflow, overflow) on axes = HOST float64[n_fields][2] (lo, hi); NaN
 * entries are replaced by the in-band min / max (hi <= lo -> lo + 1). */
int lrcvt_aggregate(int64_t n, int32_t n_fields, const float *const *field_ptrs,
                    const int32_t *d_component, const int32_t *d_site_of, int32_t n_sites,
                    int32_t n_components, int32_t n_pairs, const int32_t *pairs, int32_t n_bins,
                    double *axes, int64_t *d_count, double *d_sums, double *d_minmax,
                    int64_t *d_hist, void *stream);

/* Seeding masses (seeding.py:71-107 component_masses; SURVEY.md §8(f) rank
 * 1). In-band voxels (d_component >= 0) grouped by (component, block) --
 * block = (x/bs) + nbx*((y/bs) + nby*(z/bs)), nbx = ceil(nx/bs), nby =
 * ceil(ny/bs) -- voxels increasing inside a group, groups ordered by
 * component then block (= np.lexsort((voxel, block, comp))). Weights m_v**gamma
 * by weight_mode (LRCVT_W_*; d_weights NULL for ONES). Outputs (device):
 * d_voxels int32[max_inband] the grouped voxel list, d_weights_sorted
 * float64[max_inband] their weights (may be NULL), per group r < *n_runs:
 * d_run_key int64 = comp * n_blocks + block, d_run_start int64, d_run_len
 * int64, d_run_mass float64 = np.sum of the group's weights (numpy pairwise
 * order, bit-exact). Host outputs: *n_inband, *n_runs, *total_mass = np.sum
 * of all in-band weights in voxel order. Returns LRCVT_E_ARG (and the needed
 * sizes in *n_inband / *n_runs) when max_inband or max_runs is too small. */
int lrcvt_seed_masses(int64_t nx, int64_t ny, int64_t nz, int32_t block_size,
                      const int32_t *d_component, int32_t n_components, int32_t weight_mode,
                      const void *d_weights, int64_t max_inband, int64_t max_runs,
                      int32_t *d_voxels, double *d_weights_sorted, int64_t *d_run_key,
                      int64_t *d_run_start, int64_t *d_run_len, double *d_run_mass,
                      int64_t *n_inband, int64_t *n_runs, double *total_mass, void *stream);

/* Record block of the .lrcvt layout (layout.py:123-200 build_and_write):
 * in-band voxels ordered by (component, region = site_of with unassigned ->
 * 0xFFFFFFFF, voxel), packed as records {u32 x, y, z; f32 field[n_fields]}
 * (little-endian, 12 + 4 * n_fields bytes each) into d_records; field_ptrs
 * is a HOST array of n_fields DEVICE float32[n] pointers. Also per record
 * its region key (d_region_key, u32) and per component its first record and
 * record count (d_comp_first / d_comp_count int64[n_components]; 0 / 0 when
 * empty). *n_records = the in-band count; LRCVT_E_ARG when it exceeds
 * max_records or a site_of entry is >= n_sites. */
int lrcvt_layout_records(int64_t nx, int64_t ny, int64_t nz, int32_t n_fields,
                         const float *const *field_ptrs, const int32_t *d_component,
                         const int32_t *d_site_of, int32_t n_components, int32_t n_sites,
                         int64_t max_records,
                         void *d_records, uint32_t *d_region_key, int64_t *d_comp_first,
                         int64_t *d_comp_count, int64_t *n_records, void *stream);

/* Site adjacency (sitegraph.py:46-82 region_adjacency): the sorted,
 * de-duplicated (lo, hi) site pairs, lo < hi, of face-neighbouring voxels
 * (+x, +y, +z) with different assigned sites in the same component.
 * d_edges int64[max_edges][2] (device); *n_edges = the edge count
 * (LRCVT_E_ARG when it exceeds max_edges; call again with room). */
int lrcvt_region_adjacency(int64_t nx, int64_t ny, int64_t nz, const int32_t *d_site_of,
                           const int32_t *d_component, int64_t n_sites, int64_t max_edges,
                           int64_t *d_edges, int64_t *n_edges, void *stream);

/* Multi-GPU global mode: ONE volume in
 * z-slabs, one plan per rank. A rank owns planes [zlo, zhi); its own slab and
 * one halo plane on each side are kept current locally, the rare far reads
 * (phase-2 shortcut nodes, phi chains of the vote) go to the owning rank's
 * state buffer through peer pointers (same device, CUDA IPC, or NVLink P2P).
 * The caller drives the rounds and the collectives:
 *   set_slab, set_peers -> begin -> { eval -> exchange boundary proposals
 *   (lo -> rank-1, hi -> rank+1) -> commit(halo) -> all-reduce frontier }*
 *   -> phase2 -> { rounds, sweep (eval/commit with sweep=1) }* -> finish.
 * Proposals are 24-byte records {f64 d; i32 v, site, src, pad}. Results,
 * rounds, sweeps and the summed evaluation / commit counters equal
 * lrcvt_classify on one domain bit for bit. */
int lrcvt_mg_set_slab(lrcvt_plan *plan, int64_t zlo, int64_t zhi);
/* plan-owned full-volume (site_of, src) int32[N][2] / dist float64[N]
 * buffers (allocated on first call; base allocations, IPC-exportable) */
int lrcvt_mg_state(lrcvt_plan *plan, void **d_ss, void **d_dist);
/* z_bounds int64[world + 1] (rank r owns [z_bounds[r], z_bounds[r+1]));
 * peer_ss / peer_dist: HOST arrays of `world` device pointers, valid in this
 * process, to every rank's state buffers (this rank's own included) */
int lrcvt_mg_set_peers(lrcvt_plan *plan, int32_t world, const int64_t *z_bounds, void *const *peer_ss,
                       void *const *peer_dist);
int lrcvt_mg_begin(lrcvt_plan *plan, int64_t n_sites, const double *d_site_pos,
                   const int32_t *d_site_comp, int32_t *d_site_src, double *d_dist,
                   int64_t *n_frontier, void *stream);
int lrcvt_mg_phase2(lrcvt_plan *plan, int64_t n_sites, const int32_t *d_site_comp,
                    int64_t *n_frontier, void *stream);
/* evaluate the own frontier (sweep: the own eligible list); *n_lo / *n_hi
 * = the improved proposals on planes zlo / zhi - 1, at
 * lrcvt_mg_boundary(plan, 0 / 1) for rank - 1 / rank + 1 (the eval kernels
 * write them there as they go) */
int lrcvt_mg_eval(lrcvt_plan *plan, int32_t phase, int32_t sweep, int64_t *n_evaluated,
                  int64_t *n_lo, int64_t *n_hi, void *stream);
void *lrcvt_mg_boundary(lrcvt_plan *plan, int32_t side);
/* commit the own proposals and the n_halo proposals received from the
 * neighbour ranks (one launch, which also ends the round); *n_next = the own
 * next frontier, *n_committed = own proposals committed (= improved) */
int lrcvt_mg_commit(lrcvt_plan *plan, const void *d_halo, int64_t n_halo, int32_t sweep,
                    int64_t *n_next, int64_t *n_committed, void *stream);
/* state bits of the own slab; *assigned = own assigned voxels */
int lrcvt_mg_finish(lrcvt_plan *plan, const int32_t *d_site_src, uint8_t *d_state,
                    int64_t *assigned, void *stream);
/* vote over the own slab. Unit weights (exact integers): vote_exact writes
 * d_acc uint64[4][S] partial sums; all-reduce (sum) them, then
 * vote_exact_finish -> d_sums float64[4][S]. Any weights (voxel-order
 * chains): vote_box writes the own per-site boxes int32[6][S] (x0,y0,z0
 * min; x1,y1,z1 max) -> all-reduce min / max; vote_scan mode 1 (sites whose
 * box starts in this slab, chains from 0) and mode 2 (box starts earlier,
 * chains continue from d_init = the running sums after the previous slab)
 * write d_out float64[4][S]; vote_carry builds the running sums after this
 * slab for the next rank; the last rank's are the sums. */
int lrcvt_mg_vote_exact(lrcvt_plan *plan, int64_t n_sites, const int32_t *d_site_src, uint64_t *d_acc,
                        void *stream);
int lrcvt_mg_vote_exact_finish(lrcvt_plan *plan, int64_t n_sites, const uint64_t *d_acc, double *d_sums,
                               void *stream);
int lrcvt_mg_vote_box(lrcvt_plan *plan, int64_t n_sites, const int32_t *d_site_src, int32_t *d_box,
                      void *stream);
int lrcvt_mg_vote_scan(lrcvt_plan *plan, int64_t n_sites, const int32_t *d_site_comp, int32_t weight_mode,
                       const void *d_weights, int32_t mode, const int32_t *d_box, const double *d_init,
                       double *d_out, void *stream);
int lrcvt_mg_vote_carry(lrcvt_plan *plan, int64_t n_sites, const int32_t *d_box, const double *d_res,
                        const double *d_carry_in, double *d_carry_out, void *stream);
/* _move_sites on every rank from the identical reduced sums */
int lrcvt_mg_move(lrcvt_plan *plan, int64_t n_sites, const double *d_site_pos, const int32_t *d_site_comp,
                  const double *d_sums, double backoff, double *d_new_pos, double *d_disp,
                  int64_t *empty_regions, void *stream);
/* device milliseconds of this plan's synchronising mg steps (begin, phase2,
 * eval, commit, finish, move) since the last call: CUDA events around their
 * kernels, the host round trip of each step excluded. enable = 0 stops. */
int lrcvt_mg_timing(lrcvt_plan *plan, int32_t enable, double *ms);
/* CUDA IPC of a base device allocation (64-byte handle) */
int lrcvt_ipc_export(const void *d_ptr, uint8_t *handle64);
int lrcvt_ipc_open(const uint8_t *handle64, void **d_ptr);
int lrcvt_ipc_close(void *d_ptr);

/* Output buffers passed to consecutive lrcvt_classify calls of this plan
 * are the same and untouched in between (a Lloyd loop over one engine's
 * buffers), and lrcvt_plan_reuse_eligible holds: the classify then resets
 * and rewrites only the eligible voxels. */
int lrcvt_plan_persistent_outputs(lrcvt_plan *plan, int enable);

/* Instrumentation for bench.py: enable CUDA-event timing of every k_eval
 * launch (the dominant kernel) on the plan; read back launches, voxels
 * evaluated and summed device milliseconds. lrcvt_launch_count() counts this
 * library's own kernel launches (CUB-internal kernels excluded). */
int lrcvt_plan_set_timing(lrcvt_plan *plan, int enable);
int lrcvt_plan_timing(const lrcvt_plan *plan, int64_t *launches, int64_t *items, double *ms);
unsigned long long lrcvt_launch_count(void);
/* with timing enabled: out6 = {phase-1 eval ms, phase-2 eval ms, commit ms,
 * phase-1 voxels evaluated, phase-2 voxels evaluated, proposals committed} */
int lrcvt_plan_profile(const lrcvt_plan *plan, double *out6);

/* Size classes of the device-side relaxation round loop (host-only, no GPU
 * needed): returns the number of classes for a plan of n_inband in-band
 * voxels and writes each class's launch size (voxels its eval launch covers,
 * clamped to [1, n_inband], < 2^31) into launch_items[0..max_classes). */
int32_t lrcvt_round_classes(int64_t n_inband, int64_t *launch_items, int32_t max_classes);

const char *lrcvt_last_error(void);
int lrcvt_version(void);

#ifdef __cplusplus
}
#endif
#endif /* LRCVT_CUDA_H */
