/* fmm2d.h -- C ABI of the B200-native adaptive 2-D FMM (libfmm2d.so).
 *
 * The reference package (/root/reference/pkg, python `fmm2d` 0.1.0) has no
 * FFI; its drop-in boundary is the Python call
 *     fmm_evaluate(points: ParticleSet, cfg: TreeConfig, *, parallel, n_workers)
 *         -> (values complex128[M] in input order, EngineReport)
 * (pkg/src/fmm2d/engine.py:207-279).  Each entry point below replaces one
 * reference interface; the Python host package `paper_1205_4611_b200` binds
 * them with ctypes and keeps the reference's Python signatures (see
 * INTEGRATION.md for the binding a maintainer of the reference would add).
 *
 * Conventions: complex arrays are interleaved (re, im) doubles, i.e. the
 * memory of a numpy complex128 array.  Host pointers unless the function name
 * says `_device`.  The library never frees caller memory.  A context is not
 * thread-safe; one in-flight call per context.  Every call is synchronous.
 * Return codes map to the reference's exception types:
 *   FMM2D_EBADARG -> ValueError, FMM2D_EDEGENERATE -> DegenerateInputError
 *   (tree.py:20-21), FMM2D_ESINGULAR -> ValueError with the reference message,
 *   FMM2D_ECUDA / FMM2D_ENCCL -> RuntimeError, FMM2D_EOOM -> MemoryError.
 * fmm2d_last_error() returns the message (same text as the reference raises).
 */
#ifndef FMM2D_H
#define FMM2D_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define FMM2D_OK 0
#define FMM2D_EBADARG 2
#define FMM2D_EDEGENERATE 3
#define FMM2D_ESINGULAR 5
#define FMM2D_ECUDA 6
#define FMM2D_ENCCL 7
#define FMM2D_EOOM 8

#define FMM2D_NPHASES 9 /* engine.py:28 PHASE_NAMES order:
                           sort connect p2m m2m m2l l2l l2p p2p other */

typedef struct fmm2d_ctx fmm2d_ctx;

/* EngineReport (engine.py:34-47) plus device-side extras */
typedef struct fmm2d_report {
  double phase_ms[FMM2D_NPHASES]; /* CUDA-event time per phase; other = copies */
  double device_ms;               /* first tree kernel .. last P2P kernel */
  double total_ms;                /* whole call incl. H2D/D2H */
  int32_t n_levels;
  int32_t retries;                /* list-capacity regrow reruns */
  int64_t n_boxes;
  int64_t finest_src_min;
  int64_t finest_src_max;
  double finest_src_mean;
  int64_t p2p_skips;              /* raw coincident pairs skipped (self included) */
  int64_t list_totals[4];         /* weak, p2p, p2l, m2p entries */
  int32_t max_len[4];             /* longest list of each kind */
  int64_t h2d_bytes;
  int64_t d2h_bytes;
  int64_t kernel_launches;        /* engine kernels launched by the last attempt
                                     (excludes the CUB radix-sort kernels) */
} fmm2d_report;

/* context on CUDA device `device` (buffers, stream, events grow monotonically) */
int fmm2d_create(fmm2d_ctx** out, int device);
void fmm2d_destroy(fmm2d_ctx* ctx);
const char* fmm2d_last_error(const fmm2d_ctx* ctx);

/* tree.py:86-94 num_levels + tree.py:186-192 clamp (4^L <= n) */
int fmm2d_num_levels(int64_t n_sources, int n_desired);
/* tree.py:86-94 unclamped Eq. (6); -1 on bad input */
int fmm2d_num_levels_raw(int64_t n_sources, int n_desired);

/* replaces fmm2d.engine.fmm_evaluate (engine.py:207-279).
 * pos_xy: c128[n]; gamma: f64[n]; eval_xy: c128[m] or NULL (evaluation points
 * alias the sources, m must equal n); out_xy: c128[m] in input order. */
int fmm2d_evaluate(fmm2d_ctx* ctx, int64_t n, const double* pos_xy, const double* gamma,
                   int64_t m, const double* eval_xy, int p, double theta, int n_desired,
                   double* out_xy, fmm2d_report* rep);

/* same pipeline with inputs/outputs already resident in device memory of the
 * context's device (used by the bench's device-resident measurement) */
int fmm2d_evaluate_device(fmm2d_ctx* ctx, int64_t n, const double* d_pos_xy,
                          const double* d_gamma, int64_t m, const double* d_eval_xy, int p,
                          double theta, int n_desired, double* d_out_xy, fmm2d_report* rep);

/* replaces fmm2d.tree.build_tree (tree.py:230-334): builds on the device and
 * keeps the tree in the context; fetch it with fmm2d_export_tree */
int fmm2d_build_tree(fmm2d_ctx* ctx, int64_t n, const double* pos_xy, const double* gamma,
                     int64_t m, const double* eval_xy, int n_desired, int32_t* n_levels);

/* after FMM2D_EDEGENERATE: info = {points in box, box, level, levels still
 * required}, xy = the common coordinate (tree.py:285-291 message fields) */
int fmm2d_degenerate_info(fmm2d_ctx* ctx, int64_t info[4], double xy[2]);

/* copy the context's current tree (after build_tree or evaluate).  Level
 * arrays are concatenated over levels 0..L: boxes ((4^l-1)/3 + k), offsets
 * (sum_{l'<l}(4^l'+1) + k).  Any output pointer may be NULL. */
int fmm2d_export_tree(fmm2d_ctx* ctx, double* center_xy, double* half_width, double* half_height,
                      int64_t* src_offsets, int64_t* eval_offsets, int64_t* src_perm,
                      int64_t* eval_perm, double* src_pos_xy, double* src_strength,
                      double* eval_pos_xy);

/* replaces fmm2d.connectivity.build_connectivity (connectivity.py:99-114)
 * for a tree given by its per-level geometry (concatenated as above) */
int fmm2d_build_connectivity(fmm2d_ctx* ctx, int n_levels, const double* center_xy,
                             const double* half_width, const double* half_height, double theta);

/* totals of the context's current lists: weak (all levels), p2p, p2l, m2p */
int fmm2d_list_sizes(fmm2d_ctx* ctx, int64_t totals[4]);

/* CSR copies; weak_* over all boxes of all levels (global box ids as above),
 * p2p/p2l/m2p over finest boxes (finest-level ids). */
int fmm2d_export_lists(fmm2d_ctx* ctx, int64_t* weak_off, int64_t* weak_idx, int64_t* p2p_off,
                       int64_t* p2p_idx, int64_t* p2l_off, int64_t* p2l_idx, int64_t* m2p_off,
                       int64_t* m2p_idx);

/* list-length histogram of the last evaluate: kind 0 weak, 1 p2p, 2 p2l, 3 m2p;
 * out[len] = number of lists of that length for len < nbins */
int fmm2d_histogram(fmm2d_ctx* ctx, int kind, int64_t* out, int nbins);

/* debug seams for per-phase parity: expansions of the last evaluate
 * (c128[n_boxes * (p+1)], global box ids) and tree-ordered potentials */
int fmm2d_export_expansions(fmm2d_ctx* ctx, double* mult_xy, double* local_xy);
int fmm2d_export_phi(fmm2d_ctx* ctx, double* phi_xy);

/* replaces fmm2d.engine.direct_evaluate (engine.py:282-300), asymmetric mode */
int fmm2d_direct(fmm2d_ctx* ctx, int64_t n, const double* pos_xy, const double* gamma,
                 int64_t m, const double* eval_xy, double* out_xy);
/* replaces direct_evaluate(points, symmetric=True) (engine.py:302-323): evaluation
 * points alias the n sources; each pairwise reciprocal serves both directions */
int fmm2d_direct_symmetric(fmm2d_ctx* ctx, int64_t n, const double* pos_xy,
                           const double* gamma, double* out_xy);

/* ---------------------------------------------------------------------------
 * Unit operators (replace fmm2d.operators, operators.py:63-297) on the GPU.
 * Batched, any order p; coefficient arrays are c128[rows, p+1] row-major.
 * Singular inputs return FMM2D_ESINGULAR with the reference's message.
 * --------------------------------------------------------------------------- */
/* operators.py:63-75 p2m over nbox boxes of points off[b]..off[b+1] -> c128[nbox, p+1] */
int fmm2d_op_p2m(fmm2d_ctx* ctx, int64_t nbox, const int64_t* off, const double* pos_xy,
                 const double* gamma, const double* center_xy, int p, double* out_xy);
/* operators.py:78-93 p2l, same layout */
int fmm2d_op_p2l(fmm2d_ctx* ctx, int64_t nbox, const int64_t* off, const double* pos_xy,
                 const double* gamma, const double* center_xy, int p, double* out_xy);
/* operators.py:127-148 m2m in place; variant 0 = "scaled" (unscaled fallback
 * outside [1e-12, 1e12]), 1 = "unscaled" */
int fmm2d_op_m2m(fmm2d_ctx* ctx, int64_t rows, int p, double* coeffs_xy, const double* shift_xy,
                 int variant);
/* operators.py:171-186 l2l in place */
int fmm2d_op_l2l(fmm2d_ctx* ctx, int64_t rows, int p, double* coeffs_xy, const double* shift_xy);
/* operators.py:189-220 m2l -> out c128[rows, p+1] */
int fmm2d_op_m2l(fmm2d_ctx* ctx, int64_t rows, int p, const double* coeffs_xy,
                 const double* shift_xy, double* out_xy);
/* operators.py:227-234 l2p / 237-255 m2p of one expansion at nt targets */
int fmm2d_op_l2p(fmm2d_ctx* ctx, int p, const double* coeffs_xy, const double* center_xy,
                 int64_t nt, const double* tgt_xy, double* out_xy);
int fmm2d_op_m2p(fmm2d_ctx* ctx, int p, const double* coeffs_xy, const double* center_xy,
                 int64_t nt, const double* tgt_xy, double* out_xy);
/* operators.py:258-277 reciprocal_parts -> re, im f64[nt, ns] and the skip count */
int fmm2d_op_reciprocal_parts(fmm2d_ctx* ctx, int64_t ns, const double* src_xy, int64_t nt,
                              const double* tgt_xy, double* re, double* im, int64_t* n_skip);
/* operators.py:280-292 kernel_block -> phi c128[nt] and the skip count */
int fmm2d_op_kernel_block(fmm2d_ctx* ctx, int64_t ns, const double* src_xy, const double* gamma,
                          int64_t nt, const double* tgt_xy, double* out_xy, int64_t* n_skip);

/* connectivity.py:47-68 classify_level: level geometry (nbox = 4^l boxes),
 * parent strong CSR (local ids of level l-1); writes weak and strong CSR
 * (offsets [nbox+1]; index arrays sized 16 * parent_off[nbox/4]) */
int fmm2d_classify_level(fmm2d_ctx* ctx, int64_t nbox, const double* center_xy,
                         const double* half_width, const double* half_height,
                         const int64_t* parent_off, const int64_t* parent_idx, double theta,
                         int64_t* weak_off, int64_t* weak_idx, int64_t* strong_off,
                         int64_t* strong_idx);
/* connectivity.py:71-96 reclassify_finest: finest geometry + strong CSR ->
 * p2p / p2l / m2p CSR (index arrays sized strong_off[nbox]) */
int fmm2d_reclassify_finest(fmm2d_ctx* ctx, int64_t nbox, const double* center_xy,
                            const double* half_width, const double* half_height,
                            const int64_t* strong_off, const int64_t* strong_idx, double theta,
                            int64_t* p2p_off, int64_t* p2p_idx, int64_t* p2l_off,
                            int64_t* p2l_idx, int64_t* m2p_off, int64_t* m2p_idx);

/* ---------------------------------------------------------------------------
 * Distributed evaluation (the reference is single-process,
 * SPEC.md:409).  One context per rank, one rank per GPU.  The library runs the
 * compute phases; the caller (paper_1205_4611_b200/distributed.py, through
 * torch.distributed: NCCL over NVLink / NVSwitch) runs the collectives between
 * them on `stream`.  All d_* arguments are device pointers; every phase
 * function enqueues on `stream` and returns when host-visible results (counts)
 * are ready.  Sequence per evaluation:
 *   setup -> load -> [allreduce MIN bbox] -> root
 *   for s < log2 G: (s even, s>0: segbox -> [allreduce MIN] -> check_segbox)
 *                   8 x (hist -> [allreduce SUM] -> pick)
 *                   eqcount -> [allgather] -> partition
 *   send_counts -> [all-to-all records]
 *   (separate evaluation points: load_evals right after load -- the box
 *    allreduce then covers both -- and eval_route -> [all-to-all] after the
 *    top split; reference tree.py:205-215 / engine.py:207-279)
 *   -> build -> geom_pack -> [allgather]
 *   -> connect -> 2 x request exchange [all-to-all ids, pack, all-to-all, unpack]
 *      (particles before upward, multipoles after upward_top)
 *   -> upward -> [allgather top multipoles] -> upward_top -> downward -> end
 * --------------------------------------------------------------------------- */
int fmm2d_dist_setup(fmm2d_ctx* ctx, int world_size, int rank, int64_t n_total, int p,
                     double theta, int n_desired, void* stream, int32_t* n_levels);
int fmm2d_dist_load(fmm2d_ctx* ctx, int64_t n_local, const double* d_pos_xy,
                    const double* d_gamma, int64_t index_base, double* d_bbox4);
int fmm2d_dist_load_evals(fmm2d_ctx* ctx, int64_t m_total, int64_t m_local,
                          const double* d_eval_xy, int64_t index_base, double* d_bbox4);
int fmm2d_dist_root(fmm2d_ctx* ctx, const double* d_bbox4);
int fmm2d_dist_segbox(fmm2d_ctx* ctx, int step, double* d_box);
int fmm2d_dist_check_segbox(fmm2d_ctx* ctx, int step, const double* d_box);
int fmm2d_dist_hist(fmm2d_ctx* ctx, int step, int round, int32_t* d_hist);
int fmm2d_dist_pick(fmm2d_ctx* ctx, int step, int round, const int32_t* d_hist);
int fmm2d_dist_eqcount(fmm2d_ctx* ctx, int step, int32_t* d_eq);
int fmm2d_dist_partition(fmm2d_ctx* ctx, int step, const int32_t* d_eq_all);
int fmm2d_dist_send_counts(fmm2d_ctx* ctx, int64_t* counts, void** d_records);
int fmm2d_dist_eval_route(fmm2d_ctx* ctx, int64_t* counts, void** d_records);
/* d_eval_records / n_eval_records: the evaluation records this rank received
 * (NULL / 0 when the evaluation points alias the sources) */
int fmm2d_dist_build(fmm2d_ctx* ctx, const double* d_records, int64_t n_records,
                     const double* d_eval_records, int64_t n_eval_records,
                     int64_t* owned_boxes);
int fmm2d_dist_geom_pack(fmm2d_ctx* ctx, double* d_send);
int fmm2d_dist_connect(fmm2d_ctx* ctx, const double* d_geometry_all, int64_t* request_counts);
int fmm2d_dist_requests(fmm2d_ctx* ctx, int kind, const int32_t** d_ids);
int fmm2d_dist_item_doubles(fmm2d_ctx* ctx, int kind, int64_t* n_doubles);
int fmm2d_dist_pack(fmm2d_ctx* ctx, int kind, const int32_t* d_ids, int64_t n_ids,
                    double* d_send);
int fmm2d_dist_unpack(fmm2d_ctx* ctx, int kind, const double* d_recv);
int fmm2d_dist_upward(fmm2d_ctx* ctx, double* d_top_send, int64_t* top_boxes);
int fmm2d_dist_upward_top(fmm2d_ctx* ctx, const double* d_top_all);
int fmm2d_dist_downward(fmm2d_ctx* ctx, double* d_values, int64_t* d_indices,
                        fmm2d_report* rep);
int fmm2d_scatter_values(fmm2d_ctx* ctx, int64_t n, const double* d_values,
                         const int64_t* d_indices, double* d_out);
int fmm2d_dist_end(fmm2d_ctx* ctx);

#ifdef __cplusplus
}
#endif
#endif /* FMM2D_H */
