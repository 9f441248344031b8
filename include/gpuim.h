/*
 * gpuim.h — C ABI of libgpuim.so, the B200 (sm_100a) GPU-IM process-mapping
 * hot path.  Drop-in boundary for the reference package `promap`
 * (/root/reference/pkg/src/promap), whose public entry point for this path is
 *
 *     promap.pipelines.integrated_map(g, t, eps, seed=0, *, coarsest_factor,
 *         phi, rho, filter_mode, jet_filter_c, sigma_coarse, sigma_fine,
 *         iw_max_finest) -> Mapping                       (pipelines.py:221-235)
 *
 * The reference is pure Python with no FFI; every entry point below cites the
 * reference function it replaces.  The Python host (paper_2510_12196_b200/)
 * binds these with ctypes.
 *
 * Conventions
 *   - Every call returns int status: 0 = GIM_OK, >0 = GIM_E_*; the message of
 *     the last failure on the calling thread is gim_last_error().
 *   - `stream` is a cudaStream_t passed as void* (NULL = legacy default).
 *   - Unless a parameter says "host", pointers are DEVICE pointers owned by
 *     the caller; the library never frees caller memory.  Device graphs use
 *     int32 ids/weights (checked on upload: 2m, n, total vertex weight and
 *     total edge weight must be < 2^31), int64 for J, gains, block weights.
 *   - Kernel-level calls are asynchronous on `stream` unless they return a
 *     host scalar (documented per call), which synchronizes `stream`.
 */
#ifndef GPUIM_H_
#define GPUIM_H_

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define GIM_OK 0
#define GIM_E_INVALID 1     /* bad argument / violated precondition        */
#define GIM_E_CUDA 2        /* CUDA runtime error                          */
#define GIM_E_UNSUPPORTED 3 /* input outside the implemented envelope       */
#define GIM_E_OVERFLOW 4    /* value does not fit the int32 device layout   */
#define GIM_E_INTERNAL 5    /* unexpected internal failure                 */
#define GIM_E_EMPTY 6       /* empty graph (reference raises ValueError)     */
#define GIM_E_FORMAT 7      /* malformed METIS file (MetisFormatError)       */
#define GIM_E_IO 8          /* file cannot be opened / read                  */
#define GIM_E_CALLBACK 9    /* a caller callback returned nonzero (plugin)   */

#define GIM_MAX_LEVELS 32

/* Device-resident CSR graph (graph.py:17-39 `Graph`, int32 on device). */
typedef struct gim_graph {
  int32_t n;                /* vertices                                    */
  int64_t m2;               /* directed slots = 2m                         */
  const int32_t* offsets;   /* [n+1]                                       */
  const int32_t* targets;   /* [m2]                                        */
  const int32_t* weights;   /* [m2]  edge weights (> 0)                    */
  const int32_t* vweights;  /* [n]   vertex weights (> 0)                  */
  const int32_t* sources;   /* [m2]  edge sources (`edge_sources`, E_u)    */
} gim_graph;

/* Machine hierarchy a_1:...:a_l and distances d_1:...:d_l (topology.py:25-58
 * `Topology`), l <= GIM_MAX_LEVELS.  Distances may be non-integral
 * (Topology.integral_distances false): the device works on d * 2^s as exact
 * int64 (s = the smallest shift making every d integral when the d are
 * dyadic rationals — then every gain, J and decision equals the reference's
 * float arithmetic — else s chosen so that J fits int64, with the d rounded:
 * tolerance parity); gain-bucket bounds and the Jet filter are scaled by
 * 2^s.  gim_im_stats reports s, whether it is exact, and J in float64. */
typedef struct gim_topology {
  int32_t levels;
  int64_t hierarchy[GIM_MAX_LEVELS];
  double distances[GIM_MAX_LEVELS];
} gim_topology;

/* Keyword arguments of integrated_map (pipelines.py:221-235). */
typedef struct gim_im_params {
  int64_t coarsest_factor; /* 128   */
  double phi;              /* 0.999 */
  int32_t rho;             /* 2     */
  int32_t filter_mode;     /* 0 = "nonneg", 1 = "jet" */
  double jet_filter_c;     /* 0.25  */
  double sigma_coarse;     /* 0.065 */
  double sigma_fine;       /* 0.005 */
  int32_t iw_max_finest;   /* 10    */
  /* mode flags of THIS call (GIM_RUN_* bits), or GIM_RUN_DEFAULT = the
   * process defaults set by gim_set_* when the call starts.  Every mode
   * gives identical results; they exist for A/B measurement and tests. */
  int32_t run_flags;
  /* GIM_ISOLATED_KEEP (0, the reference's algorithm, bit-exact) or
   * GIM_ISOLATED_STRIP (1): degree-0 vertices are removed before the level
   * stack (they can never be matched, so on skewed graphs they stall the
   * coarsening, coarsening.py:289-290), the rest is mapped with the same
   * L_max, and the isolated vertices are water-filled into the lightest
   * blocks.  They add nothing to J wherever they go: tolerance parity
   * (every block <= L_max; J compared by geometric mean). */
  int32_t isolated;
} gim_im_params;

#define GIM_ISOLATED_KEEP 0
#define GIM_ISOLATED_STRIP 1

#define GIM_RUN_DEFAULT (-1)
#define GIM_RUN_FUSED 1    /* Alg. 4 as one persistent kernel per level     */
#define GIM_RUN_ROWWISE 2  /* row-wise contraction (else radix sort)        */
#define GIM_RUN_BATCH 4    /* batched multisection leaf-parent partitioning */
#define GIM_RUN_FANOUT 8   /* sibling subtrees on host threads / streams    */
#define GIM_RUN_PROFILE 16 /* per-class CUDA-event profiling (prof_* stats) */

/* Refinement counters (gim_im_stats.acct), summed over the IM levels'
 * refinement launches; SURVEY §8(d) algorithmic bytes are computed from
 * them. */
#define GIM_ACCT_SCAN 0       /* vertices swept by list-building passes     */
#define GIM_ACCT_BND 1        /* boundary vertices found (locked included)  */
#define GIM_ACCT_EVAL_V 2     /* vertices evaluated by the LP first filter  */
#define GIM_ACCT_EVAL_SLOTS 3 /* their row slots                            */
#define GIM_ACCT_EVAL_S 4     /* their distinct adjacent blocks (S)         */
#define GIM_ACCT_CAND_V 5     /* second-filter candidates                   */
#define GIM_ACCT_CAND_SLOTS 6 /* their row slots                            */
#define GIM_ACCT_MOV_V 7      /* movers applied                             */
#define GIM_ACCT_MOV_SLOTS 8  /* their row slots                            */
#define GIM_ACCT_OVL_V 9      /* rebalance: vertices of overloaded blocks   */
#define GIM_ACCT_OVL_SLOTS 10 /* rebalance: row slots walked                */
#define GIM_ACCT_OVL_S 11     /* rebalance: distinct adjacent blocks        */
#define GIM_ACCT_LP_IT 12     /* LP iterations                              */
#define GIM_ACCT_WEAK_IT 13   /* weak-rebalance iterations                  */
#define GIM_ACCT_BARRIERS 14  /* grid / cluster / CTA barriers (CTA 0)      */
#define GIM_ACCT_SWEEPS 15    /* entry sweeps over the whole CSR            */

/* Counters of one integrated_map run (for roofline accounting). */
typedef struct gim_im_stats {
  int32_t n_levels;            /* IM level-stack height                     */
  int64_t level_n[64];         /* vertices per level (finest first)         */
  int64_t level_m2[64];        /* directed slots per level                  */
  int64_t refine_iterations;   /* Alg. 4 iterations, IM levels              */
  int64_t lp_passes, weak_passes, strong_passes;
  int64_t init_refine_iterations; /* inside the initial multisection        */
  int64_t partitioner_calls;
  int64_t kernel_launches;     /* kernels launched by the whole call         */
  int64_t final_j;
  int64_t max_block_weight;
  double l_max;
  double ms_coarsen, ms_initial, ms_refine, ms_total; /* device-event times */
  /* per kernel class (only when profiling is on, see gim_set_profiling):
   * 0 J-eval, 1 HEM, 2 contraction, 3 LP first filter, 4 LP second filter,
   * 5 apply moves, 6 rebalance, 7 greedy growing, 8 subgraph extraction,
   * 9 two-hop matching.  ms from CUDA events on the launching stream,
   * bytes = algorithmic bytes, count = timed scopes. */
  double prof_ms[16];
  double prof_bytes[16];
  int64_t prof_count[16];
  /* the single timed scope with the most algorithmic bytes (profiling on):
   * its class, device ms and bytes — the finest-level refinement launch */
  int32_t top_class;
  double top_ms, top_bytes;
  /* host-array entry (gim_integrated_map) only: wall ms of the upload
   * (host narrowing + H2D) and of the download (D2H + widening) */
  double ms_upload, ms_download;
  /* host-array entry only: bytes copied host -> device (int32 CSR; weight
   * chunks holding one value are filled on the device instead) and back */
  int64_t bytes_h2d, bytes_d2h;
  /* refinement of each IM level (finest first): Alg. 4 iterations, device
   * ms (events around the level's refinement), SURVEY §8(d) algorithmic
   * bytes from the device counters, barriers executed */
  int64_t level_iters[64];
  double level_refine_ms[64];
  double level_bytes[64];
  int64_t level_barriers[64];
  /* GIM_ACCT_* counters summed over the IM levels */
  int64_t acct[16];
  /* distances as device integers d * 2^dist_shift (exact when dist_exact);
   * final_j above is in those units, final_j_f64 = J with the caller's
   * float distances (mapping.py:76-91 float path) */
  int32_t dist_shift;
  int32_t dist_exact;
  double final_j_f64;
  /* isolated-vertex strip mode: vertices set aside and mapped by the fill */
  int64_t isolated_vertices;
} gim_im_stats;

/* ---- library ---------------------------------------------------------- */
int gim_version(void);
const char* gim_last_error(void);

/* ---- objective ---------------------------------------------------------- */
/* J = sum over directed slots of w * D[Pi(src), Pi(tgt)]   (mapping.py:76-91).
 * *j_out (device int64) is OVERWRITTEN, in units of 2^-s (s = the
 * topology's distance shift, 0 for integral distances). */
int gim_total_cost(const gim_graph* g, const int32_t* assignment,
                   const gim_topology* t, int64_t* j_out, void* stream);

/* J in float64 with the topology's own distances (the reference's float J
 * for non-integral distances); *j_out device double, OVERWRITTEN. */
int gim_total_cost_f64(const gim_graph* g, const int32_t* assignment,
                       const gim_topology* t, double* j_out, void* stream);

/* Distance shift s of a topology and whether d * 2^s is exact (host ints). */
int gim_topology_scale(const gim_topology* t, int32_t* shift_out, int32_t* exact_out);

/* k-bin histogram of vertex weights, bw_out[k] overwritten (mapping.py:38-43). */
int gim_block_weights(const gim_graph* g, const int32_t* assignment, int32_t k,
                      int64_t* bw_out, void* stream);

/* ---- coarsening (coarsening.py) --------------------------------------- */
/* One heavy-edge matching round (coarsening.py:63-95).  partner[n] in/out
 * (-1 = unmatched), preferred[n] out; *matched_inout (host) is the matched
 * vertex count before/after.  Synchronizes `stream`. */
int gim_hem_round(const gim_graph* g, int32_t* partner, int32_t* preferred, double l_max,
                  uint64_t seed, int64_t* matched_inout, void* stream);

/* match_graph (coarsening.py:164-173): <= 2 HEM rounds, then two-hop
 * (leaves, twins, relatives; :113-161).  partner[n] out. Synchronizes. */
int gim_match_graph(const gim_graph* g, double l_max, uint64_t seed, int32_t* partner,
                    int64_t* matched_out, void* stream);

/* coarse_map_from_matching (coarsening.py:176-188); *n_c_out host. Syncs. */
int gim_coarse_map(int32_t n, const int32_t* partner, int32_t* coarse_map, int32_t* n_c_out,
                   void* stream);

/* contract (coarsening.py:191-249) by radix sort on (cu, cv) + segmented
 * reduce.  Output rows are sorted by target.  out_targets/out_weights/
 * out_sources need >= g->m2 slots, out_offsets n_c+1, out_vweights n_c.
 * *m2_out (host) = coarse directed slots.  Synchronizes. */
int gim_contract(const gim_graph* g, const int32_t* coarse_map, int32_t n_c,
                 int32_t* out_offsets, int32_t* out_targets, int32_t* out_weights,
                 int32_t* out_vweights, int32_t* out_sources, int64_t* m2_out, void* stream);

/* project (coarsening.py:269-277): fine_part[v] = coarse_part[coarse_map[v]]. */
int gim_project(int32_t n, const int32_t* coarse_map, const int32_t* coarse_part,
                int32_t* fine_part, void* stream);

/* ---- refinement (refinement.py, mapping.py) ---------------------------- */
/* BlockConnectivity values (mapping.py:141-158): per vertex the (block,
 * conn) list sorted by block.  out_blocks/out_weights need >= g->m2 slots.
 * *total_out (host) = number of entries.  Synchronizes. */
int gim_conn_build(const gim_graph* g, const int32_t* assignment, int32_t k,
                   int32_t* out_offsets, int32_t* out_blocks, int32_t* out_weights,
                   int64_t* total_out, void* stream);

/* label_propagation_pass (refinement.py:201-270) -> MoveProposal arrays.
 * locked may be NULL (no locks); jet = filter_mode "jet".  Synchronizes. */
int gim_lp_pass(const gim_graph* g, const int32_t* assignment, const uint8_t* locked,
                const gim_topology* t, int32_t jet, double jet_c, uint8_t* out_cand,
                int32_t* out_dest, uint8_t* out_to_move, int64_t* movers_out, void* stream);

/* weak_rebalance / strong_rebalance (refinement.py:312-386).  block_weights
 * is the device int64[k] of the current mapping.  Synchronizes. */
int gim_rebalance(const gim_graph* g, const int32_t* assignment, const int64_t* block_weights,
                  const gim_topology* t, int32_t strong, double sigma, double l_max, int32_t rho,
                  uint64_t seed, int64_t pass_counter, uint8_t* out_cand, int32_t* out_dest,
                  uint8_t* out_to_move, int32_t* incomplete_out, void* stream);

/* apply_moves (mapping.py:252-282): assignment/block_weights updated in
 * place, *delta_j_out (host) = exact change of J.  Synchronizes. */
int gim_apply_moves(const gim_graph* g, int32_t* assignment, int64_t* block_weights,
                    const uint8_t* to_move, const int32_t* dest, const gim_topology* t,
                    int64_t* delta_j_out, void* stream);

/* refine (Alg. 4, refinement.py:389-464) with an explicit RefinementConfig
 * (refinement.py:50-71).  assignment/block_weights are replaced by the best
 * mapping found.  Synchronizes. */
int gim_refine(const gim_graph* g, const gim_topology* t, int32_t* assignment,
               int64_t* block_weights, double phi, int32_t i_max, int32_t i_w_max,
               double sigma_fraction, int32_t rho, int32_t jet, double jet_c, uint64_t seed,
               double l_max, void* stream);

/* ---- initial mapping (pipelines.py) ------------------------------------ */
/* greedy_graph_growing (pipelines.py:132-188); requires n > k or k == 1. */
int gim_greedy_graph_growing(const gim_graph* g, int32_t k, int32_t* part, void* stream);

/* internal_partitioner (pipelines.py:191-218). Synchronizes. */
int gim_internal_partitioner(const gim_graph* g, int32_t k, double eps_local, uint64_t seed,
                             int32_t* part, void* stream);

/* hierarchical_multisection with the internal partitioner
 * (pipelines.py:49-110).  Synchronizes. */
int gim_hierarchical_multisection(const gim_graph* g, const gim_topology* t, double eps,
                                  uint64_t seed, int32_t* assignment, void* stream);

/* GPU-HM as a standalone algorithm on HOST int64 CSR arrays (the reference
 * Graph's own arrays): hierarchical_multisection of the whole graph with the
 * built-in partitioner (pipelines.py:49-110).  out_assignment int64[n],
 * out_block_weights int64[k] are host buffers. */
int gim_hierarchical_multisection_host(int64_t n, const int64_t* offsets, const int64_t* targets,
                                       const int64_t* edge_weights,
                                       const int64_t* vertex_weights, const gim_topology* t,
                                       double eps, uint64_t seed, int64_t* out_assignment,
                                       int64_t* out_block_weights, void* stream);

/* Plugin seam of hierarchical_multisection (pipelines.py:49-110): the
 * caller's partitioner, called once per tree node with parts > 1 in the
 * reference's depth-first order, receives the node's subgraph as HOST int64
 * CSR arrays (order-preserving local ids, graph.py:357-389), the node's
 * parts, eps_local (Eq. 2), seed and identifier, writes part[n] in
 * [0, parts) and returns 0 — nonzero aborts the call with GIM_E_CALLBACK.
 * NULL = the built-in GPU partitioner. */
typedef int (*gim_partition_fn)(void* user, int64_t n, const int64_t* offsets,
                                const int64_t* targets, const int64_t* edge_weights,
                                const int64_t* vertex_weights, int32_t parts, double eps_local,
                                uint64_t seed, const int32_t* ident, int32_t ident_len,
                                int64_t* out_part);

/* Trace record of one partitioning step (pipelines.py:36-47 SplitRecord,
 * appended at :98-104): level, identifier, parts, eps_local, subgraph
 * weight, the parts' block weights, budget met. */
typedef void (*gim_trace_fn)(void* user, int32_t level, const int32_t* ident, int32_t ident_len,
                             int32_t parts, double eps_local, int64_t subgraph_weight,
                             const int64_t* block_weights, int32_t budget_met);

/* hierarchical_multisection with the plugin seam and trace records, on HOST
 * int64 CSR arrays (depth-first, the reference's node order; each node's
 * extraction, block weights and the built-in partitioner run on the GPU).
 * partition / trace may be NULL. */
int gim_hierarchical_multisection_plugin(int64_t n, const int64_t* offsets,
                                         const int64_t* targets, const int64_t* edge_weights,
                                         const int64_t* vertex_weights, const gim_topology* t,
                                         double eps, uint64_t seed, gim_partition_fn partition,
                                         gim_trace_fn trace, void* user,
                                         int64_t* out_assignment, int64_t* out_block_weights,
                                         void* stream);

/* ---- the drop-in ------------------------------------------------------- */
/* Default keyword arguments of integrated_map. */
int gim_default_params(gim_im_params* out);

/* integrated_map on a device-resident level-0 graph (pipelines.py:221-269).
 * out_assignment int32[n], out_block_weights int64[k] (device).  params may
 * be NULL (defaults); stats may be NULL.  Synchronizes. */
int gim_integrated_map_device(const gim_graph* g, const gim_topology* t, double eps,
                              uint64_t seed, const gim_im_params* params,
                              int32_t* out_assignment, int64_t* out_block_weights,
                              gim_im_stats* stats, void* stream);

/* integrated_map on HOST int64 CSR arrays (graph.py:17-39 layout, no
 * edge_sources needed): upload, map, download.  out_assignment int64[n],
 * out_block_weights int64[k] are HOST arrays.  Returns GIM_E_EMPTY for n == 0
 * (reference: ValueError).  Synchronizes. */
int gim_integrated_map(int64_t n, const int64_t* offsets, const int64_t* targets,
                       const int64_t* edge_weights, const int64_t* vertex_weights,
                       const gim_topology* t, double eps, uint64_t seed,
                       const gim_im_params* params, int64_t* out_assignment,
                       int64_t* out_block_weights, gim_im_stats* stats, void* stream);

/* edge_sources from offsets (graph.py:32-36). */
int gim_fill_sources(int32_t n, const int32_t* offsets, int32_t* sources, void* stream);

/* Process defaults of the GIM_RUN_* modes, read by calls that start later
 * with run_flags = GIM_RUN_DEFAULT (calls in flight keep theirs). */
/* Per-kernel-class CUDA-event timing for integrated_map stats. */
void gim_set_profiling(int32_t on);

/* Run sibling multisection subtrees on concurrent host threads / CUDA
 * streams (default 1).  Results are identical either way. */
void gim_set_fanout(int32_t on);

/* Run Alg. 4 as one persistent cooperative kernel per level (default 1) or
 * as per-phase launches with host control.  Results are identical. */
void gim_set_fused(int32_t on);

/* Partition the small leaf-parent subgraphs of the multisection as one batch
 * (one launch per phase for all of them, default 1).  Results are identical. */
void gim_set_batch(int32_t on);

/* Contract level-stack matchings row-wise (default 1) or always with the
 * radix-sort path.  The coarse graphs are identical. */
void gim_set_rowwise_contraction(int32_t on);

/* ---- METIS input (graph.py:170-294, load_metis) -------------------------
 * gim_metis_load parses and validates a METIS ascii file with the reference's
 * rules and messages ("line N: ...", GIM_E_FORMAT) into a host CSR held by
 * *handle and reports n and 2m; gim_metis_fetch copies it into caller int64
 * arrays (offsets[n+1], targets[2m], edge weights[2m], vertex weights[n],
 * sources[2m]; any may be null) and frees the handle. */
int gim_metis_load(const char* path, void** handle, int64_t* n, int64_t* m2);
int gim_metis_fetch(void* handle, int64_t* offsets, int64_t* targets, int64_t* eweights,
                    int64_t* vweights, int64_t* sources);

/* METIS straight to a device CSR: the graph parsed by gim_metis_load is
 * narrowed to int32 and uploaded by the multi-threaded path of
 * gim_integrated_map (validation included) into caller DEVICE buffers
 * offsets[n+1], targets/weights/sources[2m], vweights[n]; *total_vweight
 * (host) = its total vertex weight.  Frees the handle. */
int gim_metis_upload(void* handle, int32_t* offsets, int32_t* targets, int32_t* weights,
                     int32_t* vweights, int32_t* sources, int64_t* total_vweight, void* stream);

/* kernels launched by kernel-level calls (outside integrated_map /
 * multisection calls, which count their own in gim_im_stats) since the last
 * reset (evidence). */
int64_t gim_launch_count(void);
void gim_reset_launch_count(void);

/* Device scratch is cached per (device, stream, size class) across calls;
 * this returns every cached block to the CUDA stream-ordered pools and trims
 * them (synchronizes the devices that held cached blocks). */
void gim_release_cached_memory(void);

#ifdef __cplusplus
}
#endif
#endif /* GPUIM_H_ */
