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

#define GIM_MAX_LEVELS 8

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

/* Machine hierarchy a_1:...:a_l and integral distances d_1:...:d_l
 * (topology.py:25-58 `Topology`; integral_distances must be true). */
typedef struct gim_topology {
  int32_t levels;
  int64_t hierarchy[GIM_MAX_LEVELS];
  int64_t distances[GIM_MAX_LEVELS];
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
} gim_im_params;

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
} gim_im_stats;

/* ---- library ---------------------------------------------------------- */
int gim_version(void);
const char* gim_last_error(void);

/* ---- objective ---------------------------------------------------------- */
/* J = sum over directed slots of w * D[Pi(src), Pi(tgt)]   (mapping.py:76-91).
 * *j_out (device int64) is OVERWRITTEN. */
int gim_total_cost(const gim_graph* g, const int32_t* assignment,
                   const gim_topology* t, int64_t* j_out, void* stream);

/* k-bin histogram of vertex weights, bw_out[k] overwritten (mapping.py:38-43). */
int gim_block_weights(const gim_graph* g, const int32_t* assignment, int32_t k,
                      int64_t* bw_out, void* stream);

#ifdef __cplusplus
}
#endif
#endif /* GPUIM_H_ */
