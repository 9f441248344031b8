// Shared device/host helpers for libgpuim (GPU-IM on sm_100a).
//
// Device layout: every CSR level lives in HBM as int32
// offsets/targets/weights/vertex weights plus an int32 edge-source array
// (the reference's `edge_sources`, graph.py:25-38 / PAPER.md:411-418).
// Block ids are int32, block weights / gains / J are int64.
#pragma once
#include <cuda_runtime.h>
#include <stdint.h>
#include <atomic>
#include <mutex>
#include <string>
#include <unordered_map>
#include <vector>

#include "../../include/gpuim.h"

namespace gim {

// ---------------------------------------------------------------------------
// error state (thread-local string + status codes from gpuim.h)

void set_error(const std::string& msg);
const char* last_error();

struct Error {
  int code;
  std::string msg;
};

// a failed call also leaves its code as the thread's "last error": clear it
// so the next call's launch check does not report this one again
#define GIM_CUDA(call)                                                        \
  do {                                                                        \
    cudaError_t _e = (call);                                                  \
    if (_e != cudaSuccess) {                                                  \
      (void)cudaGetLastError();                                               \
      throw ::gim::Error{GIM_E_CUDA, std::string(#call) + ": " +              \
                                         cudaGetErrorString(_e) + " @" +      \
                                         __FILE__ + ":" +                     \
                                         std::to_string(__LINE__)};           \
    }                                                                         \
  } while (0)

#define GIM_CHECK(cond, code, msg)                                            \
  do {                                                                        \
    if (!(cond)) throw ::gim::Error{(code), (msg)};                           \
  } while (0)

#define GIM_LAUNCH_CHECK() GIM_CUDA(cudaGetLastError())

// run `body` translating exceptions to a status code (C-ABI boundary)
template <class F>
int guard(F&& body) {
  try {
    body();
    return GIM_OK;
  } catch (const Error& e) {
    set_error(e.msg);
    return e.code;
  } catch (const std::exception& e) {
    set_error(std::string("internal error: ") + e.what());
    return GIM_E_INTERNAL;
  }
}

// ---------------------------------------------------------------------------
// topology: D[x,y] from mixed-radix digits, no k x k matrix
// (topology.py:112-129: d_j for the highest differing digit j, 0 if x == y)

// Each block id b gets a 64-bit "digit code": its mixed-radix digits packed
// into fixed bit fields, highest hierarchy level in the most significant
// field.  The highest set bit of code[x] ^ code[y] then lies in the field of
// the highest differing digit, and dbit[bit] holds that level's distance.
// Both tables live in one small device array (L1-resident), built once per
// topology by get_topo() — two cached loads + xor + clz per distance.
// Non-integral distances (topology.py:56-58) are carried as d * 2^dshift
// in int64 (exact for dyadic d); dbitf holds the caller's float distances per
// bit for the float64 J.
struct Topo {
  int L;                                // hierarchy levels
  int k;                                // number of PEs
  int dshift;                           // distance scale 2^dshift
  int exact;                            // 1: d * 2^dshift is exactly integral
  const unsigned long long* code;       // [k]
  const long long* dbit;                // [64]
  const double* dbitf;                  // [64] the caller's distances, followed
                                        // in the same buffer by lv[2L] (topo_lv)
};

// per-level table after dbitf (get_topo): group sizes P_l = a_0*..*a_l, then
// the scaled distances d_l — not a Topo field, so kernels passing Topo by
// value do not grow
__host__ __device__ __forceinline__ const long long* topo_lv(const Topo& t) {
  return reinterpret_cast<const long long*>(t.dbitf + 64);
}

// cached per (device, hierarchy, distances); device tables are never freed
Topo get_topo(const gim_topology& t);
Topo get_flat_topo(int k);
void topo_scale(int levels, const double* d, int* shift, int* exact);

__device__ __forceinline__ long long dist(const Topo& t, int x, int y) {
  unsigned long long c = __ldg(t.code + x) ^ __ldg(t.code + y);
  return c ? __ldg(t.dbit + (63 - __clzll(c))) : 0ll;
}

// ---------------------------------------------------------------------------
// deterministic mixers (util.py:13-24), uint64 arithmetic

__host__ __device__ __forceinline__ uint64_t splitmix64(uint64_t x) {
  x += 0x9E3779B97F4A7C15ull;
  uint64_t z = x;
  z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ull;
  z = (z ^ (z >> 27)) * 0x94D049BB133111EBull;
  return z ^ (z >> 31);
}

__host__ __device__ __forceinline__ uint64_t hash2(uint64_t seed, uint64_t a, uint64_t b) {
  return splitmix64(splitmix64(seed ^ splitmix64(a)) ^ b);
}

// ---------------------------------------------------------------------------
// per-call run context.  Everything one integrated_map / multisection call
// accumulates or switches on — the kernel-launch count, the profiling
// records, the refinement byte counters and the mode flags — lives in a
// RunCtx owned by that call and installed on the calling thread (CtxScope);
// the worker threads the call spawns install the same context.  Concurrent
// calls on different host threads (several maps per GPU on separate
// streams) therefore neither see nor reset each other's counters, and the
// process-wide gim_set_* defaults only affect calls that start afterwards.
// Kernel-level C-ABI calls outside such a call use the process context.

// Refinement counters (device-side, summed per k_refine_* launch) from which
// the algorithmic bytes of SURVEY §8(d) are computed
enum Acct {
  A_SCAN = 0,    // vertices swept by list-building passes (ext / overload test)
  A_BND,         // boundary vertices found by those passes (locked included)
  A_EVAL_V,      // vertices whose gains were evaluated (LP first filter)
  A_EVAL_SLOTS,  // their row slots
  A_EVAL_S,      // their distinct adjacent blocks (conn-table entries, S)
  A_CAND_V,      // second-filter candidates
  A_CAND_SLOTS,  // their row slots
  A_MOV_V,       // movers applied
  A_MOV_SLOTS,   // their row slots
  A_OVL_V,       // rebalance: vertices of overloaded blocks considered
  A_OVL_SLOTS,   // rebalance: row slots walked (non-interior candidates)
  A_OVL_S,       // rebalance: distinct adjacent blocks of those
  A_LP_IT,       // LP iterations
  A_WEAK_IT,     // weak-rebalance iterations
  A_BARRIERS,    // grid/cluster/CTA barriers executed (CTA 0)
  A_SWEEPS,      // entry sweeps over the whole CSR (J of the entry mapping / ext)
  A_COUNT
};

struct ProfRec {
  int cls;
  double bytes;
  cudaEvent_t a, b;
};

struct RunFlags {
  bool fused = true;    // Alg. 4 as one persistent kernel per level
  bool rowwise = true;  // row-wise contraction (else radix sort)
  bool batch = true;    // batched multisection leaf-parent partitioning
  bool fanout = true;   // sibling subtrees on host threads / streams
  bool prof = false;    // per-class CUDA-event profiling
};

struct RunCtx {
  RunFlags f;
  std::atomic<long long> launches{0};
  std::mutex mu;  // guards recs
  std::vector<ProfRec> recs;
  std::atomic<long long> acct[A_COUNT];
  RunCtx() { reset_acct(); }
  void reset_acct() {
    for (auto& a : acct) a.store(0);
  }
};

RunCtx& ctx();             // the calling thread's current context
RunFlags default_flags();  // process defaults (gim_set_*)
void set_default_flags(const RunFlags& f);

struct CtxScope {
  RunCtx* prev;
  explicit CtxScope(RunCtx* c);
  ~CtxScope();
  CtxScope(const CtxScope&) = delete;
  CtxScope& operator=(const CtxScope&) = delete;
};

// Cooperative grids launched from concurrent multisection workers leave one
// CTA slot per SM free, so they can start beside a sibling worker's
// single-CTA kernels (greedy growing) instead of waiting for them to finish
// (a cooperative launch is dispatched only when all its CTAs fit).  Results
// do not depend on the grid size.
int coop_blocks_per_sm(int occ);
struct ConcurrentScope {
  bool prev;
  ConcurrentScope();
  ~ConcurrentScope();
  ConcurrentScope(const ConcurrentScope&) = delete;
  ConcurrentScope& operator=(const ConcurrentScope&) = delete;
};

// launch accounting (current context)
void count_launch(long long n = 1);
long long launches();
void reset_launches();

// ---------------------------------------------------------------------------
// kernel-class profiling with CUDA events on the launching stream (off by
// default; bench.py turns it on for one attribution map).  Each scope records
// a start/stop event pair plus the algorithmic bytes of what it launched;
// prof_collect() resolves the pairs once at the end (no per-scope syncs).

enum ProfClass {
  P_JEVAL = 0, P_HEM, P_CONTRACT, P_LP_EVAL, P_LP_SECOND, P_APPLY, P_REBALANCE, P_GGG,
  P_EXTRACT, P_TWO_HOP, P_COUNT
};

bool prof_on();
void prof_begin(int cls, double bytes, cudaStream_t s, void** token);
void prof_end(void* token, cudaStream_t s, double extra_bytes);
// accumulate totals per class (ms, bytes, launches); clears the records
// and the single scope with the most bytes
void prof_collect(double* ms, double* bytes, long long* count, int* top_cls, double* top_ms,
                  double* top_bytes);

struct ProfScope {
  void* tok = nullptr;
  cudaStream_t s;
  double extra = 0.0;  // bytes only known after the launches (e.g. output size)
  ProfScope(int cls, double bytes, cudaStream_t st) : s(st) {
    if (prof_on()) prof_begin(cls, bytes, st, &tok);
  }
  ~ProfScope() {
    if (tok) prof_end(tok, s, extra);
  }
};

// ---------------------------------------------------------------------------
// launch geometry

constexpr int kSMs = 148;  // B200; grid-size heuristics only
// SMs of the current device (cached per ordinal): cooperative grids must not
// exceed what is co-resident on the actual part (MIG slices, reduced SKUs)
int device_sms();

inline int grid_for(long long work, int block, int max_blocks = kSMs * 16) {
  long long g = (work + block - 1) / block;
  if (g < 1) g = 1;
  if (g > max_blocks) g = max_blocks;
  return (int)g;
}

// ---------------------------------------------------------------------------
// warp helpers

__device__ __forceinline__ long long warp_sum_ll(long long v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  return v;
}

__device__ __forceinline__ int warp_sum_i(int v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  return v;
}

__device__ __forceinline__ unsigned lane_id() { return threadIdx.x & 31u; }

// block-wide int64 sum into *out with one atomic per block
template <int BLOCK>
__device__ __forceinline__ void block_sum_atomic(long long v, long long* out) {
  __shared__ long long s[BLOCK / 32];
  v = warp_sum_ll(v);
  if (lane_id() == 0) s[threadIdx.x >> 5] = v;
  __syncthreads();
  if (threadIdx.x < 32) {
    long long x = threadIdx.x < BLOCK / 32 ? s[threadIdx.x] : 0;
    x = warp_sum_ll(x);
    if (threadIdx.x == 0 && x != 0)
      atomicAdd(reinterpret_cast<unsigned long long*>(out), (unsigned long long)x);
  }
  __syncthreads();  // s[] is reusable by the next call (persistent kernels)
}

// ---------------------------------------------------------------------------
// host waits and per-thread host resources

// Wait for `s` by polling (cudaStreamQuery) with a yield between polls: the
// multisection fan-out keeps dozens of host threads waiting at once, and
// spinning inside cudaStreamSynchronize starves the threads that launch.
cudaError_t sync_stream(cudaStream_t s);

// pinned host scratch borrowed from a process-wide free list (cudaMallocHost
// / cudaFreeHost are device-synchronising, so worker threads must not call
// them); returned to the list when the owning thread exits
void* pinned_scratch(size_t bytes);

// non-blocking streams recycled across fan-out workers
cudaStream_t acquire_stream();
void release_stream(cudaStream_t s);

// ---------------------------------------------------------------------------
// stream-ordered device memory (cudaMallocAsync pool behind a stream-keyed cache)

void* dmalloc(size_t bytes, cudaStream_t s);
void dfree(void* p, cudaStream_t s);

void release_cached_memory();

template <class T>
struct DBuf {
  T* p = nullptr;
  size_t n = 0;
  cudaStream_t s = nullptr;
  DBuf() = default;
  DBuf(size_t count, cudaStream_t st) : n(count), s(st) {
    p = count ? static_cast<T*>(dmalloc(count * sizeof(T), st)) : nullptr;
  }
  DBuf(const DBuf&) = delete;
  DBuf& operator=(const DBuf&) = delete;
  DBuf(DBuf&& o) noexcept : p(o.p), n(o.n), s(o.s) { o.p = nullptr; o.n = 0; }
  DBuf& operator=(DBuf&& o) noexcept {
    if (this != &o) {
      release();
      p = o.p; n = o.n; s = o.s;
      o.p = nullptr; o.n = 0;
    }
    return *this;
  }
  ~DBuf() { release(); }
  void release() {
    if (p) dfree(p, s);
    p = nullptr;
    n = 0;
  }
  T* get() const { return p; }
};

}  // namespace gim
