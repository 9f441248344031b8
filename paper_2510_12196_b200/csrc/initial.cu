// Initial mapping kernels: greedy graph growing (K15), subgraph extraction
// (K14) and the leaf scatter of the hierarchical multisection.
//
// Reference: pipelines.py (_multi_source_bfs :113-129, greedy_graph_growing
// :132-188, hierarchical_multisection leaf :78-80), graph.py
// (extract_subgraphs :357-389).
#include <cooperative_groups.h>

#include <algorithm>
#include <chrono>
#include <cstdio>
#include <cstdlib>
#include <mutex>
#include <vector>

#include "common.cuh"
#include "kernels.cuh"
#include "radix.cuh"
#include "scan.cuh"

namespace gim {

namespace cg = cooperative_groups;

// ---------------------------------------------------------------------------
// K15 greedy graph growing, one CTA per subgraph (the coarsest partitioner
// graphs hold a few hundred vertices).  Semantics of pipelines.py:132-188:
//  * seeds: farthest-first over hop distances (BFS from {0}; then from the
//    seed set), preferring the lowest unreachable vertex, else the first
//    vertex of maximum distance;
//  * growth: the lightest block (ties: lowest id) claims, among unassigned
//    vertices it is connected to, the one with maximum connectivity (ties:
//    lowest id) — exactly the entry its lazy max-heap would pop — or the
//    lowest unassigned vertex when it has none.
// dist[n], part[n], conn[k][n] live in shared memory when they fit (else in
// the global scratch); every selection is a CTA-wide argmax/argmin.

constexpr int kGggBlock = 256;
constexpr int kGggMaxK = 64;  // block weights in shared memory up to this k
constexpr int kGggWarps = kGggBlock / 32;

struct GggJob {
  int n;
  int k;
  const int* off;
  const int* tgt;
  const int* w;
  const int* vw;
  int* part;        // out [n]
  int* scratch;     // global fallback: dist[n] + part[n] + seeds[k] + conn[k*n]
  long long* bwork; // [k]
  int use_smem;
  int m2;
  int stage;        // 1: the graph itself is copied into shared memory too
};

// CTA-wide lexicographic max of (a, -b): larger a wins, ties -> smaller b
__device__ __forceinline__ void cta_argmax(int& a, int& b, int* sa, int* sb) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) {
    int a2 = __shfl_xor_sync(0xffffffffu, a, o), b2 = __shfl_xor_sync(0xffffffffu, b, o);
    if (a2 > a || (a2 == a && b2 < b)) { a = a2; b = b2; }
  }
  if (lane_id() == 0) { sa[threadIdx.x >> 5] = a; sb[threadIdx.x >> 5] = b; }
  __syncthreads();
  a = sa[0];
  b = sb[0];
  const int nw = (int)(blockDim.x >> 5);
  for (int i = 1; i < nw; ++i)
    if (sa[i] > a || (sa[i] == a && sb[i] < b)) { a = sa[i]; b = sb[i]; }
  __syncthreads();
}

// Level-synchronous multi-source BFS (pipelines.py:113-130).  Race-free: a
// round first READS dist and marks the next frontier in the bitmap `nxt`
// (ceil(n/32) words, zero on entry and on exit) with atomicOr, then each
// bitmap word's owner thread writes dist and clears the word.
// `fresh`: distances from the seed set from scratch; else `dist` holds the
// distances from seeds[0..ns-2] and only seeds[ns-1] is added: a pruned BFS
// that lowers distances where the new seed is closer (every vertex on a
// shortest path to an improved vertex is improved too, so the result is the
// multi-source distance) and stops when a round improves nothing.
__device__ void cta_bfs(int n, const int* off, const int* tgt, int* dist, const int* seeds,
                        int ns, unsigned* nxt, bool fresh = true) {
  if (fresh) {
    for (int v = threadIdx.x; v < n; v += blockDim.x) dist[v] = -1;
    __syncthreads();
    for (int i = threadIdx.x; i < ns; i += blockDim.x) dist[seeds[i]] = 0;
  } else if (threadIdx.x == 0) {
    dist[seeds[ns - 1]] = 0;
  }
  __syncthreads();
  const int nw = (n + 31) >> 5;
  for (int d = 0;; ++d) {
    for (int v = threadIdx.x; v < n; v += blockDim.x) {
      if (dist[v] != d) continue;
      for (int e = off[v]; e < off[v + 1]; ++e) {
        const int u = tgt[e];
        const int du = dist[u];
        if (du < 0 || du > d + 1) atomicOr(&nxt[u >> 5], 1u << (u & 31));
      }
    }
    __syncthreads();
    int changed = 0;
    for (int w = threadIdx.x; w < nw; w += blockDim.x) {
      unsigned m = nxt[w];
      if (!m) continue;
      nxt[w] = 0;
      changed = 1;
      while (m) {
        const int b = __ffs(m) - 1;
        m &= m - 1;
        dist[(w << 5) + b] = d + 1;
      }
    }
    if (!__syncthreads_or(changed)) break;
  }
}

// farthest-first seed: lowest unreached vertex if any, else first argmax
__device__ int cta_pick_seed(int n, const int* dist, int* sa, int* sb) {
  int unr = INT_MIN + 1, ubv = INT_MAX;  // max of (-v) over unreached
  int bd = -1, bv = INT_MAX;
  for (int v = threadIdx.x; v < n; v += blockDim.x) {
    int d = dist[v];
    if (d < 0) {
      if (ubv == INT_MAX) { unr = 1; ubv = v; }
    } else if (d > bd) {
      bd = d;
      bv = v;
    }
  }
  int ua = ubv == INT_MAX ? 0 : 1;
  cta_argmax(ua, ubv, sa, sb);
  if (ua) return ubv;
  cta_argmax(bd, bv, sa, sb);
  return bv;
}

__global__ void __launch_bounds__(kGggBlock) k_ggg(const GggJob* jobs, int njobs) {
  const int j = blockIdx.x;
  if (j >= njobs) return;
  const GggJob J = jobs[j];
  const int n = J.n, k = J.k;
  extern __shared__ int sm[];
  __shared__ int sa[kGggWarps], sb[kGggWarps];
  __shared__ int s_v, s_b, s_next;
  int* base = J.use_smem ? sm : J.scratch;
  int* dist = base;
  int* part = dist + n;
  int* seeds = part + n;
  int* conn = seeds + k;
  unsigned* nxt = reinterpret_cast<unsigned*>(conn + (size_t)k * n);  // BFS frontier bitmap
  const int nch = (n + 31) >> 5;
  int* cmx = reinterpret_cast<int*>(nxt) + nch;  // [k][nch] chunk maxima (upper bounds)
  if (k == 1) {
    for (int v = threadIdx.x; v < n; v += blockDim.x) J.part[v] = 0;
    return;
  }
  for (int w = threadIdx.x; w < ((n + 31) >> 5); w += blockDim.x) nxt[w] = 0;
  // small graphs: CSR staged in shared memory (every growth step walks a row
  // and reads a vertex weight on its critical path)
  const int* g_off = J.off;
  const int* g_tgt = J.tgt;
  const int* g_w = J.w;
  const int* g_vw = J.vw;
  if (J.stage) {
    int* so = cmx + (size_t)k * nch;
    int* st = so + n + 1;
    int* sw = st + J.m2;
    int* sv = sw + J.m2;
    for (int i = threadIdx.x; i <= n; i += blockDim.x) so[i] = J.off[i];
    for (int i = threadIdx.x; i < J.m2; i += blockDim.x) {
      st[i] = J.tgt[i];
      sw[i] = J.w[i];
    }
    for (int i = threadIdx.x; i < n; i += blockDim.x) sv[i] = J.vw[i];
    __syncthreads();
    g_off = so;
    g_tgt = st;
    g_w = sw;
    g_vw = sv;
  }
  // seeds (pipelines.py:143-153)
  if (threadIdx.x == 0) s_v = 0;
  __syncthreads();
  cta_bfs(n, g_off, g_tgt, dist, &s_v, 1, nxt);
  int sv = cta_pick_seed(n, dist, sa, sb);
  if (threadIdx.x == 0) seeds[0] = sv;
  __syncthreads();
  for (int ns = 1; ns < k; ++ns) {
    cta_bfs(n, g_off, g_tgt, dist, seeds, ns, nxt, ns == 1);
    sv = cta_pick_seed(n, dist, sa, sb);
    if (threadIdx.x == 0) seeds[ns] = sv;
    __syncthreads();
  }
  // growth (pipelines.py:155-188) driven by warp 0 alone, no CTA barrier per
  // claim.  conn[b][u] holds block b's connectivity to unassigned u (-1 once
  // u is assigned, in every block); cmx[b][c] >= max conn[b][u] over chunk c
  // (32 vertices) is an UPPER bound: a claim raises it (atomicMax), an
  // assignment leaves it stale and a query that finds the chunk's true max
  // below the bound repairs it and retries.  The query takes the chunk
  // attaining the largest bound (lowest chunk on ties), then the lowest
  // vertex attaining the true maximum in it: the heap pop of pipelines.py
  // (max conn, lowest id); a zero maximum means the frontier is dry and the
  // lowest unassigned vertex is claimed instead.
  __shared__ long long s_bw[kGggMaxK];
  long long* bw = k <= kGggMaxK ? s_bw : J.bwork;
  for (int v = threadIdx.x; v < n; v += blockDim.x) part[v] = -1;
  for (long long i = threadIdx.x; i < (long long)k * n; i += blockDim.x) conn[i] = 0;
  for (long long i = threadIdx.x; i < (long long)k * nch; i += blockDim.x) cmx[i] = 0;
  for (int b = threadIdx.x; b < k; b += blockDim.x) bw[b] = 0;
  __syncthreads();
  if (threadIdx.x < 32) {
    const int lane = (int)threadIdx.x;
    auto claim = [&](int v, int b) {  // warp 0
      if (lane == 0) {
        part[v] = b;
        bw[b] += g_vw[v];
      }
      for (int x = lane; x < k; x += 32) conn[(long long)x * n + v] = -1;
      __syncwarp();
      int* cb = conn + (long long)b * n;
      int* mb = cmx + (long long)b * nch;
      for (int e = g_off[v] + lane; e < g_off[v + 1]; e += 32) {
        const int u = g_tgt[e];
        const int c0 = cb[u];
        if (u == v || c0 < 0) continue;  // assigned (distinct u per row)
        const int c = c0 + g_w[e];
        cb[u] = c;
        atomicMax(mb + (u >> 5), c);
      }
      __syncwarp();
    };
    for (int b = 0; b < k; ++b) claim(seeds[b], b);
    int next_free = 0;  // lane-uniform
    for (int assigned = k; assigned < n; ++assigned) {
      // lightest block, lowest id on ties (block weights < 2^31: totals are
      // checked on upload): warp min-reduce, then the lowest lane attaining it
      unsigned bwv = 0xffffffffu;
      int bb = INT_MAX;
      for (int b = lane; b < k; b += 32) {
        const unsigned x = (unsigned)bw[b];
        if (x < bwv) { bwv = x; bb = b; }
      }
      const unsigned mn = __reduce_min_sync(0xffffffffu, bwv);
      bb = (int)__reduce_min_sync(0xffffffffu, bwv == mn ? (unsigned)bb : 0xffffffffu);
      const int* cb = conn + (long long)bb * n;
      int* mb = cmx + (long long)bb * nch;
      int gv = -1;
      for (;;) {
        int bc = 0, bch = INT_MAX;  // largest bound, lowest chunk
        for (int c = lane; c < nch; c += 32) {
          const int x = mb[c];
          if (x > bc) { bc = x; bch = c; }
        }
        const int mx = (int)__reduce_max_sync(0xffffffffu, (unsigned)bc);
        if (mx <= 0) break;  // frontier dry
        bch = (int)__reduce_min_sync(0xffffffffu, bc == mx ? (unsigned)bch : 0xffffffffu);
        const int u = (bch << 5) + lane;
        const int cu = u < n ? max(cb[u], 0) : 0;
        const int cm = (int)__reduce_max_sync(0xffffffffu, (unsigned)cu);
        if (cm == mx) {
          const int gl = __ffs(__ballot_sync(0xffffffffu, cu == cm)) - 1;
          gv = (bch << 5) + gl;
          // eager removal of gv from bb's bound of this chunk (its conn
          // becomes -1 at the claim): the next query of bb needs no repair
          const int rest = (int)__reduce_max_sync(0xffffffffu, lane == gl ? 0u : (unsigned)cu);
          if (lane == 0) mb[bch] = rest;
          __syncwarp();
          break;
        }
        if (lane == 0) mb[bch] = cm;  // stale bound: repair, retry
        __syncwarp();
      }
      if (gv < 0) {  // frontier dried up: lowest unassigned vertex
        while (part[next_free] >= 0) ++next_free;
        gv = next_free;
      }
      claim(gv, bb);
    }
  }
  __syncthreads();
  for (int v = threadIdx.x; v < n; v += blockDim.x) J.part[v] = part[v];
}

// ---------------------------------------------------------------------------
// K15' greedy graph growing for graphs too large for shared memory (the
// stalled coarsest graphs of R-MAT inputs: 10^5..10^6 vertices, many of them
// isolated).  The CTA-wide argmax over all n vertices per claimed vertex
// above is O(n^2); here every block's frontier is indexed by a two-level max
// structure — cmax[b][c] >= max conn[b][u] over the unassigned u of chunk c
// (kGgCh vertices), smax[b][s] >= max cmax[b][c] over superchunk s (kGgSc
// chunks) — kept as UPPER bounds: a claim only raises them (atomicMax), and
// an assigned vertex is dropped lazily: a query that finds no unassigned
// vertex attaining a bound recomputes that chunk/superchunk and retries.
// A claimed vertex's conn entries are set to INT_MIN in every block, so the
// query and the row update need no separate assignment lookup.
// The query walks smax -> cmax -> conn taking the lowest index attaining the
// maximum at each level, which is exactly the heap pop of pipelines.py:
// maximum connectivity, ties to the lowest vertex id.
//
// One warp drives the growth loop (lightest block, query, claim, row update
// for rows up to kGgWarpRow slots) with no CTA barrier; longer rows
// are handed to the whole CTA.  Isolated vertices claimed by the fallback
// cost one step of the warp.

static bool trace_ggg() {
  static const bool on = std::getenv("GIM_TRACE_MS") != nullptr;
  return on;
}

// chunk / superchunk sizes (GIM_GG_CH / GIM_GG_SC override for A/B builds):
// 1024-vertex chunks keep the chunk bounds of a 2M-vertex coarsest graph in
// shared memory for k = 8 (70 KB), so a query makes one global round trip
// (the conn scan of its chunk) instead of two
#ifndef GIM_GG_CH
#define GIM_GG_CH 1024
#endif
#ifndef GIM_GG_SC
#define GIM_GG_SC 32
#endif
constexpr int kGgCh = GIM_GG_CH;
constexpr int kGggMaxDry = 1024;  // known-dry flags for k up to this
constexpr int kGgSc = GIM_GG_SC;
constexpr int kGgWarpRow = 128;

__device__ __forceinline__ int warp_max_int(int v) {
  return (int)__reduce_max_sync(0xffffffffu, (unsigned)v);  // v >= 0
}

struct GggLargeJob {
  int n;
  int k;
  const int* off;
  const int* tgt;
  const int* w;
  const int* vw;
  int* part;        // out [n], also the working assignment
  int* dist;        // [n]
  int* seeds;       // [k]
  int* conn;        // [k][n], zeroed by the host
  int* cmax;        // [k][nch], zeroed by the host
  int* gsmax;       // [k][nsc] (when not in shared memory), zeroed by the host
  long long* bwork; // [k]
  int smax_smem;
  int cmax_smem;    // chunk bounds in shared memory too (after the smax words)
  long long* stat;  // [8] diagnostics (GIM_TRACE_MS) or null: frontier claims,
                    // fallback claims, known-dry skips, bound repairs, CTA hub
                    // updates, cycles in queries, cycles in claims/updates,
                    // cycles in CTA hub-row updates
};

// bound loads / stores: shared memory (volatile: other warps' atomics) or L2
__device__ __forceinline__ int bnd_ld(const int* p, bool smem) {
  return smem ? *reinterpret_cast<const volatile int*>(p) : __ldcg(p);
}
__device__ __forceinline__ void bnd_st(int* p, int x, bool smem) {
  if (smem) *reinterpret_cast<volatile int*>(p) = x;
  else __stcg(p, x);
}

__device__ __forceinline__ void gg_row_update(const GggLargeJob& J, int v, int b, int nch,
                                              int nsc, int* smax, int* cmax, int t0, int stride) {
  const int n = J.n;
  int* cb = J.conn + (size_t)b * n;
  int* mb = cmax + (size_t)b * nch;
  int* sb = smax + (size_t)b * nsc;
  const int e1 = __ldg(J.off + v + 1);
  // four slots per thread per step with their loads issued together
  // (same-address atomics stay per slot: warp aggregation with
  // __match_any_sync doubled the hub-row update time, r2j A/B)
  for (int e = __ldg(J.off + v) + t0; e < e1; e += 4 * stride) {
    int u[4], wq[4], c0[4];
#pragma unroll
    for (int q = 0; q < 4; ++q) {
      const int eq = e + q * stride;
      u[q] = eq < e1 ? __ldg(J.tgt + eq) : v;
      wq[q] = eq < e1 ? __ldg(J.w + eq) : 0;
    }
#pragma unroll
    for (int q = 0; q < 4; ++q) c0[q] = u[q] != v ? __ldcg(cb + u[q]) : -1;
#pragma unroll
    for (int q = 0; q < 4; ++q) {
      if (c0[q] < 0) continue;  // conn < 0: assigned (or padding / self)
      const int c = c0[q] + wq[q];  // distinct u per row
      __stcg(cb + u[q], c);
      atomicMax(mb + u[q] / kGgCh, c);
      atomicMax(sb + u[q] / (kGgCh * kGgSc), c);
    }
  }
}

__global__ void __launch_bounds__(kGggBlock) k_ggg_large(const GggLargeJob* jobs) {
  const GggLargeJob J = jobs[blockIdx.x];
  const int n = J.n, k = J.k;
  extern __shared__ int sm[];
  __shared__ int sa[kGggWarps], sb[kGggWarps];
  __shared__ int s_cmd, s_v, s_b;
  __shared__ long long s_bw[kGggMaxK];
  // known-dry blocks: bit b set = b's frontier was found empty and b has
  // claimed only isolated vertices since (only b's own claims can grow b's
  // frontier), so its next query can be skipped
  __shared__ unsigned s_dry[(kGggMaxDry + 31) / 32];
  const int nch = (n + kGgCh - 1) / kGgCh, nsc = (nch + kGgSc - 1) / kGgSc;
  const bool track_dry = k <= kGggMaxDry;
  for (int i = threadIdx.x; i < (kGggMaxDry + 31) / 32; i += blockDim.x) s_dry[i] = 0;
  int* smax = J.smax_smem ? sm : J.gsmax;
  int* cmax = J.cmax_smem ? sm + (size_t)k * nsc : J.cmax;
  long long* bw = k <= kGggMaxK ? s_bw : J.bwork;
  if (k == 1) {
    for (int v = threadIdx.x; v < n; v += blockDim.x) J.part[v] = 0;
    return;
  }
  if (J.smax_smem)
    for (int i = threadIdx.x; i < k * nsc; i += blockDim.x) smax[i] = 0;
  if (J.cmax_smem)
    for (int i = threadIdx.x; i < k * nch; i += blockDim.x) cmax[i] = 0;
  // seeds: k_ggg_seeds (grid-wide BFS) ran before this launch
  for (int v = threadIdx.x; v < n; v += blockDim.x) J.part[v] = -1;
  for (int b = threadIdx.x; b < k; b += blockDim.x) bw[b] = 0;
  __syncthreads();
  for (int b = 0; b < k; ++b) {  // claim the seeds in block order
    const int s = J.seeds[b];
    if (threadIdx.x == 0) {
      J.part[s] = b;
      bw[b] += J.vw[s];
    }
    for (int b2 = threadIdx.x; b2 < k; b2 += blockDim.x) J.conn[(size_t)b2 * n + s] = INT_MIN;
    __syncthreads();
    gg_row_update(J, s, b, nch, nsc, smax, cmax, threadIdx.x, blockDim.x);
    __syncthreads();
  }
  const int lane = lane_id(), warp = threadIdx.x >> 5;
  int assigned = k, next_free = 0;  // warp 0's loop state (uniform in the warp)
  // fallback window: vertices [win, win + 32) one per lane — unassigned
  // flag, degree, weight — so runs of fallback claims (the isolated vertices
  // of stalled R-MAT coarsest graphs) cost no global loads; every claim
  // inside the window clears its lane's flag
  int win = -64;
  bool w_free = false;
  int w_deg = 0, w_vw = 0;
  for (;;) {
    if (warp == 0) {
      int cmd = 2;
      while (assigned < n) {
        if (k <= 32) {
          // Isolated run: while the lightest block is known-dry and the
          // lowest unassigned vertex has no neighbours, each step is the
          // general loop's fallback claim with nothing else to do (no query,
          // no frontier change, the block stays dry) — so run it with the
          // block weights and dry flags in lane registers: one argmin, one
          // ballot, two stores per claim.  Stops at the first step the
          // general loop would handle differently.
          long long myb = lane < k ? bw[lane] : 0;
          const unsigned dry = s_dry[0];
          long long runs = 0;
          for (;;) {
            const unsigned x = lane < k ? (unsigned)myb : 0xffffffffu;
            const unsigned mn = __reduce_min_sync(0xffffffffu, x);
            const int bb = (int)__reduce_min_sync(0xffffffffu, x == mn ? (unsigned)lane : 32u);
            if (!((dry >> bb) & 1u)) break;
            if (next_free < win || next_free >= win + 32) {
              win = next_free;
              const int u = win + lane;
              w_free = u < n && __ldcg(J.conn + u) >= 0;
              w_deg = u < n ? __ldg(J.off + u + 1) - __ldg(J.off + u) : 0;
              w_vw = u < n ? __ldg(J.vw + u) : 0;
            }
            const unsigned m = __ballot_sync(0xffffffffu, w_free && win + lane >= next_free);
            if (!m) {
              next_free = win + 32;
              continue;
            }
            const int l = __ffs(m) - 1;
            if (__shfl_sync(0xffffffffu, w_deg, l) != 0) break;
            const int v = win + l;
            const int vwv = __shfl_sync(0xffffffffu, w_vw, l);
            if (lane == l) w_free = false;
            if (lane == bb) myb += vwv;
            if (lane == 0) {
              J.part[v] = bb;
              __stcg(J.conn + v, INT_MIN);
            }
            next_free = v;
            ++runs;
            if (++assigned >= n) break;
          }
          if (lane < k) bw[lane] = myb;
          if (J.stat && lane == 0) {
            J.stat[1] += runs;
            J.stat[2] += runs;
          }
          __syncwarp();
          if (assigned >= n) break;
        }
        // lightest block, lowest id on ties (weights < 2^31: totals are
        // checked on upload): warp min-reduce, lowest lane attaining it
        unsigned bwv = 0xffffffffu;
        int bb = INT_MAX;
        for (int b = lane; b < k; b += 32) {
          const unsigned x = (unsigned)bw[b];
          if (x < bwv) { bwv = x; bb = b; }
        }
        const unsigned mn = __reduce_min_sync(0xffffffffu, bwv);
        bb = (int)__reduce_min_sync(0xffffffffu, bwv == mn ? (unsigned)bb : 0xffffffffu);
        int* cb = J.conn + (size_t)bb * n;
        int* mb = cmax + (size_t)bb * nch;
        const bool cs = J.cmax_smem, ss = J.smax_smem;
        int* sbm = smax + (size_t)bb * nsc;
        int v = -1;
        const bool known_dry = track_dry && ((s_dry[bb >> 5] >> (bb & 31)) & 1u);
        const long long t_q0 = J.stat ? clock64() : 0;
        if (J.stat && known_dry && lane == 0) J.stat[2] += 1;
        for (; !known_dry;) {  // query with lazy repair of stale bounds
          int top = 0, ts = INT_MAX;
          for (int i = lane; i < nsc; i += 32) {
            const int x = bnd_ld(sbm + i, ss);
            if (x > top) { top = x; ts = i; }
          }
#pragma unroll
          for (int o = 16; o > 0; o >>= 1) {
            const int x2 = __shfl_xor_sync(0xffffffffu, top, o);
            const int s2 = __shfl_xor_sync(0xffffffffu, ts, o);
            if (x2 > top || (x2 == top && s2 < ts)) { top = x2; ts = s2; }
          }
          if (top == 0) {  // every frontier bound is empty
            if (track_dry && lane == 0) s_dry[bb >> 5] |= 1u << (bb & 31);
            __syncwarp();
            break;
          }
          // lowest chunk of superchunk ts whose bound equals top
          const int c0 = ts * kGgSc;
          int cm[kGgSc / 32];
#pragma unroll
          for (int j = 0; j < kGgSc / 32; ++j) {
            const int c = c0 + j * 32 + lane;
            cm[j] = c < nch ? bnd_ld(mb + c, cs) : 0;
          }
          int ch = -1, smx = 0;
#pragma unroll
          for (int j = 0; j < kGgSc / 32; ++j) {
            const unsigned m = __ballot_sync(0xffffffffu, cm[j] == top);
            if (ch < 0 && m) ch = c0 + j * 32 + __ffs(m) - 1;
            smx = max(smx, cm[j]);
          }
          if (ch < 0 && J.stat && lane == 0) J.stat[3] += 1;
          if (ch < 0) {  // stale superchunk bound: tighten it and retry
            smx = warp_max_int(smx);
            if (lane == 0) {
              bnd_st(sbm + ts, smx, ss);
            }
            __syncwarp();
            continue;
          }
          // lowest unassigned vertex of chunk ch with conn == top
          const int u0 = ch * kGgCh;
          int cv[kGgCh / 32];
#pragma unroll
          for (int j = 0; j < kGgCh / 32; ++j) {
            const int u = u0 + j * 32 + lane;
            cv[j] = u < n ? __ldcg(cb + u) : 0;
          }
          int cmx = 0;
#pragma unroll
          for (int j = 0; j < kGgCh / 32; ++j) {
            const unsigned m = __ballot_sync(0xffffffffu, cv[j] == top);
            if (v < 0 && m) v = u0 + j * 32 + __ffs(m) - 1;
            cmx = max(cmx, cv[j]);
          }
          if (v >= 0) {
            // eager removal of v from bb's bounds (no memory round: the
            // chunk and superchunk values are in registers), so the next
            // query of bb needs no repair for it
            const int vj = (v - u0) >> 5, vl = (v - u0) & 31;
            int c2 = 0;
#pragma unroll
            for (int j = 0; j < kGgCh / 32; ++j)
              c2 = max(c2, (j == vj && lane == vl) ? 0 : cv[j]);
            c2 = warp_max_int(c2);
            const int lj = (ch - c0) >> 5, ll = (ch - c0) & 31;
            int s2 = 0;
#pragma unroll
            for (int j = 0; j < kGgSc / 32; ++j)
              s2 = max(s2, (j == lj && lane == ll) ? c2 : cm[j]);
            s2 = warp_max_int(s2);
            if (lane == 0) {
              bnd_st(mb + ch, c2, cs);
              bnd_st(sbm + ts, s2, ss);
            }
            break;
          }
          // stale chunk bound: tighten chunk and superchunk, retry
          if (J.stat && lane == 0) J.stat[3] += 1;
          cmx = warp_max_int(cmx);
          const int lj = (ch - c0) >> 5, ll = (ch - c0) & 31;
#pragma unroll
          for (int j = 0; j < kGgSc / 32; ++j)
            if (j == lj && lane == ll) cm[j] = cmx;
          int s2 = 0;
#pragma unroll
          for (int j = 0; j < kGgSc / 32; ++j) s2 = max(s2, cm[j]);
          s2 = warp_max_int(s2);
          if (lane == 0) {
            bnd_st(mb + ch, cmx, cs);
            bnd_st(sbm + ts, s2, ss);
          }
          __syncwarp();
        }
        const long long t_q1 = J.stat ? clock64() : 0;
        if (J.stat && lane == 0) {
          J.stat[v < 0 ? 1 : 0] += 1;
          J.stat[5] += t_q1 - t_q0;
        }
        int vwv, deg;
        if (v < 0) {  // frontier dried up: lowest unassigned vertex
          for (;;) {
            if (next_free < win || next_free >= win + 32) {
              win = next_free;
              const int u = win + lane;
              w_free = u < n && __ldcg(J.conn + u) >= 0;  // block 0's row marks assigned
              w_deg = u < n ? __ldg(J.off + u + 1) - __ldg(J.off + u) : 0;
              w_vw = u < n ? __ldg(J.vw + u) : 0;
            }
            const unsigned m = __ballot_sync(0xffffffffu, w_free && win + lane >= next_free);
            if (m) {
              const int l = __ffs(m) - 1;
              v = win + l;
              deg = __shfl_sync(0xffffffffu, w_deg, l);
              vwv = __shfl_sync(0xffffffffu, w_vw, l);
              next_free = v;
              break;
            }
            next_free = win + 32;
          }
        } else {
          vwv = __ldg(J.vw + v);
          deg = __ldg(J.off + v + 1) - __ldg(J.off + v);
        }
        if (v >= win && v < win + 32 && lane == v - win) w_free = false;
        if (lane == 0) {
          J.part[v] = bb;
          bw[bb] += vwv;
          // bb may have a frontier after a claim with neighbours
          if (deg > 0 && track_dry) s_dry[bb >> 5] &= ~(1u << (bb & 31));
        }
        // assigned marks: an isolated vertex never enters a frontier (no
        // neighbour raises its conn), so only block 0's row — the fallback
        // scan's "unassigned" test — needs the mark; others need all k
        if (deg > 0) {
          for (int b2 = lane; b2 < k; b2 += 32) __stcg(J.conn + (size_t)b2 * n + v, INT_MIN);
        } else if (lane == 0) {
          __stcg(J.conn + v, INT_MIN);
        }
        ++assigned;
        __syncwarp();
        if (J.stat && lane == 0) {
          J.stat[4] += deg > kGgWarpRow;
          J.stat[6] += clock64() - t_q1;
        }
        if (deg > kGgWarpRow) {  // hub row: the whole CTA updates it
          if (lane == 0) {
            s_v = v;
            s_b = bb;
          }
          cmd = 1;
          break;
        }
        if (deg > 0) {  // isolated claims (deg known) skip the offsets round trip
          gg_row_update(J, v, bb, nch, nsc, smax, cmax, lane, 32);
          __syncwarp();
        }
      }
      if (lane == 0) s_cmd = cmd;
    }
    __syncthreads();
    const int cmd = s_cmd;
    if (cmd == 2) break;
    const long long t_h0 = J.stat ? clock64() : 0;
    gg_row_update(J, s_v, s_b, nch, nsc, smax, cmax, threadIdx.x, blockDim.x);
    __syncthreads();
    if (J.stat && threadIdx.x == 0) J.stat[7] += clock64() - t_h0;
  }
}

// Farthest-first seeds of a large graph (pipelines.py:113-153) on the whole
// GPU: one cooperative launch runs the k multi-source BFS passes
// (level-synchronous frontier queues; first visit claimed by atomicCAS on
// dist, so distances are exact whatever the order; rows longer than 32 slots
// are expanded by a warp in a second pass) and after each the pick — lowest
// unreached vertex, else the first vertex of maximum distance — as grid-wide
// atomicMin / atomicMax on packed keys.
struct GgSeedArgs {
  int n, k;
  const int* off;
  const int* tgt;
  int* dist;
  int* qa;
  int* qb;
  int* heavy;
  int* ctr;                  // [0..1] queue counts, [2..3] heavy counts
  unsigned long long* keys;  // [0] lowest unreached, [1] (dist << 32 | ~v) max
  int* seeds;
};

__device__ __forceinline__ void gg_append(int* list, int* cnt, bool pred, int val) {
  const unsigned m = __ballot_sync(0xffffffffu, pred);
  if (!m) return;
  int base = 0;
  if (lane_id() == __ffs(m) - 1) base = atomicAdd(cnt, __popc(m));
  base = __shfl_sync(0xffffffffu, base, __ffs(m) - 1);
  if (pred) list[base + __popc(m & ((1u << lane_id()) - 1u))] = val;
}

__global__ void __launch_bounds__(256) k_ggg_seeds(GgSeedArgs A) {
  cg::grid_group grid = cg::this_grid();
  const long long gt = (long long)blockIdx.x * blockDim.x + threadIdx.x;
  const long long GT = (long long)gridDim.x * blockDim.x;
  const int lane = lane_id();
  const long long gw = gt >> 5, NW = GT >> 5;
  const int n = A.n;
  for (int ns = 0; ns < A.k; ++ns) {
    for (long long v = gt; v < n; v += GT) A.dist[v] = -1;
    if (gt == 0) {
      A.ctr[1] = A.ctr[2] = A.ctr[3] = 0;
      A.keys[0] = ~0ull;
      A.keys[1] = 0ull;
    }
    grid.sync();
    if (gt == 0) {
      const int ns0 = ns == 0 ? 1 : ns;
      for (int i = 0; i < ns0; ++i) {
        const int sv = ns == 0 ? 0 : A.seeds[i];
        A.dist[sv] = 0;
        A.qa[i] = sv;
      }
      A.ctr[0] = ns0;
    }
    grid.sync();
    for (int d = 0;; ++d) {
      const int cnt = __ldcg(A.ctr + (d & 1));
      if (cnt == 0) break;
      const int* cur = (d & 1) ? A.qb : A.qa;
      int* nxt = (d & 1) ? A.qa : A.qb;
      int* ncnt = A.ctr + ((d + 1) & 1);
      int* hcnt = A.ctr + 2 + (d & 1);
      for (long long b0 = gt - lane; b0 < cnt; b0 += GT) {  // warp-uniform loop
        const long long i = b0 + lane;
        int v = -1, e0 = 0, e1 = 0;
        if (i < cnt) {
          v = cur[i];
          e0 = A.off[v];
          e1 = A.off[v + 1];
        }
        const bool heavy = v >= 0 && e1 - e0 > 32;
        gg_append(A.heavy, hcnt, heavy, v);
        if (heavy) e1 = e0;
        for (int e = e0;; ++e) {  // thread per vertex, warp-converged appends
          const bool live = e < e1;
          if (!__any_sync(0xffffffffu, live)) break;
          bool fresh = false;
          int u = 0;
          if (live) {
            u = A.tgt[e];
            fresh = __ldcg(A.dist + u) < 0 && atomicCAS(A.dist + u, -1, d + 1) == -1;
          }
          gg_append(nxt, ncnt, fresh, u);
        }
      }
      grid.sync();
      // every thread has read this level's count: the count slot two levels
      // on can be reset (it is next written in level d + 1 ... d + 2)
      if (gt == 0) A.ctr[2 + ((d + 1) & 1)] = 0;
      const int hc = __ldcg(hcnt);
      for (long long h = gw; h < hc; h += NW) {
        const int v = A.heavy[h];
        const int e1 = A.off[v + 1];
        for (int eb = A.off[v]; eb < e1; eb += 32) {
          const int e = eb + lane;
          bool fresh = false;
          int u = 0;
          if (e < e1) {
            u = A.tgt[e];
            fresh = __ldcg(A.dist + u) < 0 && atomicCAS(A.dist + u, -1, d + 1) == -1;
          }
          gg_append(nxt, ncnt, fresh, u);
        }
      }
      if (gt == 0) A.ctr[d & 1] = 0;  // read by all before the barrier above
      grid.sync();
    }
    for (long long v = gt; v < n; v += GT) {
      const int dv = __ldcg(A.dist + v);
      if (dv < 0) atomicMin(A.keys, (unsigned long long)v);
      else atomicMax(A.keys + 1, ((unsigned long long)dv << 32) | (0xffffffffull - (unsigned)v));
    }
    grid.sync();
    if (gt == 0) {
      const unsigned long long ku = __ldcg(A.keys), kf = __ldcg(A.keys + 1);
      A.seeds[ns] = ku != ~0ull ? (int)ku : (int)(0xffffffffull - (kf & 0xffffffffull));
    }
    grid.sync();
  }
}

static void ggg_seeds(const DevGraph& g, int k, int* dist, int* seeds, cudaStream_t s) {
  static int occ = 0;
  static std::once_flag once;
  std::call_once(once, [] {
    GIM_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, k_ggg_seeds, 256, 0));
  });
  const int G = std::max(1, std::min(device_sms() * coop_blocks_per_sm(occ), (int)((g.n + 255) / 256)));
  const size_t n = (size_t)std::max(g.n, 1);
  DBuf<int> q(3 * n + 4, s);
  DBuf<unsigned long long> keys(2, s);
  GgSeedArgs A{g.n, k, g.off, g.tgt, dist, q.get(), q.get() + n, q.get() + 2 * n,
               q.get() + 3 * n, keys.get(), seeds};
  void* args[] = {&A};
  GIM_CUDA(cudaLaunchCooperativeKernel((const void*)k_ggg_seeds, dim3(G), dim3(256), args, 0, s));
  count_launch();
  GIM_LAUNCH_CHECK();
}

static void launch_ggg_large(const std::vector<DevGraph>& gs, int k,
                             const std::vector<int*>& parts, cudaStream_t s) {
  const int J = (int)gs.size();
  size_t total = 0, max_smax = 0, max_bnd = 0;
  std::vector<size_t> words((size_t)J);
  for (int j = 0; j < J; ++j) {
    const size_t n = (size_t)gs[(size_t)j].n;
    const size_t nch = (n + kGgCh - 1) / kGgCh, nsc = (nch + kGgSc - 1) / kGgSc;
    words[(size_t)j] = n + k + (size_t)k * n + (size_t)k * nch + (size_t)k * nsc;
    total += words[(size_t)j];
    max_smax = std::max(max_smax, (size_t)k * nsc);
    max_bnd = std::max(max_bnd, (size_t)k * (nch + nsc));
  }
  // both bound levels in shared memory when they fit, else the superchunk
  // level alone, else both in global memory
  constexpr size_t kMaxSmax = 200 * 1024;
  const bool cmax_smem = max_bnd * sizeof(int) <= kMaxSmax;
  const bool smax_smem = cmax_smem || max_smax * sizeof(int) <= kMaxSmax;
  const size_t dyn = cmax_smem ? max_bnd * sizeof(int) : smax_smem ? max_smax * sizeof(int) : 0;
  DBuf<int> scratch(std::max<size_t>(total, 1), s);
  GIM_CUDA(cudaMemsetAsync(scratch.get(), 0, sizeof(int) * total, s));
  DBuf<long long> bwork((size_t)k * J, s);
  std::vector<GggLargeJob> hj((size_t)J);
  size_t off = 0;
  for (int j = 0; j < J; ++j) {
    const DevGraph& g = gs[(size_t)j];
    const size_t n = (size_t)g.n;
    const size_t nch = (n + kGgCh - 1) / kGgCh;
    int* base = scratch.get() + off;
    GggLargeJob& q = hj[(size_t)j];
    q.n = g.n;
    q.k = k;
    q.off = g.off;
    q.tgt = g.tgt;
    q.w = g.w;
    q.vw = g.vw;
    q.part = parts[(size_t)j];
    q.dist = base;
    q.seeds = base + n;
    q.conn = q.seeds + k;
    q.cmax = q.conn + (size_t)k * n;
    q.gsmax = q.cmax + (size_t)k * nch;
    q.bwork = bwork.get() + (size_t)k * j;
    q.smax_smem = smax_smem ? 1 : 0;
    q.cmax_smem = cmax_smem ? 1 : 0;
    q.stat = nullptr;
    off += words[(size_t)j];
  }
  DBuf<long long> stat(8 * (size_t)J, s);
  if (trace_ggg()) {
    GIM_CUDA(cudaMemsetAsync(stat.get(), 0, sizeof(long long) * 8 * J, s));
    for (int j = 0; j < J; ++j) hj[(size_t)j].stat = stat.get() + 8 * j;
  }
  const auto t_seed = std::chrono::steady_clock::now();
  double ms_seed = 0.0;
  for (int j = 0; j < J; ++j)
    if (k > 1) ggg_seeds(gs[(size_t)j], k, hj[(size_t)j].dist, hj[(size_t)j].seeds, s);
  if (trace_ggg()) {
    GIM_CUDA(sync_stream(s));
    ms_seed = std::chrono::duration<double, std::milli>(std::chrono::steady_clock::now() - t_seed)
                  .count();
  }
  const auto t_grow = std::chrono::steady_clock::now();
  DBuf<GggLargeJob> dj((size_t)J, s);
  GIM_CUDA(cudaMemcpyAsync(dj.get(), hj.data(), sizeof(GggLargeJob) * (size_t)J,
                           cudaMemcpyHostToDevice, s));
  static std::once_flag once;
  std::call_once(once, [] {
    GIM_CUDA(cudaFuncSetAttribute(k_ggg_large, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                  (int)kMaxSmax));
  });
  k_ggg_large<<<J, kGggBlock, dyn, s>>>(dj.get());
  count_launch();
  GIM_LAUNCH_CHECK();
  if (trace_ggg()) {
    GIM_CUDA(sync_stream(s));
    const double ms_grow = std::chrono::duration<double, std::milli>(
                               std::chrono::steady_clock::now() - t_grow).count();
    std::vector<long long> h(8 * (size_t)J);
    GIM_CUDA(cudaMemcpy(h.data(), stat.get(), sizeof(long long) * 8 * J, cudaMemcpyDeviceToHost));
    for (int j = 0; j < J; ++j)
      std::fprintf(stderr, "ggg_large n=%d k=%d seeds %.1f ms grow %.1f ms | frontier %lld fallback %lld dry-skips %lld repairs %lld hub-updates %lld | Mcycles query %.1f claim %.1f hub %.1f\n",
                   gs[(size_t)j].n, k, ms_seed, ms_grow, h[8 * j], h[8 * j + 1], h[8 * j + 2], h[8 * j + 3],
                   h[8 * j + 4], h[8 * j + 5] / 1e6, h[8 * j + 6] / 1e6, h[8 * j + 7] / 1e6);
  }
}

// one CTA per graph; working set (and, when it fits, the graph) in shared
// memory, else a global scratch (large graphs: k_ggg_large)
static void launch_ggg(const std::vector<DevGraph>& gs, int k, const std::vector<int*>& parts,
                       cudaStream_t s) {
  const int J = (int)gs.size();
  if (J == 0) return;
  ProfScope prof(P_GGG, 0.0, s);
  constexpr size_t kMax = 160 * 1024;
  size_t max_words = 0, max_staged = 0;
  std::vector<size_t> words((size_t)J);
  for (int j = 0; j < J; ++j) {
    const DevGraph& g = gs[(size_t)j];
    words[(size_t)j] = (size_t)2 * g.n + k + (size_t)k * g.n + ((size_t)g.n + 31) / 32 +
                       (size_t)k * (((size_t)g.n + 31) / 32);
    max_words = std::max(max_words, words[(size_t)j]);
    max_staged = std::max(max_staged, words[(size_t)j] + (size_t)g.n + 1 + 2 * (size_t)g.m2 + g.n);
  }
  const bool use_smem = max_words * sizeof(int) <= kMax;
  const bool stage = max_staged * sizeof(int) <= kMax;
  const char* fl = getenv("GIM_GGG_LARGE");  // tests: force the large-graph kernel
  const bool force_large = fl && atoi(fl) != 0;
  if ((!use_smem || force_large) && k <= kGggMaxK) {
    launch_ggg_large(gs, k, parts, s);
    return;
  }
  long long scratch_words = 0;
  if (!use_smem)
    for (int j = 0; j < J; ++j) scratch_words += (long long)words[(size_t)j];
  DBuf<int> scratch((size_t)std::max(scratch_words, 1ll), s);
  DBuf<long long> bwork((size_t)k * J, s);
  // pageable staging: the call returns once the bytes are staged, so the
  // vector may die right after (pinned scratch could be overwritten early)
  std::vector<GggJob> hj((size_t)J);
  long long off = 0;
  for (int j = 0; j < J; ++j) {
    const DevGraph& g = gs[(size_t)j];
    hj[(size_t)j] = GggJob{g.n, k, g.off, g.tgt, g.w, g.vw, parts[(size_t)j],
                           use_smem ? nullptr : scratch.get() + off,
                           bwork.get() + (size_t)k * j, use_smem ? 1 : 0, (int)g.m2,
                           stage ? 1 : 0};
    if (!use_smem) off += (long long)words[(size_t)j];
  }
  DBuf<GggJob> dj((size_t)J, s);
  GIM_CUDA(cudaMemcpyAsync(dj.get(), hj.data(), sizeof(GggJob) * (size_t)J,
                           cudaMemcpyHostToDevice, s));
  const size_t smem = !use_smem ? 0 : (stage ? max_staged : max_words) * sizeof(int);
  static std::once_flag once;
  std::call_once(once, [] {
    GIM_CUDA(cudaFuncSetAttribute(k_ggg, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                  (int)(160 * 1024)));
  });
  k_ggg<<<J, kGggBlock, smem, s>>>(dj.get(), J);
  count_launch();
  GIM_LAUNCH_CHECK();
}

void greedy_graph_growing(const DevGraph& g, int k, int* part, cudaStream_t s) {
  launch_ggg(std::vector<DevGraph>{g}, k, std::vector<int*>{part}, s);
}

// all coarsest graphs of a batched partitioner step, one CTA per graph
void ggg_batch(const std::vector<DevGraph>& gs, int k, const std::vector<int*>& parts,
               cudaStream_t s) {
  launch_ggg(gs, k, parts, s);
}

// ---------------------------------------------------------------------------
// K14 extract_subgraphs (graph.py:357-389): vertices of part j keep their
// relative order (local ids), edges internal to a part keep CSR order.
// Stable radix sort of (part, v) gives the concatenated vertex order; each
// row's surviving slots are copied in order.

__global__ void k_local_ids(int n, const int* __restrict__ order, const int* __restrict__ part,
                            const int* __restrict__ pstart, int* __restrict__ local) {
  for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < n; i += gridDim.x * blockDim.x) {
    int v = order[i];
    local[v] = i - pstart[part[v]];
  }
}

__global__ void k_part_starts(int n, const unsigned* __restrict__ keys, int* __restrict__ pstart) {
  for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < n; i += gridDim.x * blockDim.x)
    if (i == 0 || keys[i] != keys[i - 1]) pstart[keys[i]] = i;
}

__global__ void k_iota_keys(int n, const int* __restrict__ part, unsigned* keys, int* vals) {
  for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < n; i += gridDim.x * blockDim.x) {
    keys[i] = (unsigned)part[i];
    vals[i] = i;
  }
}

struct KeptDeg {
  const int* order;
  const int* off;
  const int* tgt;
  const int* part;
  __device__ int operator()(long long i) const {
    int v = order[i];
    int pv = part[v], c = 0;
    for (int e = off[v]; e < off[v + 1]; ++e) c += part[tgt[e]] == pv;
    return c;
  }
};

__global__ void k_copy_rows(int n, const int* __restrict__ order, const int* __restrict__ off,
                            const int* __restrict__ tgt, const int* __restrict__ w,
                            const int* __restrict__ vw, const int* __restrict__ part,
                            const int* __restrict__ local, const int* __restrict__ pstart,
                            const int* __restrict__ noff, int* __restrict__ ntgt,
                            int* __restrict__ nw, int* __restrict__ nsrc, int* __restrict__ nvw) {
  for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < n; i += gridDim.x * blockDim.x) {
    int v = order[i];
    int pv = part[v];
    int pos = noff[i];
    int li = i - pstart[pv];
    for (int e = off[v]; e < off[v + 1]; ++e) {
      int u = tgt[e];
      if (part[u] != pv) continue;
      ntgt[pos] = local[u];
      nw[pos] = w[e];
      nsrc[pos] = li;
      ++pos;
    }
    nvw[i] = vw[v];
  }
}

__global__ void k_rebase(int cnt, const int* __restrict__ src, int base, int* __restrict__ dst) {
  for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < cnt; i += gridDim.x * blockDim.x)
    dst[i] = src[i] - base;
}

__global__ void k_gather(int n, const int* __restrict__ idx, const int* __restrict__ src,
                         int* __restrict__ dst) {
  for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < n; i += gridDim.x * blockDim.x)
    dst[i] = src[idx[i]];
}

__global__ void k_scatter_const(int n, const int* __restrict__ idx, int value, int* __restrict__ dst) {
  for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < n; i += gridDim.x * blockDim.x)
    dst[idx[i]] = value;
}

void gather(int n, const int* idx, const int* src, int* dst, cudaStream_t s) {
  if (n == 0) return;
  k_gather<<<grid_for(n, 256), 256, 0, s>>>(n, idx, src, dst);
  count_launch();
  GIM_LAUNCH_CHECK();
}

void scatter_const(int n, const int* idx, int value, int* dst, cudaStream_t s) {
  if (n == 0) return;
  k_scatter_const<<<grid_for(n, 256), 256, 0, s>>>(n, idx, value, dst);
  count_launch();
  GIM_LAUNCH_CHECK();
}

__global__ void k_leaf_scatter(int n, const int* __restrict__ idx, const int* __restrict__ part,
                               int base, int* __restrict__ dst) {
  for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < n; i += gridDim.x * blockDim.x)
    dst[idx[i]] = base + part[i];
}

// last multisection level: assignment[idx[i]] = base + part[i]
void leaf_scatter(int n, const int* idx, const int* part, int base, int* dst, cudaStream_t s) {
  if (n == 0) return;
  k_leaf_scatter<<<grid_for(n, 256), 256, 0, s>>>(n, idx, part, base, dst);
  count_launch();
  GIM_LAUNCH_CHECK();
}

// splits g by part[] into `parts` owned subgraphs + their global ids
void extract_subgraphs(const DevGraph& g, const int* part, int parts,
                       std::vector<OwnedGraph>& subs, std::vector<DBuf<int>>& ids,
                       cudaStream_t s) {
  const int n = g.n;
  ProfScope prof(P_EXTRACT, 12.0 * n + 12.0 * g.m2, s);
  subs.clear();
  ids.clear();
  subs.resize(parts);
  ids.resize(parts);
  DBuf<unsigned> keys((size_t)std::max(n, 1), s), keys2((size_t)std::max(n, 1), s);
  DBuf<int> order((size_t)std::max(n, 1), s), vals2((size_t)std::max(n, 1), s);
  DBuf<int> pstart((size_t)parts + 1, s), local((size_t)std::max(n, 1), s);
  DBuf<int> noff((size_t)n + 1, s);
  int grid = grid_for(n, 256);
  k_iota_keys<<<grid, 256, 0, s>>>(n, part, keys.get(), order.get());
  count_launch();
  radix_sort_pairs<unsigned, int>(n, keys.get(), order.get(), keys2.get(), vals2.get(),
                                  bit_length((unsigned long long)parts), s);
  // pstart[j] = first index of part j (parts without vertices: fixed below)
  GIM_CUDA(cudaMemsetAsync(pstart.get(), 0xff, sizeof(int) * ((size_t)parts + 1), s));
  k_part_starts<<<grid, 256, 0, s>>>(n, keys.get(), pstart.get());
  count_launch();
  std::vector<int> hs((size_t)parts + 1);
  GIM_CUDA(cudaMemcpyAsync(hs.data(), pstart.get(), sizeof(int) * ((size_t)parts + 1),
                           cudaMemcpyDeviceToHost, s));
  GIM_CUDA(sync_stream(s));
  hs[parts] = n;
  for (int j = parts - 1; j >= 0; --j)
    if (hs[j] < 0) hs[j] = hs[j + 1];
  GIM_CUDA(cudaMemcpyAsync(pstart.get(), hs.data(), sizeof(int) * ((size_t)parts + 1),
                           cudaMemcpyHostToDevice, s));
  k_local_ids<<<grid, 256, 0, s>>>(n, order.get(), part, pstart.get(), local.get());
  count_launch();
  DBuf<int> m2tot(1, s);
  exclusive_scan<int>(n, KeptDeg{order.get(), g.off, g.tgt, part}, StoreTo<int>{noff.get()},
                      m2tot.get(), s);
  int m2 = 0;
  GIM_CUDA(cudaMemcpyAsync(&m2, m2tot.get(), sizeof(int), cudaMemcpyDeviceToHost, s));
  GIM_CUDA(cudaMemcpyAsync(noff.get() + n, m2tot.get(), sizeof(int), cudaMemcpyDeviceToDevice, s));
  DBuf<int> ntgt((size_t)std::max(m2, 1), s), nw((size_t)std::max(m2, 1), s),
      nsrc((size_t)std::max(m2, 1), s), nvw((size_t)std::max(n, 1), s);
  k_copy_rows<<<grid, 256, 0, s>>>(n, order.get(), g.off, g.tgt, g.w, g.vw, part, local.get(),
                                   pstart.get(), noff.get(), ntgt.get(), nw.get(), nsrc.get(),
                                   nvw.get());
  count_launch();
  GIM_LAUNCH_CHECK();
  std::vector<int> hoff((size_t)n + 1);
  GIM_CUDA(cudaMemcpyAsync(hoff.data(), noff.get(), sizeof(int) * ((size_t)n + 1),
                           cudaMemcpyDeviceToHost, s));
  GIM_CUDA(sync_stream(s));
  for (int j = 0; j < parts; ++j) {
    int v0 = hs[j], v1 = hs[j + 1];
    int nj = v1 - v0;
    int e0 = hoff[v0], e1 = hoff[v1];
    OwnedGraph& sg = subs[j];
    sg.n = nj;
    int md = 0;  // exact longest row (offsets are on the host anyway)
    for (int v = v0; v < v1; ++v) md = std::max(md, hoff[(size_t)v + 1] - hoff[(size_t)v]);
    sg.maxdeg = md;
    sg.m2 = e1 - e0;
    sg.off = DBuf<int>((size_t)nj + 1, s);
    sg.tgt = DBuf<int>((size_t)std::max(e1 - e0, 1), s);
    sg.w = DBuf<int>((size_t)std::max(e1 - e0, 1), s);
    sg.src = DBuf<int>((size_t)std::max(e1 - e0, 1), s);
    sg.vw = DBuf<int>((size_t)std::max(nj, 1), s);
    ids[j] = DBuf<int>((size_t)std::max(nj, 1), s);
    k_rebase<<<grid_for(nj + 1, 256), 256, 0, s>>>(nj + 1, noff.get() + v0, e0, sg.off.get());
    count_launch();
    if (e1 > e0) {
      GIM_CUDA(cudaMemcpyAsync(sg.tgt.get(), ntgt.get() + e0, sizeof(int) * (e1 - e0), cudaMemcpyDeviceToDevice, s));
      GIM_CUDA(cudaMemcpyAsync(sg.w.get(), nw.get() + e0, sizeof(int) * (e1 - e0), cudaMemcpyDeviceToDevice, s));
      GIM_CUDA(cudaMemcpyAsync(sg.src.get(), nsrc.get() + e0, sizeof(int) * (e1 - e0), cudaMemcpyDeviceToDevice, s));
    }
    if (nj) {
      GIM_CUDA(cudaMemcpyAsync(sg.vw.get(), nvw.get() + v0, sizeof(int) * nj, cudaMemcpyDeviceToDevice, s));
      GIM_CUDA(cudaMemcpyAsync(ids[j].get(), order.get() + v0, sizeof(int) * nj, cudaMemcpyDeviceToDevice, s));
    }
  }
  GIM_LAUNCH_CHECK();
}

}  // namespace gim
