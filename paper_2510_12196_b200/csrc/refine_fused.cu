// Device-resident Alg. 4 (refinement.py:389-464): one cooperative persistent
// kernel runs the whole refinement loop of one level — label propagation
// (first filter, second filter), weak rebalancing, move application, exact
// J tracking and best-mapping bookkeeping — with grid-wide barriers between
// phases and no host round trip per iteration.
//
// Work lists.  Gains are evaluated thread-per-vertex (eval_thread): small
// levels sweep every vertex directly; large levels first compact the
// boundary vertices from ext[v] (#neighbours in another block, initialised
// per launch and kept exact by the move application), so no per-iteration
// boundary pass over the edges is needed.  The second filter, move
// application and commit run over the candidate / mover lists.  Lists are
// appended through warp-private shared-memory queues (one global atomic per
// >= 32 entries; order is irrelevant: every per-vertex result and every
// reduction is order-independent integer math).
// Invariants kept between iterations: gkey = LLONG_MIN and rtgt = -1 for
// every non-candidate; move flags are set only for the current movers and
// the lock set (= previous LP movers), both listed, so resets touch only
// listed vertices.
//
// The Alg. 4 control state (i, i_w, pass counter, best J / max weight, locks)
// is replicated in every CTA and updated identically from the same global
// counters after each barrier, so every CTA takes the same branch.  All float
// thresholds are the reference's double expressions.
//
// Weak rebalancing without a sort (refinement.py:333-346): per overloaded
// source block b the taken entries are a prefix of its (cell, vertex) order,
// cell = slot(gain)*rho + v%rho.  With W[b][c] the candidate weight per cell
// and c* the first cell whose cumulative weight exceeds excess_b, every cell
// before c* is taken whole, every cell after it not at all, and inside c* a
// vertex is taken iff P_{c*} + (weight of earlier c*-vertices of b) < excess_b.
// That in-cell prefix is a per-block running sum in vertex order: CTAs own
// contiguous vertex ranges, publish per-block partial sums (scanned across
// CTAs), and one warp per CTA walks its range with __match_any_sync ranking.
//
// Strong passes (rare: 7 of ~3,000 passes on rgg 2^20) exit the kernel
// ("yield"); the host runs the sort-based strong pass and relaunches.
#include <cooperative_groups.h>

#include <cstdio>
#include <cstdlib>
#include <map>
#include <mutex>

#include "common.cuh"
#include "kernels.cuh"
#include "refine_dev.cuh"

namespace cg = cooperative_groups;

namespace gim {

constexpr int kFusedBlock = 256;
constexpr int kFusedWarps = kFusedBlock / 32;
// co-resident CTAs per SM the grid kernels are compiled for (register cap).
// GIM build flag -DGIM_FUSED_MIN_BLOCKS overrides for A/B runs.
#ifndef GIM_FUSED_MIN_BLOCKS
#define GIM_FUSED_MIN_BLOCKS 3
#endif
constexpr int kFusedMinBlocks = GIM_FUSED_MIN_BLOCKS;
// batched cluster refinements occupy a few clusters at most: compiled for 2
// CTAs per SM, which removes the register spills (570 B per thread at 3)
constexpr int kClusterMinBlocks = 2;
constexpr int kMaxCluster = 16;
// vertex-centric first filter when a level has at most this many vertex
// groups per warp (else edge-parallel boundary pass + lists)
constexpr int kVcSteps = 2;
// longest row evaluated thread-per-vertex (longer rows: warp table path)
constexpr int kTpvMaxDeg = 64;  // non-portable cluster size (B200 allows 16)
constexpr int kCtrStride = 8;  // per-iteration-parity counters
enum { C_SMALL = 0, C_HEAVY, C_CAND, C_MOV, C_DJ, C_HUB, C_BIG, C_WIDE };

struct FusedArgs {
  int n;
  long long m2;
  const int* off;
  const int* tgt;
  const int* w;
  const int* vw;
  const int* src;
  Topo t;
  int k;
  int* part;
  long long* bw;
  int* best;
  long long* best_bw;
  int* dest;
  long long* gkey;
  unsigned char* flags0;
  unsigned char* flags1;
  int* rtgt;
  unsigned char* rcell;
  int* bstamp;         // ext: boundary counts per vertex (large levels)
  int* wdeg;           // weighted degree per vertex (with ext), else null
  int* lsmall;         // work lists
  int* lheavy;
  int* lcand;
  int* lmov0;
  int* lmov1;
  long long* W;        // [k * NC]
  long long* S;        // [k * G]
  long long* ctr;      // [2 * kCtrStride] per-parity counters, [16] = J at entry
  FusedState* st;
  int bar_mode;        // GridBarrier mode
  int smem_base;       // k_refine_smem: bytes of the regular dynamic region
  int vc_steps;        // vertex-centric first filters up to vc_steps vertices per thread
  int solo;            // 1: this CTA is a whole refinement (batched launch)
  int csize;           // >0: one cluster of csize CTAs per refinement (batched launch)
  long long* ptime;    // [16] per-phase ns (trace mode) or null
  int* hconn;          // [kHubBatch][k] conn tables of the hubs being evaluated (zeroed), or null
  int* lhub;           // medium rows (kTpvMaxDeg, hub_deg] listed by the current pass
  int* lbig;           // hub rows (> hub_deg) listed by the current pass
  int hub_deg;         // rows longer than this are hubs (cooperative grids with hconn only)
  int list_deg;        // rows longer than this are listed for the grid (<= hub_deg)
  int hub_phases;      // bit 0: first filter, bit 1: rebalance candidates
  long long* wctr;     // [1] wide LP candidates listed (in lhub) by the second filter
  long long* wacc;     // [cap] their future gains, accumulated by segments (zeroed)
  double l_max, sigma, phi, jet_c;
  int jet, rho, i_max, i_w_max;
  unsigned long long seed;
};

__device__ __forceinline__ unsigned long long globaltimer_ns() {
  unsigned long long t;
  asm volatile("mov.u64 %0, %globaltimer;" : "=l"(t));
  return t;
}

struct Ctl {
  long long J, best_j, best_maxw, maxw, pass_counter;
  long long iters, lp, weak;
  int i, i_w, best_balanced, locks_nonempty, lp_par, prev_n, it, stamp;
  int lock_stamp;  // move stamp of the locked set (previous LP movers), 0: none
  int brk, take, strong_yield;
};

// warp-aggregated counter add: every lane of the warp must execute it
__device__ __forceinline__ void acct_warp(long long* s_acct, int i, int x) {
  const int t = __reduce_add_sync(0xffffffffu, x);
  if (lane_id() == 0 && t) atomicAdd(reinterpret_cast<unsigned long long*>(&s_acct[i]),
                                     (unsigned long long)t);
}

__device__ __forceinline__ long long block_max_bw(const long long* bw, int k) {
  __shared__ long long red[kFusedWarps];
  long long m = 0;
  for (int b = threadIdx.x; b < k; b += blockDim.x) m = max(m, bw[b]);
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) m = max(m, __shfl_xor_sync(0xffffffffu, m, o));
  if (lane_id() == 0) red[threadIdx.x >> 5] = m;
  __syncthreads();
  long long r = 0;
  for (int i = 0; i < kFusedWarps; ++i) r = max(r, red[i]);
  __syncthreads();
  return r;
}

// warp-aggregated append; every lane of the warp must call it
__device__ __forceinline__ void warp_append(bool pred, int val, int* list, long long* counter) {
  const unsigned m = __ballot_sync(0xffffffffu, pred);
  if (!m) return;
  const int lane = lane_id();
  const int leader = __ffs(m) - 1;
  long long base = 0;
  if (lane == leader)
    base = (long long)atomicAdd(reinterpret_cast<unsigned long long*>(counter),
                                (unsigned long long)__popc(m));
  base = __shfl_sync(0xffffffffu, base, leader);
  if (pred) list[base + __popc(m & ((1u << lane) - 1u))] = val;
}

// Warp-private append queue in shared memory: appends cost a ballot and a
// shared store; the warp reserves list space with ONE global atomic per 32+
// entries (the list counters are single addresses every warp hits) and
// copies the entries out.  Warp-synchronous, so loops need not be
// CTA-uniform and no CTA barrier stalls the latency-bound sweeps.
struct WarpQueue {
  int* buf;   // [kQueueCap] in shared memory, private to the warp
  int cnt;    // warp-uniform
};
constexpr int kQueueCap = 64;

__device__ __forceinline__ void wq_flush(WarpQueue& q, int* list, long long* counter) {
  __syncwarp();
  if (q.cnt == 0) return;
  const unsigned lane = lane_id();
  long long base = 0;
  if (lane == 0)
    base = (long long)atomicAdd(reinterpret_cast<unsigned long long*>(counter),
                                (unsigned long long)q.cnt);
  base = __shfl_sync(0xffffffffu, base, 0);
  for (int i = lane; i < q.cnt; i += 32) list[base + i] = q.buf[i];
  __syncwarp();
  q.cnt = 0;
}

__device__ __forceinline__ void wq_push(WarpQueue& q, bool pred, int val, int* list,
                                        long long* counter) {
  const unsigned m = __ballot_sync(0xffffffffu, pred);
  if (pred) q.buf[q.cnt + __popc(m & ((1u << lane_id()) - 1u))] = val;
  q.cnt += __popc(m);
  if (q.cnt >= 32) wq_flush(q, list, counter);
}

// Barrier across the CTAs of one refinement: a one-CTA launch only needs
// __syncthreads; small graphs run as ONE thread-block cluster (plain launch,
// hardware cluster barrier with release/acquire semantics, so many
// refinements run concurrently); large graphs as a cooperative grid.
struct GridBarrier {
  int mode;            // 0 one CTA, 1 cluster, 2 cooperative grid
  long long* counter;  // shared-memory barrier count of this CTA (accounting)
  __device__ __forceinline__ void sync() const {
    if (threadIdx.x == 0) ++*counter;
    if (mode == 0) __syncthreads();
    else if (mode == 1) cg::this_cluster().sync();
    else cg::this_grid().sync();
  }
};

// Hub rows (R-MAT: 10^4-10^5 slots) would serialise a whole pass on the one
// warp that owns the vertex.  A pass lists its hubs instead; then every warp
// of the grid takes kHubSeg-slot segments of the listed hubs and adds each
// segment's conn(hub, b) into the hub's table (warp-aggregated by block),
// and after a barrier one warp per hub evaluates it from that table exactly
// like the in-warp table path.
constexpr int kHubSeg = 1024;
constexpr int kSweepWarpDeg = 128;  // entry-sweep rows longer than this: whole warp
// movers with rows longer than this (hub mode only) have their move applied
// by kHubSeg-slot segments spread over every warp of the grid, listed (in
// lsmall, free by then) by the phase that selects them
constexpr int kApplySplitDeg = 2048;
constexpr int kHubBatch = 256;  // hubs per accumulate/evaluate round
// rows longer than this are listed for the grid (shorter ones beyond
// kTpvMaxDeg stay with the owner warp: no extra barrier for a few of them);
// GIM_LIST_DEG overrides
constexpr int kListDeg = 256;

__device__ __forceinline__ void hub_accumulate(const FusedArgs& A, const int* list, long long c0,
                                               long long c1, long long gw, long long NW) {
  // (hub, segment) work items: per-CTA exclusive scan of the hubs' segment
  // counts, then grid-strided items located by binary search
  __shared__ int s_pre[kHubBatch + 1];
  __shared__ int s_wsum[kFusedWarps];
  const int lane = lane_id(), warp = threadIdx.x >> 5;
  const int nhc = (int)(c1 - c0);
  int segs = 0;
  if ((int)threadIdx.x < nhc) {
    const int v = list[c0 + threadIdx.x];
    segs = (A.off[v + 1] - A.off[v] + kHubSeg - 1) / kHubSeg;
  }
  int incl = segs;
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    const int y = __shfl_up_sync(0xffffffffu, incl, o);
    if (lane >= o) incl += y;
  }
  if (lane == 31) s_wsum[warp] = incl;
  __syncthreads();
  int base = 0;
  for (int w = 0; w < warp; ++w) base += s_wsum[w];
  if ((int)threadIdx.x <= nhc) s_pre[threadIdx.x] = base + incl - segs;  // [nhc] = total
  if (threadIdx.x == 0 && nhc == kHubBatch) {
    int tot = 0;
    for (int w = 0; w < kFusedWarps; ++w) tot += s_wsum[w];
    s_pre[kHubBatch] = tot;
  }
  __syncthreads();
  const int total = s_pre[nhc];
  for (long long j = gw; j < total; j += NW) {
    int lo = 0, hi = nhc - 1;
    while (lo < hi) {
      const int mid = (lo + hi + 1) >> 1;
      if (s_pre[mid] <= j) lo = mid;
      else hi = mid - 1;
    }
    const int v = list[c0 + lo];
    int* row = A.hconn + (size_t)lo * A.k;
    const int e1 = A.off[v + 1];
    const int sb = A.off[v] + (int)(j - s_pre[lo]) * kHubSeg, se = min(e1, sb + kHubSeg);
    for (int eb = sb; eb < se; eb += 32) {
      const int e = eb + lane;
      const int b = e < se ? A.part[A.tgt[e]] : -1;
      const int wv = e < se ? A.w[e] : 0;
      const unsigned peers = __match_any_sync(0xffffffffu, b);
      const int sum = (int)__reduce_add_sync(peers, (unsigned)wv);
      if (b >= 0 && lane == __ffs(peers) - 1) atomicAdd(row + b, sum);
    }
  }
  __syncthreads();  // s_pre / s_wsum reused by the next round
}

// warp table of a hub from its accumulated conn row (then zeroed for reuse)
__device__ __forceinline__ int hub_table(const WarpTable& wt, int k, int* row) {
  const int lane = lane_id();
  int sz = 0;
  for (int base = 0; base < k; base += 32) {
    const int i = base + lane;
    const int x = i < k ? __ldcg(row + i) : 0;
    if (i < k) {
      wt.tab[i] = x;
      row[i] = 0;
    }
    const unsigned m = __ballot_sync(0xffffffffu, x != 0);
    if (x != 0) {
      const int pos = sz + __popc(m & ((1u << lane) - 1u));
      wt.lb[pos] = i;
      wt.lw[pos] = x;
    }
    sz += __popc(m);
  }
  __syncwarp();
  return sz;
}

// one listed row, its conn table in wt: the first-filter decision (WEAK
// false, refinement.py:201-244) or the rebalance candidate (WEAK true,
// refinement.py:273-309), written exactly as the in-pass evaluation does
template <bool WEAK>
__device__ __forceinline__ void hub_eval_one(const FusedArgs& A, int u, int sz, const WarpTable& wt,
                                             int k, const Topo& T, const long long* s_dbit,
                                             long long* cnt, const unsigned char* elig,
                                             const int* elist, int n_elig,
                                             long long pass_counter, int NC) {
  const int lane = lane_id();
  const int ou = A.part[u];
  if (!WEAK) {
    const VertexEval q = eval_table(wt, sz, ou, T, s_dbit, nullptr);
    bool ok = false;
    if (q.best_b >= 0) {
      if (q.best_gain >= 0) ok = true;
      else if (A.jet) ok = jet_admits(q.best_gain, q.conn_own, A.jet_c, A.t.dshift);
    }
    if (ok && lane == 0) {
      A.dest[u] = q.best_b;
      A.gkey[u] = q.best_gain;
    }
    warp_append(ok && lane == 0, u, A.lcand, cnt + C_CAND);
  } else {
    int tb = -1;
    if (n_elig > 0) {
      const unsigned long long h = hash2(A.seed, (unsigned long long)u,
                                         (unsigned long long)pass_counter);
      tb = elist[h % (unsigned long long)n_elig];
    }
    const VertexEval q = eval_table(wt, sz, ou, T, s_dbit, elig);
    long long ctb = 0;
    if (q.best_b < 0 && tb >= 0) ctb = cost_table(wt, sz, tb, T, s_dbit);
    int target = -1;
    long long gain = 0;
    if (q.best_b >= 0) {
      target = q.best_b;
      gain = q.best_gain;
    } else if (tb >= 0) {
      target = tb;
      gain = q.cur - ctb;
    }
    if (target >= 0 && lane == 0) {
      A.rtgt[u] = target;
      const int cell = slot_for_gain(gain, A.t.dshift) * A.rho + u % A.rho;
      A.rcell[u] = (unsigned char)cell;
      atomicAdd(reinterpret_cast<unsigned long long*>(&A.W[(size_t)ou * NC + cell]),
                (unsigned long long)(long long)A.vw[u]);
    }
    warp_append(target >= 0 && lane == 0, u, A.lcand, cnt + C_CAND);
  }
}

// the rows a pass listed instead of evaluating: medium rows one warp each
// (any warp of the grid, not the owner warp), hub rows by segments
template <bool WEAK>
__device__ __forceinline__ void hub_phase(const FusedArgs& A, const GridBarrier& grid,
                                          long long* cnt, long long gw, long long NW,
                                          const WarpTable& wt, int k, const Topo& T,
                                          const long long* s_dbit, const unsigned char* elig,
                                          const int* elist, int n_elig, long long pass_counter,
                                          int NC) {
  const long long nm = cnt[C_HUB], nb = cnt[C_BIG];
  if (nm == 0 && nb == 0) return;
  for (long long i = gw; i < nm; i += NW) {
    const int u = A.lhub[i];
    const int sz = warp_build_table(wt, k, A.off[u], A.off[u + 1], A.tgt, A.w, A.part);
    hub_eval_one<WEAK>(A, u, sz, wt, k, T, s_dbit, cnt, elig, elist, n_elig, pass_counter, NC);
  }
  for (long long c0 = 0; c0 < nb; c0 += kHubBatch) {
    const long long c1 = min(nb, c0 + (long long)kHubBatch);
    hub_accumulate(A, A.lbig, c0, c1, gw, NW);
    grid.sync();
    for (long long i = c0 + gw; i < c1; i += NW) {
      const int u = A.lbig[i];
      const int sz = hub_table(wt, k, A.hconn + (size_t)(i - c0) * k);
      hub_eval_one<WEAK>(A, u, sz, wt, k, T, s_dbit, cnt, elig, elist, n_elig, pass_counter, NC);
    }
    grid.sync();
  }
  if (nb == 0) grid.sync();
}

// second filter of the listed wide LP candidates (A.lhub[0, nw)): their
// future gains (refinement.py:246-262) summed by kHubSeg-slot segments over
// every warp of the grid into A.wacc
__device__ __forceinline__ void sf_wide_accumulate(const FusedArgs& A, const Topo& T,
                                                   const long long* s_dbit, long long nw,
                                                   long long gw, long long NW) {
  __shared__ int s_pre[kHubBatch + 1];
  __shared__ int s_wsum[kFusedWarps];
  const int lane = lane_id(), warp = threadIdx.x >> 5;
  for (long long c0 = 0; c0 < nw; c0 += kHubBatch) {
    const int nhc = (int)min((long long)kHubBatch, nw - c0);
    int segs = 0;
    if ((int)threadIdx.x < nhc) {
      const int v = A.lhub[c0 + threadIdx.x];
      segs = (A.off[v + 1] - A.off[v] + kHubSeg - 1) / kHubSeg;
    }
    int incl = segs;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      const int y = __shfl_up_sync(0xffffffffu, incl, o);
      if (lane >= o) incl += y;
    }
    if (lane == 31) s_wsum[warp] = incl;
    __syncthreads();
    int base = 0, tot = 0;
    for (int w = 0; w < kFusedWarps; ++w) {
      if (w < warp) base += s_wsum[w];
      tot += s_wsum[w];
    }
    if ((int)threadIdx.x < nhc) s_pre[threadIdx.x] = base + incl - segs;
    if (threadIdx.x == 0) s_pre[nhc] = tot;
    __syncthreads();
    for (long long j = gw; j < tot; j += NW) {
      int lo = 0, hi = nhc - 1;
      while (lo < hi) {
        const int mid = (lo + hi + 1) >> 1;
        if (s_pre[mid] <= j) lo = mid;
        else hi = mid - 1;
      }
      const int v = A.lhub[c0 + lo];
      const int e1 = A.off[v + 1];
      const int sb = A.off[v] + (int)(j - s_pre[lo]) * kHubSeg, se = min(e1, sb + kHubSeg);
      const long long gv = A.gkey[v];
      const unsigned long long oc = T.code[A.part[v]];
      const unsigned long long dc = T.code[A.dest[v]];
      long long fut = 0;
      for (int e = sb + lane; e < se; e += 32) {
        const int u = A.tgt[e];
        const long long gu = A.gkey[u];
        const bool earlier = gu > gv || (gu == gv && u < v);
        const unsigned long long pc = T.code[earlier ? A.dest[u] : A.part[u]];
        fut += (long long)A.w[e] * (cdist(s_dbit, oc, pc) - cdist(s_dbit, dc, pc));
      }
      fut = warp_sum_ll(fut);
      if (lane == 0 && fut)
        atomicAdd(reinterpret_cast<unsigned long long*>(A.wacc + c0 + lo),
                  (unsigned long long)fut);
    }
    __syncthreads();  // s_pre / s_wsum reused by the next batch
  }
}

// the move application of the listed wide movers (A.lsmall[0, nw)), by
// kHubSeg-slot segments over every warp of the grid (same per-slot work as
// the mover loop in refine_body; returns this thread's share of dJ)
__device__ __forceinline__ long long apply_wide(const FusedArgs& A, const Topo& T,
                                             const long long* s_dbit, int* ext,
                                             const int* opart, const unsigned short* mstamp,
                                             unsigned short cur_stamp, long long nw,
                                             long long gw, long long NW) {
  __shared__ int s_pre[kHubBatch + 1];
  __shared__ int s_wsum[kFusedWarps];
  const int lane = lane_id(), warp = threadIdx.x >> 5;
  long long acc = 0;
  for (long long c0 = 0; c0 < nw; c0 += kHubBatch) {
    const int nhc = (int)min((long long)kHubBatch, nw - c0);
    int segs = 0;
    if ((int)threadIdx.x < nhc) {
      const int v = A.lsmall[c0 + threadIdx.x];
      segs = (A.off[v + 1] - A.off[v] + kHubSeg - 1) / kHubSeg;
    }
    int incl = segs;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      const int y = __shfl_up_sync(0xffffffffu, incl, o);
      if (lane >= o) incl += y;
    }
    if (lane == 31) s_wsum[warp] = incl;
    __syncthreads();
    int base = 0, tot = 0;
    for (int w = 0; w < kFusedWarps; ++w) {
      if (w < warp) base += s_wsum[w];
      tot += s_wsum[w];
    }
    if ((int)threadIdx.x < nhc) s_pre[threadIdx.x] = base + incl - segs;
    if (threadIdx.x == 0) s_pre[nhc] = tot;
    __syncthreads();
    for (long long j = gw; j < tot; j += NW) {
      int lo = 0, hi = nhc - 1;
      while (lo < hi) {
        const int mid = (lo + hi + 1) >> 1;
        if (s_pre[mid] <= j) lo = mid;
        else hi = mid - 1;
      }
      const int v = A.lsmall[c0 + lo];
      const int e1 = A.off[v + 1];
      const int sb = A.off[v] + (int)(j - s_pre[lo]) * kHubSeg, se = min(e1, sb + kHubSeg);
      const int ov = opart[v], nv = A.dest[v];
      const unsigned long long oc = T.code[ov], nc2 = T.code[nv];
      int dext = 0;
      for (int e = sb + lane; e < se; e += 32) {
        const int u = A.tgt[e];
        const bool um = mstamp[u] == cur_stamp;
        const int ou = um ? opart[u] : A.part[u];
        const int nu = um ? A.dest[u] : ou;
        const long long dd = cdist(s_dbit, nc2, T.code[nu]) - cdist(s_dbit, oc, T.code[ou]);
        acc += (long long)A.w[e] * dd * (um ? 1 : 2);
        if (ext) {
          const int dx = (int)(nv != nu) - (int)(ov != ou);
          dext += dx;
          if (!um && dx) atomicAdd(&ext[u], dx);
        }
      }
      dext = warp_sum_i(dext);
      if (ext && lane == 0 && dext) atomicAdd(&ext[v], dext);
    }
    __syncthreads();  // s_pre / s_wsum reused by the next batch
  }
  return acc;
}

// HUB: the skewed-degree machinery (warp entry sweeps of long rows, listed
// hub rows, grouped wide-table scoring, grid-segmented second filter and
// move application) is compiled in; the HUB = false instance (graphs without
// rows over kSweepWarpDeg slots: rgg, grids) carries none of that code
template <int VW, bool HUB>
__device__ __forceinline__ void refine_body(const FusedArgs& A) {
  // SURVEY §8(d) accounting (Acct, common.cuh): warp-aggregated (REDUX) into
  // this CTA's shared counters, added to the FusedState once at exit
  __shared__ long long s_acct[A_COUNT];
  if (threadIdx.x < A_COUNT) s_acct[threadIdx.x] = 0;
  const GridBarrier grid{A.bar_mode, &s_acct[A_BARRIERS]};
  extern __shared__ unsigned char dsm[];
  __shared__ long long s_dbit[64];
  __shared__ Ctl C;
  __shared__ int s_nelig, s_novl;
  __shared__ long long scan_tot[kFusedWarps];
  __shared__ int qbuf[kFusedWarps * 2 * kQueueCap];
  const int k = A.k;
  const int NC = 31 * A.rho;
  const int n = A.n;
  // a batched shared-memory launch runs one independent refinement per CTA
  // (or one thread-block cluster per refinement: csize CTAs each)
  const int G = A.solo ? 1 : A.csize ? A.csize : (int)gridDim.x;
  const int BX = A.solo ? 0 : A.csize ? (int)(blockIdx.x % A.csize) : (int)blockIdx.x;
  // dynamic smem: pstar[k] | run[k] | code[k] | warp tables | elist[k] | cstar[k] |
  // wrun[warps*k] | ovl[k] | elig[k]
  long long* pstar = reinterpret_cast<long long*>(dsm);
  long long* run = pstar + k;
  unsigned long long* s_code = reinterpret_cast<unsigned long long*>(run + k);
  int* tables = reinterpret_cast<int*>(s_code + k);
  int* elist = tables + (size_t)kFusedWarps * 3 * k;
  int* cstar = elist + k;
  int* olist = cstar + k;
  int* wrun = olist + k;
  unsigned char* ovl = reinterpret_cast<unsigned char*>(wrun + (size_t)kFusedWarps * k);
  unsigned char* elig = ovl + k;

  load_dbit(s_dbit, A.t);
  for (int b = threadIdx.x; b < k; b += blockDim.x) s_code[b] = A.t.code[b];
  Topo T = A.t;  // digit codes from shared memory
  T.code = s_code;
  __syncthreads();
  const long long flatd = A.t.L == 1 ? s_dbit[0] : 0;  // single-level topology
  const int lane = lane_id();
  const int warp = threadIdx.x >> 5;
  const long long gw = ((long long)BX * blockDim.x + threadIdx.x) >> 5;
  const long long NW = ((long long)G * blockDim.x) >> 5;
  const long long gt = (long long)BX * blockDim.x + threadIdx.x;
  const long long GT = (long long)G * blockDim.x;
  constexpr int GPW = 32 / VW;
  const int gi = lane / VW, li = lane % VW;
  WarpTable wt;
  wt.tab = tables + (size_t)warp * 3 * k;
  wt.lb = wt.tab + k;
  wt.lw = wt.lb + k;
  const int R = (n + G - 1) / G;  // contiguous vertex range of this CTA
  const int r0 = min(n, BX * R), r1 = min(n, r0 + R);

  // thread-per-vertex first filters straight over the vertex range when the
  // level is small; otherwise the filters run over compact lists built from
  // ext[v] = #neighbours in another block (bstamp), which the move
  // application keeps exact (more memory-level parallelism for big levels)
  const bool vcent = A.src == nullptr || (long long)n <= (long long)A.vc_steps * GT;
  int* const ext = vcent ? nullptr : A.bstamp;

  // ---- entry
  const bool first = !A.st->started;
  const bool reinit = first || A.st->reinit;
  if (reinit) {  // (re)establish the list invariants
    for (long long v = gt; v < n; v += GT) {
      A.gkey[v] = kGainNone;
      A.rtgt[v] = -1;
      reinterpret_cast<unsigned short*>(A.flags0)[v] = 0;  // move stamp
    }
    for (long long i = gt; i < (long long)k * NC; i += GT) A.W[i] = 0;
  }
  if (ext || first) {
    // one row sweep: boundary counts of the entry mapping + weighted degrees
    // (large levels) and, on the first launch, J of the entry mapping
    // (mapping.py:76-91), four slots' loads in flight per step
    // Rows longer than kSweepWarpDeg slots (R-MAT hubs: up to 10^5) are
    // swept by their whole warp instead of one thread, so no thread walks a
    // hub row alone while the grid waits at the next barrier.
    long long acc = 0;
    for (long long vb = gt & ~31ll; vb < n; vb += GT) {  // warp-uniform
      const long long v = vb + lane;
      const bool live = v < n;
      const int e0 = live ? A.off[v] : 0, e1 = live ? A.off[v + 1] : 0;
      const bool wide = HUB && e1 - e0 > kSweepWarpDeg;
      if (live && !wide) {
        const int pv = A.part[v];
        const unsigned long long pc = T.code[pv];
        int c = 0, wd = 0;
        for (int e = e0; e < e1; e += 4) {
          int tg[4], wg[4], pb[4];
#pragma unroll
          for (int q = 0; q < 4; ++q) {
            tg[q] = e + q < e1 ? A.tgt[e + q] : -1;
            wg[q] = e + q < e1 ? A.w[e + q] : 0;
          }
#pragma unroll
          for (int q = 0; q < 4; ++q) pb[q] = tg[q] >= 0 ? A.part[tg[q]] : pv;
#pragma unroll
          for (int q = 0; q < 4; ++q) {
            c += pb[q] != pv;
            wd += wg[q];
            if (first && pb[q] != pv) acc += (long long)wg[q] * cdist(s_dbit, pc, T.code[pb[q]]);
          }
        }
        if (ext) {
          ext[v] = c;
          A.wdeg[v] = wd;
        }
      }
      unsigned wm = __ballot_sync(0xffffffffu, live && wide);
      while (wm) {
        const int l = __ffs(wm) - 1;
        wm &= wm - 1;
        const int u = (int)(vb + l);
        const int f0 = __shfl_sync(0xffffffffu, e0, l), f1 = __shfl_sync(0xffffffffu, e1, l);
        const int pu = A.part[u];
        const unsigned long long pc = T.code[pu];
        int c = 0, wd = 0;
        long long a2 = 0;
        for (int e = f0 + lane; e < f1; e += 4 * 32) {
          int tg[4], wg[4], pb[4];
#pragma unroll
          for (int q = 0; q < 4; ++q) {
            const int eq = e + 32 * q;
            tg[q] = eq < f1 ? A.tgt[eq] : -1;
            wg[q] = eq < f1 ? A.w[eq] : 0;
          }
#pragma unroll
          for (int q = 0; q < 4; ++q) pb[q] = tg[q] >= 0 ? A.part[tg[q]] : pu;
#pragma unroll
          for (int q = 0; q < 4; ++q) {
            c += pb[q] != pu;
            wd += wg[q];
            if (first && pb[q] != pu) a2 += (long long)wg[q] * cdist(s_dbit, pc, T.code[pb[q]]);
          }
        }
        c = warp_sum_i(c);
        wd = warp_sum_i(wd);
        acc += a2;  // summed over the CTA below
        if (ext && lane == 0) {
          ext[u] = c;
          A.wdeg[u] = wd;
        }
      }
    }
    if (first) block_sum_atomic<kFusedBlock>(acc, A.ctr + 16);
    if (BX == 0 && threadIdx.x == 0) s_acct[A_SWEEPS] += 1;
  }
  if (first) {
    for (long long v = gt; v < n; v += GT) A.best[v] = A.part[v];
    if (BX == 0)
      for (int b = threadIdx.x; b < k; b += blockDim.x) A.best_bw[b] = A.bw[b];
  }
  grid.sync();
  if (first) {
    long long mx = block_max_bw(A.bw, k);
    if (threadIdx.x == 0) {
      C.J = A.ctr[16];
      C.maxw = mx;
      C.best_balanced = (double)mx <= A.l_max;
      C.best_j = C.J;
      C.best_maxw = mx;
      C.i = C.i_w = 0;
      C.pass_counter = 0;
      C.locks_nonempty = 0;
      C.lp_par = 0;
      C.prev_n = 0;
      C.stamp = 0;
    }
  } else if (threadIdx.x == 0) {
    const FusedState& S0 = *A.st;
    C.J = S0.J;
    C.best_j = S0.best_j;
    C.best_maxw = S0.best_maxw;
    C.maxw = S0.maxw;
    C.pass_counter = S0.pass_counter;
    C.i = S0.i;
    C.i_w = S0.i_w;
    C.best_balanced = S0.best_balanced;
    C.locks_nonempty = S0.locks_nonempty;
    C.lp_par = S0.lp_par;
    C.prev_n = S0.prev_n;
    C.stamp = S0.stamp;
  }
  if (threadIdx.x == 0) {
    C.it = 0;
    C.lock_stamp = 0;  // every launch starts without locks (after a rebalance pass)
    C.iters = C.lp = C.weak = 0;
    C.brk = 0;
    C.strong_yield = 0;
  }
  __syncthreads();
  // optional per-phase wall-clock accounting (GIM_TRACE_REFINE): CTA 0,
  // thread 0 adds %globaltimer deltas between barriers into A.ptime[phase]
  unsigned long long t_last = 0;
  if (A.ptime && BX == 0 && threadIdx.x == 0) t_last = globaltimer_ns();
#define PHASE_MARK(id)                                                   \
  do {                                                                   \
    if (A.ptime && BX == 0 && threadIdx.x == 0) {                \
      const unsigned long long t_now = globaltimer_ns();                 \
      A.ptime[(id)] += (long long)(t_now - t_last);                      \
      t_last = t_now;                                                    \
    }                                                                    \
  } while (0)

  // Move stamps (uint16 over the two flag bytes of a vertex): a vertex moves
  // in iteration `it` iff mstamp == stamp_of(it); the locked set is the
  // previous LP pass's movers (stamp C.lock_stamp), so nothing is ever
  // cleared.  The old part of a mover lives in opart, so the move
  // application can commit in place while others read it.
  unsigned short* const mstamp = reinterpret_cast<unsigned short*>(A.flags0);
  int* const opart = A.lmov1;
  while (C.i < A.i_max) {
    const bool balanced_now = (double)C.maxw <= A.l_max;
    if (C.it > 0 && C.it % 65534 == 0) {  // stamp wrap: keep only the locks
      const unsigned short ls = (unsigned short)C.lock_stamp;
      for (long long v = gt; v < n; v += GT)
        mstamp[v] = (ls && mstamp[v] == ls) ? 1 : 0;
      grid.sync();
      if (threadIdx.x == 0 && ls) C.lock_stamp = 1;
      __syncthreads();
    }
    const unsigned short cur_stamp = (unsigned short)(2 + C.it % 65534);
    const unsigned short lock_stamp = (unsigned short)C.lock_stamp;
    const bool entry_locks_empty = lock_stamp == 0;
    if (!balanced_now && !(C.i_w < A.i_w_max)) {  // strong pass: hand back to the host
      if (threadIdx.x == 0) C.strong_yield = 1;
      __syncthreads();
      break;
    }
    const int q = C.it & 1;
    long long* cnt = A.ctr + q * kCtrStride;          // this iteration (zeroed beforehand)
    long long* cnt_next = A.ctr + (q ^ 1) * kCtrStride;
    int* lmov = A.lmov0;
    const bool use_locks = lock_stamp != 0;
    const int stamp = C.stamp + 1;
    bool incomplete = false;
    // thread-per-vertex first filters straight over the vertex range when
    // the level is small; otherwise an edge-parallel boundary pass + a
    // compact list first (more memory-level parallelism for large levels)
    WarpQueue qa{qbuf + warp * 2 * kQueueCap, 0}, qb{qbuf + (warp * 2 + 1) * kQueueCap, 0};
    if (balanced_now) {
      // ---- K9 first filter (refinement.py:201-244)
      long long ns = n;  // items: vertices (vcent) or the boundary list
      if (!vcent) {
        // boundary list (unlocked): ext[v] > 0; four vertices per thread
        // per step with their loads issued together
        int nbnd = 0;
        for (long long b0 = (gt - lane) * 4; b0 < n; b0 += GT * 4) {
          bool bnd[4];
#pragma unroll
          for (int q = 0; q < 4; ++q) {
            const long long v = b0 + q * 32 + lane;
            bnd[q] = v < n && ext[v] > 0;
            nbnd += bnd[q];
          }
#pragma unroll
          for (int q = 0; q < 4; ++q) {
            const long long v = b0 + q * 32 + lane;
            if (bnd[q] && use_locks && mstamp[v] == lock_stamp) bnd[q] = false;
            wq_push(qa, bnd[q], (int)v, A.lsmall, cnt + C_SMALL);
          }
        }
        acct_warp(s_acct, A_BND, nbnd);
        if (BX == 0 && threadIdx.x == 0) s_acct[A_SCAN] += n;
        wq_flush(qa, A.lsmall, cnt + C_SMALL);
        grid.sync();
        PHASE_MARK(1);
        ns = cnt[C_SMALL];
      }
      for (long long b0 = gt - lane; b0 < ns; b0 += GT) {
        const long long idx = b0 + lane;
        bool live = idx < ns;
        int v = 0, own = 0, e0 = 0, e1 = 0;
        if (live) {
          v = vcent ? (int)idx : A.lsmall[idx];
          if (vcent && use_locks && mstamp[v] == lock_stamp) live = false;
        }
        ThreadEval r{};
        r.best_b = -1;
        bool ovf = false;
        bool hub = false, big = false;
        if (live) {
          own = A.part[v];
          e0 = A.off[v];
          e1 = A.off[v + 1];
          if ((HUB && A.hconn) && (A.hub_phases & 1) && e1 - e0 > A.list_deg) {
            // evaluated by the grid after this pass
            if (e1 - e0 > A.hub_deg) big = true;
            else hub = true;
          } else if (e1 - e0 > kTpvMaxDeg) {
            ovf = true;
          } else {
            r = eval_thread(e0, e1, own, A.tgt, A.w, A.part, T, s_dbit, nullptr, -1, flatd);
            ovf = r.overflow;
          }
        }
        wq_push(qb, hub, v, A.lhub, cnt + C_HUB);
        warp_append(big, v, A.lbig, cnt + C_BIG);
        // rows too long / too many distinct blocks: the warp evaluates them
        // one by one with the shared-memory block table
        unsigned om = __ballot_sync(0xffffffffu, live && ovf);
        while (om) {
          const int l = __ffs(om) - 1;
          om &= om - 1;
          const int u = __shfl_sync(0xffffffffu, v, l);
          const int ou = __shfl_sync(0xffffffffu, own, l);
          const int sz = warp_build_table(wt, k, A.off[u], A.off[u + 1], A.tgt, A.w, A.part);
          const VertexEval q = eval_table<HUB>(wt, sz, ou, T, s_dbit, nullptr);
          if (lane == l) {
            r.best_b = q.best_b;
            r.best_gain = q.best_gain;
            r.conn_own = q.conn_own;
            r.nblk = sz;
          }
        }
        acct_warp(s_acct, A_EVAL_V, live);
        acct_warp(s_acct, A_EVAL_SLOTS, live ? e1 - e0 : 0);
        acct_warp(s_acct, A_EVAL_S, live ? r.nblk : 0);
        bool ok = false;
        if (live && r.best_b >= 0) {
          if (r.best_gain >= 0) ok = true;
          else if (A.jet) ok = jet_admits(r.best_gain, r.conn_own, A.jet_c, A.t.dshift);
        }
        if (ok) {
          A.dest[v] = r.best_b;
          A.gkey[v] = r.best_gain;
        }
        wq_push(qa, ok, v, A.lcand, cnt + C_CAND);
      }
      wq_flush(qa, A.lcand, cnt + C_CAND);
      wq_flush(qb, A.lhub, cnt + C_HUB);
      grid.sync();
      if ((HUB && A.hconn) && (A.hub_phases & 1))  // rows listed by this first filter
        hub_phase<false>(A, grid, cnt, gw, NW, wt, k, T, s_dbit, nullptr, nullptr, 0, 0, NC);
      PHASE_MARK(2);
      // every CTA has read the previous iteration's counters by now (they
      // were consumed before this iteration's first barrier)
      if (BX == 0 && threadIdx.x < kCtrStride) cnt_next[threadIdx.x] = 0;
      // ---- K10 second filter over the candidates
      const long long nc = cnt[C_CAND];
      for (long long ib = gw * GPW; ib < nc; ib += NW * GPW) {
        const long long idx = ib + gi;
        const bool live = idx < nc;
        const int v = live ? A.lcand[idx] : 0;
        long long fut = 0;
        int csl = 0;
        // rows over kApplySplitDeg slots: decided after the grid-wide
        // segment pass below (hub mode only)
        const bool wide = live && (HUB && A.hconn) && A.off[v + 1] - A.off[v] > kApplySplitDeg;
        if (live) {
          const long long gv = A.gkey[v];
          const unsigned long long oc = T.code[A.part[v]];
          const unsigned long long dc = T.code[A.dest[v]];
          if (li == 0) csl = A.off[v + 1] - A.off[v];
          for (int e = A.off[v] + li; e < (wide ? 0 : A.off[v + 1]); e += VW) {
            int u = A.tgt[e];
            long long gu = A.gkey[u];
            bool earlier = gu > gv || (gu == gv && u < v);
            int pos = earlier ? A.dest[u] : A.part[u];
            unsigned long long pc = T.code[pos];
            fut += (long long)A.w[e] * (cdist(s_dbit, oc, pc) - cdist(s_dbit, dc, pc));
          }
        }
#pragma unroll
        for (int o = VW / 2; o > 0; o >>= 1) fut += __shfl_xor_sync(0xffffffffu, fut, o);
        const bool m = live && !wide && li == 0 && fut >= 0;
        acct_warp(s_acct, A_CAND_SLOTS, csl);
        if (m) {
          mstamp[v] = cur_stamp;
          opart[v] = A.part[v];
        }
        wq_push(qa, m, v, lmov, cnt + C_MOV);
        if ((HUB && A.hconn)) warp_append(wide && li == 0, v, A.lhub, A.wctr);
      }
      wq_flush(qa, lmov, cnt + C_MOV);
      grid.sync();
      if ((HUB && A.hconn)) {
        const long long nwc = __ldcg(A.wctr);
        if (nwc > 0) {  // wide candidates: future gains by segments, then decide
          sf_wide_accumulate(A, T, s_dbit, nwc, gw, NW);
          grid.sync();
          for (long long b0 = gt - lane; b0 < nwc; b0 += GT) {
            const long long i = b0 + lane;
            const int v = i < nwc ? A.lhub[i] : 0;
            bool m = false;
            if (i < nwc) {
              m = (long long)__ldcg(reinterpret_cast<unsigned long long*>(A.wacc + i)) >= 0;
              A.wacc[i] = 0;
              if (m) {
                mstamp[v] = cur_stamp;
                opart[v] = A.part[v];
              }
            }
            warp_append(m, v, lmov, cnt + C_MOV);
            warp_append(m, v, A.lsmall, cnt + C_WIDE);  // applied by segments too
          }
          grid.sync();
        }
      }
      PHASE_MARK(3);
    } else {
      // ---- K11 weak rebalance candidates (refinement.py:273-309)
      for (int b = threadIdx.x; b < k; b += blockDim.x) {
        ovl[b] = (double)A.bw[b] > A.l_max;
        elig[b] = (double)A.bw[b] < A.sigma;
      }
      __syncthreads();
      if (warp == 0) {  // ascending eligible / overloaded lists (ballot compaction)
        int ne = 0, no = 0;
        for (int b0 = 0; b0 < k; b0 += 32) {
          const int b = b0 + lane;
          const bool e = b < k && elig[b], o = b < k && ovl[b];
          const unsigned me = __ballot_sync(0xffffffffu, e), mo = __ballot_sync(0xffffffffu, o);
          const unsigned lt = (1u << lane) - 1u;
          if (e) elist[ne + __popc(me & lt)] = b;
          if (o) olist[no + __popc(mo & lt)] = b;
          ne += __popc(me);
          no += __popc(mo);
        }
        if (lane == 0) {
          s_nelig = ne;
          s_novl = no;
        }
      }
      __syncthreads();
      const int n_elig = s_nelig;
      incomplete = n_elig == 0;
      long long ns = n;
      if (!vcent) {  // vertices of overloaded blocks
        for (long long b0 = (gt - lane) * 4; b0 < n; b0 += GT * 4) {
          int pv[4];
#pragma unroll
          for (int q = 0; q < 4; ++q) {
            const long long v = b0 + q * 32 + lane;
            pv[q] = v < n ? A.part[v] : -1;
          }
#pragma unroll
          for (int q = 0; q < 4; ++q) {
            const long long v = b0 + q * 32 + lane;
            wq_push(qa, pv[q] >= 0 && ovl[pv[q]], (int)v, A.lsmall, cnt + C_SMALL);
          }
        }
        wq_flush(qa, A.lsmall, cnt + C_SMALL);
        grid.sync();
        PHASE_MARK(4);
        ns = cnt[C_SMALL];
      }
      for (long long b0 = gt - lane; b0 < ns; b0 += GT) {
        const long long idx = b0 + lane;
        bool live = idx < ns;
        int v = 0, own = 0;
        if (live) {
          v = vcent ? (int)idx : A.lsmall[idx];
          own = A.part[v];
          live = ovl[own] != 0;
        }
        int tb = -1;  // random eligible target if no adjacent block qualifies
        if (live && n_elig > 0) {
          unsigned long long h = hash2(A.seed, (unsigned long long)v,
                                       (unsigned long long)C.pass_counter);
          tb = elist[h % (unsigned long long)n_elig];
        }
        ThreadEval r{};
        r.best_b = -1;
        bool ovf = false, hub = false, big = false;
        int osl = 0;
        if (live && ext && ext[v] == 0) {
          // interior vertex (every neighbour in its own block): no adjacent
          // candidate, cur = 0, cost(tb) = wdeg * D(tb, own) — no row walk
          r.nblk = 1;
          if (tb >= 0)
            r.cost_tb = (long long)A.wdeg[v] * cdist(s_dbit, T.code[tb], T.code[own]);
        } else if (live) {
          const int e0 = A.off[v], e1 = A.off[v + 1];
          osl = e1 - e0;
          if ((HUB && A.hconn) && (A.hub_phases & 2) && e1 - e0 > A.list_deg) {
            // evaluated by the grid after this pass
            if (e1 - e0 > A.hub_deg) big = true;
            else hub = true;
          } else if (e1 - e0 > kTpvMaxDeg) {
            ovf = true;
          } else {
            r = eval_thread(e0, e1, own, A.tgt, A.w, A.part, T, s_dbit, elig, tb, flatd);
            ovf = r.overflow;
          }
        }
        wq_push(qb, hub, v, A.lhub, cnt + C_HUB);
        warp_append(big, v, A.lbig, cnt + C_BIG);
        unsigned om = __ballot_sync(0xffffffffu, live && ovf);
        while (om) {
          const int l = __ffs(om) - 1;
          om &= om - 1;
          const int u = __shfl_sync(0xffffffffu, v, l);
          const int ou = __shfl_sync(0xffffffffu, own, l);
          const int tbl = __shfl_sync(0xffffffffu, tb, l);
          const int sz = warp_build_table(wt, k, A.off[u], A.off[u + 1], A.tgt, A.w, A.part);
          const VertexEval q = eval_table<HUB>(wt, sz, ou, T, s_dbit, elig);
          long long ctb = 0;
          if (q.best_b < 0 && tbl >= 0) ctb = cost_table(wt, sz, tbl, T, s_dbit);  // warp-uniform
          if (lane == l) {
            r.best_b = q.best_b;
            r.best_gain = q.best_gain;
            r.cur = q.cur;
            r.cost_tb = ctb;
            r.nblk = sz;
          }
        }
        acct_warp(s_acct, A_OVL_V, live);
        acct_warp(s_acct, A_OVL_SLOTS, osl);
        acct_warp(s_acct, A_OVL_S, live ? r.nblk : 0);
        int target = -1;
        long long gain = 0;
        if (live && !hub && !big) {  // listed rows: decided by the grid below
          if (r.best_b >= 0) {
            target = r.best_b;
            gain = r.best_gain;
          } else if (tb >= 0) {
            target = tb;
            gain = r.cur - r.cost_tb;
          }
        }
        const bool isc = target >= 0;
        int wkey = -1;
        unsigned vwv = 0;
        if (isc) {
          A.rtgt[v] = target;
          const int cell = slot_for_gain(gain, A.t.dshift) * A.rho + v % A.rho;
          A.rcell[v] = (unsigned char)cell;
          wkey = own * NC + cell;
          vwv = (unsigned)A.vw[v];
        }
        // warp-aggregated W update: list neighbours mostly share (block,
        // cell), so one 64-bit atomic per distinct key instead of per vertex
        // (the 16-bit split keeps the 32-bit reductions exact)
        const unsigned peers = __match_any_sync(0xffffffffu, wkey);
        const unsigned wlo = __reduce_add_sync(peers, vwv & 0xffffu);
        const unsigned whi = __reduce_add_sync(peers, vwv >> 16);
        if (isc && lane == __ffs(peers) - 1)
          atomicAdd(reinterpret_cast<unsigned long long*>(&A.W[wkey]),
                    (unsigned long long)wlo + ((unsigned long long)whi << 16));
        wq_push(qa, isc, v, A.lcand, cnt + C_CAND);
      }
      wq_flush(qa, A.lcand, cnt + C_CAND);
      wq_flush(qb, A.lhub, cnt + C_HUB);
      // the lock set is cleared on every rebalance pass (refinement.py:425):
      // lock_stamp becomes 0 at the end of this iteration
      grid.sync();
      if ((HUB && A.hconn) && (A.hub_phases & 2))  // rows listed by this candidate pass
        hub_phase<true>(A, grid, cnt, gw, NW, wt, k, T, s_dbit, elig, elist, s_nelig,
                        C.pass_counter, NC);
      PHASE_MARK(5);
      if (BX == 0 && threadIdx.x < kCtrStride) cnt_next[threadIdx.x] = 0;
      // ---- K12 weak selection, step A: c*, P_{c*} per overloaded block (every
      // CTA redundantly; one warp per overloaded block, all cell chunks
      // loaded before the shuffle prefix) and per-(warp, block) weights of
      // c*-cell vertices over the warp's slice of this CTA's vertex range.
      // Only overloaded blocks have a c* cell (cstar = NC elsewhere).
      const int n_ovl = s_novl;
      for (int b = threadIdx.x; b < k; b += blockDim.x) {
        cstar[b] = NC;
        pstar[b] = 0;
      }
      __syncthreads();
      for (int i = warp; i < n_ovl; i += kFusedWarps) {
        const int b = olist[i];
        const double excess = (double)A.bw[b] - A.l_max;
        constexpr int kMaxChunks = 8;  // NC = 31 * rho <= 248
        long long x[kMaxChunks];
#pragma unroll
        for (int h = 0; h < kMaxChunks; ++h) {
          const int cc = h * 32 + lane;
          x[h] = cc < NC ? A.W[(size_t)b * NC + cc] : 0;
        }
        long long P = 0;
        int c = NC;
#pragma unroll
        for (int h = 0; h < kMaxChunks; ++h) {
          if (h * 32 >= NC || c < NC) break;  // warp-uniform
          long long incl = x[h];
#pragma unroll
          for (int o = 1; o < 32; o <<= 1) {
            const long long y = __shfl_up_sync(0xffffffffu, incl, o);
            if (lane >= o) incl += y;
          }
          const int cc = h * 32 + lane;
          const unsigned over = __ballot_sync(0xffffffffu, cc < NC && (double)(P + incl) > excess);
          if (over) {
            const int l = __ffs(over) - 1;
            c = h * 32 + l;
            P += __shfl_sync(0xffffffffu, incl - x[h], l);
          } else {
            P += __shfl_sync(0xffffffffu, incl, 31);
          }
        }
        if (lane == 0) { cstar[b] = c; pstar[b] = P; }
      }
      for (int i = threadIdx.x; i < kFusedWarps * k; i += blockDim.x) wrun[i] = 0;
      __syncthreads();
      const int RW = (r1 - r0 + kFusedWarps - 1) / kFusedWarps;  // warp slice
      const int w0 = min(r1, r0 + warp * RW), w1 = min(r1, w0 + RW);
      // the c*-cell ("partial") candidates of the warp's slice, in vertex
      // order, are compacted into lheavy[w0 ..) for the walk in step C
      int n_part = 0;
      if (n_ovl > 0) {
        const unsigned lt = (1u << lane) - 1u;
        for (int v0 = w0; v0 < w1; v0 += 128) {  // warp-uniform, four chunks in flight
          int tq[4];
#pragma unroll
          for (int q = 0; q < 4; ++q) {
            const int vq = v0 + q * 32 + lane;
            tq[q] = vq < w1 ? A.rtgt[vq] : -1;
          }
          int bq[4];
          bool pq[4];
#pragma unroll
          for (int q = 0; q < 4; ++q) {
            const int vq = v0 + q * 32 + lane;
            bq[q] = tq[q] >= 0 ? A.part[vq] : 0;
            pq[q] = tq[q] >= 0 && (int)A.rcell[vq] == cstar[bq[q]];
          }
#pragma unroll
          for (int q = 0; q < 4; ++q) {
            const int vq = v0 + q * 32 + lane;
            if (pq[q]) atomicAdd(&wrun[warp * k + bq[q]], A.vw[vq]);
            const unsigned mq = __ballot_sync(0xffffffffu, pq[q]);
            if (pq[q]) A.lheavy[w0 + n_part + __popc(mq & lt)] = vq;
            n_part += __popc(mq);
          }
        }
      }
      __syncthreads();
      for (int i = threadIdx.x; i < n_ovl; i += blockDim.x) {  // CTA total; warp prefix
        const int b = olist[i];
        int acc = 0;
        for (int w = 0; w < kFusedWarps; ++w) {
          const int x = wrun[w * k + b];
          wrun[w * k + b] = acc;
          acc += x;
        }
        A.S[(size_t)b * G + BX] = acc;
      }
      grid.sync();
      PHASE_MARK(6);
      // step B: exclusive scan of S over CTAs for every overloaded block,
      // one CTA per row (<= 3 entries per thread + a block-wide scan)
      for (int i = BX; i < n_ovl; i += G) {
        long long* row = A.S + (size_t)olist[i] * G;
        const int E = (G + kFusedBlock - 1) / kFusedBlock;  // <= 3
        const int c0 = threadIdx.x * E;
        long long v3[3] = {0, 0, 0};
        long long tsum = 0;
#pragma unroll
        for (int j = 0; j < 3; ++j)
          if (j < E && c0 + j < G) {
            v3[j] = row[c0 + j];
            tsum += v3[j];
          }
        long long incl = tsum;
#pragma unroll
        for (int o = 1; o < 32; o <<= 1) {
          const long long y = __shfl_up_sync(0xffffffffu, incl, o);
          if (lane >= o) incl += y;
        }
        if (lane == 31) scan_tot[warp] = incl;
        __syncthreads();
        long long base = 0;
        for (int w = 0; w < warp; ++w) base += scan_tot[w];
        long long run_ex = base + incl - tsum;
#pragma unroll
        for (int j = 0; j < 3; ++j)
          if (j < E && c0 + j < G) {
            row[c0 + j] = run_ex;
            run_ex += v3[j];
          }
        __syncthreads();
      }
      grid.sync();
      PHASE_MARK(7);
      // step C: in-cell prefix in vertex order — every warp walks its slice
      // with __match_any_sync ranking, starting from (earlier CTAs) +
      // (earlier warps of this CTA); whole cells before c* everywhere else
      for (int i = threadIdx.x; i < n_ovl; i += blockDim.x) {
        const int b = olist[i];
        run[b] = A.S[(size_t)b * G + BX];
      }
      __syncthreads();
      for (int i0 = 0; i0 < n_part; i0 += 32) {  // warp-uniform, listed partials only
        const bool live = i0 + lane < n_part;
        const int v = live ? A.lheavy[w0 + i0 + lane] : 0;
        bool partial = false;
        int b = 0;
        int wv = 0;
        if (live) {
          b = A.part[v];
          partial = true;
          wv = A.vw[v];
        }
        const unsigned act = __ballot_sync(0xffffffffu, partial);
        bool take = false;
        if (partial) {
          const unsigned peers = __match_any_sync(act, b);
          const int leader = __ffs(peers) - 1;
          long long before = 0, total = 0;
          unsigned mm = peers;
          while (mm) {
            const int l = __ffs(mm) - 1;
            mm &= mm - 1;
            const long long x = __shfl_sync(peers, (long long)wv, l);
            if (l < (int)lane) before += x;
            total += x;
          }
          const double excess = (double)A.bw[b] - A.l_max;
          take = (double)(pstar[b] + run[b] + wrun[warp * k + b] + before) < excess;
          __syncwarp(peers);
          if ((int)lane == leader) wrun[warp * k + b] += (int)total;
        }
        if (take) {
          mstamp[v] = cur_stamp;
          opart[v] = A.part[v];
          A.dest[v] = A.rtgt[v];
        }
        wq_push(qa, take, v, lmov, cnt + C_MOV);
        if ((HUB && A.hconn))
          warp_append(take && A.off[v + 1] - A.off[v] > kApplySplitDeg, v, A.lsmall,
                      cnt + C_WIDE);
      }
      const long long nc = cnt[C_CAND];
      for (long long b0 = gt - lane; b0 < nc; b0 += GT) {
        const long long idx = b0 + lane;
        bool take = false;
        int v = 0;
        if (idx < nc) {
          v = A.lcand[idx];
          take = (int)A.rcell[v] < cstar[A.part[v]];
          if (take) {
            mstamp[v] = cur_stamp;
            opart[v] = A.part[v];
            A.dest[v] = A.rtgt[v];
          }
        }
        wq_push(qa, take, v, lmov, cnt + C_MOV);
        if ((HUB && A.hconn))
          warp_append(take && A.off[v + 1] - A.off[v] > kApplySplitDeg, v, A.lsmall,
                      cnt + C_WIDE);
      }
      wq_flush(qa, lmov, cnt + C_MOV);
      grid.sync();
      PHASE_MARK(8);
    }
    // ---- K13 apply + commit over the movers: exact dJ, block weights, ext
    // counts, part[v] = dest[v] in place (a mover's neighbours read its old
    // block from opart), then restore the list invariants
    {
      const long long nm = cnt[C_MOV], nc = cnt[C_CAND];
      long long acc = 0;
      if ((HUB && A.hconn) && BX == 0 && threadIdx.x == 0) *A.wctr = 0;  // read before the last barrier
      for (long long ib = gw * GPW; ib < nm; ib += NW * GPW) {
        const long long idx = ib + gi;
        int msl = 0;
        if (idx < nm) {
          const int v = lmov[idx];
          if (li == 0) msl = A.off[v + 1] - A.off[v];
          const int ov = opart[v], nv = A.dest[v];
          const unsigned long long oc = T.code[ov], nc2 = T.code[nv];
          int dext = 0;
          const int ea = A.off[v], eb = A.off[v + 1];
          const bool split = (HUB && A.hconn) && eb - ea > kApplySplitDeg;  // segments below
          for (int e = ea + li; e < (split ? ea : eb); e += VW) {
            const int u = A.tgt[e];
            const bool um = mstamp[u] == cur_stamp;
            const int ou = um ? opart[u] : A.part[u];
            const int nu = um ? A.dest[u] : ou;
            const long long dd = cdist(s_dbit, nc2, T.code[nu]) -
                                 cdist(s_dbit, oc, T.code[ou]);
            acc += (long long)A.w[e] * dd * (um ? 1 : 2);
            if (ext) {  // boundary counts: edge (v,u) before / after the moves
              const int dx = (int)(nv != nu) - (int)(ov != ou);
              dext += dx;
              if (!um && dx) atomicAdd(&ext[u], dx);  // movers update their own
            }
          }
          if (ext && dext) atomicAdd(&ext[v], dext);
          if (li == 0) {
            A.part[v] = nv;
            if (ov != nv) {
              atomicAdd(reinterpret_cast<unsigned long long*>(&A.bw[ov]),
                        (unsigned long long)(-(long long)A.vw[v]));
              atomicAdd(reinterpret_cast<unsigned long long*>(&A.bw[nv]),
                        (unsigned long long)(long long)A.vw[v]);
            }
          }
        }
        acct_warp(s_acct, A_MOV_SLOTS, msl);
      }
      if ((HUB && A.hconn) && cnt[C_WIDE] > 0)
        acc += apply_wide(A, T, s_dbit, ext, opart, mstamp, cur_stamp, cnt[C_WIDE], gw, NW);
      block_sum_atomic<kFusedBlock>(acc, cnt + C_DJ);
      if (balanced_now) {
        for (long long i = gt; i < nc; i += GT) A.gkey[A.lcand[i]] = kGainNone;
      } else {
        for (long long i = gt; i < nc; i += GT) A.rtgt[A.lcand[i]] = -1;
        for (long long i = gt; i < (long long)k * NC; i += GT) A.W[i] = 0;
      }
    }
    grid.sync();
    PHASE_MARK(9);
    // ---- Alg. 4 control (refinement.py:433-463), replicated per CTA
    const long long mx = block_max_bw(A.bw, k);
    if (threadIdx.x == 0) {
      const long long mv = cnt[C_MOV];
      if (BX == 0) {
        s_acct[A_MOV_V] += mv;
        if (balanced_now) {
          s_acct[A_CAND_V] += cnt[C_CAND];
          s_acct[A_LP_IT] += 1;
        } else {
          s_acct[A_WEAK_IT] += 1;
        }
      }
      C.take = 0;
      C.iters++;
      C.stamp = stamp;
      if (balanced_now) {
        C.lp++;
        C.i_w = 0;
      } else {
        C.weak++;
        C.i_w++;
        C.pass_counter++;
      }
      // this pass's movers become the next locks (LP) or there are none
      C.lock_stamp = (balanced_now && mv > 0) ? cur_stamp : 0;
      C.locks_nonempty = C.lock_stamp != 0;
      C.prev_n = 0;
      if (mv == 0 && ((balanced_now && entry_locks_empty) || (!balanced_now && incomplete))) {
        C.brk = 1;
      } else {
        C.J += cnt[C_DJ];
        C.maxw = mx;
        int reset = 0;
        if ((double)C.maxw <= A.l_max) {
          if (!C.best_balanced) {
            C.best_balanced = 1;
            C.best_j = C.J;
            C.best_maxw = C.maxw;
            reset = C.take = 1;
          } else if (C.J < C.best_j) {
            reset = (double)C.J < A.phi * (double)C.best_j;
            C.best_j = C.J;
            C.best_maxw = C.maxw;
            C.take = 1;
          }
        } else if (!C.best_balanced && C.maxw < C.best_maxw) {
          C.best_maxw = C.maxw;
          reset = C.take = 1;
        }
        C.i = reset ? 0 : C.i + 1;
      }
      C.it++;
    }
    __syncthreads();
    PHASE_MARK(11);
    if (C.brk) break;
    if (C.take) {
      for (long long v = gt; v < n; v += GT) A.best[v] = A.part[v];
      if (BX == 0)
        for (int b = threadIdx.x; b < k; b += blockDim.x) A.best_bw[b] = A.bw[b];
    }
  }
  // ---- exit: persist the control state; on completion restore the best
  grid.sync();
  if (threadIdx.x < A_COUNT && (threadIdx.x != A_BARRIERS || BX == 0) && s_acct[threadIdx.x])
    atomicAdd(reinterpret_cast<unsigned long long*>(&A.st->acct[threadIdx.x]),
              (unsigned long long)s_acct[threadIdx.x]);
  if (BX == 0 && threadIdx.x == 0) {
    FusedState& S1 = *A.st;
    S1.started = 1;
    S1.reinit = 0;
    S1.J = C.J;
    S1.best_j = C.best_j;
    S1.best_maxw = C.best_maxw;
    S1.maxw = C.maxw;
    S1.pass_counter = C.pass_counter;
    S1.i = C.i;
    S1.i_w = C.i_w;
    S1.best_balanced = C.best_balanced;
    S1.locks_nonempty = C.locks_nonempty;
    S1.lp_par = C.lp_par;
    S1.prev_n = C.prev_n;
    S1.stamp = C.stamp;
    S1.status = C.strong_yield ? 1 : 0;
    S1.iters += C.iters;
    S1.lp += C.lp;
    S1.weak += C.weak;
  }
  if (!C.strong_yield) {
    for (long long v = gt; v < n; v += GT) A.part[v] = A.best[v];
    if (BX == 0)
      for (int b = threadIdx.x; b < k; b += blockDim.x) A.bw[b] = A.best_bw[b];
  }
}

template <int VW, bool HUB>
__global__ void __launch_bounds__(kFusedBlock, kFusedMinBlocks) k_refine_fused(FusedArgs A) {
  refine_body<VW, HUB>(A);
}

// one thread-block cluster per independent refinement (batched launch)
template <int VW>
__global__ void __launch_bounds__(kFusedBlock, kClusterMinBlocks) k_refine_cluster_batch(const FusedArgs* args,
                                                                      int csize) {
  refine_body<VW, false>(args[blockIdx.x / csize]);
}

// Shared-memory-resident refinement of a small graph: ONE CTA copies the
// CSR, the mapping and every per-vertex work array into shared memory and
// runs the same Alg. 4 loop on them (generic pointers), so every gather in
// the latency-bound phases is a shared-memory access instead of an L2 round
// trip.  Layout after the regular dynamic region (A.smem_base bytes):
//   int64: gkey[n] bw[k] best_bw[k] W[k*NC] S[k] ctr[17]
//   int32: off[n+1] tgt[m2] w[m2] vw[n] part[n] best[n] dest[n] rtgt[n]
//          lheavy[n] lcand[n] lmov0[n] lmov1[n]
//   uint8: flags0[n] flags1[n] rcell[n]
template <int VW>
__device__ __forceinline__ void refine_smem_run(const FusedArgs& A) {
  extern __shared__ __align__(16) unsigned char dsm[];
  __shared__ FusedArgs SA;
  const int n = A.n, k = A.k, NC = 31 * A.rho;
  const long long m2 = A.m2;
  long long* q = reinterpret_cast<long long*>(dsm + A.smem_base);
  long long* gkey = q;
  long long* bw = gkey + n;
  long long* best_bw = bw + k;
  long long* W = best_bw + k;
  long long* S = W + (size_t)k * NC;
  long long* ctr = S + k;
  int* ip = reinterpret_cast<int*>(ctr + 17);
  int* off = ip;
  int* tgt = off + n + 1;
  int* w = tgt + m2;
  int* vw = w + m2;
  int* part = vw + n;
  int* best = part + n;
  int* dest = best + n;
  int* rtgt = dest + n;
  int* lheavy = rtgt + n;
  int* lcand = lheavy + n;
  int* lmov0 = lcand + n;
  int* lmov1 = lmov0 + n;
  unsigned char* f0 = reinterpret_cast<unsigned char*>(lmov1 + n);
  unsigned char* f1 = f0 + n;
  unsigned char* rcell = f1 + n;
  const bool first = !A.st->started;
  for (int i = threadIdx.x; i <= n; i += blockDim.x) off[i] = A.off[i];
  for (long long e = threadIdx.x; e < m2; e += blockDim.x) {
    tgt[e] = A.tgt[e];
    w[e] = A.w[e];
  }
  for (int v = threadIdx.x; v < n; v += blockDim.x) {
    vw[v] = A.vw[v];
    part[v] = A.part[v];
    if (!first) best[v] = A.best[v];
  }
  for (int b = threadIdx.x; b < k; b += blockDim.x) {
    bw[b] = A.bw[b];
    if (!first) best_bw[b] = A.best_bw[b];
  }
  for (int i = threadIdx.x; i < 17; i += blockDim.x) ctr[i] = 0;
  if (threadIdx.x == 0) {
    SA = A;
    SA.off = off; SA.tgt = tgt; SA.w = w; SA.vw = vw; SA.src = nullptr;
    SA.part = part; SA.bw = bw; SA.best = best; SA.best_bw = best_bw;
    SA.dest = dest; SA.gkey = gkey; SA.flags0 = f0; SA.flags1 = f1;
    SA.rtgt = rtgt; SA.rcell = rcell; SA.bstamp = nullptr; SA.lsmall = nullptr;
    SA.lheavy = lheavy; SA.lcand = lcand; SA.lmov0 = lmov0; SA.lmov1 = lmov1;
    SA.W = W; SA.S = S; SA.ctr = ctr;
    SA.bar_mode = 0;
  }
  __syncthreads();
  refine_body<VW, false>(SA);
  __syncthreads();
  const bool yielded = A.st->status != 0;  // strong pass due: the host needs everything
  for (int v = threadIdx.x; v < n; v += blockDim.x) {
    A.part[v] = part[v];
    if (yielded) A.best[v] = best[v];
  }
  for (int b = threadIdx.x; b < k; b += blockDim.x) {
    A.bw[b] = bw[b];
    if (yielded) A.best_bw[b] = best_bw[b];
  }
}

template <int VW>
__global__ void __launch_bounds__(kFusedBlock) k_refine_smem(FusedArgs A) {
  refine_smem_run<VW>(A);
}

// one CTA per independent refinement (the batched multisection leaves)
template <int VW>
__global__ void __launch_bounds__(kFusedBlock) k_refine_smem_batch(const FusedArgs* args) {
  refine_smem_run<VW>(args[blockIdx.x]);
}

// shared-memory bytes of k_refine_smem beyond the regular dynamic region
static size_t smem_resident_bytes(long long n, long long m2, int k, int NC) {
  return 8 * ((size_t)n + 2 * (size_t)k + (size_t)k * NC + (size_t)k + 17) +
         4 * ((size_t)n + 1 + 2 * (size_t)m2 + 11 * (size_t)n) + 3 * (size_t)n;
}

// ---------------------------------------------------------------------------
// host side

// GIM_TRACE_REFINE for batched launches: per-phase times of job 0 and the
// batch's device time, printed after the batch finished
struct BatchTrace {
  bool on = false;
  DBuf<long long> pt;
  cudaEvent_t e[2]{};
  void begin(long long** job0_ptime, cudaStream_t s) {
    static const bool env = std::getenv("GIM_TRACE_REFINE") != nullptr;
    on = env;
    if (!on) return;
    pt = DBuf<long long>(16, s);
    GIM_CUDA(cudaMemsetAsync(pt.get(), 0, 16 * sizeof(long long), s));
    *job0_ptime = pt.get();
    GIM_CUDA(cudaEventCreate(&e[0]));
    GIM_CUDA(cudaEventCreate(&e[1]));
    GIM_CUDA(cudaEventRecord(e[0], s));
  }
  void end(const char* kind, int jobs, int n0, long long m20, long long it0, cudaStream_t s) {
    if (!on) return;
    GIM_CUDA(cudaEventRecord(e[1], s));
    GIM_CUDA(cudaEventSynchronize(e[1]));
    float ms = 0;
    cudaEventElapsedTime(&ms, e[0], e[1]);
    long long h[16];
    GIM_CUDA(cudaMemcpy(h, pt.get(), sizeof(h), cudaMemcpyDeviceToHost));
    std::fprintf(stderr, "%s jobs=%d job0 n=%d m2=%lld iters=%lld batch_ms=%.3f us/iter(job0)=%.1f |",
                 kind, jobs, n0, m20, it0, ms, it0 ? 1000.0 * ms / (double)it0 : 0.0);
    static const char* nm[12] = {"stamp", "blist", "ff", "sf", "wlist", "wcand", "wA", "wB",
                                 "wsel", "apply", "commit", "ctl"};
    for (int i = 0; i < 12; ++i) std::fprintf(stderr, " %s=%.1f", nm[i], h[i] / 1000.0);
    std::fprintf(stderr, "\n");
    cudaEventDestroy(e[0]);
    cudaEventDestroy(e[1]);
  }
};

// Raise a kernel's dynamic shared-memory limit to the device's opt-in
// maximum (minus its static shared memory) once per (device, kernel).  The
// limit is never lowered afterwards: launches of the same kernel with
// different k (different dynamic sizes) from other calls / threads must all
// stay valid.
static void raise_dyn_smem_limit(const void* fn) {
  static std::mutex mu;
  static std::map<std::pair<int, const void*>, bool> done;
  int dev = 0;
  GIM_CUDA(cudaGetDevice(&dev));
  std::lock_guard<std::mutex> lk(mu);
  if (done.count({dev, fn})) return;
  int optin = 0;
  GIM_CUDA(cudaDeviceGetAttribute(&optin, cudaDevAttrMaxSharedMemoryPerBlockOptin, dev));
  cudaFuncAttributes fa;
  GIM_CUDA(cudaFuncGetAttributes(&fa, fn));
  const int lim = optin > (int)fa.sharedSizeBytes ? optin - (int)fa.sharedSizeBytes : 0;
  GIM_CUDA(cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize, lim));
  GIM_CUDA(cudaFuncSetAttribute(fn, cudaFuncAttributeNonPortableClusterSizeAllowed, 1));
  done[{dev, fn}] = true;
}

// co-resident CTAs per SM for (VW, smem), queried once per device
template <int VW>
static int coop_max_blocks(size_t smem) {
  static std::mutex mu;
  static std::map<std::pair<int, size_t>, int> cache;
  int dev = 0;
  GIM_CUDA(cudaGetDevice(&dev));
  std::lock_guard<std::mutex> lk(mu);
  auto key = std::make_pair(dev, smem);
  auto it = cache.find(key);
  if (it != cache.end()) return it->second;
  int sms = 0, per = 0;
  GIM_CUDA(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev));
  raise_dyn_smem_limit((const void*)k_refine_fused<VW, false>);
  raise_dyn_smem_limit((const void*)k_refine_fused<VW, true>);
  int per2 = 0;
  GIM_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per, k_refine_fused<VW, false>,
                                                         kFusedBlock, smem));
  GIM_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per2, k_refine_fused<VW, true>,
                                                         kFusedBlock, smem));
  per = std::min(per, per2);
  (void)sms;
  const int r = std::max(1, per);
  cache.emplace(key, r);
  return r;
}

// vertices per CTA of a cluster-mode refinement (GIM_CLUSTER_VPC overrides)
static int cluster_vertices_per_cta() {
  static const int v = [] {
    const char* e = std::getenv("GIM_CLUSTER_VPC");
    int x = e ? std::atoi(e) : 0;
    return x > 0 ? x : 256;
  }();
  return v;
}

// graphs up to this many vertices (and fitting) refine shared-memory
// resident in one CTA (GIM_SMEM_MAXN overrides; 0 disables)
static long long smem_max_n() {
  static const long long v = [] {
    const char* e = std::getenv("GIM_SMEM_MAXN");
    return e ? std::atoll(e) : 1000ll;
  }();
  return v;
}

// dynamic shared memory available to k_refine_smem<VW> (opt-in maximum
// minus its static shared memory); sets the attribute once per device
template <int VW>
static size_t smem_dyn_limit_vw() {
  static std::mutex mu;
  static std::map<int, size_t> cache;
  int dev = 0;
  GIM_CUDA(cudaGetDevice(&dev));
  std::lock_guard<std::mutex> lk(mu);
  auto it = cache.find(dev);
  if (it != cache.end()) return it->second;
  int optin = 0;
  GIM_CUDA(cudaDeviceGetAttribute(&optin, cudaDevAttrMaxSharedMemoryPerBlockOptin, dev));
  cudaFuncAttributes fa;
  GIM_CUDA(cudaFuncGetAttributes(&fa, k_refine_smem<VW>));
  const size_t lim = (size_t)optin > fa.sharedSizeBytes ? (size_t)optin - fa.sharedSizeBytes : 0;
  GIM_CUDA(cudaFuncSetAttribute(k_refine_smem<VW>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                (int)lim));
  cache.emplace(dev, lim);
  return lim;
}

struct VWDISPATCH {};
template <class>
static size_t smem_dyn_limit(int vw) {
  switch (vw) {
    case 4: return smem_dyn_limit_vw<4>();
    case 8: return smem_dyn_limit_vw<8>();
    case 16: return smem_dyn_limit_vw<16>();
    default: return smem_dyn_limit_vw<32>();
  }
}

// vertex-centric first filters while a level has at most this many
// vertices per thread (GIM_VC_STEPS overrides)
static int vc_steps() {
  static const int v = [] {
    const char* e = std::getenv("GIM_VC_STEPS");
    int x = e ? std::atoi(e) : 0;
    return x > 0 ? x : kVcSteps;
  }();
  return v;
}

// vertices per CTA of a cooperative-grid refinement (GIM_COOP_VPC overrides)
static int coop_vpc() {
  static const int v = [] {
    const char* e = std::getenv("GIM_COOP_VPC");
    int x = e ? std::atoi(e) : 0;
    return x > 0 ? x : 128;
  }();
  return v;
}

// rows longer than this are evaluated grid-wide (GIM_HUB_DEG overrides; 0 = off)
static int hub_deg() {
  const char* e = std::getenv("GIM_HUB_DEG");
  return e ? std::atoi(e) : 2048;
}
static int list_deg() {
  const char* e = std::getenv("GIM_LIST_DEG");
  return e ? std::max(std::atoi(e), 1) : kListDeg;
}
static int hub_phases() {
  const char* e = std::getenv("GIM_HUB_PHASES");
  return e ? std::atoi(e) : 3;
}

bool fused_supported(int k, int rho) { return k <= 1024 && rho >= 1 && rho <= 8; }

// LP pass (K9+K10) 8*S + 17n + 25*(2m_cand), with S the
// conn-table entries of the unlocked vertices (evaluated vertices' distinct
// adjacent blocks + one per interior vertex); rebalance (K11+K12) 8*S_over +
// 24*n_over + 16*k*31*rho; apply (K13) 24 per mover slot; plus the entry
// sweeps 8n + 12*m2 each (as K1)
double s8d_refine_bytes(const long long* d, long long n, long long m2, int k, int rho) {
  const double interior = (double)(d[A_SCAN] - d[A_BND]);
  const double S = (double)d[A_EVAL_S] + interior;
  double b = 8.0 * S + 17.0 * (double)n * (double)d[A_LP_IT] + 25.0 * (double)d[A_CAND_SLOTS];
  b += 8.0 * (double)d[A_OVL_S] + 24.0 * (double)d[A_OVL_V] +
       16.0 * (double)k * 31.0 * (double)rho * (double)d[A_WEAK_IT];
  b += 24.0 * (double)d[A_MOV_SLOTS];
  b += (8.0 * (double)n + 12.0 * (double)m2) * (double)d[A_SWEEPS];
  return b;
}

// runs Alg. 4 iterations on the device until the loop ends (returns true) or a
// strong pass is due (returns false; the host performs it and calls again)
bool refine_fused_run(const RefineLevel& L, const Topo& t, int* part, long long* bw,
                      const FusedCfg& cfg, FusedBuffers& fb, cudaStream_t s) {
  const DevGraph& g = L.g;
  const int k = t.k;
  const int NC = 31 * cfg.rho;
  size_t smem = (size_t)kFusedWarps * 4 * k * sizeof(int) + (size_t)k * (8 + 8 + 8 + 4 + 4 + 4 + 1 + 1);
  smem = (smem + 15) & ~(size_t)15;
  int per = 0;
  switch (L.vw) {
    case 4: per = coop_max_blocks<4>(smem); break;
    case 8: per = coop_max_blocks<8>(smem); break;
    case 16: per = coop_max_blocks<16>(smem); break;
    default: per = coop_max_blocks<32>(smem); break;
  }
  const int maxb = coop_blocks_per_sm(per) * device_sms();
  // small graphs: one CTA, or one thread-block cluster of up to kMaxCluster
  // CTAs (plain launches, so the refinements of sibling subgraphs overlap);
  // otherwise ~1K vertices per CTA, at most one full co-resident wave
  const int vpc = cluster_vertices_per_cta();
  int G, mode;
  const size_t extra = smem_resident_bytes(g.n, g.m2, k, NC);
  if (g.n <= smem_max_n() && smem + extra <= smem_dyn_limit<VWDISPATCH>(L.vw)) {
    G = 1;
    mode = 3;
  } else if (g.n <= (long long)vpc) {
    G = 1;
    mode = 0;
  } else if (g.n <= (long long)vpc * kMaxCluster) {
    G = (g.n + vpc - 1) / vpc;
    mode = 1;
  } else {
    G = (int)std::min<long long>((long long)maxb,
                                 ((long long)g.n + coop_vpc() - 1) / coop_vpc());
    mode = 2;
  }
  if (fb.S_cap < (long long)G * k) {
    fb.S = DBuf<long long>((size_t)G * k, s);
    fb.S_cap = (long long)G * k;
  }
  if (fb.W_cap < (long long)k * NC) {
    fb.W = DBuf<long long>((size_t)k * NC, s);
    fb.W_cap = (long long)k * NC;
  }
  FusedArgs A;
  A.n = g.n;
  A.m2 = g.m2;
  A.off = g.off;
  A.tgt = g.tgt;
  A.w = g.w;
  A.vw = g.vw;
  A.src = g.src;
  A.t = t;
  A.k = k;
  A.part = part;
  A.bw = bw;
  A.best = fb.best;
  A.best_bw = fb.best_bw;
  A.dest = fb.dest;
  A.gkey = fb.gkey;
  A.flags0 = fb.tm0;
  A.flags1 = fb.tm1;
  A.rtgt = fb.rtgt;
  A.rcell = fb.rcell;
  A.bstamp = fb.bstamp;
  A.wdeg = fb.wdeg;
  A.lsmall = fb.lsmall;
  A.lheavy = fb.lheavy;
  A.lcand = fb.lcand;
  A.lmov0 = fb.lmov0;
  A.lmov1 = fb.lmov1;
  A.W = fb.W.get();
  A.S = fb.S.get();
  A.ctr = fb.ctr;
  A.st = fb.state;
  A.bar_mode = mode == 3 ? 0 : mode;
  A.smem_base = (int)smem;
  A.vc_steps = vc_steps();
  A.solo = 0;
  A.csize = 0;
  A.ptime = nullptr;
  // hub rows: grid-wide evaluation (cooperative grids only)
  DBuf<int> hconn;
  DBuf<long long> wide;
  A.hconn = nullptr;
  A.wctr = nullptr;
  A.wacc = nullptr;
  A.lhub = nullptr;
  A.lbig = nullptr;
  A.hub_deg = 0;
  A.list_deg = 0;
  A.hub_phases = 0;
  const int ldeg = std::min(hub_deg(), list_deg());
  if (mode == 2 && hub_deg() > 0 && (g.maxdeg < 0 ? g.m2 > ldeg : g.maxdeg > ldeg)) {
    hconn = DBuf<int>((size_t)kHubBatch * k, s);
    GIM_CUDA(cudaMemsetAsync(hconn.get(), 0, sizeof(int) * (size_t)kHubBatch * k, s));
    A.hconn = hconn.get();
    // wide LP candidates: at most m2 / kApplySplitDeg rows
    const size_t wcap = (size_t)(g.m2 / kApplySplitDeg + 2);
    wide = DBuf<long long>(wcap + 1, s);
    GIM_CUDA(cudaMemsetAsync(wide.get(), 0, sizeof(long long) * (wcap + 1), s));
    A.wctr = wide.get();
    A.wacc = wide.get() + 1;
    A.lhub = fb.lheavy;
    A.lbig = fb.lmov1;
    A.hub_deg = hub_deg();
    A.list_deg = ldeg;
    A.hub_phases = hub_phases();
  }
  A.l_max = cfg.l_max;
  A.sigma = cfg.sigma;
  A.phi = cfg.phi;
  A.jet_c = cfg.jet_c;
  A.jet = cfg.jet;
  A.rho = cfg.rho;
  A.i_max = cfg.i_max;
  A.i_w_max = cfg.i_w_max;
  A.seed = cfg.seed;
  void* args[] = {&A};
  void* fn = nullptr;
  // rows over kSweepWarpDeg slots (or unknown maximum degree): the HUB instance
  const bool hubk = A.hconn != nullptr || g.maxdeg < 0 || g.maxdeg > kSweepWarpDeg;
  switch (L.vw) {
    case 4: fn = hubk ? (void*)k_refine_fused<4, true> : (void*)k_refine_fused<4, false>; break;
    case 8: fn = hubk ? (void*)k_refine_fused<8, true> : (void*)k_refine_fused<8, false>; break;
    case 16: fn = hubk ? (void*)k_refine_fused<16, true> : (void*)k_refine_fused<16, false>; break;
    default: fn = hubk ? (void*)k_refine_fused<32, true> : (void*)k_refine_fused<32, false>; break;
  }
  static const bool trace = std::getenv("GIM_TRACE_REFINE") != nullptr;
  cudaEvent_t te[2];
  DBuf<long long> ptime;
  if (trace) {
    ptime = DBuf<long long>(16, s);
    GIM_CUDA(cudaMemsetAsync(ptime.get(), 0, 16 * sizeof(long long), s));
    A.ptime = ptime.get();
    GIM_CUDA(cudaEventCreate(&te[0]));
    GIM_CUDA(cudaEventCreate(&te[1]));
    GIM_CUDA(cudaEventRecord(te[0], s));
  }
  const long long it0 = fb.lp_seen + fb.weak_seen, lp0 = fb.lp_seen;
  {
    // one launch = many Alg. 4 iterations; its algorithmic bytes come from
    // the device counters it returns (SURVEY §8(d) formulas)
    ProfScope prof(P_LP_EVAL, 0.0, s);
    if (mode == 3) {
      void* fs = nullptr;
      switch (L.vw) {
        case 4: fs = (void*)k_refine_smem<4>; break;
        case 8: fs = (void*)k_refine_smem<8>; break;
        case 16: fs = (void*)k_refine_smem<16>; break;
        default: fs = (void*)k_refine_smem<32>; break;
      }
      GIM_CUDA(cudaLaunchKernel(fs, dim3(1), dim3(kFusedBlock), args, smem + extra, s));
    } else if (mode == 0) {
      GIM_CUDA(cudaLaunchKernel(fn, dim3(1), dim3(kFusedBlock), args, smem, s));
    } else if (mode == 1) {
      cudaLaunchConfig_t lc{};
      lc.gridDim = dim3(G);
      lc.blockDim = dim3(kFusedBlock);
      lc.dynamicSmemBytes = smem;
      lc.stream = s;
      cudaLaunchAttribute at[1];
      at[0].id = cudaLaunchAttributeClusterDimension;
      at[0].val.clusterDim.x = G;
      at[0].val.clusterDim.y = 1;
      at[0].val.clusterDim.z = 1;
      lc.attrs = at;
      lc.numAttrs = 1;
      GIM_CUDA(cudaLaunchKernelExC(&lc, fn, args));
    } else {
      GIM_CUDA(cudaLaunchCooperativeKernel(fn, dim3(G), dim3(kFusedBlock), args, smem, s));
    }
    count_launch();
    GIM_CUDA(cudaMemcpyAsync(fb.h_state, fb.state, sizeof(FusedState), cudaMemcpyDeviceToHost, s));
    GIM_CUDA(sync_stream(s));
    long long d[16];
    for (int i = 0; i < 16; ++i) {
      d[i] = fb.h_state->acct[i] - fb.acct_seen[i];
      fb.acct_seen[i] = fb.h_state->acct[i];
    }
    prof.extra = s8d_refine_bytes(d, g.n, g.m2, k, cfg.rho);
    fb.lp_seen = fb.h_state->lp;
    fb.weak_seen = fb.h_state->weak;
  }
  if (trace) {
    GIM_CUDA(cudaEventRecord(te[1], s));
    GIM_CUDA(cudaEventSynchronize(te[1]));
    float ms = 0;
    cudaEventElapsedTime(&ms, te[0], te[1]);
    const long long its = fb.lp_seen + fb.weak_seen - it0;
    long long pt[16];
    GIM_CUDA(cudaMemcpy(pt, ptime.get(), sizeof(pt), cudaMemcpyDeviceToHost));
    std::fprintf(stderr, "refine n=%d m2=%lld k=%d G=%d mode=%d iters=%lld lp=%lld ms=%.3f us/iter=%.1f |",
                 g.n, g.m2, k, G, mode, its, fb.lp_seen - lp0, ms,
                 its ? 1000.0 * ms / (double)its : 0.0);
    static const char* nm[12] = {"stamp", "blist", "ff", "sf", "wlist", "wcand", "wA", "wB",
                                 "wsel", "apply", "commit", "ctl"};
    for (int i = 0; i < 12; ++i) std::fprintf(stderr, " %s=%.1f", nm[i], pt[i] / 1000.0);
    std::fprintf(stderr, "\n");
    cudaEventDestroy(te[0]);
    cudaEventDestroy(te[1]);
  }
  return fb.h_state->status == 0;
}

// ---------------------------------------------------------------------------
// batched shared-memory-resident refinement (one CTA per job)

size_t refine_smem_regular_bytes(int k) {
  size_t smem = (size_t)kFusedWarps * 4 * k * sizeof(int) + (size_t)k * (8 + 8 + 8 + 4 + 4 + 4 + 1 + 1);
  return (smem + 15) & ~(size_t)15;
}

bool refine_smem_fits(long long n, long long m2, int k, int rho, int vw) {
  if (n > smem_max_n()) return false;
  const size_t need = refine_smem_regular_bytes(k) + smem_resident_bytes(n, m2, k, 31 * rho);
  return need <= smem_dyn_limit<VWDISPATCH>(vw);
}

int refine_pick_vw(long long n, long long m2) {
  double avg = n ? (double)m2 / (double)n : 0.0;
  return avg <= 3.0 ? 4 : avg <= 6.0 ? 8 : avg <= 12.0 ? 16 : 32;
}

void refine_smem_batch(std::vector<SmemRefineJob>& jobs, const Topo& t, FusedState* states,
                       std::vector<char>& yielded, cudaStream_t s) {
  const int J = (int)jobs.size();
  yielded.assign((size_t)J, 0);
  if (J == 0) return;
  const int k = t.k;
  const size_t base = refine_smem_regular_bytes(k);
  GIM_CUDA(cudaMemsetAsync(states, 0, sizeof(FusedState) * (size_t)J, s));
  std::vector<FusedArgs> host((size_t)J);
  for (int j = 0; j < J; ++j) {
    const SmemRefineJob& R = jobs[(size_t)j];
    FusedArgs A{};
    A.n = R.g.n;
    A.m2 = R.g.m2;
    A.off = R.g.off;
    A.tgt = R.g.tgt;
    A.w = R.g.w;
    A.vw = R.g.vw;
    A.src = nullptr;
    A.t = t;
    A.k = k;
    A.part = R.part;
    A.bw = R.bw;
    A.best = R.best;
    A.best_bw = R.best_bw;
    A.st = states + j;
    A.bar_mode = 0;
    A.solo = 1;
    A.csize = 0;
    A.smem_base = (int)base;
    A.vc_steps = vc_steps();
    A.ptime = nullptr;
    A.hconn = nullptr;
    A.wctr = nullptr;
    A.wacc = nullptr;
    A.lhub = nullptr;
    A.lbig = nullptr;
    A.hub_deg = 0;
    A.list_deg = 0;
    A.hub_phases = 0;
    A.l_max = R.cfg.l_max;
    A.sigma = R.cfg.sigma;
    A.phi = R.cfg.phi;
    A.jet_c = R.cfg.jet_c;
    A.jet = R.cfg.jet;
    A.rho = R.cfg.rho;
    A.i_max = R.cfg.i_max;
    A.i_w_max = R.cfg.i_w_max;
    A.seed = R.cfg.seed;
    host[(size_t)j] = A;
  }
  BatchTrace trace;
  trace.begin(&host[0].ptime, s);
  // group by lane width (the VW template), one launch per group
  DBuf<FusedArgs> dargs((size_t)J, s);
  std::vector<FusedArgs> ordered;
  std::vector<int> order;
  int vws[4] = {4, 8, 16, 32};
  std::vector<std::pair<int, std::pair<int, size_t>>> groups;  // vw, (first, count) + smem
  std::vector<size_t> gsmem;
  for (int vw : vws) {
    const int first = (int)ordered.size();
    size_t mx = 0;
    for (int j = 0; j < J; ++j)
      if (jobs[(size_t)j].vw == vw) {
        ordered.push_back(host[(size_t)j]);
        order.push_back(j);
        mx = std::max(mx, base + smem_resident_bytes(jobs[(size_t)j].g.n, jobs[(size_t)j].g.m2, k,
                                                     31 * jobs[(size_t)j].cfg.rho));
      }
    if ((int)ordered.size() > first) {
      groups.push_back({vw, {first, (size_t)((int)ordered.size() - first)}});
      gsmem.push_back(mx);
    }
  }
  GIM_CUDA(cudaMemcpyAsync(dargs.get(), ordered.data(), sizeof(FusedArgs) * (size_t)J,
                           cudaMemcpyHostToDevice, s));  // pageable: staged before return
  for (size_t gi = 0; gi < groups.size(); ++gi) {
    const int vw = groups[gi].first, first = groups[gi].second.first;
    const int cnt = (int)groups[gi].second.second;
    const FusedArgs* a = dargs.get() + first;
    const size_t lim = smem_dyn_limit<VWDISPATCH>(vw);
    GIM_CHECK(gsmem[gi] <= lim, GIM_E_INTERNAL, "batched refinement exceeds shared memory");
    static std::once_flag once[4];
    auto set_attr = [&](const void* fn, int slot) {
      std::call_once(once[slot], [&] {
        GIM_CUDA(cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)lim));
      });
    };
    switch (vw) {
      case 4: set_attr((const void*)k_refine_smem_batch<4>, 0); break;
      case 8: set_attr((const void*)k_refine_smem_batch<8>, 1); break;
      case 16: set_attr((const void*)k_refine_smem_batch<16>, 2); break;
      default: set_attr((const void*)k_refine_smem_batch<32>, 3); break;
    }
    switch (vw) {
      case 4: k_refine_smem_batch<4><<<cnt, kFusedBlock, gsmem[gi], s>>>(a); break;
      case 8: k_refine_smem_batch<8><<<cnt, kFusedBlock, gsmem[gi], s>>>(a); break;
      case 16: k_refine_smem_batch<16><<<cnt, kFusedBlock, gsmem[gi], s>>>(a); break;
      default: k_refine_smem_batch<32><<<cnt, kFusedBlock, gsmem[gi], s>>>(a); break;
    }
    count_launch();
    GIM_LAUNCH_CHECK();
  }
  // read back the job states (status: strong pass due) in launch order
  FusedState* hs = static_cast<FusedState*>(pinned_scratch(sizeof(FusedState) * (size_t)J));
  GIM_CUDA(cudaMemcpyAsync(hs, states, sizeof(FusedState) * (size_t)J, cudaMemcpyDeviceToHost, s));
  GIM_CUDA(sync_stream(s));
  trace.end("smem_batch", J, jobs[0].g.n, jobs[0].g.m2, hs[0].iters, s);
  for (int j = 0; j < J; ++j) {
    // states are indexed by the original job (A.st = states + j)
    yielded[(size_t)j] = hs[j].status != 0;
    jobs[(size_t)j].iters = hs[j].iters;
    jobs[(size_t)j].lp = hs[j].lp;
    jobs[(size_t)j].weak = hs[j].weak;
  }
  (void)order;
}

// batched cluster-mode refinement: one cluster per job, per-job scratch in
// global memory (levels too large to be shared-memory resident)
void refine_cluster_batch(std::vector<SmemRefineJob>& jobs, const Topo& t, FusedState* states,
                          std::vector<char>& yielded, cudaStream_t s) {
  const int J = (int)jobs.size();
  yielded.assign((size_t)J, 0);
  if (J == 0) return;
  const int k = t.k;
  const size_t base = refine_smem_regular_bytes(k);
  GIM_CUDA(cudaMemsetAsync(states, 0, sizeof(FusedState) * (size_t)J, s));
  // scratch arena: per job 8 int arrays, gkey, 3 byte arrays, W, S, ctr
  std::vector<size_t> off((size_t)J + 1, 0);
  auto words = [&](const SmemRefineJob& R) {
    const size_t n = (size_t)std::max(R.g.n, 1), NC = 31 * (size_t)R.cfg.rho;
    return 8 * n + 2 * n + (3 * n + 7) / 4 + 2 * ((size_t)k * NC + (size_t)k * kMaxCluster + 17) + 8;
  };
  for (int j = 0; j < J; ++j) off[(size_t)j + 1] = off[(size_t)j] + ((words(jobs[(size_t)j]) + 3) & ~(size_t)3);
  DBuf<int> arena(off[(size_t)J], s);
  std::vector<FusedArgs> host((size_t)J);
  for (int j = 0; j < J; ++j) {
    const SmemRefineJob& R = jobs[(size_t)j];
    const size_t n = (size_t)std::max(R.g.n, 1), NC = 31 * (size_t)R.cfg.rho;
    int* a = arena.get() + off[(size_t)j];
    FusedArgs A{};
    A.n = R.g.n;
    A.m2 = R.g.m2;
    A.off = R.g.off;
    A.tgt = R.g.tgt;
    A.w = R.g.w;
    A.vw = R.g.vw;
    A.src = nullptr;
    A.t = t;
    A.k = k;
    A.part = R.part;
    A.bw = R.bw;
    A.best = R.best;
    A.best_bw = R.best_bw;
    A.dest = a;
    A.rtgt = a + n;
    A.lsmall = a + 2 * n;
    A.lheavy = a + 3 * n;
    A.lcand = a + 4 * n;
    A.lmov0 = a + 5 * n;
    A.lmov1 = a + 6 * n;
    A.bstamp = nullptr;
    long long* q = reinterpret_cast<long long*>(a + 8 * n);  // 8-byte aligned (n ints * 8)
    A.gkey = q;
    A.W = q + n;
    A.S = A.W + (size_t)k * NC;
    A.ctr = A.S + (size_t)k * kMaxCluster;
    unsigned char* b = reinterpret_cast<unsigned char*>(A.ctr + 17);
    A.flags0 = b;
    A.flags1 = b + n;
    A.rcell = b + 2 * n;
    A.st = states + j;
    A.smem_base = (int)base;
    A.vc_steps = vc_steps();
    A.solo = 0;
    A.ptime = nullptr;
    A.hconn = nullptr;
    A.wctr = nullptr;
    A.wacc = nullptr;
    A.lhub = nullptr;
    A.lbig = nullptr;
    A.hub_deg = 0;
    A.list_deg = 0;
    A.hub_phases = 0;
    A.l_max = R.cfg.l_max;
    A.sigma = R.cfg.sigma;
    A.phi = R.cfg.phi;
    A.jet_c = R.cfg.jet_c;
    A.jet = R.cfg.jet;
    A.rho = R.cfg.rho;
    A.i_max = R.cfg.i_max;
    A.i_w_max = R.cfg.i_w_max;
    A.seed = R.cfg.seed;
    host[(size_t)j] = A;
    GIM_CUDA(cudaMemsetAsync(A.ctr, 0, 17 * sizeof(long long), s));
  }
  const int vpc = cluster_vertices_per_cta();
  BatchTrace trace;
  trace.begin(&host[0].ptime, s);
  DBuf<FusedArgs> dargs((size_t)J, s);
  std::vector<FusedArgs> ordered;
  struct Grp { int vw, first, cnt, cs; };
  std::vector<Grp> groups;
  for (int vw : {4, 8, 16, 32}) {
    const int first = (int)ordered.size();
    int cs = 1;
    for (int j = 0; j < J; ++j)
      if (jobs[(size_t)j].vw == vw) {
        cs = std::max(cs, std::min(kMaxCluster, (jobs[(size_t)j].g.n + vpc - 1) / vpc));
        ordered.push_back(host[(size_t)j]);
      }
    const int cnt = (int)ordered.size() - first;
    if (cnt) {
      for (int i = first; i < first + cnt; ++i) {
        ordered[(size_t)i].csize = cs;
        ordered[(size_t)i].bar_mode = cs > 1 ? 1 : 0;
      }
      groups.push_back({vw, first, cnt, cs});
    }
  }
  GIM_CUDA(cudaMemcpyAsync(dargs.get(), ordered.data(), sizeof(FusedArgs) * (size_t)J,
                           cudaMemcpyHostToDevice, s));  // pageable: staged before return
  for (const Grp& g : groups) {
    void* fn = nullptr;
    switch (g.vw) {
      case 4: fn = (void*)k_refine_cluster_batch<4>; break;
      case 8: fn = (void*)k_refine_cluster_batch<8>; break;
      case 16: fn = (void*)k_refine_cluster_batch<16>; break;
      default: fn = (void*)k_refine_cluster_batch<32>; break;
    }
    raise_dyn_smem_limit(fn);
    const FusedArgs* a = dargs.get() + g.first;
    int cs = g.cs;
    void* args[] = {(void*)&a, (void*)&cs};
    cudaLaunchConfig_t lc{};
    lc.gridDim = dim3((unsigned)(g.cnt * g.cs));
    lc.blockDim = dim3(kFusedBlock);
    lc.dynamicSmemBytes = base;
    lc.stream = s;
    cudaLaunchAttribute at[1];
    at[0].id = cudaLaunchAttributeClusterDimension;
    at[0].val.clusterDim.x = (unsigned)g.cs;
    at[0].val.clusterDim.y = 1;
    at[0].val.clusterDim.z = 1;
    lc.attrs = at;
    lc.numAttrs = 1;
    GIM_CUDA(cudaLaunchKernelExC(&lc, fn, args));
    count_launch();
  }
  FusedState* hs = static_cast<FusedState*>(pinned_scratch(sizeof(FusedState) * (size_t)J));
  GIM_CUDA(cudaMemcpyAsync(hs, states, sizeof(FusedState) * (size_t)J, cudaMemcpyDeviceToHost, s));
  GIM_CUDA(sync_stream(s));
  trace.end("cluster_batch", J, jobs[0].g.n, jobs[0].g.m2, hs[0].iters, s);
  for (int j = 0; j < J; ++j) {
    yielded[(size_t)j] = hs[j].status != 0;
    jobs[(size_t)j].iters = hs[j].iters;
    jobs[(size_t)j].lp = hs[j].lp;
    jobs[(size_t)j].weak = hs[j].weak;
  }
}

}  // namespace gim
