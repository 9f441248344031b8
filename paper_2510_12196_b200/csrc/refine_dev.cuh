// Device helpers shared by the per-phase refinement kernels (refine.cu)
// and the device-resident Alg. 4 loop (refine_fused.cu).
#pragma once
#include "common.cuh"

namespace gim {

constexpr long long kGainNone = LLONG_MIN;

// distance between two digit codes (see Topo)
__device__ __forceinline__ long long cdist(const long long* dbit, unsigned long long a,
                                           unsigned long long b) {
  unsigned long long c = a ^ b;
  return c ? dbit[63 - __clzll(c)] : 0ll;
}

struct Best {
  long long gain;
  int b;
};

// (gain desc, block asc); b < 0 = none
__device__ __forceinline__ bool best_better(long long g1, int b1, long long g2, int b2) {
  if (b1 < 0) return false;
  if (b2 < 0) return true;
  if (g1 != g2) return g1 > g2;
  return b1 < b2;
}

// shared per-block copy of dbit
__device__ __forceinline__ void load_dbit(long long* s_dbit, const Topo& t) {
  for (int i = threadIdx.x; i < 64; i += blockDim.x) s_dbit[i] = t.dbit[i];
}

// ---------------------------------------------------------------------------
// Per-vertex gain evaluation, register path (degree <= VW).
// Lane j of the group holds neighbour j: its block code and edge weight.
// cost(b_j) = sum_i w_i D(b_j, b_i) by a VW-step shuffle broadcast;
// gain(b_j) = cur - cost(b_j), cur = cost(own)  (Eq. 1, refinement.py:171-186).

struct VertexEval {
  long long cur;       // sum_u w D(own, Pi u)
  long long conn_own;  // conn(v, own)
  long long best_gain;
  int best_b;          // -1: no admissible adjacent block
};

// Neighbours in the same block are merged first: __match_any_sync groups the
// lanes of a vertex group by block, the first lane of each block (the
// "leader") gets conn(v, b) by a redux over its peers, and the cost sweep
// runs over the leaders only — the number of DISTINCT adjacent blocks
// (typically 1-3) instead of the degree.  Non-leader lanes hold the same
// block as their leader, so dropping them changes no (gain, block) maximum.
// `dmax` (max degree over the warp's groups) is unused but kept for callers.
// Interior vertices (every neighbour in the own block) are the common case
// after the first iterations: a warp whose groups have no candidate lane
// skips the whole evaluation.
template <int VW>
__device__ __forceinline__ VertexEval eval_regs(bool valid, int own, int myb, int myw, int dmax,
                                                const Topo& t, const long long* s_dbit,
                                                const unsigned char* allowed, bool need_conn) {
  (void)dmax;
  VertexEval r;
  r.cur = 0;
  r.conn_own = 0;
  r.best_gain = kGainNone;
  r.best_b = -1;
  const bool cand0 = valid && myb >= 0 && myb != own && (allowed == nullptr || allowed[myb]);
  if (!__any_sync(0xffffffffu, cand0)) return r;
  const int lane = (int)lane_id();
  const unsigned gmask =
      VW == 32 ? 0xffffffffu : (((1u << VW) - 1u) << (lane & ~(VW - 1)));
  const int key = valid ? myb : -1 - lane;
  const unsigned peers = __match_any_sync(0xffffffffu, key) & gmask;
  const bool leader = valid && lane == __ffs(peers) - 1;
  const int conn = (int)__reduce_add_sync(peers, valid ? (unsigned)myw : 0u);
  const unsigned lm = __ballot_sync(0xffffffffu, leader) & gmask;
  const int trips = __reduce_max_sync(0xffffffffu, (unsigned)__popc(lm));
  const unsigned long long ocode = t.code[(own < 0 ? 0 : own)];
  const unsigned long long mycode = myb >= 0 ? t.code[myb] : 0ull;
  const long long cl = leader ? (long long)conn : 0;
  long long cur = cl * cdist(s_dbit, ocode, mycode);
  long long co = (need_conn && leader && myb == own) ? cl : 0;
  long long cost = 0;
  unsigned rem = lm;
  for (int i = 0; i < trips; ++i) {
    const int src = rem ? __ffs(rem) - 1 : lane;
    const bool use = rem != 0;
    rem &= rem - 1;
    const unsigned long long ci = __shfl_sync(0xffffffffu, mycode, src);
    const int wi = __shfl_sync(0xffffffffu, conn, src);
    if (use) cost += (long long)wi * cdist(s_dbit, mycode, ci);
  }
#pragma unroll
  for (int o = VW / 2; o > 0; o >>= 1) {
    cur += __shfl_xor_sync(0xffffffffu, cur, o);
    if (need_conn) co += __shfl_xor_sync(0xffffffffu, co, o);
  }
  const bool cand = cand0 && leader;
  long long g = cand ? cur - cost : kGainNone;
  int b = cand ? myb : -1;
#pragma unroll
  for (int o = VW / 2; o > 0; o >>= 1) {
    long long g2 = __shfl_xor_sync(0xffffffffu, g, o);
    int b2 = __shfl_xor_sync(0xffffffffu, b, o);
    if (best_better(g2, b2, g, b)) { g = g2; b = b2; }
  }
  r.cur = cur;
  r.conn_own = co;
  r.best_gain = g;
  r.best_b = b;
  return r;
}

// ---------------------------------------------------------------------------
// Per-vertex gain evaluation, thread-per-vertex path.  One thread walks the
// row and merges neighbours by block into at most TPV_DISTINCT (block, conn)
// pairs held in registers (unrolled, statically indexed); then
// cur = sum_j conn_j D(own, b_j), cost(b_i) = sum_j conn_j D(b_i, b_j) and
// the best admissible b_i by (gain desc, block asc) — exactly Eq. 1 over the
// reference's slot table (refinement.py:168-198).  No shuffles: a warp
// evaluates 32 vertices at once with independent instruction streams, which
// is what the latency-bound refinement phases need.  A vertex with more
// distinct adjacent blocks than TPV_DISTINCT reports `overflow` and is
// handed to the warp-per-vertex table path.  `tb` >= 0 also returns the
// cost of moving to tb (rebalance fallback target).

constexpr int TPV_DISTINCT = 4;

#ifndef GIM_EVAL_CHUNK
#define GIM_EVAL_CHUNK 4
#endif
constexpr int kEvalChunk = GIM_EVAL_CHUNK;  // row slots per load batch

struct ThreadEval {
  long long cur, conn_own, best_gain, cost_tb;
  int best_b;
  int nblk;  // distinct adjacent blocks found (conn-table entries, S_v)
  bool overflow;
};

// `flatd` > 0: single-level topology (the internal partitioner's), D(x,y) =
// flatd * [x != y], so cost(b) = flatd * (W - conn(b)) and
// gain(b) = flatd * (conn(b) - conn(own)) — no distance lookups at all.
__device__ __forceinline__ ThreadEval eval_thread(int e0, int e1, int own, const int* tgt,
                                                  const int* w, const int* part, const Topo& t,
                                                  const long long* s_dbit,
                                                  const unsigned char* allowed, int tb,
                                                  long long flatd = 0) {
  ThreadEval r;
  r.cur = 0;
  r.conn_own = 0;
  r.best_gain = kGainNone;
  r.best_b = -1;
  r.cost_tb = 0;
  r.nblk = 0;
  r.overflow = false;
  int nb[TPV_DISTINCT];
  long long cw[TPV_DISTINCT];
#pragma unroll
  for (int j = 0; j < TPV_DISTINCT; ++j) {
    nb[j] = -1;
    cw[j] = 0;
  }
  int cnt = 0;
  // rows in chunks of kEvalChunk: the target / weight loads and then the
  // block gathers of a chunk are independent, so they overlap
  for (int e = e0; e < e1; e += kEvalChunk) {
    int tg[kEvalChunk], wg[kEvalChunk], pb[kEvalChunk];
#pragma unroll
    for (int q = 0; q < kEvalChunk; ++q)
      if (e + q < e1) {
        tg[q] = tgt[e + q];
        wg[q] = w[e + q];
      }
#pragma unroll
    for (int q = 0; q < kEvalChunk; ++q)
      if (e + q < e1) pb[q] = part[tg[q]];
#pragma unroll
    for (int q = 0; q < kEvalChunk; ++q) {
      if (e + q >= e1) break;
      const int b = pb[q];
      const long long ww = wg[q];
      bool found = false;
#pragma unroll
      for (int j = 0; j < TPV_DISTINCT; ++j)
        if (nb[j] == b) {
          cw[j] += ww;
          found = true;
        }
      if (!found) {
        if (cnt == TPV_DISTINCT) {
          r.overflow = true;
          return r;
        }
#pragma unroll
        for (int j = 0; j < TPV_DISTINCT; ++j)
          if (j == cnt) {
            nb[j] = b;
            cw[j] = ww;
          }
        ++cnt;
      }
    }
  }
  r.nblk = cnt;
  if (flatd > 0) {
    long long W = 0, ctb = 0;
#pragma unroll
    for (int j = 0; j < TPV_DISTINCT; ++j) {
      if (j < cnt) {
        W += cw[j];
        if (nb[j] == own) r.conn_own = cw[j];
        if (nb[j] == tb) ctb = cw[j];
      }
    }
    r.cur = flatd * (W - r.conn_own);
    if (tb >= 0) r.cost_tb = flatd * (W - ctb);
#pragma unroll
    for (int i = 0; i < TPV_DISTINCT; ++i) {
      if (i < cnt && nb[i] != own && (allowed == nullptr || allowed[nb[i]])) {
        const long long g = flatd * (cw[i] - r.conn_own);
        if (best_better(g, nb[i], r.best_gain, r.best_b)) {
          r.best_gain = g;
          r.best_b = nb[i];
        }
      }
    }
    return r;
  }
  unsigned long long code[TPV_DISTINCT];
  bool adm[TPV_DISTINCT];
  bool any = false;
  const unsigned long long oc = t.code[own];
#pragma unroll
  for (int j = 0; j < TPV_DISTINCT; ++j) {
    code[j] = j < cnt ? t.code[nb[j]] : oc;
    adm[j] = j < cnt && nb[j] != own && (allowed == nullptr || allowed[nb[j]]);
    any |= adm[j];
    if (j < cnt) {
      r.cur += cw[j] * cdist(s_dbit, oc, code[j]);
      if (nb[j] == own) r.conn_own = cw[j];
    }
  }
  if (tb >= 0) {
    const unsigned long long tc = t.code[tb];
#pragma unroll
    for (int j = 0; j < TPV_DISTINCT; ++j)
      if (j < cnt) r.cost_tb += cw[j] * cdist(s_dbit, tc, code[j]);
  }
  if (!any) return r;  // interior vertex / nothing admissible: no candidate
#pragma unroll
  for (int i = 0; i < TPV_DISTINCT; ++i) {
    if (adm[i]) {
      long long cost = 0;
#pragma unroll
      for (int j = 0; j < TPV_DISTINCT; ++j)
        if (j < cnt && j != i) cost += cw[j] * cdist(s_dbit, code[i], code[j]);
      const long long g = r.cur - cost;
      if (best_better(g, nb[i], r.best_gain, r.best_b)) {
        r.best_gain = g;
        r.best_b = nb[i];
      }
    }
  }
  return r;
}

// cur = sum_u w D(own, Pi u) alone (rebalance fallback when no candidate)
template <int VW>
__device__ __forceinline__ long long cur_regs(bool valid, int own, int myb, int myw,
                                              const Topo& t, const long long* s_dbit) {
  const unsigned long long ocode = t.code[(own < 0 ? 0 : own)];
  const unsigned long long mycode = myb >= 0 ? t.code[myb] : 0ull;
  long long cur = valid ? (long long)myw * cdist(s_dbit, ocode, mycode) : 0;
#pragma unroll
  for (int o = VW / 2; o > 0; o >>= 1) cur += __shfl_xor_sync(0xffffffffu, cur, o);
  return cur;
}

// cost of moving to a fixed block `tb` (for the rebalance hash fallback)
template <int VW>
__device__ __forceinline__ long long cost_regs(bool valid, int myb, int myw, int tb,
                                               const Topo& t, const long long* s_dbit) {
  unsigned long long tc = t.code[(tb < 0 ? 0 : tb)];
  unsigned long long mc = myb >= 0 ? t.code[myb] : 0ull;
  long long c = valid ? (long long)myw * cdist(s_dbit, tc, mc) : 0;
#pragma unroll
  for (int o = VW / 2; o > 0; o >>= 1) c += __shfl_xor_sync(0xffffffffu, c, o);
  return c;
}

// ---------------------------------------------------------------------------
// Per-vertex gain evaluation, shared-memory path (degree > VW): one warp per
// vertex, conn(v, b) accumulated into a dense per-warp block table with
// shared atomics, compacted to the nonzero (block, conn) list, then
// cost(b) = sum_j conn_j D(b, b_j) over the list.

struct WarpTable {
  int* tab;    // [k]
  int* lb;     // [k] nonzero blocks
  int* lw;     // [k] their conn
};

__device__ __forceinline__ int warp_build_table(const WarpTable& wt, int k, int e0, int e1,
                                                const int* __restrict__ tgt,
                                                const int* __restrict__ w,
                                                const int* __restrict__ part) {
  const int lane = lane_id();
  __syncwarp();  // every lane is done reading the previous vertex's table
  for (int i = lane; i < k; i += 32) wt.tab[i] = 0;
  __syncwarp();
  for (int e = e0 + lane; e < e1; e += 32) atomicAdd(&wt.tab[part[tgt[e]]], w[e]);
  __syncwarp();
  int s = 0;
  for (int base = 0; base < k; base += 32) {
    int i = base + lane;
    int x = i < k ? wt.tab[i] : 0;
    unsigned m = __ballot_sync(0xffffffffu, x != 0);
    if (x != 0) {
      int pos = s + __popc(m & ((1u << lane) - 1u));
      wt.lb[pos] = i;
      wt.lw[pos] = x;
    }
    s += __popc(m);
  }
  __syncwarp();
  return s;
}

// Wide tables (many distinct adjacent blocks, R-MAT hubs): the O(s^2)
// candidate costs below become O(L) each.  With mixed-radix block ids the
// blocks within distance d_l of b form the contiguous range of b's level-l
// group (size P_l), so cost(b) = sum_l d_l * (S_l(b) - S_{l-1}(b)) with
// S_l(b) the table's sum over that group (S_{-1}(b) = conn(b), S_{L-1} = the
// total) — read from an in-place exclusive prefix sum of the dense table.
// Integer regrouping of the same sum: the gains are identical.
#ifndef GIM_GROUPED_MIN_S
#define GIM_GROUPED_MIN_S 16
#endif
constexpr int kGroupedMinS = GIM_GROUPED_MIN_S;

__device__ __forceinline__ long long grouped_cost(const int* pre, int k, int L,
                                                  const long long* lv, int total, int b,
                                                  long long cb) {
  long long c = 0, prev = cb;
  for (int l = 0; l < L; ++l) {
    long long S = total;
    if (l < L - 1) {
      const long long P = __ldg(lv + l);
      const long long g0 = (b / P) * P, g1 = g0 + P;
      S = (long long)(g1 >= k ? total : pre[g1]) - pre[g0];
    }
    c += __ldg(lv + L + l) * (S - prev);
    prev = S;
  }
  return c;
}

__device__ __forceinline__ VertexEval eval_table_grouped(int* tab, const int* lb, const int* lw,
                                                      int s, int own, int k, int L,
                                                      const long long* lv,
                                                      const unsigned char* allowed) {
  const int lane = lane_id();
  const int conn_own = tab[own];
  // in-place exclusive prefix of tab[0..k): contiguous chunk per lane
  const int per = (k + 31) >> 5, c0 = min(k, lane * per), c1 = min(k, c0 + per);
  int run = 0;
  for (int c = c0; c < c1; ++c) run += tab[c];
  int incl = run;
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    const int y = __shfl_up_sync(0xffffffffu, incl, o);
    if (lane >= o) incl += y;
  }
  const int total = __shfl_sync(0xffffffffu, incl, 31);
  int ex = incl - run;
  __syncwarp();
  for (int c = c0; c < c1; ++c) {
    const int x = tab[c];
    tab[c] = ex;
    ex += x;
  }
  __syncwarp();
  const long long cur = grouped_cost(tab, k, L, lv, total, own, conn_own);
  long long g = kGainNone;
  int b = -1;
  for (int i = lane; i < s; i += 32) {
    const int bi = lb[i];
    if (bi == own || (allowed && !allowed[bi])) continue;
    const long long gi = cur - grouped_cost(tab, k, L, lv, total, bi, lw[i]);
    if (best_better(gi, bi, g, b)) { g = gi; b = bi; }
  }
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) {
    long long g2 = __shfl_xor_sync(0xffffffffu, g, o);
    int b2 = __shfl_xor_sync(0xffffffffu, b, o);
    if (best_better(g2, b2, g, b)) { g = g2; b = b2; }
  }
  __syncwarp();
  VertexEval r;
  r.cur = cur;
  r.conn_own = conn_own;
  r.best_gain = g;
  r.best_b = b;
  return r;
}

template <bool WIDE = true>
__device__ __forceinline__ VertexEval eval_table(const WarpTable& wt, int s, int own,
                                                 const Topo& t, const long long* s_dbit,
                                                 const unsigned char* allowed) {
  // wide tables: O(L) per candidate (leaves wt.tab as a prefix sum; callers
  // use only lb / lw afterwards and the next table build re-zeroes it)
  if (WIDE && s > kGroupedMinS)
    return eval_table_grouped(wt.tab, wt.lb, wt.lw, s, own, t.k, t.L, topo_lv(t), allowed);
  const int lane = lane_id();
  const unsigned long long oc = t.code[own];
  long long cur = 0;
  for (int j = lane; j < s; j += 32)
    cur += (long long)wt.lw[j] * cdist(s_dbit, oc, t.code[wt.lb[j]]);
  cur = warp_sum_ll(cur);
  long long g = kGainNone;
  int b = -1;
  for (int i = lane; i < s; i += 32) {
    int bi = wt.lb[i];
    if (bi == own || (allowed && !allowed[bi])) continue;
    unsigned long long ci = t.code[bi];
    long long cost = 0;
    for (int j = 0; j < s; ++j)
      cost += (long long)wt.lw[j] * cdist(s_dbit, ci, t.code[wt.lb[j]]);
    long long gi = cur - cost;
    if (best_better(gi, bi, g, b)) { g = gi; b = bi; }
  }
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) {
    long long g2 = __shfl_xor_sync(0xffffffffu, g, o);
    int b2 = __shfl_xor_sync(0xffffffffu, b, o);
    if (best_better(g2, b2, g, b)) { g = g2; b = b2; }
  }
  VertexEval r;
  r.cur = cur;
  r.conn_own = wt.tab[own];
  r.best_gain = g;
  r.best_b = b;
  return r;
}

__device__ __forceinline__ long long cost_table(const WarpTable& wt, int s, int tb,
                                                const Topo& t, const long long* s_dbit) {
  const unsigned long long tc = t.code[tb];
  long long c = 0;
  for (int j = lane_id(); j < s; j += 32)
    c += (long long)wt.lw[j] * cdist(s_dbit, tc, t.code[wt.lb[j]]);
  return warp_sum_ll(c);
}

// ---------------------------------------------------------------------------
// shared per-vertex decisions

struct LpOut {
  unsigned char* cand;
  int* dest;
  long long* gkey;  // gain for candidates, kGainNone otherwise
};

struct LpParams {
  const unsigned char* locked;  // null = no locks
  int jet;
  double jet_c;
  int dshift;  // distances scaled by 2^dshift (Topo::dshift)
};

// Jet filter (refinement.py:236-240): -gain < floor(c * conn(v, own)); gains
// carry the 2^dshift distance scale, conn is a weight
__device__ __forceinline__ bool jet_admits(long long gain, long long conn_own, double c,
                                          int dshift) {
  return (double)(-gain) < ldexp(floor(c * (double)conn_own), dshift);
}

__device__ __forceinline__ void lp_decide(int v, int own, const VertexEval& r,
                                          const LpParams& p, const LpOut& o) {
  bool ok = false;
  if (r.best_b >= 0) {
    if (r.best_gain >= 0) ok = true;
    else if (p.jet) ok = jet_admits(r.best_gain, r.conn_own, p.jet_c, p.dshift);
  }
  o.cand[v] = ok ? 1 : 0;
  o.dest[v] = ok ? r.best_b : own;
  o.gkey[v] = ok ? r.best_gain : kGainNone;
}

struct RbParams {
  const unsigned char* ovl;    // [k] overloaded blocks
  const unsigned char* elig;   // [k] eligible blocks (bw < sigma)
  const int* elig_list;        // ascending eligible ids
  int n_elig;
  unsigned long long seed;
  long long pass_counter;
};

struct RbOut {
  int* target;      // -1: not a rebalance candidate
  long long* gain;
  unsigned char* to_move;  // zeroed by the candidate pass
};


// bucket slot of a gain (refinement.py:41-47): bisect_right over
// [0, 1..10, 20..100, 200..1000] of -gain; slot 0 = positive, 30 = <= -1000
__device__ __forceinline__ int slot_for_gain(long long g) {
  if (g > 0) return 0;
  if (g <= -1000) return 30;
  long long x = -g;  // bisect_right over [0,1..10,20..100,200..1000]
  if (x <= 10) return (int)x + 1;
  if (x < 100) return 10 + (int)(x / 10);
  if (x < 1000) return 19 + (int)(x / 100);
  return 30;
}

// the same bucket for a gain in units of 2^-sh (scaled distances): the slot
// bounds are integers b, and b * 2^sh <= -g  <=>  b <= floor(-g / 2^sh)
__device__ __forceinline__ int slot_for_gain(long long g, int sh) {
  return slot_for_gain(g > 0 ? g : -((-g) >> sh));
}

}  // namespace gim
