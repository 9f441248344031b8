// Coarsening: heavy-edge matching (K3/K4), two-hop matching (K5), coarse ids,
// contraction by hand-rolled radix sort + segmented reduce (K6), projection (K7).
//
// Reference: coarsening.py (match rounds :63-95, two-hop :98-161,
// match_graph :164-173, coarse ids :176-188, contract :191-249, project
// :269-277, build_level_stack :280-295).
#include <cooperative_groups.h>

#include <mutex>

#include "common.cuh"
#include "kernels.cuh"
#include "radix.cuh"
#include "scan.cuh"
#include "coarsen_dev.cuh"

namespace gim {

namespace cg = cooperative_groups;

// device-side "round 2 only below 40 % matched" (coarsening.py:167-170):
// `gate` is a snapshot of the matched count after round 1
__device__ __forceinline__ bool hem_gated(const long long* gate, int n) {
  return gate && (n ? (double)*gate / (double)n : 1.0) >= 0.40;
}


// ---------------------------------------------------------------------------
// K3 heavy-edge preference: per unmatched v, argmax over eligible unmatched
// neighbours u (c_v + c_u <= l_max) of (w^2/(c_v c_u), hash2(seed,min,max)),
// first CSR slot on a full tie (coarsening.py:72-90).  The rational is
// compared exactly by 128-bit cross multiplication (c_v cancels).

// VW lanes per vertex; loop bounds are warp-uniform so the shuffles in the
// group reduction always run with the full mask
template <int VW>
__global__ void __launch_bounds__(256) k_hem_pref(int n, const int* __restrict__ off,
                                                  const int* __restrict__ tgt,
                                                  const int* __restrict__ w,
                                                  const int* __restrict__ vw,
                                                  const int* __restrict__ partner, double l_max,
                                                  unsigned long long seed, int* __restrict__ pref) {
  constexpr int GPW = 32 / VW;
  const long long wid = ((long long)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  const long long nw = ((long long)gridDim.x * blockDim.x) >> 5;
  const int lane = lane_id();
  const int gi = lane / VW, li = lane % VW;
  for (long long vb = wid * GPW; vb < n; vb += nw * GPW) {
    const int v = (int)(vb + gi);
    HemCand best;
    best.u = -1;
    best.w = best.c = best.slot = 0;
    best.h = 0;
    const bool active = v < n && partner[v] < 0;
    if (active) {
      const long long cv = vw[v];
      const int e1 = off[v + 1];
      for (int e = off[v] + li; e < e1; e += VW) {
        int u = tgt[e];
        if (partner[u] >= 0) continue;
        int cu = vw[u];
        if ((double)(cv + cu) > l_max) continue;
        HemCand c;
        c.w = w[e];
        c.c = cu;
        c.slot = e;
        c.u = u;
        c.h = hash2(seed, (unsigned long long)min(v, u), (unsigned long long)max(v, u));
        if (hem_better(c, best)) best = c;
      }
    }
#pragma unroll
    for (int o = VW / 2; o > 0; o >>= 1) {
      HemCand y = hem_shfl(best, o);
      if (hem_better(y, best)) best = y;
    }
    if (li == 0 && v < n) pref[v] = active ? best.u : -1;
  }
}

// K4 mutual matching: v and u match iff they prefer each other (snapshot
// semantics: preferences were all computed first, coarsening.py:91-94)
template <int BLOCK>
__global__ void __launch_bounds__(BLOCK) k_hem_mutual(int n, const int* __restrict__ pref,
                                                      int* __restrict__ partner,
                                                      long long* __restrict__ matched,
                                                      const long long* gate = nullptr) {
  if (hem_gated(gate, n)) return;
  long long cnt = 0;
  for (int v = blockIdx.x * BLOCK + threadIdx.x; v < n; v += gridDim.x * BLOCK) {
    int u = pref[v];
    if (u >= 0 && v < u && pref[u] == v) {
      partner[v] = u;
      partner[u] = v;
      cnt += 2;
    }
  }
  block_sum_atomic<BLOCK>(cnt, matched);
}

// Thread-per-vertex preference (rows up to kHemTpv slots): one thread walks
// its row in chunks of 4 (the target / weight loads, then the eligibility
// gathers of a chunk, are independent and overlap) — no shuffles, 32
// vertices per warp in flight.  elig_c[u] = c_u for unmatched u, -1 for
// matched u (one gather instead of partner[u] + vw[u]).  Longer rows are
// evaluated in place by the whole warp (strided slots + shuffle argmax).
constexpr int kHemTpv = 32;
constexpr int kHemHuge = 1024;

// Per-round eligibility: elig[u] = c_u for unmatched u, -1 for matched u —
// ONE 4-byte gather per candidate slot (the array stays L2-resident: 16.8 MB
// at 2^22).  The tie-break hash2(seed, min, max) = splitmix64(S_min ^ max),
// S_a = splitmix64(seed ^ splitmix64(a)), is recomputed from the ids (pure
// ALU) and only when a candidate's rating ties the current best's.
__device__ __forceinline__ unsigned long long hem_s(unsigned long long seed, int a) {
  return splitmix64(seed ^ splitmix64((unsigned long long)a));
}

__device__ __forceinline__ unsigned long long hem_hash(unsigned long long seed, int v, int u) {
  const int a = min(v, u), b = max(v, u);
  return splitmix64(hem_s(seed, a) ^ (unsigned long long)b);
}

// rating order of coarsening.py:52-60 with the hash computed lazily:
// returns true when `c` beats `best` (both hashes filled in on a tie)
__device__ __forceinline__ bool hem_better_lazy(HemCand& c, bool& c_h, HemCand& best,
                                                bool& best_h, unsigned long long seed, int v) {
  c_h = false;
  if (best.u < 0) return true;
  const unsigned long long cw2 = (unsigned long long)c.w * (unsigned long long)c.w;
  const unsigned long long bw2 = (unsigned long long)best.w * (unsigned long long)best.w;
  const unsigned __int128 lhs = (unsigned __int128)cw2 * (unsigned)best.c;
  const unsigned __int128 rhs = (unsigned __int128)bw2 * (unsigned)c.c;
  if (lhs != rhs) return lhs > rhs;
  if (!best_h) {
    best.h = hem_hash(seed, v, best.u);
    best_h = true;
  }
  c.h = hem_hash(seed, v, c.u);
  c_h = true;
  if (c.h != best.h) return c.h > best.h;
  return c.slot < best.slot;
}

__global__ void k_hem_elig(int n, const int* __restrict__ partner, const int* __restrict__ vw,
                           int* __restrict__ elig, const long long* gate, int* huge_cnt) {
  if (huge_cnt && blockIdx.x == 0 && threadIdx.x == 0) *huge_cnt = 0;
  if (hem_gated(gate, n)) return;
  for (int v = blockIdx.x * blockDim.x + threadIdx.x; v < n; v += gridDim.x * blockDim.x)
    elig[v] = partner[v] < 0 ? vw[v] : -1;
}

__global__ void __launch_bounds__(256) k_hem_pref_tpv(int n, const int* __restrict__ off,
                                                      const int* __restrict__ tgt,
                                                      const int* __restrict__ w,
                                                      const int* __restrict__ elig,
                                                      unsigned long long seed,
                                                      double l_max, int* __restrict__ pref,
                                                      const long long* gate,
                                                      int* __restrict__ huge,
                                                      int* __restrict__ huge_cnt) {
  if (hem_gated(gate, n)) return;
  const int lane = lane_id();
  const long long T = (long long)gridDim.x * blockDim.x;
  for (long long b0 = (long long)blockIdx.x * blockDim.x + threadIdx.x - lane; b0 < n; b0 += T) {
    const int v = (int)(b0 + lane);
    const bool inr = v < n;
    const int cvv = inr ? elig[v] : -1;
    const bool active = cvv >= 0;  // unmatched
    int e0 = 0, e1 = 0;
    if (active) {
      e0 = off[v];
      e1 = off[v + 1];
    }
    // hub rows: one CTA each in k_hem_pref_huge
    const bool hugerow = active && e1 - e0 > kHemHuge;
    if (hugerow) huge[atomicAdd(huge_cnt, 1)] = v;
    const bool longrow = active && e1 - e0 > kHemTpv && !hugerow;
    HemCand best;
    best.u = -1;
    best.w = best.c = best.slot = 0;
    best.h = 0;
    bool best_h = false;
    if (active && !longrow) {
      const long long cv = cvv;
      for (int e = e0; e < e1; e += 4) {
        int tg[4], wg[4], cg[4];
#pragma unroll
        for (int q = 0; q < 4; ++q)
          if (e + q < e1) {
            tg[q] = tgt[e + q];
            wg[q] = w[e + q];
          }
#pragma unroll
        for (int q = 0; q < 4; ++q)
          if (e + q < e1) cg[q] = elig[tg[q]];
#pragma unroll
        for (int q = 0; q < 4; ++q) {
          if (e + q >= e1) break;
          const int cu = cg[q];
          if (cu < 0 || (double)(cv + cu) > l_max) continue;
          HemCand c;
          c.w = wg[q];
          c.c = cu;
          c.slot = e + q;
          c.u = tg[q];
          c.h = 0;
          bool c_h;
          if (hem_better_lazy(c, c_h, best, best_h, seed, v)) {
            best = c;
            best_h = c_h;
          }
        }
      }
    }
    // long rows: the warp evaluates them one by one
    unsigned lm = __ballot_sync(0xffffffffu, longrow);
    while (lm) {
      const int l = __ffs(lm) - 1;
      lm &= lm - 1;
      const int x = __shfl_sync(0xffffffffu, v, l);
      const int xb = __shfl_sync(0xffffffffu, e0, l), xe = __shfl_sync(0xffffffffu, e1, l);
      const long long cx = __shfl_sync(0xffffffffu, cvv, l);
      HemCand bx;
      bx.u = -1;
      bx.w = bx.c = bx.slot = 0;
      bx.h = 0;
      for (int e = xb + lane; e < xe; e += 32) {
        const int u = tgt[e];
        const int cu = elig[u];
        if (cu < 0 || (double)(cx + cu) > l_max) continue;
        HemCand c;
        c.w = w[e];
        c.c = cu;
        c.slot = e;
        c.u = u;
        c.h = hem_hash(seed, x, u);
        if (hem_better(c, bx)) bx = c;
      }
#pragma unroll
      for (int o = 16; o > 0; o >>= 1) {
        HemCand y = hem_shfl(bx, o);
        if (hem_better(y, bx)) bx = y;
      }
      if (lane == l) best = bx;
    }
    if (inr && !hugerow) pref[v] = active ? best.u : -1;
  }
}

// hub rows (> kHemHuge slots, R-MAT): one CTA per row, strided slots, warp
// shuffle argmax then across the CTA's warps
__global__ void __launch_bounds__(256) k_hem_pref_huge(const int* __restrict__ off,
                                                       const int* __restrict__ tgt,
                                                       const int* __restrict__ w,
                                                       const int* __restrict__ elig,
                                                       unsigned long long seed, double l_max,
                                                       int* __restrict__ pref,
                                                       const long long* gate, int n,
                                                       const int* __restrict__ huge,
                                                       const int* __restrict__ huge_cnt) {
  if (hem_gated(gate, n)) return;
  __shared__ HemCand sb[8];
  const int cnt = *huge_cnt;
  for (int h = blockIdx.x; h < cnt; h += gridDim.x) {
    const int x = huge[h];
    const long long cx = elig[x];
    HemCand bx;
    bx.u = -1;
    bx.w = bx.c = bx.slot = 0;
    bx.h = 0;
    for (int e = off[x] + threadIdx.x; e < off[x + 1]; e += blockDim.x) {
      const int u = tgt[e];
      const int cu = elig[u];
      if (cu < 0 || (double)(cx + cu) > l_max) continue;
      HemCand c;
      c.w = w[e];
      c.c = cu;
      c.slot = e;
      c.u = u;
      c.h = hem_hash(seed, x, u);
      if (hem_better(c, bx)) bx = c;
    }
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) {
      HemCand y = hem_shfl(bx, o);
      if (hem_better(y, bx)) bx = y;
    }
    if (lane_id() == 0) sb[threadIdx.x >> 5] = bx;
    __syncthreads();
    if (threadIdx.x == 0) {
      HemCand b = sb[0];
      for (int i = 1; i < (int)(blockDim.x >> 5); ++i)
        if (hem_better(sb[i], b)) b = sb[i];
      pref[x] = b.u;
    }
    __syncthreads();
  }
}

static int pick_vw(long long m2, int n) {
  double avg = n ? (double)m2 / n : 0.0;
  if (avg <= 3.0) return 4;
  if (avg <= 7.0) return 8;
  if (avg <= 20.0) return 16;
  return 32;
}

void hem_round(const DevGraph& g, int* partner, int* pref, double l_max,
               unsigned long long seed, long long* matched, cudaStream_t s,
               const long long* gate) {
  if (g.n == 0) return;
  // 16 B per vertex, 16 B per slot
  ProfScope prof(P_HEM, 16.0 * g.n + 16.0 * g.m2, s);
  constexpr int B = 256;
  DBuf<int> ev((size_t)g.n, s);
  // a row can exceed kHemHuge (row-length bound known for uploaded and
  // matching-contracted levels; otherwise only the total bounds it)
  const bool hubs = g.maxdeg >= 0 ? g.maxdeg > kHemHuge : g.m2 > (long long)kHemHuge;
  DBuf<int> huge(hubs ? (size_t)g.n + 1 : 1, s);
  int* hcnt = hubs ? huge.get() + g.n : nullptr;
  k_hem_elig<<<grid_for(g.n, B, kSMs * 8), B, 0, s>>>(g.n, partner, g.vw, ev.get(), gate, hcnt);
  k_hem_pref_tpv<<<grid_for(g.n, B, kSMs * 16), B, 0, s>>>(g.n, g.off, g.tgt, g.w, ev.get(), seed,
                                                           l_max, pref, gate, huge.get(), hcnt);
  if (hubs) {
    k_hem_pref_huge<<<kSMs, B, 0, s>>>(g.off, g.tgt, g.w, ev.get(), seed, l_max, pref, gate, g.n,
                                       huge.get(), hcnt);
    count_launch();
  }
  k_hem_mutual<B><<<grid_for(g.n, B, kSMs * 8), B, 0, s>>>(g.n, pref, partner, matched, gate);
  GIM_LAUNCH_CHECK();
  count_launch(3);
}



// ---------------------------------------------------------------------------
// K5 two-hop matching (coarsening.py:98-161).  Leaves and twins form
// disjoint groups: group members are compacted in vertex order, stably
// sorted by group key, and each group runs the sequential `_pair_up`
// automaton on one thread.  Relatives have overlapping groups visited in
// matchmaker order, so they run as one sequential device thread.

__device__ void pair_up_seq(const int* grp, int len, int* partner, const int* vw, double l_max,
                            long long* cnt) {
  int i = 0;
  while (i + 1 < len) {
    int a = grp[i], b = grp[i + 1];
    if (partner[a] >= 0) { ++i; continue; }
    if (partner[b] >= 0 || (double)((long long)vw[a] + vw[b]) > l_max) { ++i; continue; }
    partner[a] = b;
    partner[b] = a;
    *cnt += 2;
    i += 2;
  }
}

struct LeafFlag {
  const int* off;
  const int* partner;
  __device__ int operator()(long long v) const {
    return (off[v + 1] - off[v] == 1 && partner[v] < 0) ? 1 : 0;
  }
};
struct TwinFlag {
  const int* off;
  const int* partner;
  __device__ int operator()(long long v) const {
    return (off[v + 1] - off[v] >= 1 && partner[v] < 0) ? 1 : 0;
  }
};
template <class Flag>
struct CompactOut {
  Flag f;
  int* out;
  __device__ void operator()(long long v, int pos) const {
    if (f(v)) out[pos] = (int)v;
  }
};

// group key per compacted member: leaves -> the single neighbour;
// twins -> order-independent 64-bit hash of the neighbourhood (+ degree)
__global__ void k_leaf_keys(int cnt, const int* __restrict__ mem, const int* __restrict__ off,
                            const int* __restrict__ tgt, unsigned long long* keys, int* vals) {
  for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < cnt; i += gridDim.x * blockDim.x) {
    int v = mem[i];
    keys[i] = (unsigned long long)tgt[off[v]];
    vals[i] = v;
  }
}

__global__ void k_twin_keys(int cnt, const int* __restrict__ mem, const int* __restrict__ off,
                            const int* __restrict__ tgt, unsigned long long* keys, int* vals) {
  for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < cnt; i += gridDim.x * blockDim.x) {
    int v = mem[i];
    unsigned long long h1 = 0, h2 = 0;
    for (int e = off[v]; e < off[v + 1]; ++e) {
      unsigned long long x = splitmix64((unsigned long long)tgt[e]);
      h1 += x;
      h2 ^= splitmix64(x ^ 0x5851F42D4C957F2Dull);
    }
    keys[i] = splitmix64(h1 ^ (h2 * 0x9E3779B97F4A7C15ull) ^ (unsigned long long)(off[v + 1] - off[v]));
    vals[i] = v;
  }
}

__device__ bool same_neighbourhood(int a, int b, const int* off, const int* tgt) {
  int da = off[a + 1] - off[a], db = off[b + 1] - off[b];
  if (da != db) return false;
  for (int e = off[a]; e < off[a + 1]; ++e) {
    int x = tgt[e];
    bool found = false;
    for (int f = off[b]; f < off[b + 1]; ++f)
      if (tgt[f] == x) { found = true; break; }
    if (!found) return false;
  }
  return true;
}

// one thread per group start (head of a run of equal keys)
__global__ void k_pair_groups(int cnt, const unsigned long long* __restrict__ keys,
                              const int* __restrict__ mem, int* partner, const int* vw,
                              double l_max, int verify_twins, const int* off, const int* tgt,
                              long long* matched, int* collision) {
  long long local = 0;
  for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < cnt; i += gridDim.x * blockDim.x) {
    if (i > 0 && keys[i] == keys[i - 1]) continue;
    int j = i + 1;
    while (j < cnt && keys[j] == keys[i]) ++j;
    if (verify_twins)
      for (int q = i + 1; q < j; ++q)
        if (!same_neighbourhood(mem[i], mem[q], off, tgt)) atomicExch(collision, 1);
    pair_up_seq(mem + i, j - i, partner, vw, l_max, &local);
  }
  if (local) atomicAdd(reinterpret_cast<unsigned long long*>(matched), (unsigned long long)local);
}

// relatives (coarsening.py:148-158): sequential over matchmakers with degree
// <= 8; each sorts its currently unmatched neighbours and pairs them up
__global__ void k_relatives(int n, const int* __restrict__ off, const int* __restrict__ tgt,
                            int* partner, const int* vw, double l_max, long long* matched,
                            int* progressed) {
  if (blockIdx.x != 0 || threadIdx.x != 0) return;
  long long local = 0;
  int prog = 0;
  int grp[8];
  for (int mm = 0; mm < n; ++mm) {
    int d = off[mm + 1] - off[mm];
    if (d > 8) continue;
    int len = 0;
    for (int e = off[mm]; e < off[mm + 1]; ++e) {
      int u = tgt[e];
      if (partner[u] < 0) {
        int p = len++;
        while (p > 0 && grp[p - 1] > u) { grp[p] = grp[p - 1]; --p; }  // insertion sort
        grp[p] = u;
      }
    }
    long long before = local;
    pair_up_seq(grp, len, partner, vw, l_max, &local);
    if (local > before) prog = 1;
  }
  *matched += local;
  *progressed = prog;
}

// relatives in parallel, with the sequential result.  Matchmaker mm only
// reads and writes the partner state of its currently unmatched neighbours,
// so two matchmakers interact only through a shared unmatched neighbour.
// Rounds: every live matchmaker (degree <= 8, >= 2 unmatched neighbours)
// stamps its unmatched neighbours with atomicMin((round tag) | mm); a
// matchmaker is ready when it owns all of them — no earlier pending
// matchmaker can change its group, and the ready ones touch disjoint
// vertex sets — and runs its pair-up; the rest retry next round.  The
// lowest pending matchmaker is always ready.  A matchmaker seeing fewer
// than two unmatched neighbours is dropped: the set only shrinks, so at its
// sequential turn it would pair nothing either.  The tag decreases per
// round, so stale stamps never need clearing (owner >= key <=> not claimed
// by an earlier matchmaker this round).  One cooperative launch, two grid
// barriers per round; state written by other CTAs is read through L2.
__device__ __forceinline__ int rel_unmatched(const int* off, const int* tgt, const int* partner,
                                             int mm, int* grp) {
  int len = 0;
  for (int e = off[mm]; e < off[mm + 1]; ++e) {
    const int u = tgt[e];
    if (__ldcg(partner + u) < 0) {
      if (grp) {
        int p = len;
        while (p > 0 && grp[p - 1] > u) { grp[p] = grp[p - 1]; --p; }  // insertion sort
        grp[p] = u;
      }
      ++len;
    }
  }
  return len;
}

__global__ void __launch_bounds__(256) k_relatives_par(int n, const int* __restrict__ off,
                                                       const int* __restrict__ tgt, int* partner,
                                                       const int* __restrict__ vw, double l_max,
                                                       long long* matched, int* progressed,
                                                       int* la, int* lb,
                                                       unsigned long long* owner, int* ctr) {
  cg::grid_group grid = cg::this_grid();
  const long long gt = (long long)blockIdx.x * blockDim.x + threadIdx.x;
  const long long GT = (long long)gridDim.x * blockDim.x;
  for (long long v = gt; v < n; v += GT) {
    const int d = off[v + 1] - off[v];
    if (d < 2 || d > 8) continue;
    if (rel_unmatched(off, tgt, partner, (int)v, nullptr) >= 2) la[atomicAdd(&ctr[0], 1)] = (int)v;
  }
  grid.sync();
  long long local = 0;
  int* cur = la;
  int* nxt = lb;
  for (int r = 0;; ++r) {
    const int cnt = __ldcg(ctr + (r & 1));
    if (cnt == 0) break;
    const unsigned long long tag = (unsigned long long)(0x7fffffff - r) << 32;
    for (long long i = gt; i < cnt; i += GT) {
      const int mm = cur[i];
      if (rel_unmatched(off, tgt, partner, mm, nullptr) < 2) {
        cur[i] = -1;
        continue;
      }
      for (int e = off[mm]; e < off[mm + 1]; ++e) {
        const int u = tgt[e];
        if (__ldcg(partner + u) < 0) atomicMin(owner + u, tag | (unsigned)mm);
      }
    }
    if (gt == 0) ctr[(r + 1) & 1] = 0;  // last read in the previous round
    grid.sync();
    for (long long i = gt; i < cnt; i += GT) {
      const int mm = cur[i];
      if (mm < 0) continue;
      const unsigned long long key = tag | (unsigned)mm;
      bool ready = true;
      for (int e = off[mm]; e < off[mm + 1]; ++e) ready &= __ldcg(owner + tgt[e]) >= key;
      if (!ready) {
        nxt[atomicAdd(&ctr[(r + 1) & 1], 1)] = mm;
        continue;
      }
      int grp[8];
      const int len = rel_unmatched(off, tgt, partner, mm, grp);
      int i2 = 0;
      while (i2 + 1 < len) {  // _pair_up (coarsening.py:98-110)
        const int a = grp[i2], b = grp[i2 + 1];
        if (__ldcg(partner + a) >= 0) { ++i2; continue; }
        if (__ldcg(partner + b) >= 0 || (double)((long long)vw[a] + vw[b]) > l_max) { ++i2; continue; }
        __stcg(partner + a, b);
        __stcg(partner + b, a);
        local += 2;
        i2 += 2;
      }
    }
    grid.sync();
    int* t = cur;
    cur = nxt;
    nxt = t;
  }
  local = warp_sum_ll(local);
  if (lane_id() == 0 && local) {
    atomicAdd(reinterpret_cast<unsigned long long*>(matched), (unsigned long long)local);
    atomicExch(progressed, 1);
  }
}

static void relatives_parallel(const DevGraph& g, int* partner, double l_max, long long* matched_d,
                               int* progressed, cudaStream_t s) {
  static int occ = 0;
  static std::once_flag once;
  std::call_once(once, [] {
    GIM_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, k_relatives_par, 256, 0));
  });
  const int G = std::max(1, std::min(device_sms() * coop_blocks_per_sm(occ), (int)((g.n + 255) / 256)));
  DBuf<int> la((size_t)std::max(g.n, 1), s), lb((size_t)std::max(g.n, 1), s), ctr(2, s);
  DBuf<unsigned long long> owner((size_t)std::max(g.n, 1), s);
  GIM_CUDA(cudaMemsetAsync(ctr.get(), 0, 2 * sizeof(int), s));
  GIM_CUDA(cudaMemsetAsync(owner.get(), 0xff, sizeof(unsigned long long) * (size_t)g.n, s));
  GIM_CUDA(cudaMemsetAsync(progressed, 0, sizeof(int), s));
  int n = g.n;
  const int* off = g.off;
  const int* tgt = g.tgt;
  const int* vwp = g.vw;
  int* pa = la.get();
  int* pb = lb.get();
  unsigned long long* ow = owner.get();
  int* ct = ctr.get();
  void* args[] = {&n, &off, &tgt, &partner, &vwp, &l_max, &matched_d, &progressed,
                  &pa, &pb, &ow, &ct};
  GIM_CUDA(cudaLaunchCooperativeKernel((const void*)k_relatives_par, dim3(G), dim3(256), args, 0, s));
  count_launch();
  GIM_LAUNCH_CHECK();
}

// sort-and-pair one two-hop phase; returns after the pairing kernel
static void two_hop_phase(const DevGraph& g, int* partner, double l_max, long long* matched,
                          bool twins, int* collision, cudaStream_t s) {
  DBuf<int> cnt_d(1, s);
  DBuf<int> mem((size_t)g.n, s);
  if (twins) {
    TwinFlag f{g.off, partner};
    exclusive_scan<int>(g.n, f, CompactOut<TwinFlag>{f, mem.get()}, cnt_d.get(), s);
  } else {
    LeafFlag f{g.off, partner};
    exclusive_scan<int>(g.n, f, CompactOut<LeafFlag>{f, mem.get()}, cnt_d.get(), s);
  }
  int cnt = 0;
  GIM_CUDA(cudaMemcpyAsync(&cnt, cnt_d.get(), sizeof(int), cudaMemcpyDeviceToHost, s));
  GIM_CUDA(sync_stream(s));
  if (cnt < 2) return;
  DBuf<unsigned long long> keys(cnt, s), keys2(cnt, s);
  DBuf<int> vals(cnt, s), vals2(cnt, s);
  int grid = grid_for(cnt, 256);
  if (twins)
    k_twin_keys<<<grid, 256, 0, s>>>(cnt, mem.get(), g.off, g.tgt, keys.get(), vals.get());
  else
    k_leaf_keys<<<grid, 256, 0, s>>>(cnt, mem.get(), g.off, g.tgt, keys.get(), vals.get());
  count_launch();
  GIM_LAUNCH_CHECK();
  radix_sort_pairs<unsigned long long, int>(cnt, keys.get(), vals.get(), keys2.get(),
                                            vals2.get(), twins ? 64 : bit_length(g.n), s);
  k_pair_groups<<<grid, 256, 0, s>>>(cnt, keys.get(), vals.get(), partner, g.vw, l_max,
                                     twins ? 1 : 0, g.off, g.tgt, matched, collision);
  count_launch();
  GIM_LAUNCH_CHECK();
}

// GIM_RELATIVES_SEQ=1: the single-thread sequential relatives (tests)
static bool relatives_seq() {
  const char* e = getenv("GIM_RELATIVES_SEQ");
  return e && atoi(e) != 0;
}

// returns the matched count after two-hop (coarsening.py:113-161)
long long two_hop(const DevGraph& g, int* partner, double l_max, long long matched_now,
                  long long* matched_d, cudaStream_t s) {
  const double target = 0.40;
  auto frac = [&](long long m) { return g.n ? (double)m / (double)g.n : 1.0; };
  DBuf<int> flags(2, s);  // [collision, progressed]
  GIM_CUDA(cudaMemsetAsync(flags.get(), 0, 2 * sizeof(int), s));
  auto read = [&]() {
    long long m = 0;
    GIM_CUDA(cudaMemcpyAsync(&m, matched_d, sizeof(long long), cudaMemcpyDeviceToHost, s));
    GIM_CUDA(sync_stream(s));
    return m;
  };
  GIM_CUDA(cudaMemcpyAsync(matched_d, &matched_now, sizeof(long long), cudaMemcpyHostToDevice, s));
  long long m = matched_now;
  ProfScope prof(P_TWO_HOP, 0.0, s);
  for (int rep = 0; rep < 3; ++rep) {
    if (frac(m) >= target) return m;
    two_hop_phase(g, partner, l_max, matched_d, false, flags.get(), s);
    m = read();
    if (frac(m) >= target) return m;
    two_hop_phase(g, partner, l_max, matched_d, true, flags.get(), s);
    m = read();
    int coll = 0;
    GIM_CUDA(cudaMemcpy(&coll, flags.get(), sizeof(int), cudaMemcpyDeviceToHost));
    GIM_CHECK(coll == 0, GIM_E_INTERNAL, "two-hop twin hash collision (non-identical "
                                         "neighbourhoods share a 64-bit key)");
    if (frac(m) >= target) return m;
    if (relatives_seq()) {
      k_relatives<<<1, 1, 0, s>>>(g.n, g.off, g.tgt, partner, g.vw, l_max, matched_d,
                                  flags.get() + 1);
      count_launch();
      GIM_LAUNCH_CHECK();
    } else {
      relatives_parallel(g, partner, l_max, matched_d, flags.get() + 1, s);
    }
    m = read();
    int prog = 0;
    GIM_CUDA(cudaMemcpy(&prog, flags.get() + 1, sizeof(int), cudaMemcpyDeviceToHost));
    if (!prog) return m;
  }
  return m;
}

// ---------------------------------------------------------------------------
// coarse ids (coarsening.py:176-188): root = min(v, partner); ids by an
// exclusive scan over is_root in vertex order

struct IsRoot {
  const int* partner;
  __device__ int operator()(long long v) const {
    int p = partner[v];
    return (p < 0 || v < p) ? 1 : 0;
  }
};

__global__ void k_coarse_map(int n, const int* __restrict__ partner, const int* __restrict__ ids,
                             int* __restrict__ cmap) {
  for (int v = blockIdx.x * blockDim.x + threadIdx.x; v < n; v += gridDim.x * blockDim.x) {
    int p = partner[v];
    cmap[v] = (p >= 0 && p < v) ? ids[p] : ids[v];
  }
}

int coarse_map(int n, const int* partner, int* cmap, cudaStream_t s) {
  if (n == 0) return 0;
  DBuf<int> ids((size_t)n, s), tot(1, s);
  exclusive_scan<int>(n, IsRoot{partner}, StoreTo<int>{ids.get()}, tot.get(), s);
  k_coarse_map<<<grid_for(n, 256), 256, 0, s>>>(n, partner, ids.get(), cmap);
  count_launch();
  GIM_LAUNCH_CHECK();
  int n_c = 0;
  GIM_CUDA(cudaMemcpyAsync(&n_c, tot.get(), sizeof(int), cudaMemcpyDeviceToHost, s));
  GIM_CUDA(sync_stream(s));
  return n_c;
}

// ---------------------------------------------------------------------------
// K6 contraction (coarsening.py:191-249): key (cu, cv) = cu * n_c + cv per
// fine slot, self loops keyed past the end, radix sort, segmented sum of
// equal keys -> coarse CSR sorted by (source, target).

template <int BLOCK>
__global__ void __launch_bounds__(BLOCK) k_contract_keys(long long m2, const int* __restrict__ src,
                                                         const int* __restrict__ tgt,
                                                         const int* __restrict__ w,
                                                         const int* __restrict__ cmap, int n_c,
                                                         unsigned long long* __restrict__ keys,
                                                         int* __restrict__ vals,
                                                         long long* __restrict__ selfloops) {
  const unsigned long long sent = (unsigned long long)n_c * (unsigned long long)n_c;
  long long cnt = 0;
  for (long long e = (long long)blockIdx.x * BLOCK + threadIdx.x; e < m2;
       e += (long long)gridDim.x * BLOCK) {
    int cu = cmap[src[e]], cv = cmap[tgt[e]];
    if (cu == cv) {
      keys[e] = sent;
      ++cnt;
    } else {
      keys[e] = (unsigned long long)cu * (unsigned long long)n_c + (unsigned long long)cv;
    }
    vals[e] = w[e];
  }
  block_sum_atomic<BLOCK>(cnt, selfloops);
}

struct KeyHead {
  const unsigned long long* keys;
  __device__ int operator()(long long i) const { return (i == 0 || keys[i] != keys[i - 1]) ? 1 : 0; }
};

struct KeyHeadOut {
  const unsigned long long* keys;
  const int* vals;
  long long valid;
  int n_c;
  int* ctgt;
  int* cw;
  int* csrc;
  int* deg;
  __device__ void operator()(long long i, int uid) const {
    if (i > 0 && keys[i] == keys[i - 1]) return;
    long long sum = 0;
    long long j = i;
    while (j < valid && keys[j] == keys[i]) sum += vals[j++];
    unsigned long long k = keys[i];
    int cu = (int)(k / (unsigned long long)n_c);
    ctgt[uid] = (int)(k % (unsigned long long)n_c);
    cw[uid] = (int)sum;
    csrc[uid] = cu;
    atomicAdd(&deg[cu], 1);
  }
};

__global__ void k_coarse_vw(int n, const int* __restrict__ cmap, const int* __restrict__ vw,
                            int* __restrict__ cvw) {
  for (int v = blockIdx.x * blockDim.x + threadIdx.x; v < n; v += gridDim.x * blockDim.x)
    atomicAdd(&cvw[cmap[v]], vw[v]);
}

// returns m2 of the coarse graph; out arrays must hold >= g.m2 slots
long long contract_into(const DevGraph& g, const int* cmap, int n_c, int* c_off, int* c_tgt,
                        int* c_w, int* c_vw, int* c_src, cudaStream_t s) {
  ProfScope prof(P_CONTRACT, 12.0 * g.n + 12.0 * g.m2 + 8.0 * n_c, s);
  GIM_CUDA(cudaMemsetAsync(c_vw, 0, sizeof(int) * (size_t)n_c, s));
  if (n_c > 0) {
    k_coarse_vw<<<grid_for(g.n, 256), 256, 0, s>>>(g.n, cmap, g.vw, c_vw);
    count_launch();
  }
  if (g.m2 == 0) {
    GIM_CUDA(cudaMemsetAsync(c_off, 0, sizeof(int) * ((size_t)n_c + 1), s));
    return 0;
  }
  DBuf<unsigned long long> keys((size_t)g.m2, s), keys2((size_t)g.m2, s);
  DBuf<int> vals((size_t)g.m2, s), vals2((size_t)g.m2, s);
  DBuf<long long> selfl(1, s);
  GIM_CUDA(cudaMemsetAsync(selfl.get(), 0, sizeof(long long), s));
  constexpr int B = 256;
  k_contract_keys<B><<<grid_for(g.m2, B, kSMs * 8), B, 0, s>>>(
      g.m2, g.src, g.tgt, g.w, cmap, n_c, keys.get(), vals.get(), selfl.get());
  count_launch();
  GIM_LAUNCH_CHECK();
  int bits = bit_length((unsigned long long)n_c * (unsigned long long)n_c);
  radix_sort_pairs<unsigned long long, int>(g.m2, keys.get(), vals.get(), keys2.get(),
                                            vals2.get(), bits, s);
  long long self = 0;
  GIM_CUDA(cudaMemcpyAsync(&self, selfl.get(), sizeof(long long), cudaMemcpyDeviceToHost, s));
  GIM_CUDA(sync_stream(s));
  long long valid = g.m2 - self;
  DBuf<int> deg((size_t)n_c + 1, s), m2c_d(1, s);
  GIM_CUDA(cudaMemsetAsync(deg.get(), 0, sizeof(int) * ((size_t)n_c + 1), s));
  KeyHeadOut out{keys.get(), vals.get(), valid, n_c, c_tgt, c_w, c_src, deg.get()};
  exclusive_scan<int>(valid, KeyHead{keys.get()}, out, m2c_d.get(), s);
  exclusive_scan<int>((long long)n_c + 1, LoadAs<int, int>{deg.get()}, StoreTo<int>{c_off},
                      (int*)nullptr, s);
  int m2c = 0;
  GIM_CUDA(cudaMemcpyAsync(&m2c, m2c_d.get(), sizeof(int), cudaMemcpyDeviceToHost, s));
  GIM_CUDA(sync_stream(s));
  prof.extra = 8.0 * m2c;
  return m2c;
}

void contract(const DevGraph& g, const int* cmap, int n_c, OwnedGraph& out, cudaStream_t s) {
  DBuf<int> t((size_t)std::max<long long>(g.m2, 1), s), w((size_t)std::max<long long>(g.m2, 1), s),
      sr((size_t)std::max<long long>(g.m2, 1), s);
  out.n = n_c;
  out.maxdeg = -1;  // unknown (radix path)
  out.off = DBuf<int>((size_t)n_c + 1, s);
  out.vw = DBuf<int>((size_t)std::max(n_c, 1), s);
  long long m2c = contract_into(g, cmap, n_c, out.off.get(), t.get(), w.get(), out.vw.get(),
                                sr.get(), s);
  out.m2 = m2c;
  out.tgt = DBuf<int>((size_t)std::max<long long>(m2c, 1), s);
  out.w = DBuf<int>((size_t)std::max<long long>(m2c, 1), s);
  out.src = DBuf<int>((size_t)std::max<long long>(m2c, 1), s);
  if (m2c) {
    GIM_CUDA(cudaMemcpyAsync(out.tgt.get(), t.get(), sizeof(int) * m2c, cudaMemcpyDeviceToDevice, s));
    GIM_CUDA(cudaMemcpyAsync(out.w.get(), w.get(), sizeof(int) * m2c, cudaMemcpyDeviceToDevice, s));
    GIM_CUDA(cudaMemcpyAsync(out.src.get(), sr.get(), sizeof(int) * m2c, cudaMemcpyDeviceToDevice, s));
  }
}

// ---------------------------------------------------------------------------
// K6' contraction of a MATCHING (the level-stack case): every coarse vertex c
// has one or two members, so its row is the union of <= 2 fine rows mapped
// through M.  One warp per coarse vertex stages those L = deg(v1) + deg(v2)
// (cv, w) pairs in shared memory, drops the self loop cv == c, and
// deduplicates / ranks them in O(L^2 / 32): the output row is sorted by
// target and parallel edges are summed — the same labelled graph as the
// sort path, with two row sweeps instead of six radix passes.  Rows longer
// than kRowCap (hubs, R-MAT) route the whole level to the radix-sort path.

constexpr int kRowCap = 256;
constexpr int kRowWarps = 8;

// member table: per coarse vertex c the rows of its <= 2 fine members as
// (begin0, len0, begin1, len1) — one 16-byte load in the row kernels, which
// then start from the slots without a dependent offsets gather
__global__ void k_members(int n, const int* __restrict__ partner, const int* __restrict__ cmap,
                          const int* __restrict__ off, const int* __restrict__ vw,
                          int4* __restrict__ mem, int* __restrict__ rowlen, int* __restrict__ cvw,
                          int* __restrict__ maxlen) {
  int mx = 0;
  for (int v = blockIdx.x * blockDim.x + threadIdx.x; v < n; v += gridDim.x * blockDim.x) {
    const int p = partner[v];
    if (p >= 0 && p < v) continue;  // not the root of its pair
    const int c = cmap[v];
    const int b0 = off[v], d0 = off[v + 1] - b0;
    int b1 = 0, d1 = 0, wsum = vw[v];
    if (p >= 0) {
      b1 = off[p];
      d1 = off[p + 1] - b1;
      wsum += vw[p];
    }
    mem[c] = make_int4(b0, d0, b1, d1);
    rowlen[c] = d0 + d1;
    cvw[c] = wsum;
    mx = max(mx, d0 + d1);
  }
  mx = __reduce_max_sync(0xffffffffu, mx);
  if (lane_id() == 0 && mx) atomicMax(maxlen, mx);
}

// stage the row of coarse vertex c in K/Wt (self loops -> INT_MAX)
__device__ __forceinline__ int stage_row(int c, const int4* mem, const int* tgt, const int* w,
                                         const int* cmap, int* K, int* Wt) {
  const int4 m = mem[c];
  const int L = m.y + m.w;
  for (int i = lane_id(); i < L; i += 32) {
    const int e = i < m.y ? m.x + i : m.z + (i - m.y);
    const int key = cmap[tgt[e]];
    K[i] = key == c ? INT_MAX : key;
    Wt[i] = w[e];
  }
  __syncwarp();
  return L;
}

// Warp-per-coarse-vertex contraction (rows of L <= kCtTpv = 32 staged
// entries): lane i stages entry i of the <= 2 member rows (coalesced target /
// weight loads straight from the member table's row ranges, then the M
// gather), self loops drop out, __match_any_sync groups equal coarse
// targets, __reduce_add_sync sums their weights (parallel edges) and each
// group's lowest lane writes the entry at its rank among the group leaders —
// the deduplicated row in first-occurrence order, at its upper-bound offset
// (compacted afterwards).  Within-row order is irrelevant to every consumer
// (the pipeline is invariant to it; the ABI's gim_contract keeps
// sorted rows).  No shared memory, ~20 instructions per row.  Longer rows go
// through the shared-memory warp path (k_row_long) into the same buffers.
constexpr int kCtTpv = 32;
constexpr int kCtBlock = 256;

// one row's staged entry for this lane (key -1: none / self loop)
__device__ __forceinline__ void row_entry(const int4 m, int c, int lane, const int* __restrict__ tgt,
                                          const int* __restrict__ w, int& t, int& wt) {
  t = -1;
  wt = 0;
  if (lane < m.y + m.w) {
    const int e = lane < m.y ? m.x + lane : m.z + (lane - m.y);
    t = tgt[e];
    wt = w[e];
  }
}

__device__ __forceinline__ void row_emit(int c, int key, int wt, int lane, const int* __restrict__ ub,
                                         int* __restrict__ t_tgt, int* __restrict__ t_w,
                                         int* __restrict__ cdeg) {
  const unsigned peers = __match_any_sync(0xffffffffu, key);
  const int sum = (int)__reduce_add_sync(peers, (unsigned)wt);
  const bool lead = key >= 0 && lane == __ffs(peers) - 1;
  const unsigned leads = __ballot_sync(0xffffffffu, lead);
  if (lead) {
    const int pos = ub[c] + __popc(leads & ((1u << lane) - 1u));
    t_tgt[pos] = key;
    t_w[pos] = sum;
  }
  if (lane == 0) cdeg[c] = __popc(leads);
}

// two rows per warp per step: both rows' loads are in flight together (the
// kernel is bound by the dependent member -> slots -> M chain per row)
__global__ void __launch_bounds__(kCtBlock) k_row_warp(int n_c, const int4* __restrict__ mem,
                                                       const int* __restrict__ ub,
                                                       const int* __restrict__ tgt,
                                                       const int* __restrict__ w,
                                                       const int* __restrict__ cmap,
                                                       int* __restrict__ t_tgt,
                                                       int* __restrict__ t_w,
                                                       int* __restrict__ cdeg) {
  const int lane = lane_id();
  const long long nw = ((long long)gridDim.x * blockDim.x) >> 5;
  for (long long c0 = ((long long)blockIdx.x * blockDim.x + threadIdx.x) >> 5; c0 < n_c;
       c0 += 2 * nw) {
    const int ca = (int)c0;
    const long long cbl = c0 + nw;
    const int cb = cbl < n_c ? (int)cbl : -1;
    const int4 ma = mem[ca];
    const int4 mb = cb >= 0 ? mem[cb] : make_int4(0, 0, 0, 0);
    const bool la = ma.y + ma.w <= kCtTpv, lb = cb >= 0 && mb.y + mb.w <= kCtTpv;
    int ta = -1, wa = 0, tb = -1, wb = 0;
    if (la) row_entry(ma, ca, lane, tgt, w, ta, wa);
    if (lb) row_entry(mb, cb, lane, tgt, w, tb, wb);
    int ka = ta >= 0 ? cmap[ta] : -1;
    int kb = tb >= 0 ? cmap[tb] : -1;
    if (ka == ca) { ka = -1; wa = 0; }  // self loops
    if (kb == cb) { kb = -1; wb = 0; }
    if (la) row_emit(ca, ka, wa, lane, ub, t_tgt, t_w, cdeg);  // warp-uniform
    if (lb) row_emit(cb, kb, wb, lane, ub, t_tgt, t_w, cdeg);
  }
}

// long rows (kCtTpv < L <= kRowCap): warp per row, shared-memory staging
__global__ void __launch_bounds__(kRowWarps * 32) k_row_long(int n_c, const int4* __restrict__ mem,
                                                            const int* __restrict__ rowlen,
                                                            const int* __restrict__ ub,
                                                            const int* __restrict__ tgt,
                                                            const int* __restrict__ w,
                                                            const int* __restrict__ cmap,
                                                            int* __restrict__ t_tgt,
                                                            int* __restrict__ t_w,
                                                            int* __restrict__ cdeg) {
  __shared__ int sK[kRowWarps][kRowCap], sW[kRowWarps][kRowCap];
  __shared__ unsigned char sF[kRowWarps][kRowCap];
  const int warp = threadIdx.x >> 5, lane = lane_id();
  int* K = sK[warp];
  int* Wt = sW[warp];
  unsigned char* F = sF[warp];
  for (long long c0 = ((long long)blockIdx.x * blockDim.x + threadIdx.x) >> 5; c0 < n_c;
       c0 += ((long long)gridDim.x * blockDim.x) >> 5) {
    const int c = (int)c0;
    if (rowlen[c] <= kCtTpv) continue;  // warp-uniform
    const int L = stage_row(c, mem, tgt, w, cmap, K, Wt);
    int nf = 0;
    for (int i = lane; i < L; i += 32) {
      const int key = K[i];
      bool first = key != INT_MAX;
      for (int j = 0; j < i && first; ++j)
        if (K[j] == key) first = false;
      F[i] = first;
      nf += first;
    }
    nf = warp_sum_i(nf);
    __syncwarp();
    const int base = ub[c];
    for (int i = lane; i < L; i += 32) {
      if (!F[i]) continue;
      const int key = K[i];
      long long sum = 0;
      int rank = 0;
      for (int j = 0; j < L; ++j) {
        const int kj = K[j];
        if (kj == key) sum += Wt[j];
        rank += (F[j] && kj < key);
      }
      t_tgt[base + rank] = key;
      t_w[base + rank] = (int)sum;
    }
    if (lane == 0) cdeg[c] = nf;
    __syncwarp();
  }
}

// compaction: row c moves from its upper-bound slot to its final offset
__global__ void k_row_compact(int n_c, const int* __restrict__ ub, const int* __restrict__ c_off,
                              const int* __restrict__ t_tgt, const int* __restrict__ t_w,
                              int* __restrict__ c_tgt, int* __restrict__ c_w,
                              int* __restrict__ c_src) {
  const int lane = lane_id();
  // warp per 32 rows: each row copied by lanes in turn (coalesced per row)
  for (long long r0 = ((long long)blockIdx.x * blockDim.x + threadIdx.x) - lane; r0 < n_c;
       r0 += (long long)gridDim.x * blockDim.x) {
    const int myc = (int)(r0 + lane);
    int mb = 0, mo = 0, md = 0;
    if (myc < n_c) {
      mb = ub[myc];
      mo = c_off[myc];
      md = c_off[myc + 1] - mo;
    }
    for (int j = 0; j < 32; ++j) {
      const int b = __shfl_sync(0xffffffffu, mb, j), o = __shfl_sync(0xffffffffu, mo, j),
                d = __shfl_sync(0xffffffffu, md, j);
      for (int i = lane; i < d; i += 32) {
        c_tgt[o + i] = t_tgt[b + i];
        c_w[o + i] = t_w[b + i];
        c_src[o + i] = (int)r0 + j;
      }
    }
  }
}

// contraction of a matching (partner[] given); falls back to the radix-sort
// path when some coarse row exceeds kRowCap
void contract_matching(const DevGraph& g, const int* cmap, const int* partner, int n_c,
                       OwnedGraph& out, cudaStream_t s) {
  if (g.m2 == 0 || n_c == 0) {
    contract(g, cmap, n_c, out, s);
    return;
  }
  DBuf<int4> mem((size_t)std::max(n_c, 1), s);
  DBuf<int> rowlen((size_t)n_c + 1, s);
  DBuf<int> cdeg((size_t)n_c + 1, s), ub((size_t)n_c + 1, s), scal(3, s);  // maxlen, m2c, ub total
  DBuf<int> cvw((size_t)n_c, s);
  GIM_CUDA(cudaMemsetAsync(scal.get(), 0, 3 * sizeof(int), s));
  GIM_CUDA(cudaMemsetAsync(cdeg.get() + n_c, 0, sizeof(int), s));
  k_members<<<grid_for(g.n, 256), 256, 0, s>>>(g.n, partner, cmap, g.off, g.vw, mem.get(),
                                               rowlen.get(), cvw.get(), scal.get());
  count_launch();
  GIM_LAUNCH_CHECK();
  exclusive_scan<int>((long long)n_c, LoadAs<int, int>{rowlen.get()}, StoreTo<int>{ub.get()},
                      scal.get() + 2, s);
  int hs[3] = {0, 0, 0};
  int* hp = static_cast<int*>(pinned_scratch(sizeof(hs)));
  GIM_CUDA(cudaMemcpyAsync(hp, scal.get(), sizeof(hs), cudaMemcpyDeviceToHost, s));
  GIM_CUDA(sync_stream(s));
  std::copy(hp, hp + 3, hs);
  const int maxlen = hs[0], ubtot = hs[2];
  if (maxlen > kRowCap) {  // hub rows: radix-sort path for this level
    contract(g, cmap, n_c, out, s);
    return;
  }
  ProfScope prof(P_CONTRACT, 12.0 * g.n + 12.0 * g.m2 + 8.0 * n_c, s);
  out.n = n_c;
  out.maxdeg = maxlen;  // rows of the merged members: an upper bound
  out.vw = std::move(cvw);
  out.off = DBuf<int>((size_t)n_c + 1, s);
  DBuf<int> t_tgt((size_t)std::max(ubtot, 1), s), t_w((size_t)std::max(ubtot, 1), s);
  k_row_warp<<<grid_for((long long)n_c * 32, kCtBlock, kSMs * 32), kCtBlock, 0, s>>>(
      n_c, mem.get(), ub.get(), g.tgt, g.w, cmap, t_tgt.get(), t_w.get(), cdeg.get());
  count_launch();
  if (maxlen > kCtTpv) {
    const int grid = grid_for((long long)n_c * 32, kRowWarps * 32, kSMs * 8);
    k_row_long<<<grid, kRowWarps * 32, 0, s>>>(n_c, mem.get(), rowlen.get(), ub.get(),
                                               g.tgt, g.w, cmap, t_tgt.get(), t_w.get(),
                                               cdeg.get());
    count_launch();
  }
  GIM_LAUNCH_CHECK();
  exclusive_scan<int>((long long)n_c + 1, LoadAs<int, int>{cdeg.get()},
                      StoreTo<int>{out.off.get()}, scal.get() + 1, s);
  GIM_CUDA(cudaMemcpyAsync(hp, out.off.get() + n_c, sizeof(int), cudaMemcpyDeviceToHost, s));
  GIM_CUDA(sync_stream(s));
  const int m2c = hp[0];
  out.m2 = m2c;
  out.tgt = DBuf<int>((size_t)std::max(m2c, 1), s);
  out.w = DBuf<int>((size_t)std::max(m2c, 1), s);
  out.src = DBuf<int>((size_t)std::max(m2c, 1), s);
  k_row_compact<<<grid_for(n_c, 256, kSMs * 16), 256, 0, s>>>(
      n_c, ub.get(), out.off.get(), t_tgt.get(), t_w.get(), out.tgt.get(), out.w.get(),
      out.src.get());
  count_launch();
  GIM_LAUNCH_CHECK();
  prof.extra = 8.0 * m2c;
}

// K7 projection (coarsening.py:269-277): Pi_f = Pi_c[M]
__global__ void k_project(int n, const int* __restrict__ cmap, const int* __restrict__ pc,
                          int* __restrict__ pf) {
  for (int v = blockIdx.x * blockDim.x + threadIdx.x; v < n; v += gridDim.x * blockDim.x)
    pf[v] = pc[cmap[v]];
}

void project(int n, const int* cmap, const int* pc, int* pf, cudaStream_t s) {
  if (n == 0) return;
  k_project<<<grid_for(n, 256), 256, 0, s>>>(n, cmap, pc, pf);
  count_launch();
  GIM_LAUNCH_CHECK();
}

__global__ void k_copy_ll(const long long* src, long long* dst) { *dst = *src; }

__global__ void k_pack4(const long long* a, const int* b, const int* c, const int* d,
                        long long* out) {
  out[0] = *a;
  out[1] = *b;
  out[2] = *c;
  out[3] = d ? *d : -1;
}

// ---------------------------------------------------------------------------
// One level of the stack with a single host round trip (the common case):
// both matching rounds (round 2 gated on the device), the coarse ids and the
// member table speculatively, then ONE read of (matched, n_c, max row).
// The contraction then runs without waiting: arrays are sized by the upper
// bound m2 and the true 2m_c stays on the device (*m2c_dev) until the
// caller reads every level's at once.  Returns false (nothing allocated
// for the coarse level) when the level needs the general path: < 40 %
// matched (two-hop), or hub rows > kRowCap.
bool coarsen_level_fast(const DevGraph& g_in, double l_max, unsigned long long lseed,
                        int* partner, int* cmap, int* n_c_out, long long* matched_out,
                        OwnedGraph& out, int* m2c_dev, bool* stalled, const int* g_m2_dev,
                        long long* g_m2_out, cudaStream_t s) {
  DevGraph g = g_in;
  const int n = g.n;
  *stalled = false;
  GIM_CUDA(cudaMemsetAsync(partner, 0xff, sizeof(int) * (size_t)std::max(n, 1), s));
  DBuf<int> pref((size_t)std::max(n, 1), s);
  DBuf<long long> cnt(2, s);  // [matched, matched after round 1]
  GIM_CUDA(cudaMemsetAsync(cnt.get(), 0, 2 * sizeof(long long), s));
  hem_round(g, partner, pref.get(), l_max, splitmix64(lseed ^ 1ull), cnt.get(), s, nullptr);
  k_copy_ll<<<1, 1, 0, s>>>(cnt.get(), cnt.get() + 1);
  hem_round(g, partner, pref.get(), l_max, splitmix64(lseed ^ 2ull), cnt.get(), s,
            cnt.get() + 1);
  // speculative coarse ids + members (valid unless two-hop changes partner)
  DBuf<int> ids((size_t)std::max(n, 1), s), tot(1, s);
  exclusive_scan<int>(n, IsRoot{partner}, StoreTo<int>{ids.get()}, tot.get(), s);
  k_coarse_map<<<grid_for(n, 256), 256, 0, s>>>(n, partner, ids.get(), cmap);
  DBuf<int4> mem((size_t)std::max(n, 1), s);
  DBuf<int> rowlen((size_t)n + 1, s), cvw((size_t)std::max(n, 1), s);
  DBuf<int> scal(3, s);  // maxlen, ubtot, m2c
  GIM_CUDA(cudaMemsetAsync(scal.get(), 0, 3 * sizeof(int), s));
  k_members<<<grid_for(n, 256), 256, 0, s>>>(n, partner, cmap, g.off, g.vw, mem.get(),
                                             rowlen.get(), cvw.get(), scal.get());
  DBuf<long long> pack(4, s);
  k_pack4<<<1, 1, 0, s>>>(cnt.get(), tot.get(), scal.get(), g_m2_dev, pack.get());
  count_launch(5);
  GIM_LAUNCH_CHECK();
  long long* hp = static_cast<long long*>(pinned_scratch(4 * sizeof(long long)));
  GIM_CUDA(cudaMemcpyAsync(hp, pack.get(), 4 * sizeof(long long), cudaMemcpyDeviceToHost, s));
  GIM_CUDA(sync_stream(s));
  const long long matched = hp[0];
  const int n_c = (int)hp[1], maxlen = (int)hp[2];
  if (g_m2_dev) {  // this level's own 2m was still on the device
    g.m2 = hp[3];
    *g_m2_out = hp[3];
  }
  *matched_out = matched;
  *n_c_out = n_c;
  const double frac = n ? (double)matched / (double)n : 1.0;
  if (frac < 0.40 || maxlen > kRowCap) return false;
  if ((double)n_c * 1.02 > (double)n) {  // stall guard
    *stalled = true;
    return true;
  }
  ProfScope prof(P_CONTRACT, 12.0 * n + 12.0 * g.m2 + 8.0 * n_c, s);
  const long long cap = std::max<long long>(g.m2, 1);
  out.n = n_c;
  out.maxdeg = maxlen;  // rows of the merged members: an upper bound
  out.vw = std::move(cvw);
  out.off = DBuf<int>((size_t)n_c + 1, s);
  out.tgt = DBuf<int>((size_t)cap, s);
  out.w = DBuf<int>((size_t)cap, s);
  out.src = DBuf<int>((size_t)cap, s);
  DBuf<int> ub((size_t)n_c + 1, s), cdeg((size_t)n_c + 1, s);
  DBuf<int> t_tgt((size_t)cap, s), t_w((size_t)cap, s);
  GIM_CUDA(cudaMemsetAsync(cdeg.get() + n_c, 0, sizeof(int), s));
  exclusive_scan<int>((long long)n_c, LoadAs<int, int>{rowlen.get()}, StoreTo<int>{ub.get()},
                      scal.get() + 1, s);
  k_row_warp<<<grid_for((long long)n_c * 32, kCtBlock, kSMs * 32), kCtBlock, 0, s>>>(
      n_c, mem.get(), ub.get(), g.tgt, g.w, cmap, t_tgt.get(), t_w.get(), cdeg.get());
  count_launch();
  if (maxlen > kCtTpv) {
    const int grid = grid_for((long long)n_c * 32, kRowWarps * 32, kSMs * 8);
    k_row_long<<<grid, kRowWarps * 32, 0, s>>>(n_c, mem.get(), rowlen.get(), ub.get(),
                                               g.tgt, g.w, cmap, t_tgt.get(), t_w.get(),
                                               cdeg.get());
    count_launch();
  }
  exclusive_scan<int>((long long)n_c + 1, LoadAs<int, int>{cdeg.get()},
                      StoreTo<int>{out.off.get()}, m2c_dev, s);
  k_row_compact<<<grid_for(n_c, 256, kSMs * 16), 256, 0, s>>>(
      n_c, ub.get(), out.off.get(), t_tgt.get(), t_w.get(), out.tgt.get(), out.w.get(),
      out.src.get());
  count_launch();
  GIM_LAUNCH_CHECK();
  out.m2 = cap;  // upper bound until the next level's round trip reads *m2c_dev
  return true;
}

}  // namespace gim
