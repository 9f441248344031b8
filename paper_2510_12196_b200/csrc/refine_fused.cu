// Device-resident Alg. 4 (refinement.py:389-464): one cooperative persistent
// kernel runs the whole refinement loop of one level — label propagation
// (first filter, second filter), weak rebalancing, move application, exact
// J tracking and best-mapping bookkeeping — with grid-wide barriers between
// phases and no host round trip per iteration.
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
// contiguous vertex ranges, publish per-block partial sums, and one warp per
// CTA walks its range with __match_any_sync ranking.
//
// Strong passes (rare: 7 of ~3,000 passes on rgg 2^20) exit the kernel
// ("yield"); the host runs the sort-based strong pass and relaunches.
#include <cooperative_groups.h>

#include "common.cuh"
#include "kernels.cuh"
#include "refine_dev.cuh"

namespace cg = cooperative_groups;

namespace gim {

constexpr int kFusedBlock = 256;
constexpr int kFusedWarps = kFusedBlock / 32;

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
  unsigned char* cand;
  int* dest;
  long long* gkey;
  unsigned char* tm0;
  unsigned char* tm1;
  int* rtgt;             // rebalance target per vertex (-1 = none)
  unsigned char* rcell;  // rebalance cell per vertex
  long long* W;          // [k * C] candidate weight per (source block, cell)
  long long* S;          // [G * k] per-CTA partial sums of c*-cell weights
  long long* ctr;        // [movers0, dj0, movers1, dj1, J]
  const int* heavy;
  int n_heavy;
  FusedState* st;
  double l_max, sigma, phi, jet_c;
  int jet, rho, i_max, i_w_max;
  unsigned long long seed;
};

// per-CTA replicated control state
struct Ctl {
  long long J, best_j, best_maxw, maxw, pass_counter;
  int i, i_w, best_balanced, locks_nonempty, lp_par, it, brk, take, strong_yield;
  long long iters, lp, weak;
};

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

template <int VW>
__global__ void __launch_bounds__(kFusedBlock) k_refine_fused(FusedArgs A) {
  cg::grid_group grid = cg::this_grid();
  extern __shared__ unsigned char dsm[];
  __shared__ long long s_dbit[64];
  __shared__ Ctl C;
  __shared__ int s_nelig;
  const int k = A.k;
  const int NC = 31 * A.rho;
  const int n = A.n;
  // dynamic smem: warp tables | ovl[k] | elig[k] | elist[k] | cstar[k] | pstar[k] | run[k]
  int* tables = reinterpret_cast<int*>(dsm);
  long long* pstar = reinterpret_cast<long long*>(tables + (size_t)kFusedWarps * 3 * k);
  long long* run = pstar + k;
  int* elist = reinterpret_cast<int*>(run + k);
  int* cstar = elist + k;
  unsigned char* ovl = reinterpret_cast<unsigned char*>(cstar + k);
  unsigned char* elig = ovl + k;

  load_dbit(s_dbit, A.t);
  const int lane = lane_id();
  const int warp = threadIdx.x >> 5;
  const long long gw = ((long long)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  const long long NW = ((long long)gridDim.x * blockDim.x) >> 5;
  const long long gt = (long long)blockIdx.x * blockDim.x + threadIdx.x;
  const long long GT = (long long)gridDim.x * blockDim.x;
  constexpr int GPW = 32 / VW;
  const int gi = lane / VW, li = lane % VW;
  WarpTable wt;
  wt.tab = tables + (size_t)warp * 3 * k;
  wt.lb = wt.tab + k;
  wt.lw = wt.lb + k;
  // contiguous vertex range of this CTA (weak selection walk)
  const int R = (n + gridDim.x - 1) / gridDim.x;
  const int r0 = min(n, (int)blockIdx.x * R), r1 = min(n, r0 + R);

  // ---- entry: J, best := current (first launch only)
  if (!A.st->started) {
    long long acc = 0;
    for (long long e = gt; e < A.m2; e += GT)
      acc += (long long)A.w[e] * dist(A.t, A.part[A.src[e]], A.part[A.tgt[e]]);
    block_sum_atomic<kFusedBlock>(acc, A.ctr + 4);
    for (long long v = gt; v < n; v += GT) A.best[v] = A.part[v];
    for (long long i = gt; i < (long long)k * NC; i += GT) A.W[i] = 0;
    if (blockIdx.x == 0)
      for (int b = threadIdx.x; b < k; b += blockDim.x) A.best_bw[b] = A.bw[b];
    grid.sync();
    long long mx = block_max_bw(A.bw, k);
    if (threadIdx.x == 0) {
      C.J = A.ctr[4];
      C.maxw = mx;
      C.best_balanced = (double)mx <= A.l_max;
      C.best_j = C.J;
      C.best_maxw = mx;
      C.i = C.i_w = 0;
      C.pass_counter = 0;
      C.locks_nonempty = 0;
      C.lp_par = 0;
      C.it = 0;
      C.iters = C.lp = C.weak = 0;
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
    C.it = 0;
    C.iters = C.lp = C.weak = 0;
  }
  if (threadIdx.x == 0) {
    C.brk = 0;
    C.strong_yield = 0;
  }
  __syncthreads();

  while (C.i < A.i_max) {
    const bool balanced_now = (double)C.maxw <= A.l_max;
    const bool entry_locks_empty = !C.locks_nonempty;
    if (!balanced_now && !(C.i_w < A.i_w_max)) {  // strong pass: hand back to the host
      if (threadIdx.x == 0) C.strong_yield = 1;
      __syncthreads();
      break;
    }
    const int q = C.it & 1;
    long long* movers = A.ctr + 2 * q;
    long long* dj = A.ctr + 2 * q + 1;
    unsigned char* tm = C.lp_par ? A.tm1 : A.tm0;
    const unsigned char* locks = C.locks_nonempty ? (C.lp_par ? A.tm0 : A.tm1) : nullptr;
    bool incomplete = false;
    if (balanced_now) {
      // ---- K9 first filter
      LpParams lp{locks, A.jet, A.jet_c};
      LpOut lo{A.cand, A.dest, A.gkey};
      for (long long vb = gw * GPW; vb < n; vb += NW * GPW) {
        const int v = (int)(vb + gi);
        bool live = v < n;
        int e0 = 0, d = 0, own = 0;
        if (live) {
          e0 = A.off[v];
          d = A.off[v + 1] - e0;
          own = A.part[v];
          if (d > VW) live = false;
          else if (locks && locks[v]) {
            live = false;
            if (li == 0) { lo.cand[v] = 0; lo.dest[v] = own; lo.gkey[v] = kGainNone; }
          }
        }
        const bool valid = live && li < d;
        int myb = -1, myw = 0;
        if (valid) {
          myb = A.part[A.tgt[e0 + li]];
          myw = A.w[e0 + li];
        }
        const int dmax = __reduce_max_sync(0xffffffffu, live ? d : 0);
        VertexEval r = eval_regs<VW>(valid, live ? own : 0, myb, myw, dmax, A.t, s_dbit, nullptr,
                                     A.jet != 0);
        if (live && li == 0) lp_decide(v, own, r, lp, lo);
      }
      for (long long hi = gw; hi < A.n_heavy; hi += NW) {
        const int v = A.heavy[hi];
        const int own = A.part[v];
        if (locks && locks[v]) {
          if (lane == 0) { lo.cand[v] = 0; lo.dest[v] = own; lo.gkey[v] = kGainNone; }
          continue;
        }
        int s = warp_build_table(wt, k, A.off[v], A.off[v + 1], A.tgt, A.w, A.part);
        VertexEval r = eval_table(wt, s, own, A.t, s_dbit, nullptr);
        if (lane == 0) lp_decide(v, own, r, lp, lo);
        __syncwarp();
      }
      grid.sync();
      if (blockIdx.x == 0 && threadIdx.x < 2) A.ctr[2 * (q ^ 1) + threadIdx.x] = 0;
      // ---- K10 second filter
      long long moved = 0;
      for (long long vb = gw * GPW; vb < n; vb += NW * GPW) {
        const int v = (int)(vb + gi);
        const bool c = v < n && A.cand[v];
        long long fut = 0;
        if (c) {
          const long long gv = A.gkey[v];
          const unsigned long long oc = __ldg(A.t.code + A.part[v]);
          const unsigned long long dc = __ldg(A.t.code + A.dest[v]);
          for (int e = A.off[v] + li; e < A.off[v + 1]; e += VW) {
            int u = A.tgt[e];
            long long gu = A.gkey[u];
            bool earlier = gu > gv || (gu == gv && u < v);
            int pos = earlier ? A.dest[u] : A.part[u];
            unsigned long long pc = __ldg(A.t.code + pos);
            fut += (long long)A.w[e] * (cdist(s_dbit, oc, pc) - cdist(s_dbit, dc, pc));
          }
        }
#pragma unroll
        for (int o = VW / 2; o > 0; o >>= 1) fut += __shfl_xor_sync(0xffffffffu, fut, o);
        if (v < n && li == 0) {
          bool m = c && fut >= 0;
          tm[v] = m ? 1 : 0;
          moved += m;
        }
      }
      block_sum_atomic<kFusedBlock>(moved, movers);
      grid.sync();
    } else {
      // ---- K11 weak rebalance candidates (refinement.py:273-309); locks are
      // cleared by the control update below (locks_nonempty = 0)
      for (int b = threadIdx.x; b < k; b += blockDim.x) {
        ovl[b] = (double)A.bw[b] > A.l_max;
        elig[b] = (double)A.bw[b] < A.sigma;
      }
      __syncthreads();
      if (threadIdx.x == 0) {  // ascending eligible list
        int ne = 0;
        for (int b = 0; b < k; ++b)
          if (elig[b]) elist[ne++] = b;
        s_nelig = ne;
      }
      __syncthreads();
      const int n_elig = s_nelig;
      incomplete = n_elig == 0;
      RbParams rp{ovl, elig, elist, n_elig, A.seed, C.pass_counter};
      for (long long vb = gw * GPW; vb < n; vb += NW * GPW) {
        const int v = (int)(vb + gi);
        bool live = v < n;
        int e0 = 0, d = 0, own = 0;
        if (live) {
          e0 = A.off[v];
          d = A.off[v + 1] - e0;
          own = A.part[v];
          if (li == 0) tm[v] = 0;
          if (d > VW) live = false;
          else if (!ovl[own]) {
            live = false;
            if (li == 0) A.rtgt[v] = -1;
          }
        }
        const bool valid = live && li < d;
        int myb = -1, myw = 0;
        if (valid) {
          myb = A.part[A.tgt[e0 + li]];
          myw = A.w[e0 + li];
        }
        const int dmax = __reduce_max_sync(0xffffffffu, live ? d : 0);
        VertexEval r = eval_regs<VW>(valid, live ? own : 0, myb, myw, dmax, A.t, s_dbit, elig,
                                     false);
        bool need = live && r.best_b < 0 && n_elig > 0;
        unsigned any = __ballot_sync(0xffffffffu, need);
        int tb = -1;
        if (need) {
          unsigned long long h = hash2(rp.seed, (unsigned long long)v,
                                       (unsigned long long)rp.pass_counter);
          tb = elist[h % (unsigned long long)n_elig];
        }
        long long cost = 0, cur = 0;
        if (any) {
          cost = cost_regs<VW>(valid && need, myb, myw, need ? tb : 0, A.t, s_dbit);
          cur = cur_regs<VW>(valid && need, own, myb, myw, A.t, s_dbit);
        }
        if (live && li == 0) {
          int target = -1;
          long long gain = 0;
          if (r.best_b >= 0) {
            target = r.best_b;
            gain = r.best_gain;
          } else if (need) {
            target = tb;
            gain = cur - cost;
          }
          A.rtgt[v] = target;
          if (target >= 0) {
            int cell = slot_for_gain(gain) * A.rho + v % A.rho;
            A.rcell[v] = (unsigned char)cell;
            atomicAdd(reinterpret_cast<unsigned long long*>(&A.W[(size_t)own * NC + cell]),
                      (unsigned long long)(long long)A.vw[v]);
          }
        }
      }
      for (long long hi = gw; hi < A.n_heavy; hi += NW) {
        const int v = A.heavy[hi];
        const int own = A.part[v];
        if (!ovl[own]) {
          if (lane == 0) A.rtgt[v] = -1;
          continue;
        }
        int s = warp_build_table(wt, k, A.off[v], A.off[v + 1], A.tgt, A.w, A.part);
        VertexEval r = eval_table(wt, s, own, A.t, s_dbit, elig);
        int target = -1;
        long long gain = 0;
        if (r.best_b >= 0) {
          target = r.best_b;
          gain = r.best_gain;
        } else if (n_elig > 0) {
          unsigned long long h = hash2(rp.seed, (unsigned long long)v,
                                       (unsigned long long)rp.pass_counter);
          target = elist[h % (unsigned long long)n_elig];
          gain = r.cur - cost_table(wt, s, target, A.t, s_dbit);
        }
        if (lane == 0) {
          A.rtgt[v] = target;
          if (target >= 0) {
            int cell = slot_for_gain(gain) * A.rho + v % A.rho;
            A.rcell[v] = (unsigned char)cell;
            atomicAdd(reinterpret_cast<unsigned long long*>(&A.W[(size_t)own * NC + cell]),
                      (unsigned long long)(long long)A.vw[v]);
          }
        }
        __syncwarp();
      }
      grid.sync();
      if (blockIdx.x == 0 && threadIdx.x < 2) A.ctr[2 * (q ^ 1) + threadIdx.x] = 0;
      // ---- K12 weak selection, step A: c*, P_{c*} per overloaded block and
      // this CTA's per-block weight of c*-cell candidates
      for (int b = threadIdx.x; b < k; b += blockDim.x) {
        run[b] = 0;
        if (!ovl[b]) { cstar[b] = NC; pstar[b] = 0; continue; }
        const double excess = (double)A.bw[b] - A.l_max;
        long long P = 0;
        int c = 0;
        for (; c < NC; ++c) {
          long long wc = A.W[(size_t)b * NC + c];
          if ((double)(P + wc) > excess) break;
          P += wc;
        }
        cstar[b] = c;
        pstar[b] = P;
      }
      __syncthreads();
      for (int v = r0 + threadIdx.x; v < r1; v += blockDim.x) {
        int tb = A.rtgt[v];
        if (tb < 0) continue;
        int b = A.part[v];
        if ((int)A.rcell[v] == cstar[b])
          atomicAdd(reinterpret_cast<unsigned long long*>(&run[b]), (unsigned long long)(long long)A.vw[v]);
      }
      __syncthreads();
      for (int b = threadIdx.x; b < k; b += blockDim.x) A.S[(size_t)blockIdx.x * k + b] = run[b];
      grid.sync();
      // step B: in-cell prefix in vertex order, then the take decisions
      for (int b = threadIdx.x; b < k; b += blockDim.x) {
        long long base = 0;
        for (int c2 = 0; c2 < (int)blockIdx.x; ++c2) base += A.S[(size_t)c2 * k + b];
        run[b] = base;
      }
      __syncthreads();
      long long moved = 0;
      if (warp == 0) {
        for (int v0 = r0; v0 < r1; v0 += 32) {
          const int v = v0 + lane;
          bool partial = false;
          int b = 0;
          long long wv = 0;
          if (v < r1) {
            int tb = A.rtgt[v];
            if (tb >= 0) {
              b = A.part[v];
              partial = (int)A.rcell[v] == cstar[b];
              wv = A.vw[v];
            }
          }
          unsigned act = __ballot_sync(0xffffffffu, partial);
          if (partial) {
            unsigned peers = __match_any_sync(act, b);
            int leader = __ffs(peers) - 1;
            long long before = 0, total = 0;
            unsigned m = peers;
            while (m) {
              int l = __ffs(m) - 1;
              m &= m - 1;
              long long x = __shfl_sync(peers, wv, l);
              if (l < (int)lane) before += x;
              total += x;
            }
            const long long q0 = run[b] + before;
            const double excess = (double)A.bw[b] - A.l_max;
            if ((double)(pstar[b] + q0) < excess) {
              tm[v] = 1;
              A.dest[v] = A.rtgt[v];
              ++moved;
            }
            __syncwarp(peers);
            if ((int)lane == leader) run[b] += total;
          }
          __syncwarp();
        }
      } else {
        for (int v = r0 + threadIdx.x - 32; v < r1; v += blockDim.x - 32) {
          int tb = A.rtgt[v];
          if (tb < 0) continue;
          int b = A.part[v];
          if ((int)A.rcell[v] < cstar[b]) {
            tm[v] = 1;
            A.dest[v] = tb;
            ++moved;
          }
        }
      }
      block_sum_atomic<kFusedBlock>(moved, movers);
      grid.sync();
      for (long long i = gt; i < (long long)k * NC; i += GT) A.W[i] = 0;  // next weak pass
    }
    // ---- K13 apply moves: exact dJ + block weights
    {
      long long acc = 0;
      for (long long vb = gw * GPW; vb < n; vb += NW * GPW) {
        const int v = (int)(vb + gi);
        if (v < n && tm[v]) {
          const int ov = A.part[v], nv = A.dest[v];
          const unsigned long long oc = __ldg(A.t.code + ov), nc = __ldg(A.t.code + nv);
          for (int e = A.off[v] + li; e < A.off[v + 1]; e += VW) {
            int u = A.tgt[e];
            bool um = tm[u];
            int ou = A.part[u];
            int nu = um ? A.dest[u] : ou;
            long long dd = cdist(s_dbit, nc, __ldg(A.t.code + nu)) -
                           cdist(s_dbit, oc, __ldg(A.t.code + ou));
            acc += (long long)A.w[e] * dd * (um ? 1 : 2);
          }
          if (li == 0 && ov != nv) {
            atomicAdd(reinterpret_cast<unsigned long long*>(&A.bw[ov]),
                      (unsigned long long)(-(long long)A.vw[v]));
            atomicAdd(reinterpret_cast<unsigned long long*>(&A.bw[nv]),
                      (unsigned long long)(long long)A.vw[v]);
          }
        }
      }
      block_sum_atomic<kFusedBlock>(acc, dj);
    }
    grid.sync();
    for (long long v = gt; v < n; v += GT)
      if (tm[v]) A.part[v] = A.dest[v];
    grid.sync();
    // ---- Alg. 4 control (refinement.py:433-463), replicated per CTA
    long long mx = block_max_bw(A.bw, k);
    if (threadIdx.x == 0) {
      const long long mv = *movers;
      C.take = 0;
      C.iters++;
      if (balanced_now) C.lp++; else { C.weak++; C.i_w++; C.pass_counter++; }
      if (balanced_now) C.i_w = 0;
      if (mv == 0 && ((balanced_now && entry_locks_empty) || (!balanced_now && incomplete))) {
        C.brk = 1;
      } else {
        C.J += *dj;
        C.maxw = mx;
        if (balanced_now) {
          C.locks_nonempty = mv > 0;
          C.lp_par ^= 1;
        } else {
          C.locks_nonempty = 0;
        }
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
        C.it++;
      }
    }
    __syncthreads();
    if (C.brk) break;
    if (C.take) {
      for (long long v = gt; v < n; v += GT) A.best[v] = A.part[v];
      if (blockIdx.x == 0)
        for (int b = threadIdx.x; b < k; b += blockDim.x) A.best_bw[b] = A.bw[b];
    }
  }
  // ---- exit: persist the control state; on completion restore the best
  grid.sync();
  if (blockIdx.x == 0 && threadIdx.x == 0) {
    FusedState& S1 = *A.st;
    S1.started = 1;
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
    S1.status = C.strong_yield ? 1 : 0;
    S1.iters += C.iters;
    S1.lp += C.lp;
    S1.weak += C.weak;
  }
  if (!C.strong_yield) {
    for (long long v = gt; v < n; v += GT) A.part[v] = A.best[v];
    if (blockIdx.x == 0)
      for (int b = threadIdx.x; b < k; b += blockDim.x) A.bw[b] = A.best_bw[b];
  }
}

// ---------------------------------------------------------------------------
// host side

template <int VW>
static int coop_max_blocks(size_t smem) {
  int dev = 0, sms = 0, per = 0;
  GIM_CUDA(cudaGetDevice(&dev));
  GIM_CUDA(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev));
  if (smem > 48 * 1024)
    GIM_CUDA(cudaFuncSetAttribute(k_refine_fused<VW>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                  (int)smem));
  GIM_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per, k_refine_fused<VW>, kFusedBlock,
                                                         smem));
  return std::max(1, per) * sms;
}

bool fused_supported(int k, int rho) { return k <= 1024 && rho >= 1 && rho <= 8; }

// runs Alg. 4 iterations on the device until the loop ends (returns true) or a
// strong pass is due (returns false; the host performs it and calls again)
bool refine_fused_run(const RefineLevel& L, const Topo& t, int* part, long long* bw,
                      const FusedCfg& cfg, FusedBuffers& fb, cudaStream_t s) {
  const DevGraph& g = L.g;
  const int k = t.k;
  const int NC = 31 * cfg.rho;
  size_t smem = (size_t)kFusedWarps * 3 * k * sizeof(int) + (size_t)k * (8 + 8 + 4 + 4 + 1 + 1);
  smem = (smem + 15) & ~(size_t)15;
  int maxb = 0;
  switch (L.vw) {
    case 4: maxb = coop_max_blocks<4>(smem); break;
    case 8: maxb = coop_max_blocks<8>(smem); break;
    case 16: maxb = coop_max_blocks<16>(smem); break;
    default: maxb = coop_max_blocks<32>(smem); break;
  }
  // ~2K vertices per CTA, at most one full co-resident wave
  int G = (int)std::min<long long>((long long)maxb, std::max<long long>(1, ((long long)g.n + 2047) / 2048));
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
  A.cand = fb.cand;
  A.dest = fb.dest;
  A.gkey = fb.gkey;
  A.tm0 = fb.tm0;
  A.tm1 = fb.tm1;
  A.rtgt = fb.rtgt;
  A.rcell = fb.rcell;
  A.W = fb.W.get();
  A.S = fb.S.get();
  A.ctr = fb.ctr;
  A.heavy = L.heavy.get();
  A.n_heavy = L.n_heavy;
  A.st = fb.state;
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
  switch (L.vw) {
    case 4: fn = (void*)k_refine_fused<4>; break;
    case 8: fn = (void*)k_refine_fused<8>; break;
    case 16: fn = (void*)k_refine_fused<16>; break;
    default: fn = (void*)k_refine_fused<32>; break;
  }
  {
    ProfScope prof(P_LP_EVAL, 0.0, s);
    GIM_CUDA(cudaLaunchCooperativeKernel(fn, dim3(G), dim3(kFusedBlock), args, smem, s));
  }
  count_launch();
  GIM_CUDA(cudaMemcpyAsync(fb.h_state, fb.state, sizeof(FusedState), cudaMemcpyDeviceToHost, s));
  GIM_CUDA(cudaStreamSynchronize(s));
  return fb.h_state->status == 0;
}

}  // namespace gim
