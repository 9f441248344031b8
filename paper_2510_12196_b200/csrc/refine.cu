// Refinement kernels: Jet-style label propagation (K9/K10), weak/strong
// rebalancing (K11/K12), move application with exact J delta (K13), and the
// block-connectivity table (K8, parity unit).
//
// Reference: refinement.py (_best_target :168-190, _gain_to :193-198,
// label_propagation_pass :201-270, _rebalance_candidates :273-309,
// weak_rebalance :312-347, strong_rebalance :350-386), mapping.py
// (BlockConnectivity :124-249, apply_moves :252-282).
//
// Per-vertex connectivity is never stored between iterations: every pass
// rebuilds conn(v, .) on chip from the CSR row and Pi (registers for
// degree <= VW, a per-warp shared-memory block table otherwise), which is
// exact and keeps the HBM traffic at one row sweep per pass.
#include "common.cuh"
#include "kernels.cuh"
#include "radix.cuh"
#include "refine_dev.cuh"
#include "scan.cuh"

namespace gim {

// ---------------------------------------------------------------------------
// K9 first filter / K11 candidates, register path.  mode 0 = LP, 1 = rebalance

template <int VW>
__global__ void __launch_bounds__(256) k_eval_regs(int mode, int n, const int* __restrict__ off,
                                                   const int* __restrict__ tgt,
                                                   const int* __restrict__ w,
                                                   const int* __restrict__ part, Topo t,
                                                   LpParams lp, LpOut lo, RbParams rb, RbOut ro,
                                                   long long* __restrict__ ctr) {
  __shared__ long long s_dbit[64];
  load_dbit(s_dbit, t);
  __syncthreads();
  constexpr int GPW = 32 / VW;
  const long long wid = ((long long)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  const long long nw = ((long long)gridDim.x * blockDim.x) >> 5;
  const int lane = lane_id();
  const int gi = lane / VW, li = lane % VW;
  // per-iteration counters are zeroed here instead of by separate memsets
  if (ctr && blockIdx.x == 0 && threadIdx.x < 2) ctr[threadIdx.x] = 0;
  for (long long vb = wid * GPW; vb < n; vb += nw * GPW) {
    const int v = (int)(vb + gi);
    bool live = v < n;
    int e0 = 0, d = 0, own = 0;
    if (live) {
      e0 = off[v];
      d = off[v + 1] - e0;
      own = part[v];
      if (mode == 1 && li == 0) ro.to_move[v] = 0;
      if (d > VW) live = false;  // handled by the shared-memory path
      else if (mode == 0 && lp.locked && lp.locked[v]) {
        live = false;
        if (li == 0) { lo.cand[v] = 0; lo.dest[v] = own; lo.gkey[v] = kGainNone; }
      } else if (mode == 1 && !rb.ovl[own]) {
        live = false;
        if (li == 0) ro.target[v] = -1;
      }
    }
    const bool valid = live && li < d;
    int myb = -1, myw = 0;
    if (valid) {
      myb = part[tgt[e0 + li]];
      myw = w[e0 + li];
    }
    const int dmax = __reduce_max_sync(0xffffffffu, live ? d : 0);
    VertexEval r = eval_regs<VW>(valid, live ? own : 0, myb, myw, dmax, t, s_dbit,
                                 mode == 1 ? rb.elig : nullptr, mode == 0 && lp.jet);
    if (mode == 0) {
      if (live && li == 0) lp_decide(v, own, r, lp, lo);
    } else {
      // fallback target: eligible[hash2(seed, v, pass) % n_elig] (refinement.py:302-307)
      bool need = live && r.best_b < 0 && rb.n_elig > 0;
      unsigned any = __ballot_sync(0xffffffffu, need);
      int tb = -1;
      if (need) {
        unsigned long long h = hash2(rb.seed, (unsigned long long)v,
                                     (unsigned long long)rb.pass_counter);
        tb = rb.elig_list[h % (unsigned long long)rb.n_elig];
      }
      long long cost = 0, cur = 0;
      if (any) {
        cost = cost_regs<VW>(valid && need, myb, myw, need ? tb : 0, t, s_dbit);
        cur = cur_regs<VW>(valid && need, own, myb, myw, t, s_dbit);
      }
      if (live && li == 0) {
        if (r.best_b >= 0) {
          ro.target[v] = r.best_b;
          ro.gain[v] = r.best_gain;
        } else if (need) {
          ro.target[v] = tb;
          ro.gain[v] = cur - cost;
        } else {
          ro.target[v] = -1;  // no eligible block anywhere: incomplete
        }
      }
    }
  }
}

// K9/K11 for heavy vertices (degree > VW): one warp per listed vertex
__global__ void __launch_bounds__(128) k_eval_table(int mode, int n_heavy,
                                                    const int* __restrict__ heavy, int k,
                                                    const int* __restrict__ off,
                                                    const int* __restrict__ tgt,
                                                    const int* __restrict__ w,
                                                    const int* __restrict__ part, Topo t,
                                                    LpParams lp, LpOut lo, RbParams rb,
                                                    RbOut ro) {
  extern __shared__ int smem[];
  __shared__ long long s_dbit[64];
  load_dbit(s_dbit, t);
  __syncthreads();
  const int warp = threadIdx.x >> 5;
  WarpTable wt;
  wt.tab = smem + (size_t)warp * 3 * k;
  wt.lb = wt.tab + k;
  wt.lw = wt.lb + k;
  const int lane = lane_id();
  const int nwarps = (gridDim.x * blockDim.x) >> 5;
  for (int i = (blockIdx.x * blockDim.x + threadIdx.x) >> 5; i < n_heavy; i += nwarps) {
    const int v = heavy[i];
    const int own = part[v];
    if (mode == 0 && lp.locked && lp.locked[v]) {
      if (lane == 0) { lo.cand[v] = 0; lo.dest[v] = own; lo.gkey[v] = kGainNone; }
      continue;
    }
    if (mode == 1 && !rb.ovl[own]) {
      if (lane == 0) ro.target[v] = -1;
      continue;
    }
    int s = warp_build_table(wt, k, off[v], off[v + 1], tgt, w, part);
    VertexEval r = eval_table(wt, s, own, t, s_dbit, mode == 1 ? rb.elig : nullptr);
    if (mode == 0) {
      if (lane == 0) lp_decide(v, own, r, lp, lo);
    } else {
      if (r.best_b >= 0) {
        if (lane == 0) { ro.target[v] = r.best_b; ro.gain[v] = r.best_gain; }
      } else if (rb.n_elig > 0) {
        unsigned long long h = hash2(rb.seed, (unsigned long long)v,
                                     (unsigned long long)rb.pass_counter);
        int tb = rb.elig_list[h % (unsigned long long)rb.n_elig];
        long long cost = cost_table(wt, s, tb, t, s_dbit);
        if (lane == 0) { ro.target[v] = tb; ro.gain[v] = r.cur - cost; }
      } else if (lane == 0) {
        ro.target[v] = -1;
      }
    }
    __syncwarp();
  }
}

// ---------------------------------------------------------------------------
// K10 second filter (refinement.py:246-269): candidate v is re-evaluated as if
// every candidate neighbour ordered before it (higher gain, then lower id)
// had moved; kept iff the re-evaluated gain is >= 0.

template <int VW>
__global__ void __launch_bounds__(256) k_lp_second(int n, const int* __restrict__ off,
                                                   const int* __restrict__ tgt,
                                                   const int* __restrict__ w,
                                                   const int* __restrict__ part, Topo t,
                                                   const unsigned char* __restrict__ cand,
                                                   const int* __restrict__ dest,
                                                   const long long* __restrict__ gkey,
                                                   unsigned char* __restrict__ to_move,
                                                   long long* __restrict__ movers) {
  __shared__ long long s_dbit[64];
  load_dbit(s_dbit, t);
  __syncthreads();
  constexpr int GPW = 32 / VW;
  const long long wid = ((long long)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  const long long nw = ((long long)gridDim.x * blockDim.x) >> 5;
  const int lane = lane_id();
  const int gi = lane / VW, li = lane % VW;
  long long moved = 0;
  for (long long vb = wid * GPW; vb < n; vb += nw * GPW) {
    const int v = (int)(vb + gi);
    const bool c = v < n && cand[v];
    long long fut = 0;
    if (c) {
      const long long gv = gkey[v];
      const unsigned long long oc = __ldg(t.code + part[v]);
      const unsigned long long dc = __ldg(t.code + dest[v]);
      for (int e = off[v] + li; e < off[v + 1]; e += VW) {
        int u = tgt[e];
        long long gu = gkey[u];
        bool earlier = gu > gv || (gu == gv && u < v);  // kGainNone never earlier
        int pos = earlier ? dest[u] : part[u];
        unsigned long long pc = __ldg(t.code + pos);
        fut += (long long)w[e] * (cdist(s_dbit, oc, pc) - cdist(s_dbit, dc, pc));
      }
    }
#pragma unroll
    for (int o = VW / 2; o > 0; o >>= 1) fut += __shfl_xor_sync(0xffffffffu, fut, o);
    if (v < n && li == 0) {
      bool m = c && fut >= 0;
      to_move[v] = m ? 1 : 0;
      moved += m;
    }
  }
  block_sum_atomic<256>(moved, movers);
}

// ---------------------------------------------------------------------------
// K13 apply moves (mapping.py:252-282) with the exact J delta:
// dJ = sum over movers v, neighbours u of w (D(new v, new u) - D(old v, old u)),
// doubled when u stays (its mirror slot (u, v) changes identically).
// Block weights by warp-aggregated atomics.

template <int VW>
__global__ void __launch_bounds__(256) k_apply_delta(int n, const int* __restrict__ off,
                                                     const int* __restrict__ tgt,
                                                     const int* __restrict__ w,
                                                     const int* __restrict__ vw,
                                                     const int* __restrict__ part, Topo t,
                                                     const unsigned char* __restrict__ to_move,
                                                     const int* __restrict__ dest,
                                                     long long* __restrict__ bw,
                                                     long long* __restrict__ dj) {
  __shared__ long long s_dbit[64];
  load_dbit(s_dbit, t);
  __syncthreads();
  constexpr int GPW = 32 / VW;
  const long long wid = ((long long)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  const long long nw = ((long long)gridDim.x * blockDim.x) >> 5;
  const int lane = lane_id();
  const int gi = lane / VW, li = lane % VW;
  long long acc = 0;
  for (long long vb = wid * GPW; vb < n; vb += nw * GPW) {
    const int v = (int)(vb + gi);
    if (v < n && to_move[v]) {
      const int ov = part[v], nv = dest[v];
      const unsigned long long oc = __ldg(t.code + ov), nc = __ldg(t.code + nv);
      for (int e = off[v] + li; e < off[v + 1]; e += VW) {
        int u = tgt[e];
        bool um = to_move[u];
        int ou = part[u];
        int nu = um ? dest[u] : ou;
        long long d = cdist(s_dbit, nc, __ldg(t.code + nu)) - cdist(s_dbit, oc, __ldg(t.code + ou));
        acc += (long long)w[e] * d * (um ? 1 : 2);
      }
      if (li == 0 && ov != nv) {
        atomicAdd(reinterpret_cast<unsigned long long*>(&bw[ov]), (unsigned long long)(-(long long)vw[v]));
        atomicAdd(reinterpret_cast<unsigned long long*>(&bw[nv]), (unsigned long long)(long long)vw[v]);
      }
    }
  }
  block_sum_atomic<256>(acc, dj);
}

__global__ void k_commit(int n, const unsigned char* __restrict__ to_move,
                         const int* __restrict__ dest, int* __restrict__ part) {
  for (int v = blockIdx.x * blockDim.x + threadIdx.x; v < n; v += gridDim.x * blockDim.x)
    if (to_move[v]) part[v] = dest[v];
}

// ---------------------------------------------------------------------------
// K12 rebalance selection (refinement.py:333-346 weak, 371-385 strong).
// Candidates are compacted in vertex order (the reference visits source
// blocks ascending, vertices ascending; since the sort key starts with the
// block this is equivalent), stably radix-sorted by
//   weak:   (source, cell)            cell = slot(gain) * rho + v % rho
//   strong: (target, cell, source)
// and a segmented prefix of vertex weights selects the taken prefix:
//   weak: exclusive prefix < bw[src] - l_max;  strong: inclusive <= l_max - bw[tgt].


struct RbFlag {
  const int* part;
  const unsigned char* ovl;
  const int* target;
  __device__ int operator()(long long v) const { return (ovl[part[v]] && target[v] >= 0) ? 1 : 0; }
};

struct RbKeyOut {
  RbFlag f;
  const long long* gain;
  int rho, k, strong, dshift;
  unsigned int* keys;
  int* vals;
  __device__ void operator()(long long v, int pos) const {
    if (!f(v)) return;
    int src = f.part[v];
    int tb = f.target[v];
    unsigned cell = (unsigned)(slot_for_gain(gain[v], dshift) * rho + (int)(v % rho));
    unsigned ncell = 31u * (unsigned)rho;
    unsigned key = strong ? ((unsigned)tb * ncell + cell) * (unsigned)k + (unsigned)src
                          : (unsigned)src * ncell + cell;
    keys[pos] = key;
    vals[pos] = (int)v;
  }
};

struct RbWeight {
  const int* vals;
  const int* vw;
  __device__ long long operator()(long long i) const { return vw[vals[i]]; }
};

__global__ void k_rb_group_start(int cnt, const unsigned int* __restrict__ keys, unsigned div,
                                 int* __restrict__ gstart) {
  for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < cnt; i += gridDim.x * blockDim.x) {
    unsigned gcur = keys[i] / div;
    if (i == 0 || keys[i - 1] / div != gcur) gstart[gcur] = i;
  }
}

__global__ void k_rb_select(int cnt, int strong, const unsigned int* __restrict__ keys,
                            unsigned div, const int* __restrict__ vals,
                            const long long* __restrict__ excl, const int* __restrict__ vw,
                            const int* __restrict__ gstart, const long long* __restrict__ bw,
                            double l_max, const int* __restrict__ target,
                            unsigned char* __restrict__ to_move, int* __restrict__ dest,
                            long long* __restrict__ movers) {
  long long moved = 0;
  for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < cnt; i += gridDim.x * blockDim.x) {
    unsigned grp = keys[i] / div;
    long long before = excl[i] - excl[gstart[grp]];
    int v = vals[i];
    bool take;
    if (strong) {
      double room = l_max - (double)bw[grp];
      take = (double)(before + vw[v]) <= room;
    } else {
      double excess = (double)bw[grp] - l_max;
      take = (double)before < excess;
    }
    if (take) {
      to_move[v] = 1;
      dest[v] = target[v];
      ++moved;
    }
  }
  if (moved) atomicAdd(reinterpret_cast<unsigned long long*>(movers), (unsigned long long)moved);
}

// ---------------------------------------------------------------------------
// host wrappers

static void launch_eval(const RefineLevel& L, int mode, const Topo& t, const int* part,
                        const LpParams& lp, const LpOut& lo, const RbParams& rb,
                        const RbOut& ro, long long* ctr, cudaStream_t s) {
  const DevGraph& g = L.g;
  // LP first filter / rebalance candidates: every CSR row once (target,
  // weight, Pi[target] = 12 B/slot) + offsets, Pi, lock and the three
  // per-vertex outputs (22 B/vertex)
  ProfScope prof(mode == 0 ? P_LP_EVAL : P_REBALANCE, 22.0 * g.n + 12.0 * g.m2, s);
  constexpr int B = 256;
  long long groups = (long long)g.n * L.vw;
  int grid = grid_for(groups, B, kSMs * 8);
  switch (L.vw) {
    case 4: k_eval_regs<4><<<grid, B, 0, s>>>(mode, g.n, g.off, g.tgt, g.w, part, t, lp, lo, rb, ro, ctr); break;
    case 8: k_eval_regs<8><<<grid, B, 0, s>>>(mode, g.n, g.off, g.tgt, g.w, part, t, lp, lo, rb, ro, ctr); break;
    case 16: k_eval_regs<16><<<grid, B, 0, s>>>(mode, g.n, g.off, g.tgt, g.w, part, t, lp, lo, rb, ro, ctr); break;
    default: k_eval_regs<32><<<grid, B, 0, s>>>(mode, g.n, g.off, g.tgt, g.w, part, t, lp, lo, rb, ro, ctr); break;
  }
  count_launch();
  if (L.n_heavy > 0) {
    int k = t.k;
    size_t smem = (size_t)4 * 3 * k * sizeof(int);
    // dynamic + the kernel's static shared memory may pass 48 KB before the
    // dynamic part alone does (k = 1024): always raise the opt-in limit
    static int configured_smem = 0;
    if ((int)smem > configured_smem) {
      GIM_CUDA(cudaFuncSetAttribute(k_eval_table, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                    (int)smem));
      configured_smem = (int)smem;
    }
    int hgrid = grid_for((long long)L.n_heavy * 32, 128, kSMs * 4);
    k_eval_table<<<hgrid, 128, smem, s>>>(mode, L.n_heavy, L.heavy.get(), k, g.off, g.tgt, g.w,
                                          part, t, lp, lo, rb, ro);
    count_launch();
  }
  GIM_LAUNCH_CHECK();
}

struct HeavyFlag {
  const int* off;
  int vw;
  __device__ int operator()(long long v) const { return off[v + 1] - off[v] > vw ? 1 : 0; }
};
struct HeavyOut {
  HeavyFlag f;
  int* out;
  __device__ void operator()(long long v, int pos) const {
    if (f(v)) out[pos] = (int)v;
  }
};

void prepare_level_vw(RefineLevel& L) {
  const DevGraph& g = L.g;
  double avg = g.n ? (double)g.m2 / g.n : 0.0;
  L.vw = avg <= 3.0 ? 4 : avg <= 6.0 ? 8 : avg <= 12.0 ? 16 : 32;
}

void prepare_level(RefineLevel& L, int k, cudaStream_t s) {
  const DevGraph& g = L.g;
  prepare_level_vw(L);
  GIM_CHECK((long long)k * 12 * 4 <= 200 * 1024 || g.n == 0, GIM_E_UNSUPPORTED,
            "k too large for the shared-memory connectivity table (k <= 4266)");
  L.heavy = DBuf<int>((size_t)std::max(g.n, 1), s);
  DBuf<int> cnt(1, s);
  HeavyFlag f{g.off, L.vw};
  exclusive_scan<int>(g.n, f, HeavyOut{f, L.heavy.get()}, cnt.get(), s);
  int h = 0;
  if (g.n) {
    GIM_CUDA(cudaMemcpyAsync(&h, cnt.get(), sizeof(int), cudaMemcpyDeviceToHost, s));
    GIM_CUDA(sync_stream(s));
  }
  L.n_heavy = h;
}

void lp_pass(const RefineLevel& L, const Topo& t, const int* part, const unsigned char* locked,
             int jet, double jet_c, RefineBuffers& rb, cudaStream_t s) {
  const DevGraph& g = L.g;
  LpParams lp{locked, jet, jet_c, t.dshift};
  LpOut lo{rb.cand.get(), rb.dest.get(), rb.gkey.get()};
  RbParams rp{};
  RbOut ro{};
  launch_eval(L, 0, t, part, lp, lo, rp, ro, rb.ctr.get(), s);
  ProfScope prof(P_LP_SECOND, 6.0 * g.n, s);  // lower bound: candidate rows not counted
  constexpr int B = 256;
  int grid = grid_for((long long)g.n * L.vw, B, kSMs * 8);
  switch (L.vw) {
    case 4: k_lp_second<4><<<grid, B, 0, s>>>(g.n, g.off, g.tgt, g.w, part, t, rb.cand.get(), rb.dest.get(), rb.gkey.get(), rb.to_move.get(), rb.movers); break;
    case 8: k_lp_second<8><<<grid, B, 0, s>>>(g.n, g.off, g.tgt, g.w, part, t, rb.cand.get(), rb.dest.get(), rb.gkey.get(), rb.to_move.get(), rb.movers); break;
    case 16: k_lp_second<16><<<grid, B, 0, s>>>(g.n, g.off, g.tgt, g.w, part, t, rb.cand.get(), rb.dest.get(), rb.gkey.get(), rb.to_move.get(), rb.movers); break;
    default: k_lp_second<32><<<grid, B, 0, s>>>(g.n, g.off, g.tgt, g.w, part, t, rb.cand.get(), rb.dest.get(), rb.gkey.get(), rb.to_move.get(), rb.movers); break;
  }
  count_launch();
  GIM_LAUNCH_CHECK();
}

void rebalance_pass(const RefineLevel& L, const Topo& t, const int* part, const long long* bw,
                    bool strong, double l_max, int rho, unsigned long long seed,
                    long long pass_counter, const unsigned char* ovl, const unsigned char* elig,
                    const int* elig_list, int n_elig, RefineBuffers& rb, cudaStream_t s) {
  const DevGraph& g = L.g;
  const int k = t.k;
  LpParams lp{};
  LpOut lo{};
  RbParams rp{ovl, elig, elig_list, n_elig, seed, pass_counter};
  RbOut ro{rb.dest2.get(), rb.gkey.get(), rb.to_move.get()};
  launch_eval(L, 1, t, part, lp, lo, rp, ro, rb.ctr.get(), s);
  // compaction in vertex order + keys
  RbFlag f{part, ovl, rb.dest2.get()};
  RbKeyOut ko{f, rb.gkey.get(), rho, k, strong ? 1 : 0, t.dshift, rb.rkeys.get(), rb.rvals.get()};
  exclusive_scan<int>(g.n, f, ko, rb.count.get(), s);
  int cnt = 0;
  GIM_CUDA(cudaMemcpyAsync(&cnt, rb.count.get(), sizeof(int), cudaMemcpyDeviceToHost, s));
  GIM_CUDA(sync_stream(s));
  if (cnt == 0) return;
  unsigned ncell = 31u * (unsigned)rho;
  unsigned long long maxkey = strong ? (unsigned long long)k * ncell * k : (unsigned long long)k * ncell;
  GIM_CHECK(maxkey < (1ull << 32), GIM_E_UNSUPPORTED, "rebalance key exceeds 32 bits");
  radix_sort_pairs<unsigned int, int>(cnt, rb.rkeys.get(), rb.rvals.get(), rb.rkeys2.get(),
                                      rb.rvals2.get(), bit_length(maxkey), s);
  unsigned div = strong ? ncell * (unsigned)k : ncell;
  exclusive_scan<long long>(cnt, RbWeight{rb.rvals.get(), g.vw}, StoreTo<long long>{rb.rexcl.get()},
                            (long long*)nullptr, s);
  int grid = grid_for(cnt, 256);
  k_rb_group_start<<<grid, 256, 0, s>>>(cnt, rb.rkeys.get(), div, rb.gstart.get());
  k_rb_select<<<grid, 256, 0, s>>>(cnt, strong ? 1 : 0, rb.rkeys.get(), div, rb.rvals.get(),
                                   rb.rexcl.get(), g.vw, rb.gstart.get(), bw, l_max,
                                   rb.dest2.get(), rb.to_move.get(), rb.dest.get(),
                                   rb.movers);
  count_launch(2);
  GIM_LAUNCH_CHECK();
}

void apply_moves(const RefineLevel& L, const Topo& t, int* part, long long* bw,
                 RefineBuffers& rb, cudaStream_t s) {
  const DevGraph& g = L.g;
  // rb.dj was zeroed by the candidate pass of this iteration
  ProfScope prof(P_APPLY, 6.0 * g.n, s);  // lower bound: mover rows not counted
  constexpr int B = 256;
  int grid = grid_for((long long)g.n * L.vw, B, kSMs * 8);
  switch (L.vw) {
    case 4: k_apply_delta<4><<<grid, B, 0, s>>>(g.n, g.off, g.tgt, g.w, g.vw, part, t, rb.to_move.get(), rb.dest.get(), bw, rb.dj); break;
    case 8: k_apply_delta<8><<<grid, B, 0, s>>>(g.n, g.off, g.tgt, g.w, g.vw, part, t, rb.to_move.get(), rb.dest.get(), bw, rb.dj); break;
    case 16: k_apply_delta<16><<<grid, B, 0, s>>>(g.n, g.off, g.tgt, g.w, g.vw, part, t, rb.to_move.get(), rb.dest.get(), bw, rb.dj); break;
    default: k_apply_delta<32><<<grid, B, 0, s>>>(g.n, g.off, g.tgt, g.w, g.vw, part, t, rb.to_move.get(), rb.dest.get(), bw, rb.dj); break;
  }
  k_commit<<<grid_for(g.n, 256), 256, 0, s>>>(g.n, rb.to_move.get(), rb.dest.get(), part);
  count_launch(2);
  GIM_LAUNCH_CHECK();
}

// (re)allocate only when the buffers are smaller than needed, so one set
// serves every level of a mapping (finest level first in size order)
void alloc_refine_buffers(RefineBuffers& rb, int n, int k, cudaStream_t s) {
  if (rb.cap_n >= std::max(n, 1) && rb.cap_k >= k && rb.ctr.get()) return;
  rb.cap_n = std::max(n, 1);
  rb.cap_k = k;
  size_t nn = (size_t)std::max(n, 1);
  rb.cand = DBuf<unsigned char>(nn, s);
  rb.to_move = DBuf<unsigned char>(2 * nn, s);  // 2 bytes per vertex: fused-loop move stamps
  rb.locks = DBuf<unsigned char>(nn, s);
  rb.dest = DBuf<int>(nn, s);
  rb.dest2 = DBuf<int>(nn, s);
  rb.gkey = DBuf<long long>(nn, s);
  rb.rkeys = DBuf<unsigned int>(nn, s);
  rb.rkeys2 = DBuf<unsigned int>(nn, s);
  rb.rvals = DBuf<int>(nn, s);
  rb.rvals2 = DBuf<int>(nn, s);
  rb.rexcl = DBuf<long long>(nn, s);
  rb.gstart = DBuf<int>((size_t)k * 31 * 8 + 1, s);
  rb.count = DBuf<int>(1, s);
  rb.ctr = DBuf<long long>(2, s);
  rb.movers = rb.ctr.get();
  rb.dj = rb.ctr.get() + 1;
  GIM_CUDA(cudaMemsetAsync(rb.ctr.get(), 0, 2 * sizeof(long long), s));
  rb.masks = DBuf<unsigned char>((size_t)k * 2, s);
  rb.elist = DBuf<int>((size_t)k, s);
  rb.jtmp = DBuf<long long>(1, s);
  rb.best = DBuf<int>(nn, s);
  rb.best_bw = DBuf<long long>((size_t)k, s);
  rb.fctr = DBuf<long long>(17, s);
  rb.bstamp = DBuf<int>(nn, s);
  rb.lists = DBuf<int>(nn * 5, s);
  rb.rcell = DBuf<unsigned char>(nn, s);
  rb.fstate = DBuf<unsigned char>(sizeof(FusedState), s);
}

// ---------------------------------------------------------------------------
// K8 connectivity table (parity unit; mapping.py:141-158): per vertex the
// sorted (block, conn) list, built by the same key-sort + segmented reduce
// as contraction with key (v, Pi(u)).

__global__ void k_conn_keys(long long m2, const int* __restrict__ src, const int* __restrict__ tgt,
                            const int* __restrict__ w, const int* __restrict__ part, int k,
                            unsigned long long* __restrict__ keys, int* __restrict__ vals) {
  for (long long e = (long long)blockIdx.x * blockDim.x + threadIdx.x; e < m2;
       e += (long long)gridDim.x * blockDim.x) {
    keys[e] = (unsigned long long)src[e] * (unsigned long long)k + (unsigned long long)part[tgt[e]];
    vals[e] = w[e];
  }
}

struct ConnHead {
  const unsigned long long* keys;
  __device__ int operator()(long long i) const { return (i == 0 || keys[i] != keys[i - 1]) ? 1 : 0; }
};
struct ConnOut {
  const unsigned long long* keys;
  const int* vals;
  long long m2;
  int k;
  int* blocks;
  int* cw;
  int* deg;
  __device__ void operator()(long long i, int uid) const {
    if (i > 0 && keys[i] == keys[i - 1]) return;
    long long sum = 0;
    long long j = i;
    while (j < m2 && keys[j] == keys[i]) sum += vals[j++];
    blocks[uid] = (int)(keys[i] % (unsigned long long)k);
    cw[uid] = (int)sum;
    atomicAdd(&deg[keys[i] / (unsigned long long)k], 1);
  }
};

long long conn_build(const DevGraph& g, const int* part, int k, int* c_off, int* c_blocks,
                     int* c_w, cudaStream_t s) {
  if (g.m2 == 0) {
    GIM_CUDA(cudaMemsetAsync(c_off, 0, sizeof(int) * ((size_t)g.n + 1), s));
    return 0;
  }
  DBuf<unsigned long long> keys((size_t)g.m2, s), keys2((size_t)g.m2, s);
  DBuf<int> vals((size_t)g.m2, s), vals2((size_t)g.m2, s), deg((size_t)g.n + 1, s), tot(1, s);
  k_conn_keys<<<grid_for(g.m2, 256), 256, 0, s>>>(g.m2, g.src, g.tgt, g.w, part, k, keys.get(),
                                                  vals.get());
  count_launch();
  GIM_LAUNCH_CHECK();
  radix_sort_pairs<unsigned long long, int>(g.m2, keys.get(), vals.get(), keys2.get(), vals2.get(),
                                            bit_length((unsigned long long)g.n * k), s);
  GIM_CUDA(cudaMemsetAsync(deg.get(), 0, sizeof(int) * ((size_t)g.n + 1), s));
  ConnOut out{keys.get(), vals.get(), g.m2, k, c_blocks, c_w, deg.get()};
  exclusive_scan<int>(g.m2, ConnHead{keys.get()}, out, tot.get(), s);
  exclusive_scan<int>((long long)g.n + 1, LoadAs<int, int>{deg.get()}, StoreTo<int>{c_off},
                      (int*)nullptr, s);
  int total = 0;
  GIM_CUDA(cudaMemcpyAsync(&total, tot.get(), sizeof(int), cudaMemcpyDeviceToHost, s));
  GIM_CUDA(sync_stream(s));
  return total;
}

}  // namespace gim
