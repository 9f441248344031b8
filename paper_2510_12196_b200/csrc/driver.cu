// Host driver (native runtime): level stack, Alg. 4 refinement control,
// hierarchical multisection with the internal partitioner, integrated_map —
// plus the C-ABI entry points of include/gpuim.h.
//
// All float threshold math (l_max, sigma, excess/room, phi * J, match
// fractions, Eq. 2) is evaluated on the host in IEEE double with the same
// operation order as the reference's Python float expressions, so control
// decisions agree bit-for-bit; kernels only see the resulting doubles.
#include <array>
#include <atomic>
#include <cstdio>
#include <cstdlib>
#include <chrono>
#include <cmath>
#include <exception>
#include <thread>
#include <queue>
#include <algorithm>
#include <vector>

#include "common.cuh"
#include "kernels.cuh"
#include "scan.cuh"

namespace gim {

void greedy_graph_growing(const DevGraph& g, int k, int* part, cudaStream_t s);
void fill_sources(int n, const int* off, int* src, cudaStream_t s);
void extract_subgraphs(const DevGraph& g, const int* part, int parts,
                       std::vector<OwnedGraph>& subs, std::vector<DBuf<int>>& ids,
                       cudaStream_t s);
void gather(int n, const int* idx, const int* src, int* dst, cudaStream_t s);
void scatter_const(int n, const int* idx, int value, int* dst, cudaStream_t s);
void leaf_scatter(int n, const int* idx, const int* part, int base, int* dst, cudaStream_t s);

// ---------------------------------------------------------------------------
// run statistics

struct RunStats {  // shared by the multisection worker threads
  std::atomic<long long> refine_iterations{0}, lp{0}, weak{0}, strong{0};
  std::atomic<long long> init_refine_iterations{0}, partitioner_calls{0};
  std::atomic<bool> in_initial{false};
};

// pinned host scratch (process-wide free list, leased per host thread)
struct Pinned {
  void* get(size_t need) { return pinned_scratch(need); }
};
static Pinned g_pin;

template <class T>
static T read_scalar(const T* d, cudaStream_t s) {
  T* h = static_cast<T*>(g_pin.get(sizeof(T)));
  GIM_CUDA(cudaMemcpyAsync(h, d, sizeof(T), cudaMemcpyDeviceToHost, s));
  GIM_CUDA(sync_stream(s));
  return *h;
}

__global__ void k_sum_vw(int n, const int* __restrict__ vw, long long* out) {
  long long acc = 0;
  for (int v = blockIdx.x * blockDim.x + threadIdx.x; v < n; v += gridDim.x * blockDim.x)
    acc += vw[v];
  block_sum_atomic<256>(acc, out);
}

static long long total_vertex_weight(const DevGraph& g, cudaStream_t s) {
  DBuf<long long> d(1, s);
  GIM_CUDA(cudaMemsetAsync(d.get(), 0, sizeof(long long), s));
  if (g.n) {
    k_sum_vw<<<grid_for(g.n, 256, kSMs * 2), 256, 0, s>>>(g.n, g.vw, d.get());
    count_launch();
  }
  return read_scalar(d.get(), s);
}

__global__ void k_iota(int n, int* p) {
  for (int v = blockIdx.x * blockDim.x + threadIdx.x; v < n; v += gridDim.x * blockDim.x) p[v] = v;
}

// ---------------------------------------------------------------------------
// refinement config (refinement.py:50-101)

struct RefCfg {
  double phi = 0.999;
  int i_max = 12;
  int i_w_max = 2;
  double sigma_fraction = 0.005;
  int rho = 2;
  int jet = 0;
  double jet_c = 0.25;
  unsigned long long seed = 0;
};

static RefCfg config_for_level(int level, int n_levels, double phi, int rho, int jet,
                               double jet_c, double sigma_coarse, double sigma_fine,
                               int iw_max_finest, unsigned long long seed) {
  int span = std::max(n_levels - 1, 1);
  double frac = n_levels > 1 ? (double)level / (double)span : 0.0;
  double delta = sigma_fine + (sigma_coarse - sigma_fine) * frac;
  RefCfg c;
  c.phi = phi;
  c.i_max = 12 + level;
  c.i_w_max = level == 0 ? iw_max_finest : 2;
  c.sigma_fraction = delta;
  c.rho = rho;
  c.jet = jet;
  c.jet_c = jet_c;
  c.seed = seed;
  return c;
}

// ---------------------------------------------------------------------------
// Alg. 4 (refinement.py:389-464).  `part`/`bw` are consumed and replaced by
// the best mapping seen.

// mode flags (RunFlags, per call): fused = device-resident loop (else per-phase
// launches), rowwise = row-wise contraction of matchings (else radix sort),
// batch / fanout = multisection scheduling; results are identical either way

static long long max_of(const std::vector<long long>& x) {
  long long m = 0;
  for (long long y : x) m = std::max(m, y);
  return m;
}

// Alg. 4 with the persistent cooperative kernel (refine_fused.cu); the host
// only performs the rare strong passes the kernel hands back.
// `resume`: continue a refinement whose fused kernel (a batched launch) handed
// back a strong pass; rb.best / rb.best_bw hold its best copy
static void refine_device_loop(RefineLevel& L, const Topo& t, int* part, long long* bw_d,
                               const RefCfg& cfg, double l_max, RunStats& st, RefineBuffers& rb,
                               cudaStream_t s, const FusedState* resume = nullptr) {
  const int n = L.g.n, k = t.k;
  FusedBuffers fb;
  fb.cand = rb.cand.get();
  fb.tm0 = rb.to_move.get();
  fb.tm1 = fb.tm0 + rb.cap_n;  // contiguous with tm0: the fused loop keeps uint16 move stamps in both
  fb.rcell = rb.rcell.get();
  fb.dest = rb.dest.get();
  fb.rtgt = rb.dest2.get();
  fb.best = rb.best.get();
  fb.gkey = rb.gkey.get();
  fb.best_bw = rb.best_bw.get();
  fb.ctr = rb.fctr.get();
  fb.bstamp = rb.bstamp.get();
  fb.wdeg = rb.rvals2.get();  // free during the fused loop (host strong passes only)
  const size_t nn = (size_t)rb.cap_n;
  fb.lsmall = rb.lists.get();
  fb.lheavy = fb.lsmall + nn;
  fb.lcand = fb.lheavy + nn;
  fb.lmov0 = fb.lcand + nn;
  fb.lmov1 = fb.lmov0 + nn;
  fb.state = reinterpret_cast<FusedState*>(rb.fstate.get());
  FusedState hs{};
  fb.h_state = &hs;
  FusedCfg fc;
  fc.l_max = l_max;
  fc.sigma = l_max * (1.0 - cfg.sigma_fraction);
  fc.phi = cfg.phi;
  fc.jet_c = cfg.jet_c;
  fc.jet = cfg.jet;
  fc.rho = cfg.rho;
  fc.i_max = cfg.i_max;
  fc.i_w_max = cfg.i_w_max;
  fc.seed = cfg.seed;
  GIM_CUDA(cudaMemsetAsync(fb.state, 0, sizeof(FusedState), s));
  GIM_CUDA(cudaMemsetAsync(fb.ctr, 0, 17 * sizeof(long long), s));
  bool skip_launch = false;
  if (resume) {
    hs = *resume;
    skip_launch = true;
  }
  long long strong = 0;
  bool host_finished = false;
  std::vector<long long> bw((size_t)k);
  std::vector<unsigned char> masks((size_t)k * 2);
  std::vector<int> el((size_t)k);
  for (;;) {
    if (!skip_launch && refine_fused_run(L, t, part, bw_d, fc, fb, s)) break;
    skip_launch = false;
    // strong pass (refinement.py:350-386) + the same Alg. 4 bookkeeping
    GIM_CUDA(cudaMemcpyAsync(bw.data(), bw_d, sizeof(long long) * k, cudaMemcpyDeviceToHost, s));
    GIM_CUDA(sync_stream(s));
    int ne = 0;
    for (int b = 0; b < k; ++b) {
      masks[b] = (double)bw[b] > l_max;
      masks[k + b] = (double)bw[b] < fc.sigma;
      if (masks[k + b]) el[ne++] = b;
    }
    const bool incomplete = ne == 0;
    if (L.heavy.get() == nullptr) prepare_level(L, k, s);  // host strong pass: heavy list
    GIM_CUDA(cudaMemcpyAsync(rb.masks.get(), masks.data(), (size_t)k * 2, cudaMemcpyHostToDevice, s));
    if (ne)
      GIM_CUDA(cudaMemcpyAsync(rb.elist.get(), el.data(), sizeof(int) * ne, cudaMemcpyHostToDevice, s));
    rebalance_pass(L, t, part, bw_d, true, l_max, cfg.rho, cfg.seed, hs.pass_counter,
                   rb.masks.get(), rb.masks.get() + k, rb.elist.get(), ne, rb, s);
    apply_moves(L, t, part, bw_d, rb, s);
    long long ctr[2];
    GIM_CUDA(cudaMemcpyAsync(bw.data(), bw_d, sizeof(long long) * k, cudaMemcpyDeviceToHost, s));
    GIM_CUDA(cudaMemcpyAsync(ctr, rb.ctr.get(), 2 * sizeof(long long), cudaMemcpyDeviceToHost, s));
    GIM_CUDA(sync_stream(s));
    ++strong;
    ++hs.iters;
    hs.i_w = 0;
    ++hs.pass_counter;
    if (ctr[0] == 0 && incomplete) {
      host_finished = true;
      break;
    }
    hs.J += ctr[1];
    hs.maxw = max_of(bw);
    hs.locks_nonempty = 0;
    bool reset = false, take = false;
    if ((double)hs.maxw <= l_max) {
      if (!hs.best_balanced) {
        hs.best_balanced = 1;
        hs.best_j = hs.J;
        hs.best_maxw = hs.maxw;
        reset = take = true;
      } else if (hs.J < hs.best_j) {
        reset = (double)hs.J < cfg.phi * (double)hs.best_j;
        hs.best_j = hs.J;
        hs.best_maxw = hs.maxw;
        take = true;
      }
    } else if (!hs.best_balanced && hs.maxw < hs.best_maxw) {
      hs.best_maxw = hs.maxw;
      reset = take = true;
    }
    if (take) {
      GIM_CUDA(cudaMemcpyAsync(fb.best, part, sizeof(int) * n, cudaMemcpyDeviceToDevice, s));
      GIM_CUDA(cudaMemcpyAsync(fb.best_bw, bw_d, sizeof(long long) * k, cudaMemcpyDeviceToDevice, s));
    }
    hs.i = reset ? 0 : hs.i + 1;
    if (hs.i >= cfg.i_max) {
      host_finished = true;
      break;
    }
    hs.status = 0;
    hs.started = 1;
    hs.reinit = 1;  // the host pass reused the per-vertex arrays
    hs.prev_n = 0;  // no locks after a rebalance pass
    GIM_CUDA(cudaMemcpyAsync(fb.state, &hs, sizeof(FusedState), cudaMemcpyHostToDevice, s));
    GIM_CUDA(cudaMemsetAsync(fb.ctr, 0, 17 * sizeof(long long), s));
  }
  if (host_finished) {  // restore the best mapping (the kernel does this itself otherwise)
    GIM_CUDA(cudaMemcpyAsync(part, fb.best, sizeof(int) * n, cudaMemcpyDeviceToDevice, s));
    GIM_CUDA(cudaMemcpyAsync(bw_d, fb.best_bw, sizeof(long long) * k, cudaMemcpyDeviceToDevice, s));
    GIM_CUDA(sync_stream(s));
  }
  st.lp += hs.lp;
  st.weak += hs.weak;
  st.strong += strong;
  if (!st.in_initial)  // IM-level refinement counters (SURVEY §8(d) accounting)
    for (int i = 0; i < A_COUNT; ++i) ctx().acct[i].fetch_add(hs.acct[i]);
  if (st.in_initial) st.init_refine_iterations += hs.iters;
  else st.refine_iterations += hs.iters;
}

static void refine(RefineLevel& L, const Topo& t, int* part, long long* bw_d, const RefCfg& cfg,
                   double l_max, RunStats& st, RefineBuffers& rb, cudaStream_t s) {
  const int n = L.g.n, k = t.k;
  prepare_level_vw(L);
  alloc_refine_buffers(rb, n, k, s);
  const bool aligned = ((reinterpret_cast<uintptr_t>(L.g.src) |
                         reinterpret_cast<uintptr_t>(L.g.tgt)) & 15) == 0;
  if (ctx().f.fused && fused_supported(k, cfg.rho) && n > 0 && aligned) {
    refine_device_loop(L, t, part, bw_d, cfg, l_max, st, rb, s);
    return;
  }
  if (L.heavy.get() == nullptr) prepare_level(L, k, s);
  // host mirrors
  size_t pin_bytes = sizeof(long long) * ((size_t)k + 2) + (size_t)k * 2 + sizeof(int) * (size_t)k;
  char* pin = static_cast<char*>(g_pin.get(pin_bytes));
  long long* h_bw = reinterpret_cast<long long*>(pin);
  long long* h_mv = h_bw + k;
  long long* h_dj = h_mv + 1;
  unsigned char* h_ovl = reinterpret_cast<unsigned char*>(h_dj + 1);
  unsigned char* h_elig = h_ovl + k;
  int* h_elist = reinterpret_cast<int*>(h_elig + k);
  unsigned char* d_masks = rb.masks.get();
  int* d_elist = rb.elist.get();

  total_cost(L.g, part, t, rb.jtmp.get(), s);
  GIM_CUDA(cudaMemcpyAsync(h_dj, rb.jtmp.get(), sizeof(long long), cudaMemcpyDeviceToHost, s));
  GIM_CUDA(cudaMemcpyAsync(h_bw, bw_d, sizeof(long long) * k, cudaMemcpyDeviceToHost, s));
  GIM_CUDA(sync_stream(s));
  long long J = *h_dj;
  std::vector<long long> bw(h_bw, h_bw + k);
  auto maxof = [&](const std::vector<long long>& x) {
    long long m = 0;
    for (long long y : x) m = std::max(m, y);
    return m;
  };
  const double sigma = l_max * (1.0 - cfg.sigma_fraction);
  DBuf<int> best((size_t)std::max(n, 1), s);
  GIM_CUDA(cudaMemcpyAsync(best.get(), part, sizeof(int) * n, cudaMemcpyDeviceToDevice, s));
  std::vector<long long> best_bw = bw;
  long long maxw = maxof(bw);
  bool best_balanced = (double)maxw <= l_max;
  long long best_j = J;
  long long best_maxw = maxw;
  bool locks_nonempty = false;
  int i = 0, i_w = 0;
  long long pass_counter = 0;
  while (i < cfg.i_max) {
    const bool balanced_now = (double)maxw <= l_max;
    const bool entry_locks_empty = !locks_nonempty;
    bool incomplete = false;
    bool is_lp = balanced_now;
    if (balanced_now) {
      lp_pass(L, t, part, locks_nonempty ? rb.locks.get() : nullptr, cfg.jet, cfg.jet_c, rb, s);
      i_w = 0;
      ++st.lp;
    } else {
      locks_nonempty = false;
      int ne = 0;
      for (int b = 0; b < k; ++b) {
        h_ovl[b] = (double)bw[b] > l_max;
        h_elig[b] = (double)bw[b] < sigma;
        if (h_elig[b]) h_elist[ne++] = b;
      }
      incomplete = ne == 0;
      GIM_CUDA(cudaMemcpyAsync(d_masks, h_ovl, (size_t)k * 2, cudaMemcpyHostToDevice, s));
      if (ne)
        GIM_CUDA(cudaMemcpyAsync(d_elist, h_elist, sizeof(int) * ne, cudaMemcpyHostToDevice, s));
      bool strong = !(i_w < cfg.i_w_max);
      rebalance_pass(L, t, part, bw_d, strong, l_max, cfg.rho, cfg.seed, pass_counter,
                     d_masks, d_masks + k, d_elist, ne, rb, s);
      if (strong) {
        i_w = 0;
        ++st.strong;
      } else {
        ++i_w;
        ++st.weak;
      }
      ++pass_counter;
    }
    apply_moves(L, t, part, bw_d, rb, s);
    GIM_CUDA(cudaMemcpyAsync(h_bw, bw_d, sizeof(long long) * k, cudaMemcpyDeviceToHost, s));
    GIM_CUDA(cudaMemcpyAsync(h_mv, rb.ctr.get(), 2 * sizeof(long long), cudaMemcpyDeviceToHost, s));
    GIM_CUDA(sync_stream(s));
    if (st.in_initial) ++st.init_refine_iterations;
    else ++st.refine_iterations;
    const long long movers = *h_mv;
    if (movers == 0) {
      if (balanced_now && entry_locks_empty) break;   // fixed point
      if (!balanced_now && incomplete) break;         // rebalancing is stuck
    }
    J += *h_dj;
    bw.assign(h_bw, h_bw + k);
    maxw = maxof(bw);
    if (is_lp) {
      std::swap(rb.locks, rb.to_move);  // locks for the next pass = the moved set
      locks_nonempty = movers > 0;
    } else {
      locks_nonempty = false;
    }
    bool reset = false;
    bool take = false;
    if ((double)maxw <= l_max) {
      if (!best_balanced) {
        best_balanced = true;
        best_j = J;
        best_maxw = maxw;
        reset = take = true;
      } else if (J < best_j) {
        reset = (double)J < cfg.phi * (double)best_j;
        best_j = J;
        best_maxw = maxw;
        take = true;
      }
    } else if (!best_balanced && maxw < best_maxw) {
      best_maxw = maxw;
      reset = take = true;
    }
    if (take) {
      GIM_CUDA(cudaMemcpyAsync(best.get(), part, sizeof(int) * n, cudaMemcpyDeviceToDevice, s));
      best_bw = bw;
    }
    i = reset ? 0 : i + 1;
  }
  GIM_CUDA(cudaMemcpyAsync(part, best.get(), sizeof(int) * n, cudaMemcpyDeviceToDevice, s));
  std::copy(best_bw.begin(), best_bw.end(), h_bw);
  GIM_CUDA(cudaMemcpyAsync(bw_d, h_bw, sizeof(long long) * k, cudaMemcpyHostToDevice, s));
  GIM_CUDA(sync_stream(s));
}

// ---------------------------------------------------------------------------
// level stack (coarsening.py:164-173, 280-295)

struct Level {
  OwnedGraph own;       // empty for the input level
  DevGraph g;
  DBuf<int> cmap;       // fine -> coarse (absent on the coarsest level)
  int n_c = 0;
  RefineLevel rl;
};

static long long match_graph(const DevGraph& g, double l_max, unsigned long long seed,
                             int* partner, cudaStream_t s) {
  GIM_CUDA(cudaMemsetAsync(partner, 0xff, sizeof(int) * (size_t)std::max(g.n, 1), s));
  DBuf<int> pref((size_t)std::max(g.n, 1), s);
  DBuf<long long> matched(1, s);
  GIM_CUDA(cudaMemsetAsync(matched.get(), 0, sizeof(long long), s));
  long long m = 0;
  auto frac = [&](long long x) { return g.n ? (double)x / (double)g.n : 1.0; };
  for (int r = 0; r < 2; ++r) {
    if (frac(m) >= 0.40) break;
    hem_round(g, partner, pref.get(), l_max, splitmix64(seed ^ (unsigned long long)(r + 1)),
              matched.get(), s);
    m = read_scalar(matched.get(), s);
  }
  if (frac(m) < 0.40) m = two_hop(g, partner, l_max, m, matched.get(), s);
  return m;
}

// `first`: index of g0 in the whole stack (a continuation of a stack whose
// first levels were built elsewhere uses the same per-level seeds)
static std::vector<Level> build_level_stack(const DevGraph& g0, double l_max, long long threshold,
                                            unsigned long long seed, cudaStream_t s,
                                            int first = 0) {
  std::vector<Level> levels;
  levels.emplace_back();
  levels.back().g = g0;
  // 2m of levels built by the one-round-trip path, read back in one copy
  constexpr int kMaxPending = 64;
  DBuf<int> m2c(kMaxPending, s);
  std::vector<int> pending;  // level indices
  auto resolve = [&] {
    if (pending.empty()) return;
    int* h = static_cast<int*>(pinned_scratch(sizeof(int) * kMaxPending));
    GIM_CUDA(cudaMemcpyAsync(h, m2c.get(), sizeof(int) * kMaxPending, cudaMemcpyDeviceToHost, s));
    GIM_CUDA(sync_stream(s));
    for (size_t i = 0; i < pending.size(); ++i) {
      Level& L = levels[(size_t)pending[i]];
      L.own.m2 = h[i];
      L.g.m2 = h[i];
    }
    pending.clear();
  };
  for (;;) {
    Level& cur = levels.back();
    if ((long long)cur.g.n < threshold) break;
    DBuf<int> partner((size_t)std::max(cur.g.n, 1), s);
    unsigned long long lseed =
        splitmix64(seed ^ (unsigned long long)(first + levels.size() - 1));
    DBuf<int> cmap((size_t)std::max(cur.g.n, 1), s);
    int n_c = 0;
    Level next;
    if (ctx().f.rowwise && (int)pending.size() < kMaxPending) {
      long long m = 0, true_m2 = -1;
      bool stalled = false;
      // the current level's 2m, if still on the device, rides on this round trip
      const bool cur_pending = !pending.empty() && pending.back() == (int)levels.size() - 1;
      const int* cur_m2_dev = cur_pending ? m2c.get() + (pending.size() - 1) : nullptr;
      const bool ok = coarsen_level_fast(cur.g, l_max, lseed, partner.get(), cmap.get(), &n_c,
                                         &m, next.own, m2c.get() + pending.size(), &stalled,
                                         cur_m2_dev, &true_m2, s);
      if (cur_pending) {
        cur.own.m2 = true_m2;
        cur.g.m2 = true_m2;
      }
      if (ok) {
        if (stalled) break;
        next.g = next.own.view();
        cur.cmap = std::move(cmap);
        cur.n_c = n_c;
        pending.push_back((int)levels.size());
        levels.push_back(std::move(next));
        continue;
      }
      // this level needs the general code: two-hop matching / hub rows
      resolve();
      Level& c2 = levels.back();
      DBuf<long long> md(1, s);
      if ((c2.g.n ? (double)m / (double)c2.g.n : 1.0) < 0.40)
        two_hop(c2.g, partner.get(), l_max, m, md.get(), s);
      n_c = coarse_map(c2.g.n, partner.get(), cmap.get(), s);
      if ((double)n_c * 1.02 > (double)c2.g.n) break;  // stall guard
      contract_matching(c2.g, cmap.get(), partner.get(), n_c, next.own, s);
      next.g = next.own.view();
      c2.cmap = std::move(cmap);
      c2.n_c = n_c;
      levels.push_back(std::move(next));
      continue;
    }
    resolve();
    match_graph(cur.g, l_max, lseed, partner.get(), s);
    n_c = coarse_map(cur.g.n, partner.get(), cmap.get(), s);
    if ((double)n_c * 1.02 > (double)cur.g.n) break;  // stall guard
    if (ctx().f.rowwise)
      contract_matching(cur.g, cmap.get(), partner.get(), n_c, next.own, s);
    else
      contract(cur.g, cmap.get(), n_c, next.own, s);
    next.g = next.own.view();
    cur.cmap = std::move(cmap);
    cur.n_c = n_c;
    levels.push_back(std::move(next));
  }
  resolve();
  return levels;
}

// ---------------------------------------------------------------------------
// GIM_TRACE_MS: host-wall ms of the multisection's tree levels and of the
// general-path partitioner's phases (stream-synchronised; diagnostics only)
static bool trace_ms() {
  static const bool on = std::getenv("GIM_TRACE_MS") != nullptr;
  return on;
}

struct MsTimer {
  bool on;
  cudaStream_t s;
  std::chrono::steady_clock::time_point t0;
  MsTimer(cudaStream_t st) : on(trace_ms()), s(st) {
    if (on) {
      sync_stream(s);
      t0 = std::chrono::steady_clock::now();
    }
  }
  double lap() {
    if (!on) return 0.0;
    sync_stream(s);
    const auto t1 = std::chrono::steady_clock::now();
    const double ms = std::chrono::duration<double, std::milli>(t1 - t0).count();
    t0 = t1;
    return ms;
  }
};

// ---------------------------------------------------------------------------
// internal partitioner (pipelines.py:191-218)

static void internal_partitioner(const DevGraph& g, long long total, int parts, double eps_local,
                                 unsigned long long seed, int* part, RunStats& st, cudaStream_t s) {
  const int n = g.n;
  ++st.partitioner_calls;
  if (parts <= 1 || n == 0) {
    GIM_CUDA(cudaMemsetAsync(part, 0, sizeof(int) * (size_t)std::max(n, 1), s));
    return;
  }
  if (n <= parts) {
    k_iota<<<grid_for(n, 256), 256, 0, s>>>(n, part);
    count_launch();
    return;
  }
  Topo tf = get_flat_topo(parts);
  const double l_max = (1.0 + eps_local) * (double)total / (double)parts;
  MsTimer tm(s);
  std::vector<Level> levels =
      build_level_stack(g, l_max, std::max<long long>(64ll * parts, 2), seed, s);
  const double t_stack = tm.lap();
  const int nl = (int)levels.size();
  DBuf<int> cur((size_t)std::max(levels.back().g.n, 1), s);
  greedy_graph_growing(levels.back().g, parts, cur.get(), s);
  const double t_ggg = tm.lap();
  DBuf<long long> bw((size_t)parts, s);
  RefineBuffers rb;
  alloc_refine_buffers(rb, g.n, parts, s);  // finest level: serves all levels
  for (int li = nl - 1; li >= 0; --li) {
    Level& L = levels[li];
    if (li < nl - 1) {
      DBuf<int> fine((size_t)std::max(L.g.n, 1), s);
      project(L.g.n, L.cmap.get(), cur.get(), fine.get(), s);
      cur = std::move(fine);
    }
    block_weights(L.g.n, L.g.vw, cur.get(), parts, bw.get(), s);
    RefCfg cfg = config_for_level(li, nl, 0.999, 2, 1, 0.25, 0.065, 0.005, 10,
                                  hash2(seed, 101, (unsigned long long)li));
    L.rl.g = L.g;
    refine(L.rl, tf, cur.get(), bw.get(), cfg, l_max, st, rb, s);
  }
  GIM_CUDA(cudaMemcpyAsync(part, cur.get(), sizeof(int) * n, cudaMemcpyDeviceToDevice, s));
  if (tm.on)
    std::fprintf(stderr, "partitioner n=%d parts=%d levels=%d coarsest=%d | stack %.3f ms ggg %.3f ms refine %.3f ms\n",
                 n, parts, nl, levels.back().g.n, t_stack, t_ggg, tm.lap());
}

// ---------------------------------------------------------------------------
// batched internal partitioner for small subgraphs (batch.cu): same results
// as internal_partitioner() per job, one launch per phase for all jobs

struct BatchPartJob {
  DevGraph g;
  long long total;
  double eps_local;
  unsigned long long seed;
  int* out_part;  // [g.n]
};

// batch-eligible: small enough that every level refines shared-memory resident
constexpr int kBatchMaxN = 16384;  // batched extraction (CTA per node)
// Tree levels whose nodes are all at most this large are partitioned by the
// batched path; larger nodes run the general path, one host thread / stream
// each.  Measured at rgg 2^22, H=4:8:6 (scripts/ab_env.sh): the six ~4K-vertex
// nodes of tree level 2 take 10 ms batched (the slowest job's refinement
// gates every per-level launch) and ~3 ms concurrently on the general path;
// initial mapping 19.5 -> 15.6 ms.  GIM_BATCH_MAXN overrides.
constexpr int kBatchPartMaxN = 2048;
static int batch_max_n() {
  static const int v = [] {
    const char* e = std::getenv("GIM_BATCH_MAXN");
    return e ? std::atoi(e) : kBatchPartMaxN;
  }();
  return v;
}

// jobs the batch hands back: general path, one host thread / stream each
static void general_parallel(const std::vector<BatchPartJob*>& jobs, int parts, RunStats& st,
                             cudaStream_t s) {
  if (jobs.empty()) return;
  if (jobs.size() == 1) {
    BatchPartJob& B = *jobs[0];
    internal_partitioner(B.g, B.total, parts, B.eps_local, B.seed, B.out_part, st, s);
    return;
  }
  int dev = 0;
  GIM_CUDA(cudaGetDevice(&dev));
  GIM_CUDA(sync_stream(s));
  std::vector<std::thread> workers;
  std::vector<std::exception_ptr> errs(jobs.size());
  RunCtx* const pc = &ctx();
  for (size_t j = 0; j < jobs.size(); ++j) {
    workers.emplace_back([&, j, pc] {
      CtxScope scope(pc);
      ConcurrentScope conc;
      cudaStream_t cs = nullptr;
      try {
        GIM_CUDA(cudaSetDevice(dev));
        cs = acquire_stream();
        BatchPartJob& B = *jobs[j];
        DBuf<int> p((size_t)std::max(B.g.n, 1), cs);
        internal_partitioner(B.g, B.total, parts, B.eps_local, B.seed, p.get(), st, cs);
        GIM_CUDA(cudaMemcpyAsync(B.out_part, p.get(), sizeof(int) * B.g.n,
                                 cudaMemcpyDeviceToDevice, cs));
        GIM_CUDA(sync_stream(cs));
      } catch (...) {
        errs[j] = std::current_exception();
      }
      release_stream(cs);
    });
  }
  for (auto& w : workers) w.join();
  for (auto& e : errs)
    if (e) std::rethrow_exception(e);
}

static void internal_partitioner_batch(std::vector<BatchPartJob>& jobs, int parts, RunStats& st,
                                       cudaStream_t s) {
  std::vector<BatchPartJob*> general;
  std::vector<int> fast;  // jobs on the batched path
  for (int j = 0; j < (int)jobs.size(); ++j) {
    BatchPartJob& B = jobs[(size_t)j];
    if (parts <= 1 || B.g.n <= parts) {  // trivial cases as internal_partitioner
      internal_partitioner(B.g, B.total, parts, B.eps_local, B.seed, B.out_part, st, s);
      continue;
    }
    fast.push_back(j);
  }
  if (fast.empty()) return;
  const int J = (int)fast.size();
  Topo tf = get_flat_topo(parts);
  std::vector<DevGraph> gs;
  std::vector<double> lmax;
  std::vector<unsigned long long> seeds;
  for (int j : fast) {
    const BatchPartJob& B = jobs[(size_t)j];
    gs.push_back(B.g);
    lmax.push_back((1.0 + B.eps_local) * (double)B.total / (double)parts);
    seeds.push_back(B.seed);
  }
  std::vector<SmallStack> stacks;
  DBuf<int> arena;
  coarsen_small_batch(gs, lmax, seeds, std::max<long long>(64ll * parts, 2), stacks, arena, s);
  // a stack that stopped at a level needing two-hop matching continues on
  // the general level-stack code from that level (same per-level seeds);
  // the job then refines in the batch like the others
  std::vector<std::vector<Level>> tails((size_t)J);
  std::vector<DBuf<int>> tail_src((size_t)J);
  for (int i = 0; i < J; ++i) {
    SmallStack& S = stacks[(size_t)i];
    if (S.status != 1) continue;
    DevGraph top = S.levels.back();
    if (!top.src) {  // arena levels carry no E_u
      tail_src[(size_t)i] = DBuf<int>((size_t)std::max<long long>(top.m2, 1), s);
      fill_sources(top.n, top.off, tail_src[(size_t)i].get(), s);
      top.src = tail_src[(size_t)i].get();
    }
    tails[(size_t)i] = build_level_stack(top, lmax[(size_t)i],
                                         std::max<long long>(64ll * parts, 2), seeds[(size_t)i],
                                         s, S.nl - 1);
    std::vector<Level>& T = tails[(size_t)i];
    S.levels.back() = top;
    S.cmap.back() = T.size() > 1 ? T[0].cmap.get() : nullptr;
    for (size_t l = 1; l < T.size(); ++l) {
      S.levels.push_back(T[l].g);
      S.cmap.push_back(l + 1 < T.size() ? T[l].cmap.get() : nullptr);
    }
    S.nl = (int)S.levels.size();
    S.status = 0;
  }
  // jobs the fast path cannot take: general path
  std::vector<int> ok;
  for (int i = 0; i < J; ++i) {
    const SmallStack& S = stacks[(size_t)i];
    if (S.status == 0) {
      ok.push_back(i);
    } else {
      BatchPartJob& B = jobs[(size_t)fast[(size_t)i]];
      if (std::getenv("GIM_BATCH_DEBUG"))
        std::fprintf(stderr, "[batch-debug] job n=%d: level stack needs the general path\n", B.g.n);
      general.push_back(&B);
    }
  }
  if (ok.empty()) {
    general_parallel(general, parts, st, s);
    return;
  }
  static const bool debug = std::getenv("GIM_BATCH_DEBUG") != nullptr;
  if (debug) {  // compare every fast-path level stack with the general one
    for (int i : ok) {
      const BatchPartJob& B = jobs[(size_t)fast[(size_t)i]];
      const SmallStack& S = stacks[(size_t)i];
      std::vector<Level> ref = build_level_stack(B.g, lmax[(size_t)i],
                                                 std::max<long long>(64ll * parts, 2), B.seed, s);
      GIM_CUDA(sync_stream(s));
      std::fprintf(stderr, "[batch-debug] job %d n=%d levels fast=%d general=%d\n", i, B.g.n,
                   S.nl, (int)ref.size());
      for (int l = 0; l < std::min(S.nl, (int)ref.size()); ++l) {
        const DevGraph& a = S.levels[(size_t)l];
        const DevGraph& b = ref[(size_t)l].g;
        auto fetch = [&](const int* p, long long cnt) {
          std::vector<int> h((size_t)std::max(cnt, 0ll));
          if (cnt > 0) GIM_CUDA(cudaMemcpy(h.data(), p, sizeof(int) * cnt, cudaMemcpyDeviceToHost));
          return h;
        };
        bool same = a.n == b.n && a.m2 == b.m2 && fetch(a.off, a.n + 1) == fetch(b.off, b.n + 1) &&
                    fetch(a.tgt, a.m2) == fetch(b.tgt, b.m2) && fetch(a.w, a.m2) == fetch(b.w, b.m2) &&
                    fetch(a.vw, a.n) == fetch(b.vw, b.n);
        if (l + 1 < S.nl && l + 1 < (int)ref.size())
          same = same && fetch(S.cmap[(size_t)l], a.n) == fetch(ref[(size_t)l].cmap.get(), a.n);
        std::fprintf(stderr, "[batch-debug]   level %d n=%d/%d m2=%lld/%lld %s\n", l, a.n, b.n,
                     a.m2, b.m2, same ? "same" : "DIFFERENT");
      }
    }
  }
  st.partitioner_calls += (long long)ok.size();
  const int K = (int)ok.size();
  // per-job ping-pong partitions, block weights, refine scratch
  int nmax = 0, lmaxn = 0;
  for (int i : ok) {
    nmax = std::max(nmax, gs[(size_t)i].n);
    lmaxn = std::max(lmaxn, stacks[(size_t)i].nl);
  }
  DBuf<int> pa((size_t)K * nmax, s), pb((size_t)K * nmax, s), best((size_t)K * nmax, s);
  DBuf<long long> bw((size_t)K * parts, s), best_bw((size_t)K * parts, s);
  DBuf<FusedState> states((size_t)2 * K, s);
  std::vector<int*> cur((size_t)K), nxt((size_t)K);
  for (int q = 0; q < K; ++q) {
    cur[(size_t)q] = pa.get() + (size_t)q * nmax;
    nxt[(size_t)q] = pb.get() + (size_t)q * nmax;
  }
  // initial partition of every coarsest graph (pipelines.py:206)
  {
    std::vector<DevGraph> coarsest;
    std::vector<int*> outs;
    for (int q = 0; q < K; ++q) {
      const SmallStack& S = stacks[(size_t)ok[(size_t)q]];
      coarsest.push_back(S.levels.back());
      outs.push_back(cur[(size_t)q]);
    }
    ggg_batch(coarsest, parts, outs, s);
  }
  std::vector<char> failed((size_t)K, 0);
  for (int t = 0; t < lmaxn; ++t) {
    std::vector<BpJob> bp;
    std::vector<SmemRefineJob> rj, rc;  // shared-memory resident / cluster
    std::vector<int> who, whoc;
    for (int q = 0; q < K; ++q) {
      if (failed[(size_t)q]) continue;
      const int i = ok[(size_t)q];
      const SmallStack& S = stacks[(size_t)i];
      const int li = S.nl - 1 - t;
      if (li < 0) continue;
      const DevGraph& g = S.levels[(size_t)li];
      const bool project = t > 0;
      if (project) std::swap(cur[(size_t)q], nxt[(size_t)q]);  // nxt = coarse part
      long long* bwq = bw.get() + (size_t)q * parts;
      bp.push_back(BpJob{g.n, parts, project ? S.cmap[(size_t)li] : nullptr,
                         project ? nxt[(size_t)q] : nullptr, cur[(size_t)q], g.vw, bwq});
      const BatchPartJob& B = jobs[(size_t)fast[(size_t)i]];
      RefCfg cfg = config_for_level(li, S.nl, 0.999, 2, 1, 0.25, 0.065, 0.005, 10,
                                    hash2(B.seed, 101, (unsigned long long)li));
      SmemRefineJob R;
      R.g = g;
      R.vw = refine_pick_vw(g.n, g.m2);
      R.part = cur[(size_t)q];
      R.bw = bwq;
      R.cfg.l_max = lmax[(size_t)i];
      R.cfg.sigma = lmax[(size_t)i] * (1.0 - cfg.sigma_fraction);
      R.cfg.phi = cfg.phi;
      R.cfg.jet_c = cfg.jet_c;
      R.cfg.jet = cfg.jet;
      R.cfg.rho = cfg.rho;
      R.cfg.i_max = cfg.i_max;
      R.cfg.i_w_max = cfg.i_w_max;
      R.cfg.seed = cfg.seed;
      R.best = best.get() + (size_t)q * nmax;
      R.best_bw = best_bw.get() + (size_t)q * parts;
      if (refine_smem_fits(g.n, g.m2, parts, R.cfg.rho, R.vw)) {
        rj.push_back(R);
        who.push_back(q);
      } else {
        rc.push_back(R);
        whoc.push_back(q);
      }
    }
    if (rj.empty() && rc.empty()) continue;
    bproj_bw_batch(bp, s);
    std::vector<char> yielded;
    // a refinement that handed back a strong pass resumes on the general
    // device loop (host strong pass, relaunches) exactly where it stopped
    auto account = [&](std::vector<SmemRefineJob>& v, const std::vector<int>& w,
                       FusedState* dstates) {
      for (size_t r = 0; r < v.size(); ++r) {
        if (!yielded[r]) {
          st.init_refine_iterations += v[r].iters;
          st.lp += v[r].lp;
          st.weak += v[r].weak;
          continue;
        }
        const int q = w[r];
        const int i = ok[(size_t)q];
        const SmallStack& S = stacks[(size_t)i];
        const int li = S.nl - 1 - t;
        const BatchPartJob& B = jobs[(size_t)fast[(size_t)i]];
        RefCfg cfg = config_for_level(li, S.nl, 0.999, 2, 1, 0.25, 0.065, 0.005, 10,
                                      hash2(B.seed, 101, (unsigned long long)li));
        FusedState hs0;
        GIM_CUDA(cudaMemcpyAsync(&hs0, dstates + r, sizeof(FusedState), cudaMemcpyDeviceToHost, s));
        RefineLevel L;
        L.g = v[r].g;
        prepare_level(L, parts, s);
        RefineBuffers rb;
        alloc_refine_buffers(rb, L.g.n, parts, s);
        GIM_CUDA(cudaMemcpyAsync(rb.best.get(), v[r].best, sizeof(int) * (size_t)L.g.n,
                                 cudaMemcpyDeviceToDevice, s));
        GIM_CUDA(cudaMemcpyAsync(rb.best_bw.get(), v[r].best_bw, sizeof(long long) * parts,
                                 cudaMemcpyDeviceToDevice, s));
        GIM_CUDA(sync_stream(s));
        if (std::getenv("GIM_BATCH_DEBUG"))
          std::fprintf(stderr, "[batch-debug] job n=%d: strong pass, resumed\n", v[r].g.n);
        refine_device_loop(L, tf, v[r].part, v[r].bw, cfg, v[r].cfg.l_max, st, rb, s, &hs0);
      }
    };
    if (!rc.empty()) {
      refine_cluster_batch(rc, tf, states.get() + K, yielded, s);
      account(rc, whoc, states.get() + K);
    }
    if (!rj.empty()) {
      refine_smem_batch(rj, tf, states.get(), yielded, s);
      account(rj, who, states.get());
    }
  }
  if (debug) {  // final partitions vs the general path
    GIM_CUDA(sync_stream(s));
    for (int q = 0; q < K; ++q) {
      if (failed[(size_t)q]) continue;
      BatchPartJob& B = jobs[(size_t)fast[(size_t)ok[(size_t)q]]];
      DBuf<int> ref((size_t)std::max(B.g.n, 1), s);
      internal_partitioner(B.g, B.total, parts, B.eps_local, B.seed, ref.get(), st, s);
      GIM_CUDA(sync_stream(s));
      std::vector<int> x((size_t)B.g.n), y((size_t)B.g.n);
      GIM_CUDA(cudaMemcpy(x.data(), cur[(size_t)q], sizeof(int) * B.g.n, cudaMemcpyDeviceToHost));
      GIM_CUDA(cudaMemcpy(y.data(), ref.get(), sizeof(int) * B.g.n, cudaMemcpyDeviceToHost));
      int diff = 0;
      for (int v = 0; v < B.g.n; ++v) diff += x[(size_t)v] != y[(size_t)v];
      std::fprintf(stderr, "[batch-debug] job %d final partition: %d of %d differ\n", q, diff,
                   B.g.n);
    }
  }
  for (int q = 0; q < K; ++q) {
    BatchPartJob& B = jobs[(size_t)fast[(size_t)ok[(size_t)q]]];
    if (failed[(size_t)q]) {
      general.push_back(&B);
      continue;
    }
    GIM_CUDA(cudaMemcpyAsync(B.out_part, cur[(size_t)q], sizeof(int) * (size_t)B.g.n,
                             cudaMemcpyDeviceToDevice, s));
  }
  general_parallel(general, parts, st, s);
}

// ---------------------------------------------------------------------------
// hierarchical multisection (pipelines.py:49-110)

struct MsCtx {
  std::vector<long long> h;  // the multisection only needs the hierarchy
  long long k;
  long long total;
  double eps;
  int* assignment;
  RunStats* st;
  bool threads;
  int device;
};


static double adaptive_imbalance(double eps, long long total, long long sub, long long k,
                                 long long k_sub, int depth) {
  double value = std::pow((1.0 + eps) * (double)(k_sub * total) / (double)(k * sub),
                          1.0 / (double)depth) - 1.0;
  return std::max(value, 0.0);
}

static int calc_id(const std::vector<long long>& h, const std::vector<int>& ident) {
  const int ell = (int)h.size();
  long long out = 0, place = 1;
  for (int i = 0; i < ell; ++i) {
    out += ident[ell - 1 - i] * place;
    place *= h[i];
  }
  return (int)out;
}

// Sibling subtrees are independent (disjoint vertex sets, seeds derived from
// the parent only), so each child subtree that still has partitioning work
// runs on its own host thread and CUDA stream; the result is identical to
// the reference's sequential recursion.
static void descend(MsCtx& C, const DevGraph& sub, long long sub_total, int level,
                    std::vector<int>& ident, const int* translation, unsigned long long node_seed,
                    cudaStream_t s) {
  if (sub.n == 0) return;
  if (level == 0) {
    scatter_const(sub.n, translation, calc_id(C.h, ident), C.assignment, s);
    return;
  }
  const int parts = (int)C.h[level - 1];
  long long k_sub = 1;
  for (int i = 0; i < level; ++i) k_sub *= C.h[i];
  double eps_local = adaptive_imbalance(C.eps, C.total, sub_total, C.k, k_sub, level);
  DBuf<int> part((size_t)std::max(sub.n, 1), s);
  if (parts == 1)
    GIM_CUDA(cudaMemsetAsync(part.get(), 0, sizeof(int) * sub.n, s));
  else
    internal_partitioner(sub, sub_total, parts, eps_local, node_seed, part.get(), *C.st, s);
  if (level == 1) {
    // the children are leaves (pipelines.py:78-80): vertex v of part j lands
    // on calc_id(ident + (j,)) = calc_id(ident + (0,)) + j — no subgraphs needed
    ident.push_back(0);
    const int base = calc_id(C.h, ident);
    ident.pop_back();
    leaf_scatter(sub.n, translation, part.get(), base, C.assignment, s);
    return;
  }
  DBuf<long long> bw((size_t)parts, s);
  block_weights(sub.n, sub.vw, part.get(), parts, bw.get(), s);
  std::vector<long long> child_total((size_t)parts);
  GIM_CUDA(cudaMemcpyAsync(child_total.data(), bw.get(), sizeof(long long) * parts,
                           cudaMemcpyDeviceToHost, s));
  std::vector<OwnedGraph> subs;
  std::vector<DBuf<int>> ids;
  extract_subgraphs(sub, part.get(), parts, subs, ids, s);  // synchronizes s
  std::vector<DBuf<int>> trans((size_t)parts);
  for (int j = 0; j < parts; ++j) {
    trans[j] = DBuf<int>((size_t)std::max(subs[j].n, 1), s);
    gather(subs[j].n, ids[j].get(), translation, trans[j].get(), s);
  }
  if (level - 1 == 1 && ctx().f.batch && C.h[0] > 1) {
    // the children split straight into leaves: partition all of them in one
    // batch (one launch per phase) when they are small
    bool small = true;
    for (int j = 0; j < parts; ++j) small = small && subs[j].n <= batch_max_n();
    if (small) {
      std::vector<BatchPartJob> jobs;
      std::vector<DBuf<int>> cparts((size_t)parts);
      const int cp = (int)C.h[0];
      for (int j = 0; j < parts; ++j) {
        cparts[(size_t)j] = DBuf<int>((size_t)std::max(subs[j].n, 1), s);
        if (subs[j].n == 0) continue;
        const double eps_child =
            adaptive_imbalance(C.eps, C.total, child_total[j], C.k, C.h[0], 1);
        jobs.push_back(BatchPartJob{subs[j].view(), child_total[j], eps_child,
                                    hash2(node_seed, (unsigned long long)level,
                                          (unsigned long long)j),
                                    cparts[(size_t)j].get()});
      }
      internal_partitioner_batch(jobs, cp, *C.st, s);
      for (int j = 0; j < parts; ++j) {
        if (subs[j].n == 0) continue;
        ident.push_back(j);
        ident.push_back(0);
        const int base = calc_id(C.h, ident);
        ident.pop_back();
        ident.pop_back();
        leaf_scatter(subs[j].n, trans[j].get(), cparts[(size_t)j].get(), base, C.assignment, s);
      }
      return;
    }
  }
  const bool fan_out = level - 1 >= 1 && parts > 1 && C.threads;
  if (!fan_out) {
    for (int j = 0; j < parts; ++j) {
      ident.push_back(j);
      descend(C, subs[j].view(), child_total[j], level - 1, ident, trans[j].get(),
              hash2(node_seed, (unsigned long long)level, (unsigned long long)j), s);
      ident.pop_back();
    }
    return;
  }
  GIM_CUDA(sync_stream(s));  // children read subs/trans from other streams
  std::vector<std::thread> workers;
  std::vector<std::exception_ptr> errs((size_t)parts);
  RunCtx* const pc = &ctx();
  for (int j = 0; j < parts; ++j) {
    workers.emplace_back([&, j, pc] {
      CtxScope scope(pc);
      ConcurrentScope conc;
      cudaStream_t cs = nullptr;
      try {
        GIM_CUDA(cudaSetDevice(C.device));
        cs = acquire_stream();
        {
          std::vector<int> id2 = ident;
          id2.push_back(j);
          descend(C, subs[j].view(), child_total[j], level - 1, id2, trans[j].get(),
                  hash2(node_seed, (unsigned long long)level, (unsigned long long)j), cs);
        }
        GIM_CUDA(sync_stream(cs));
      } catch (...) {
        errs[j] = std::current_exception();
      }
      release_stream(cs);
    });
  }
  for (auto& w : workers) w.join();
  for (auto& e : errs)
    if (e) std::rethrow_exception(e);
}

// Plugin-seam multisection (gim_hierarchical_multisection_plugin): the
// reference's depth-first recursion node by node (pipelines.py:72-107), so a
// caller's partitioner sees the nodes — and trace records are produced — in
// the reference's order.  Extraction, block weights, scatters and the
// built-in partitioner stay on the GPU; a caller partitioner gets the
// node's subgraph as host int64 arrays.
struct PluginCtx {
  MsCtx* C;
  gim_partition_fn partition;
  gim_trace_fn trace;
  void* user;
};

static void descend_plugin(PluginCtx& P, const DevGraph& sub, long long sub_total, int level,
                           std::vector<int>& ident, const int* translation,
                           unsigned long long node_seed, cudaStream_t s) {
  MsCtx& C = *P.C;
  if (sub.n == 0) return;
  if (level == 0) {
    scatter_const(sub.n, translation, calc_id(C.h, ident), C.assignment, s);
    return;
  }
  const int parts = (int)C.h[level - 1];
  long long k_sub = 1;
  for (int i = 0; i < level; ++i) k_sub *= C.h[i];
  const double eps_local = adaptive_imbalance(C.eps, C.total, sub_total, C.k, k_sub, level);
  DBuf<int> part((size_t)std::max(sub.n, 1), s);
  if (parts == 1) {
    GIM_CUDA(cudaMemsetAsync(part.get(), 0, sizeof(int) * sub.n, s));
  } else if (P.partition) {
    // the node's subgraph to the host as int64 (graph.py:17-39 layout)
    const size_t n = (size_t)sub.n, m2 = (size_t)sub.m2;
    std::vector<int> o32(n + 1), t32(m2), w32(m2), v32(n);
    GIM_CUDA(cudaMemcpyAsync(o32.data(), sub.off, sizeof(int) * (n + 1), cudaMemcpyDeviceToHost, s));
    if (m2) {
      GIM_CUDA(cudaMemcpyAsync(t32.data(), sub.tgt, sizeof(int) * m2, cudaMemcpyDeviceToHost, s));
      GIM_CUDA(cudaMemcpyAsync(w32.data(), sub.w, sizeof(int) * m2, cudaMemcpyDeviceToHost, s));
    }
    GIM_CUDA(cudaMemcpyAsync(v32.data(), sub.vw, sizeof(int) * n, cudaMemcpyDeviceToHost, s));
    GIM_CUDA(sync_stream(s));
    std::vector<int64_t> o(o32.begin(), o32.end()), tt(t32.begin(), t32.end()),
        ww(w32.begin(), w32.end()), vv(v32.begin(), v32.end()), out(n, 0);
    const int rc = P.partition(P.user, (int64_t)n, o.data(), tt.data(), ww.data(), vv.data(),
                               parts, eps_local, node_seed, ident.data(), (int32_t)ident.size(),
                               out.data());
    GIM_CHECK(rc == 0, GIM_E_CALLBACK, "partitioner callback failed");
    std::vector<int> p32(n);
    for (size_t i = 0; i < n; ++i) {
      GIM_CHECK(out[i] >= 0 && out[i] < parts, GIM_E_CALLBACK, "partitioner returned an invalid assignment");
      p32[i] = (int)out[i];
    }
    GIM_CUDA(cudaMemcpyAsync(part.get(), p32.data(), sizeof(int) * n, cudaMemcpyHostToDevice, s));
    GIM_CUDA(sync_stream(s));
  } else {
    internal_partitioner(sub, sub_total, parts, eps_local, node_seed, part.get(), *C.st, s);
  }
  DBuf<long long> bw((size_t)parts, s);
  block_weights(sub.n, sub.vw, part.get(), parts, bw.get(), s);
  std::vector<long long> child_total((size_t)parts);
  GIM_CUDA(cudaMemcpyAsync(child_total.data(), bw.get(), sizeof(long long) * parts,
                           cudaMemcpyDeviceToHost, s));
  GIM_CUDA(sync_stream(s));
  if (P.trace) {
    long long mx = 0;
    for (long long x : child_total) mx = std::max(mx, x);
    const double budget = (1.0 + eps_local) * (double)sub_total / (double)parts;
    std::vector<int64_t> bw64(child_total.begin(), child_total.end());
    P.trace(P.user, level, ident.data(), (int32_t)ident.size(), parts, eps_local, sub_total,
            bw64.data(), (double)mx <= budget ? 1 : 0);
  }
  std::vector<OwnedGraph> subs;
  std::vector<DBuf<int>> ids;
  extract_subgraphs(sub, part.get(), parts, subs, ids, s);
  for (int j = 0; j < parts; ++j) {
    DBuf<int> tr((size_t)std::max(subs[j].n, 1), s);
    gather(subs[j].n, ids[j].get(), translation, tr.get(), s);
    ident.push_back(j);
    descend_plugin(P, subs[j].view(), child_total[j], level - 1, ident, tr.get(),
                   hash2(node_seed, (unsigned long long)level, (unsigned long long)j), s);
    ident.pop_back();
  }
}

// Breadth-first multisection: all nodes of one tree level are partitioned
// together — as one batch when they are small (internal_partitioner_batch),
// else one host thread per node — then all their children are extracted.
// Every node computes exactly what descend() computes for it; only the
// order of independent work changes.
struct MsNode {
  OwnedGraph own;  // empty for the root
  DevGraph g;
  DBuf<int> trans_own;
  const int* trans = nullptr;
  long long total = 0;
  std::vector<int> ident;
  unsigned long long seed = 0;
};

static void multisection_bfs(MsCtx& C, const DevGraph& root, long long total, const int* ids,
                             unsigned long long seed, cudaStream_t s) {
  std::vector<MsNode> nodes(1);
  std::vector<DBuf<int>> arenas;  // batched extractions: children live here
  nodes[0].g = root;
  nodes[0].trans = ids;
  nodes[0].total = total;
  nodes[0].seed = seed;
  MsTimer tm(s);
  for (int level = (int)C.h.size(); level >= 1; --level) {
    const int parts = (int)C.h[level - 1];
    long long k_sub = 1;
    for (int i = 0; i < level; ++i) k_sub *= C.h[i];
    const int N = (int)nodes.size();
    if (tm.on && level < (int)C.h.size())
      std::fprintf(stderr, "ms extraction into tree level %d: %.3f ms\n", level, tm.lap());
    std::vector<DBuf<int>> part((size_t)N);
    for (int j = 0; j < N; ++j) part[(size_t)j] = DBuf<int>((size_t)std::max(nodes[(size_t)j].g.n, 1), s);
    bool small = parts > 1;
    for (const MsNode& nd : nodes) small = small && nd.g.n <= batch_max_n();
    if (parts == 1) {
      for (int j = 0; j < N; ++j)
        GIM_CUDA(cudaMemsetAsync(part[(size_t)j].get(), 0, sizeof(int) * nodes[(size_t)j].g.n, s));
    } else if (small) {
      std::vector<BatchPartJob> jobs;
      for (int j = 0; j < N; ++j) {
        const MsNode& nd = nodes[(size_t)j];
        jobs.push_back(BatchPartJob{nd.g, nd.total,
                                    adaptive_imbalance(C.eps, C.total, nd.total, C.k, k_sub, level),
                                    nd.seed, part[(size_t)j].get()});
      }
      internal_partitioner_batch(jobs, parts, *C.st, s);
    } else if (N == 1 || !C.threads) {
      for (int j = 0; j < N; ++j) {
        const MsNode& nd = nodes[(size_t)j];
        internal_partitioner(nd.g, nd.total, parts,
                             adaptive_imbalance(C.eps, C.total, nd.total, C.k, k_sub, level),
                             nd.seed, part[(size_t)j].get(), *C.st, s);
      }
    } else {  // large nodes: one host thread / stream each
      GIM_CUDA(sync_stream(s));
      std::vector<std::thread> workers;
      std::vector<std::exception_ptr> errs((size_t)N);
      RunCtx* const pc = &ctx();
      for (int j = 0; j < N; ++j) {
        workers.emplace_back([&, j, pc] {
          CtxScope scope(pc);
          ConcurrentScope conc;
          cudaStream_t cs = nullptr;
          try {
            GIM_CUDA(cudaSetDevice(C.device));
            cs = acquire_stream();
            const MsNode& nd = nodes[(size_t)j];
            DBuf<int> p((size_t)std::max(nd.g.n, 1), cs);
            internal_partitioner(nd.g, nd.total, parts,
                                 adaptive_imbalance(C.eps, C.total, nd.total, C.k, k_sub, level),
                                 nd.seed, p.get(), *C.st, cs);
            GIM_CUDA(cudaMemcpyAsync(part[(size_t)j].get(), p.get(), sizeof(int) * nd.g.n,
                                     cudaMemcpyDeviceToDevice, cs));
            GIM_CUDA(sync_stream(cs));
          } catch (...) {
            errs[(size_t)j] = std::current_exception();
          }
          release_stream(cs);
        });
      }
      for (auto& w : workers) w.join();
      for (auto& e : errs)
        if (e) std::rethrow_exception(e);
    }
    if (tm.on) {
      long long tot_n = 0;
      int mx = 0;
      for (const MsNode& nd : nodes) {
        tot_n += nd.g.n;
        mx = std::max(mx, nd.g.n);
      }
      std::fprintf(stderr, "ms tree level %d: %d nodes (sum n %lld, max %d, parts %d) %s: %.3f ms\n",
                   level, N, tot_n, mx, parts, small ? "batch" : "general", tm.lap());
    }
    if (level == 1) {  // leaves (pipelines.py:78-80)
      for (int j = 0; j < N; ++j) {
        MsNode& nd = nodes[(size_t)j];
        nd.ident.push_back(0);
        const int base = calc_id(C.h, nd.ident);
        leaf_scatter(nd.g.n, nd.trans, part[(size_t)j].get(), base, C.assignment, s);
      }
      return;
    }
    std::vector<MsNode> next;
    bool small_nodes = parts <= 64;
    for (const MsNode& nd : nodes) small_nodes = small_nodes && nd.g.n <= kBatchMaxN;
    if (small_nodes) {  // all children of this tree level in one launch (CTA per node)
      std::vector<DevGraph> gs;
      std::vector<const int*> pp, tr;
      for (int j = 0; j < N; ++j) {
        gs.push_back(nodes[(size_t)j].g);
        pp.push_back(part[(size_t)j].get());
        tr.push_back(nodes[(size_t)j].trans);
      }
      std::vector<ExChild> kids;
      arenas.emplace_back();
      extract_batch(gs, pp, tr, parts, kids, arenas.back(), s);
      for (const ExChild& x : kids) {
        if (x.g.n == 0) continue;  // descend() returns at once for empty nodes
        const MsNode& nd = nodes[(size_t)x.node];
        MsNode ch;
        ch.g = x.g;
        ch.trans = x.trans;
        ch.total = x.total;
        ch.ident = nd.ident;
        ch.ident.push_back(x.part);
        ch.seed = hash2(nd.seed, (unsigned long long)level, (unsigned long long)x.part);
        next.push_back(std::move(ch));
      }
      nodes = std::move(next);
      continue;
    }
    for (int j = 0; j < N; ++j) {
      MsNode& nd = nodes[(size_t)j];
      DBuf<long long> bw((size_t)parts, s);
      block_weights(nd.g.n, nd.g.vw, part[(size_t)j].get(), parts, bw.get(), s);
      std::vector<long long> child_total((size_t)parts);
      GIM_CUDA(cudaMemcpyAsync(child_total.data(), bw.get(), sizeof(long long) * parts,
                               cudaMemcpyDeviceToHost, s));
      std::vector<OwnedGraph> subs;
      std::vector<DBuf<int>> sids;
      extract_subgraphs(nd.g, part[(size_t)j].get(), parts, subs, sids, s);  // synchronizes s
      for (int c = 0; c < parts; ++c) {
        if (subs[(size_t)c].n == 0) continue;  // descend() returns at once for empty nodes
        MsNode ch;
        ch.own = std::move(subs[(size_t)c]);
        ch.g = ch.own.view();
        ch.trans_own = DBuf<int>((size_t)std::max(ch.g.n, 1), s);
        gather(ch.g.n, sids[(size_t)c].get(), nd.trans, ch.trans_own.get(), s);
        ch.trans = ch.trans_own.get();
        ch.total = child_total[(size_t)c];
        ch.ident = nd.ident;
        ch.ident.push_back(c);
        ch.seed = hash2(nd.seed, (unsigned long long)level, (unsigned long long)c);
        next.push_back(std::move(ch));
      }
    }
    nodes = std::move(next);
  }
}

static void hierarchical_multisection(const DevGraph& g, long long total,
                                      const std::vector<long long>& h,
                                      double eps,
                                      unsigned long long seed, int* assignment, RunStats& st,
                                      cudaStream_t s) {
  GIM_CHECK(g.n > 0, GIM_E_EMPTY, "cannot map an empty graph");
  MsCtx C;
  C.h = h;
  C.k = 1;
  for (long long a : h) C.k *= a;
  C.total = total;
  C.eps = eps;
  C.assignment = assignment;
  C.st = &st;
  C.threads = ctx().f.fanout;
  GIM_CUDA(cudaGetDevice(&C.device));
  GIM_CUDA(cudaMemsetAsync(assignment, 0, sizeof(int) * g.n, s));
  DBuf<int> ident_ids((size_t)g.n, s);
  k_iota<<<grid_for(g.n, 256), 256, 0, s>>>(g.n, ident_ids.get());
  count_launch();
  if (ctx().f.batch) {
    multisection_bfs(C, g, total, ident_ids.get(), seed, s);
    return;
  }
  std::vector<int> ident;
  descend(C, g, total, (int)h.size(), ident, ident_ids.get(), seed, s);
}

// ---------------------------------------------------------------------------
// integrated_map (pipelines.py:221-269)

struct ImTimes {
  cudaEvent_t e[4];
};

// `l_max_in` >= 0: the caller's L_max (isolated-vertex strip mode maps the
// reduced graph against the full graph's L_max)
static void integrated_map_device(const DevGraph& g0, long long total, const gim_topology& tt,
                                  double eps, unsigned long long seed, const gim_im_params& P,
                                  int* out_part, long long* out_bw, gim_im_stats* stats,
                                  cudaStream_t s, double l_max_in = -1.0) {
  GIM_CHECK(g0.n > 0, GIM_E_EMPTY, "cannot map an empty graph");
  const auto th0 = std::chrono::steady_clock::now();
  Topo t = get_topo(tt);
  std::vector<long long> h(tt.hierarchy, tt.hierarchy + tt.levels);
  const long long k = t.k;
  RunStats st;
  reset_launches();
  cudaEvent_t ev[4];
  for (auto& e : ev) GIM_CUDA(cudaEventCreate(&e));
  GIM_CUDA(cudaEventRecord(ev[0], s));
  const double l_max = l_max_in >= 0.0 ? l_max_in : (1.0 + eps) * (double)total / (double)k;
  std::vector<Level> levels = build_level_stack(
      g0, l_max, std::max<long long>(P.coarsest_factor * k, 1), seed, s);
  const int nl = (int)levels.size();
  std::vector<long long> level_n, level_m2;
  for (auto& L : levels) {
    level_n.push_back(L.g.n);
    level_m2.push_back(L.g.m2);
  }
  GIM_CUDA(cudaEventRecord(ev[1], s));
  DBuf<int> cur((size_t)std::max(levels.back().g.n, 1), s);
  st.in_initial = true;
  hierarchical_multisection(levels.back().g, total, h, eps,
                            hash2(seed, 7, 7), cur.get(), st, s);
  st.in_initial = false;
  GIM_CUDA(cudaEventRecord(ev[2], s));
  RefineBuffers rb;
  alloc_refine_buffers(rb, g0.n, (int)k, s);  // sized for level 0, reused by every level
  // per-level refinement accounting: events around each level's refine and
  // the device counters it added (SURVEY §8(d) bytes)
  std::vector<cudaEvent_t> lev((size_t)2 * nl);
  for (auto& e : lev) GIM_CUDA(cudaEventCreate(&e));
  std::vector<std::array<long long, A_COUNT>> lacct((size_t)nl);
  std::vector<long long> liters((size_t)nl);
  ctx().reset_acct();
  for (int li = nl - 1; li >= 0; --li) {
    Level& L = levels[li];
    if (li < nl - 1) {
      DBuf<int> fine((size_t)std::max(L.g.n, 1), s);
      project(L.g.n, L.cmap.get(), cur.get(), fine.get(), s);
      cur = std::move(fine);
      levels[li + 1] = Level();  // release the coarser level
    }
    block_weights(L.g.n, L.g.vw, cur.get(), (int)k, out_bw, s);
    RefCfg cfg = config_for_level(li, nl, P.phi, P.rho, P.filter_mode, P.jet_filter_c,
                                  P.sigma_coarse, P.sigma_fine, P.iw_max_finest,
                                  hash2(seed, 211, (unsigned long long)li));
    L.rl.g = L.g;
    long long a0[A_COUNT];
    for (int i = 0; i < A_COUNT; ++i) a0[i] = ctx().acct[i].load();
    const long long it0 = st.refine_iterations.load();
    GIM_CUDA(cudaEventRecord(lev[(size_t)2 * li], s));
    refine(L.rl, t, cur.get(), out_bw, cfg, l_max, st, rb, s);
    GIM_CUDA(cudaEventRecord(lev[(size_t)2 * li + 1], s));
    for (int i = 0; i < A_COUNT; ++i) lacct[(size_t)li][(size_t)i] = ctx().acct[i].load() - a0[i];
    liters[(size_t)li] = st.refine_iterations.load() - it0;
  }
  GIM_CUDA(cudaMemcpyAsync(out_part, cur.get(), sizeof(int) * g0.n, cudaMemcpyDeviceToDevice, s));
  GIM_CUDA(cudaEventRecord(ev[3], s));
  GIM_CUDA(cudaEventSynchronize(ev[3]));
  const auto th3 = std::chrono::steady_clock::now();
  if (stats) {
    float a = 0, b = 0, c = 0, tot = 0;
    cudaEventElapsedTime(&a, ev[0], ev[1]);
    cudaEventElapsedTime(&b, ev[1], ev[2]);
    cudaEventElapsedTime(&c, ev[2], ev[3]);
    cudaEventElapsedTime(&tot, ev[0], ev[3]);
    stats->n_levels = nl;
    stats->isolated_vertices = 0;
    for (int i = 0; i < 64; ++i) {
      stats->level_n[i] = i < nl ? level_n[i] : 0;
      stats->level_m2[i] = i < nl ? level_m2[i] : 0;
      stats->level_iters[i] = i < nl ? liters[(size_t)i] : 0;
      stats->level_refine_ms[i] = 0.0;
      stats->level_bytes[i] = 0.0;
      stats->level_barriers[i] = 0;
      if (i < nl) {
        float lm = 0.f;
        cudaEventElapsedTime(&lm, lev[(size_t)2 * i], lev[(size_t)2 * i + 1]);
        stats->level_refine_ms[i] = lm;
        stats->level_bytes[i] = s8d_refine_bytes(lacct[(size_t)i].data(), level_n[i],
                                                 level_m2[i], (int)k, P.rho);
        stats->level_barriers[i] = lacct[(size_t)i][A_BARRIERS];
      }
    }
    for (int i = 0; i < 16; ++i) stats->acct[i] = i < A_COUNT ? ctx().acct[i].load() : 0;
    stats->ms_upload = stats->ms_download = 0.0;
    stats->bytes_h2d = stats->bytes_d2h = 0;
    stats->ms_coarsen = a;
    stats->ms_initial = b;
    stats->ms_refine = c;
    stats->ms_total = tot;
    stats->refine_iterations = st.refine_iterations;
    stats->lp_passes = st.lp;
    stats->weak_passes = st.weak;
    stats->strong_passes = st.strong;
    stats->init_refine_iterations = st.init_refine_iterations;
    stats->partitioner_calls = st.partitioner_calls;
    stats->kernel_launches = launches();
    stats->l_max = l_max;
    double pms[P_COUNT] = {0}, pby[P_COUNT] = {0};
    long long pct[P_COUNT] = {0};
    int tcls = -1;
    double tms = 0, tby = 0;
    prof_collect(pms, pby, pct, &tcls, &tms, &tby);
    stats->top_class = tcls;
    stats->top_ms = tms;
    stats->top_bytes = tby;
    for (int c = 0; c < 16; ++c) {
      stats->prof_ms[c] = c < P_COUNT ? pms[c] : 0.0;
      stats->prof_bytes[c] = c < P_COUNT ? pby[c] : 0.0;
      stats->prof_count[c] = c < P_COUNT ? pct[c] : 0;
    }
    DBuf<long long> dj(1, s);
    total_cost(g0, out_part, t, dj.get(), s);
    stats->final_j = read_scalar(dj.get(), s);
    stats->dist_shift = t.dshift;
    stats->dist_exact = t.exact;
    if (t.exact) {
      stats->final_j_f64 = std::ldexp((double)stats->final_j, -t.dshift);
    } else {
      DBuf<double> djf(1, s);
      total_cost_f64(g0, out_part, t, djf.get(), s);
      stats->final_j_f64 = read_scalar(djf.get(), s);
    }
    std::vector<long long> bw((size_t)k);
    GIM_CUDA(cudaMemcpy(bw.data(), out_bw, sizeof(long long) * k, cudaMemcpyDeviceToHost));
    long long mx = 0;
    for (long long x : bw) mx = std::max(mx, x);
    stats->max_block_weight = mx;
  }
  for (auto& e : ev) cudaEventDestroy(e);
  for (auto& e : lev) cudaEventDestroy(e);
  if (trace_ms()) {
    const auto th4 = std::chrono::steady_clock::now();
    float dev = 0.f;
    std::fprintf(stderr, "im host ms: start->ev3 %.2f ev3->exit %.2f (seed %llu)\n",
                 std::chrono::duration<double, std::milli>(th3 - th0).count(),
                 std::chrono::duration<double, std::milli>(th4 - th3).count(), seed);
    (void)dev;
  }
}

// ---------------------------------------------------------------------------
// isolated-vertex strip mode (gim_im_params.isolated, include/gpuim.h)

__global__ void k_isolated_flag(int n, const int* __restrict__ off, int* __restrict__ flag) {
  for (int v = blockIdx.x * blockDim.x + threadIdx.x; v < n; v += gridDim.x * blockDim.x)
    flag[v] = off[v + 1] == off[v];
}

// isolated vertex of rank r (vertex order) -> the block whose fill range
// [start[b], start[b+1]) holds r
__global__ void k_fill_isolated(int n_iso, const int* __restrict__ ids,
                                const int* __restrict__ start, int k, int* __restrict__ part) {
  for (int r = blockIdx.x * blockDim.x + threadIdx.x; r < n_iso; r += gridDim.x * blockDim.x) {
    int lo = 0, hi = k;  // last b with start[b] <= r
    while (hi - lo > 1) {
      const int mid = (lo + hi) >> 1;
      if (start[mid] <= r) lo = mid;
      else hi = mid;
    }
    part[ids[r]] = lo;
  }
}

// Water-filling of `cnt` equal weights `w0` into blocks of weights bw: the
// lowest level T with sum_b max(0, floor((T - bw_b) / w0)) >= cnt, ties of
// the last unit to the lowest block ids.  Returns the per-block counts.
static std::vector<long long> water_fill(const std::vector<long long>& bw, long long cnt,
                                         long long w0) {
  const size_t k = bw.size();
  auto units = [&](long long T) {
    long long u = 0;
    for (long long b : bw) u += T > b ? (T - b) / w0 : 0;
    return u;
  };
  long long lo = *std::min_element(bw.begin(), bw.end()), hi = lo + (cnt + 1) * w0;
  while (lo < hi) {  // minimal T with units(T) >= cnt
    const long long mid = lo + (hi - lo) / 2;
    if (units(mid) >= cnt) hi = mid;
    else lo = mid + 1;
  }
  std::vector<long long> c(k);
  long long used = 0;
  for (size_t b = 0; b < k; ++b) {
    c[b] = lo - 1 > bw[b] ? (lo - 1 - bw[b]) / w0 : 0;
    used += c[b];
  }
  for (size_t b = 0; b < k && used < cnt; ++b) {
    const long long at_T = lo > bw[b] ? (lo - bw[b]) / w0 : 0;
    if (at_T > c[b]) {
      c[b] += 1;
      ++used;
    }
  }
  return c;
}

static void integrated_map_dispatch(const DevGraph& g0, long long total, const gim_topology& tt,
                                    double eps, unsigned long long seed, const gim_im_params& P,
                                    int* out_part, long long* out_bw, gim_im_stats* stats,
                                    cudaStream_t s) {
  integrated_map_device(g0, total, tt, eps, seed, P, out_part, out_bw, stats, s);
}

static void integrated_map_strip(const DevGraph& g0, long long total, const gim_topology& tt,
                                 double eps, unsigned long long seed, const gim_im_params& P,
                                 int* out_part, long long* out_bw, gim_im_stats* stats,
                                 cudaStream_t s) {
  Topo t = get_topo(tt);
  const int k = t.k;
  const int n = g0.n;
  DBuf<int> flag((size_t)n, s);
  k_isolated_flag<<<grid_for(n, 256), 256, 0, s>>>(n, g0.off, flag.get());
  count_launch();
  GIM_LAUNCH_CHECK();
  std::vector<OwnedGraph> subs;
  std::vector<DBuf<int>> ids;
  extract_subgraphs(g0, flag.get(), 2, subs, ids, s);  // 0: with edges, 1: isolated
  const OwnedGraph& R = subs[0];
  const int n_iso = subs[1].n;
  const double l_max = (1.0 + eps) * (double)total / (double)k;
  gim_im_params Q = P;
  Q.isolated = GIM_ISOLATED_KEEP;
  if (n_iso == 0 || R.n == 0) {  // nothing to strip / nothing but isolated vertices
    if (R.n == 0) {
      GIM_CUDA(cudaMemsetAsync(out_part, 0, sizeof(int) * n, s));
    } else {
      integrated_map_device(g0, total, tt, eps, seed, Q, out_part, out_bw, stats, s);
      return;
    }
  } else {
    long long total_r = 0;
    {
      DBuf<long long> d(1, s);
      GIM_CUDA(cudaMemsetAsync(d.get(), 0, sizeof(long long), s));
      k_sum_vw<<<grid_for(R.n, 256, kSMs * 2), 256, 0, s>>>(R.n, R.vw.get(), d.get());
      count_launch();
      total_r = read_scalar(d.get(), s);
    }
    // the reduced graph gets the full graph's capacity: eps_r makes every
    // multisection node's budget (Eq. 2) and L_max the same absolute weights
    // as with the isolated vertices present (they are the slack)
    const double eps_r = (1.0 + eps) * (double)total / (double)total_r - 1.0;
    DBuf<int> rp((size_t)R.n, s);
    integrated_map_device(R.view(), total_r, tt, eps_r, seed, Q, rp.get(), out_bw, stats, s, l_max);
    leaf_scatter(R.n, ids[0].get(), rp.get(), 0, out_part, s);
  }
  if (n_iso > 0) {
    // water-fill the isolated vertices into the lightest blocks
    std::vector<long long> bw((size_t)k, 0);
    if (R.n > 0)
      GIM_CUDA(cudaMemcpyAsync(bw.data(), out_bw, sizeof(long long) * k, cudaMemcpyDeviceToHost, s));
    std::vector<int> iw((size_t)n_iso);
    GIM_CUDA(cudaMemcpyAsync(iw.data(), subs[1].vw.get(), sizeof(int) * n_iso,
                             cudaMemcpyDeviceToHost, s));
    GIM_CUDA(sync_stream(s));
    const bool equal = std::all_of(iw.begin(), iw.end(), [&](int x) { return x == iw[0]; });
    if (equal) {  // unit (equal) weights: per-block counts, rank ranges on the device
      std::vector<long long> c = water_fill(bw, n_iso, iw[0]);
      std::vector<int> start((size_t)k + 1, 0);
      for (int b = 0; b < k; ++b) start[(size_t)b + 1] = start[(size_t)b] + (int)c[(size_t)b];
      DBuf<int> ds((size_t)k + 1, s);
      GIM_CUDA(cudaMemcpyAsync(ds.get(), start.data(), sizeof(int) * (k + 1),
                               cudaMemcpyHostToDevice, s));
      k_fill_isolated<<<grid_for(n_iso, 256), 256, 0, s>>>(n_iso, ids[1].get(), ds.get(), k,
                                                           out_part);
      count_launch();
      GIM_LAUNCH_CHECK();
      GIM_CUDA(sync_stream(s));
    } else {  // general weights: heaviest first into the current lightest block (LPT)
      std::vector<int> order((size_t)n_iso), blk((size_t)n_iso);
      for (int i = 0; i < n_iso; ++i) order[(size_t)i] = i;
      std::stable_sort(order.begin(), order.end(),
                       [&](int a, int b) { return iw[(size_t)a] > iw[(size_t)b]; });
      using Q2 = std::pair<long long, int>;
      std::priority_queue<Q2, std::vector<Q2>, std::greater<Q2>> heap;
      for (int b = 0; b < k; ++b) heap.push({bw[(size_t)b], b});
      for (int i : order) {
        auto top = heap.top();
        heap.pop();
        blk[(size_t)i] = top.second;
        top.first += iw[(size_t)i];
        heap.push(top);
      }
      DBuf<int> db((size_t)n_iso, s);
      GIM_CUDA(cudaMemcpyAsync(db.get(), blk.data(), sizeof(int) * n_iso, cudaMemcpyHostToDevice,
                               s));
      leaf_scatter(n_iso, ids[1].get(), db.get(), 0, out_part, s);
      GIM_CUDA(sync_stream(s));
    }
  }
  block_weights(n, g0.vw, out_part, k, out_bw, s);
  if (stats) {
    std::vector<long long> bw((size_t)k);
    GIM_CUDA(cudaMemcpyAsync(bw.data(), out_bw, sizeof(long long) * k, cudaMemcpyDeviceToHost, s));
    GIM_CUDA(sync_stream(s));
    stats->max_block_weight = *std::max_element(bw.begin(), bw.end());
    stats->l_max = l_max;
    stats->isolated_vertices = n_iso;
    if (R.n == 0) {  // no IM run filled the stats
      stats->n_levels = 0;
      stats->final_j = 0;
      stats->final_j_f64 = 0.0;
      stats->kernel_launches = launches();
    }
  }
}

// host-array upload (graph.py:17-39 int64 CSR) -> int32 device level
__global__ void k_narrow(long long n, const long long* __restrict__ in, int* __restrict__ out) {
  for (long long i = (long long)blockIdx.x * blockDim.x + threadIdx.x; i < n;
       i += (long long)gridDim.x * blockDim.x)
    out[i] = (int)in[i];
}

__global__ void k_fill_sources(int n, const int* __restrict__ off, int* __restrict__ src) {
  // one warp per vertex row
  const int lane = lane_id();
  for (long long w = ((long long)blockIdx.x * blockDim.x + threadIdx.x) >> 5; w < n;
       w += ((long long)gridDim.x * blockDim.x) >> 5) {
    int v = (int)w;
    for (int e = off[v] + lane; e < off[v + 1]; e += 32) src[e] = v;
  }
}

void fill_sources(int n, const int* off, int* src, cudaStream_t s) {
  if (n == 0) return;
  k_fill_sources<<<grid_for((long long)n * 32, 256, kSMs * 16), 256, 0, s>>>(n, off, src);
  count_launch();
  GIM_LAUNCH_CHECK();
}

// Host int64 CSR -> device int32 level (graph.py:17-39 arrays).  The
// arrays are narrowed to int32 ON THE HOST by worker threads, each writing
// into its own double-buffered pinned staging block and copying on its own
// stream, so narrowing, PCIe transfer and the other workers overlap and
// only half the bytes cross the bus.  The same pass validates what the
// device path relies on (values fit int32, positive vertex weights, total
// vertex / edge weight < 2^31).
namespace {
struct UpJob {
  const int64_t* src;
  int* dst;
  long long cnt;
  int kind;  // 0 targets, 1 edge weights, 2 vertex weights, 3 offsets
};
struct UpAcc {
  long long sum_ew = 0, sum_vw = 0, h2d = 0, maxdeg = 0;
  bool bad_range = false, bad_vw = false, bad_ew = false, bad_off = false, bad_tgt = false;
};
}  // namespace

__global__ void k_fill_i32(long long n, int v, int* __restrict__ out) {
  for (long long i = (long long)blockIdx.x * blockDim.x + threadIdx.x; i < n;
       i += (long long)gridDim.x * blockDim.x)
    out[i] = v;
}

// returns the bytes copied host -> device.  Weight chunks holding one value
// (unit-weight graphs: every chunk) are not copied: the device fills them.
static long long upload_graph(long long n, const int64_t* off, const int64_t* tgt,
                              const int64_t* ew, const int64_t* vw, OwnedGraph& G,
                              cudaStream_t s) {
  GIM_CHECK(n >= 0 && n < INT32_MAX, GIM_E_OVERFLOW, "n must be < 2^31");
  GIM_CHECK(off[0] == 0, GIM_E_INVALID, "offsets[0] must be 0");
  long long m2 = off[n];
  GIM_CHECK(m2 >= 0 && m2 < INT32_MAX, GIM_E_OVERFLOW, "2m must be < 2^31");
  G.n = (int)n;
  G.m2 = m2;
  G.off = DBuf<int>((size_t)n + 1, s);
  G.tgt = DBuf<int>((size_t)std::max(m2, 1ll), s);
  G.w = DBuf<int>((size_t)std::max(m2, 1ll), s);
  G.vw = DBuf<int>((size_t)std::max(n, 1ll), s);
  G.src = DBuf<int>((size_t)std::max(m2, 1ll), s);
  // device buffers come from `s`'s stream order: the workers' streams wait
  GIM_CUDA(sync_stream(s));
  constexpr long long kChunk = 1ll << 19;  // elements per staging buffer
  std::vector<UpJob> jobs;
  auto add = [&](const int64_t* h, long long cnt, int* d, int kind) {
    for (long long i = 0; i < cnt; i += kChunk)
      jobs.push_back(UpJob{h + i, d + i, std::min(kChunk, cnt - i), kind});
  };
  add(off, n + 1, G.off.get(), 3);
  add(tgt, m2, G.tgt.get(), 0);
  add(ew, m2, G.w.get(), 1);
  add(vw, n, G.vw.get(), 2);
  const int T = (int)std::max<size_t>(1, std::min<size_t>(jobs.size(),
                                       std::max(2u, std::min(16u, std::thread::hardware_concurrency()))));
  std::vector<UpAcc> acc((size_t)T);
  std::vector<std::exception_ptr> errs((size_t)T);
  std::atomic<size_t> next{0};
  int dev = 0;
  GIM_CUDA(cudaGetDevice(&dev));
  auto worker = [&](int t) {
    cudaStream_t ws = nullptr;
    try {
      GIM_CUDA(cudaSetDevice(dev));
      ws = acquire_stream();
      int* stage = static_cast<int*>(pinned_scratch(sizeof(int) * 2 * kChunk));
      cudaEvent_t done[2];
      GIM_CUDA(cudaEventCreateWithFlags(&done[0], cudaEventDisableTiming));
      GIM_CUDA(cudaEventCreateWithFlags(&done[1], cudaEventDisableTiming));
      bool used[2] = {false, false};
      UpAcc& a = acc[(size_t)t];
      for (int slot = 0;; slot ^= 1) {
        const size_t j = next.fetch_add(1);
        if (j >= jobs.size()) break;
        const UpJob& J = jobs[j];
        int* buf = stage + (size_t)slot * kChunk;
        if (used[slot]) GIM_CUDA(cudaEventSynchronize(done[slot]));
        long long sum = 0;
        bool bad = false, nonpos = false, same = J.kind == 1 || J.kind == 2;
        bool badt = false, bado = false;
        if (same) {  // weights: validate, and look for a constant chunk first
          const int64_t x0 = J.src[0];
          for (long long i = 0; i < J.cnt; ++i) {
            const int64_t x = J.src[i];
            bad |= x < INT32_MIN || x > INT32_MAX;
            nonpos |= x <= 0;
            sum += x;
            same &= x == x0;
          }
          if (same && !bad) {
            k_fill_i32<<<grid_for(J.cnt, 256), 256, 0, ws>>>(J.cnt, (int)x0, J.dst);
            count_launch();
            GIM_LAUNCH_CHECK();
          } else {
            for (long long i = 0; i < J.cnt; ++i) buf[i] = (int)J.src[i];
          }
        } else {
          for (long long i = 0; i < J.cnt; ++i) {
            const int64_t x = J.src[i];
            bad |= x < INT32_MIN || x > INT32_MAX;
            badt |= x < 0 || x >= n;  // targets: vertex ids (offsets: below)
            buf[i] = (int)x;
          }
          if (J.kind == 3) {  // row lengths inside the chunk (boundaries: below)
            badt = false;
            for (long long i = 1; i < J.cnt; ++i) {
              const long long len = J.src[i] - J.src[i - 1];
              bado |= len < 0;
              a.maxdeg = std::max<long long>(a.maxdeg, len);
            }
          }
        }
        a.bad_range |= bad;
        a.bad_tgt |= badt;
        a.bad_off |= bado;
        if (J.kind == 1) a.bad_ew |= nonpos;
        if (J.kind == 1) a.sum_ew += sum;
        if (J.kind == 2) { a.sum_vw += sum; a.bad_vw |= nonpos; }
        if (!(same && !bad)) {
          GIM_CUDA(cudaMemcpyAsync(J.dst, buf, sizeof(int) * J.cnt, cudaMemcpyHostToDevice, ws));
          GIM_CUDA(cudaEventRecord(done[slot], ws));
          used[slot] = true;
          a.h2d += (long long)sizeof(int) * J.cnt;
        }
      }
      GIM_CUDA(sync_stream(ws));
      cudaEventDestroy(done[0]);
      cudaEventDestroy(done[1]);
    } catch (...) {
      errs[(size_t)t] = std::current_exception();
      if (ws) sync_stream(ws);
    }
    release_stream(ws);
  };
  std::vector<std::thread> pool;
  for (int t = 1; t < T; ++t) pool.emplace_back(worker, t);
  worker(0);
  for (auto& th : pool) th.join();
  for (auto& e : errs)
    if (e) std::rethrow_exception(e);
  UpAcc tot;
  for (auto& a : acc) {
    tot.sum_ew += a.sum_ew;
    tot.sum_vw += a.sum_vw;
    tot.bad_range |= a.bad_range;
    tot.bad_vw |= a.bad_vw;
    tot.bad_ew |= a.bad_ew;
    tot.bad_off |= a.bad_off;
    tot.bad_tgt |= a.bad_tgt;
    tot.h2d += a.h2d;
    tot.maxdeg = std::max(tot.maxdeg, a.maxdeg);
  }
  for (long long b = kChunk; b <= n; b += kChunk) {  // rows across chunk boundaries
    tot.maxdeg = std::max<long long>(tot.maxdeg, off[b] - off[b - 1]);
    tot.bad_off |= off[b] < off[b - 1];
  }
  G.maxdeg = (int)std::min<long long>(tot.maxdeg, INT32_MAX);
  GIM_CHECK(!tot.bad_range, GIM_E_OVERFLOW, "CSR values must fit int32");
  GIM_CHECK(!tot.bad_off, GIM_E_INVALID, "offsets must be nondecreasing");
  GIM_CHECK(!tot.bad_tgt, GIM_E_INVALID, "edge targets must lie in [0, n)");
  GIM_CHECK(!tot.bad_ew, GIM_E_INVALID, "edge weights must be positive");
  GIM_CHECK(!tot.bad_vw, GIM_E_INVALID, "vertex weights must be positive");
  GIM_CHECK(tot.sum_vw < INT32_MAX, GIM_E_OVERFLOW, "total vertex weight must be < 2^31");
  GIM_CHECK(tot.sum_ew < INT32_MAX, GIM_E_OVERFLOW, "total edge weight must be < 2^31");
  G.total_vw = tot.sum_vw;
  fill_sources((int)n, G.off.get(), G.src.get(), s);
  GIM_LAUNCH_CHECK();
  return tot.h2d;
}

__global__ void k_widen(int n, const int* __restrict__ in, long long* __restrict__ out) {
  for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < n; i += gridDim.x * blockDim.x)
    out[i] = in[i];
}

}  // namespace gim

// ===========================================================================
// C ABI

using namespace gim;

static gim_im_params default_params() {
  gim_im_params p;
  p.coarsest_factor = 128;
  p.phi = 0.999;
  p.rho = 2;
  p.filter_mode = 0;
  p.jet_filter_c = 0.25;
  p.sigma_coarse = 0.065;
  p.sigma_fine = 0.005;
  p.iw_max_finest = 10;
  p.run_flags = GIM_RUN_DEFAULT;
  p.isolated = GIM_ISOLATED_KEEP;
  return p;
}

// the call's mode flags: explicit bits or the process defaults
static RunFlags flags_of(const gim_im_params* P) {
  RunFlags f = default_flags();
  if (P && P->run_flags >= 0) {
    f.fused = P->run_flags & GIM_RUN_FUSED;
    f.rowwise = P->run_flags & GIM_RUN_ROWWISE;
    f.batch = P->run_flags & GIM_RUN_BATCH;
    f.fanout = P->run_flags & GIM_RUN_FANOUT;
    f.prof = P->run_flags & GIM_RUN_PROFILE;
  }
  return f;
}

extern "C" int gim_default_params(gim_im_params* out) {
  return guard([&] {
    GIM_CHECK(out, GIM_E_INVALID, "null argument");
    *out = default_params();
  });
}

extern "C" int gim_hem_round(const gim_graph* g, int32_t* partner, int32_t* preferred,
                             double l_max, uint64_t seed, int64_t* matched_inout, void* stream) {
  return guard([&] {
    GIM_CHECK(g && partner && preferred && matched_inout, GIM_E_INVALID, "null argument");
    cudaStream_t s = (cudaStream_t)stream;
    DBuf<long long> m(1, s);
    long long h = *matched_inout;
    GIM_CUDA(cudaMemcpyAsync(m.get(), &h, sizeof(long long), cudaMemcpyHostToDevice, s));
    hem_round(view(*g), partner, preferred, l_max, seed, m.get(), s);
    *matched_inout = read_scalar(m.get(), s);
  });
}

extern "C" int gim_match_graph(const gim_graph* g, double l_max, uint64_t seed, int32_t* partner,
                               int64_t* matched_out, void* stream) {
  return guard([&] {
    GIM_CHECK(g && partner, GIM_E_INVALID, "null argument");
    long long m = match_graph(view(*g), l_max, seed, partner, (cudaStream_t)stream);
    if (matched_out) *matched_out = m;
  });
}

extern "C" int gim_coarse_map(int32_t n, const int32_t* partner, int32_t* cmap_out,
                              int32_t* n_c_out, void* stream) {
  return guard([&] {
    GIM_CHECK(n >= 0 && n_c_out, GIM_E_INVALID, "bad argument");
    *n_c_out = gim::coarse_map(n, partner, cmap_out, (cudaStream_t)stream);
  });
}

extern "C" int gim_contract(const gim_graph* g, const int32_t* coarse_map, int32_t n_c,
                            int32_t* out_offsets, int32_t* out_targets, int32_t* out_weights,
                            int32_t* out_vweights, int32_t* out_sources, int64_t* m2_out,
                            void* stream) {
  return guard([&] {
    GIM_CHECK(g && m2_out && n_c >= 0, GIM_E_INVALID, "bad argument");
    *m2_out = contract_into(view(*g), coarse_map, n_c, out_offsets, out_targets, out_weights,
                            out_vweights, out_sources, (cudaStream_t)stream);
  });
}

extern "C" int gim_project(int32_t n, const int32_t* coarse_map, const int32_t* coarse_part,
                           int32_t* fine_part, void* stream) {
  return guard([&] { project(n, coarse_map, coarse_part, fine_part, (cudaStream_t)stream); });
}

extern "C" int gim_conn_build(const gim_graph* g, const int32_t* assignment, int32_t k,
                              int32_t* out_offsets, int32_t* out_blocks, int32_t* out_weights,
                              int64_t* total_out, void* stream) {
  return guard([&] {
    GIM_CHECK(g && total_out && k >= 1, GIM_E_INVALID, "bad argument");
    *total_out = conn_build(view(*g), assignment, k, out_offsets, out_blocks, out_weights,
                            (cudaStream_t)stream);
  });
}

__global__ void k_lp_export(int n, const unsigned char* tm, unsigned char* out) {
  for (int v = blockIdx.x * blockDim.x + threadIdx.x; v < n; v += gridDim.x * blockDim.x)
    out[v] = tm[v];
}

extern "C" int gim_lp_pass(const gim_graph* g, const int32_t* assignment, const uint8_t* locked,
                           const gim_topology* t, int32_t jet, double jet_c, uint8_t* out_cand,
                           int32_t* out_dest, uint8_t* out_to_move, int64_t* movers_out,
                           void* stream) {
  return guard([&] {
    GIM_CHECK(g && t, GIM_E_INVALID, "null argument");
    cudaStream_t s = (cudaStream_t)stream;
    Topo tp = get_topo(*t);
    RefineLevel L;
    L.g = view(*g);
    prepare_level(L, tp.k, s);
    RefineBuffers rb;
    alloc_refine_buffers(rb, g->n, tp.k, s);
    lp_pass(L, tp, assignment, locked, jet, jet_c, rb, s);
    if (g->n) {
      GIM_CUDA(cudaMemcpyAsync(out_cand, rb.cand.get(), g->n, cudaMemcpyDeviceToDevice, s));
      GIM_CUDA(cudaMemcpyAsync(out_dest, rb.dest.get(), sizeof(int) * g->n, cudaMemcpyDeviceToDevice, s));
      GIM_CUDA(cudaMemcpyAsync(out_to_move, rb.to_move.get(), g->n, cudaMemcpyDeviceToDevice, s));
    }
    long long mv = read_scalar(rb.movers, s);
    if (movers_out) *movers_out = mv;
  });
}

__global__ void k_rb_export(int n, const int* part, const unsigned char* ovl, const int* target,
                            const unsigned char* tm, const int* dest, unsigned char* cand,
                            int* odest, unsigned char* otm) {
  for (int v = blockIdx.x * blockDim.x + threadIdx.x; v < n; v += gridDim.x * blockDim.x) {
    bool c = ovl[part[v]] && target[v] >= 0;
    cand[v] = c;
    odest[v] = c ? target[v] : part[v];
    otm[v] = tm[v];
    (void)dest;
  }
}

extern "C" int gim_rebalance(const gim_graph* g, const int32_t* assignment,
                             const int64_t* block_weights, const gim_topology* t, int32_t strong,
                             double sigma, double l_max, int32_t rho, uint64_t seed,
                             int64_t pass_counter, uint8_t* out_cand, int32_t* out_dest,
                             uint8_t* out_to_move, int32_t* incomplete_out, void* stream) {
  return guard([&] {
    GIM_CHECK(g && t && block_weights, GIM_E_INVALID, "null argument");
    GIM_CHECK(rho >= 1, GIM_E_INVALID, "rho must be >= 1");
    cudaStream_t s = (cudaStream_t)stream;
    Topo tp = get_topo(*t);
    const int k = tp.k;
    std::vector<long long> bw((size_t)k);
    GIM_CUDA(cudaMemcpyAsync(bw.data(), block_weights, sizeof(long long) * k,
                             cudaMemcpyDeviceToHost, s));
    GIM_CUDA(sync_stream(s));
    std::vector<unsigned char> masks((size_t)k * 2);
    std::vector<int> el;
    for (int b = 0; b < k; ++b) {
      masks[b] = (double)bw[b] > l_max;
      masks[k + b] = (double)bw[b] < sigma;
      if (masks[k + b]) el.push_back(b);
    }
    DBuf<unsigned char> dm((size_t)k * 2, s);
    DBuf<int> de((size_t)k, s);
    GIM_CUDA(cudaMemcpyAsync(dm.get(), masks.data(), (size_t)k * 2, cudaMemcpyHostToDevice, s));
    if (!el.empty())
      GIM_CUDA(cudaMemcpyAsync(de.get(), el.data(), sizeof(int) * el.size(), cudaMemcpyHostToDevice, s));
    RefineLevel L;
    L.g = view(*g);
    prepare_level(L, k, s);
    RefineBuffers rb;
    alloc_refine_buffers(rb, g->n, k, s);
    rebalance_pass(L, tp, assignment, reinterpret_cast<const long long*>(block_weights),
                   strong != 0, l_max, rho, seed, pass_counter,
                   dm.get(), dm.get() + k, de.get(), (int)el.size(), rb, s);
    if (g->n) {
      k_rb_export<<<grid_for(g->n, 256), 256, 0, s>>>(g->n, assignment, dm.get(), rb.dest2.get(),
                                                       rb.to_move.get(), rb.dest.get(), out_cand,
                                                       out_dest, out_to_move);
      GIM_LAUNCH_CHECK();
    }
    GIM_CUDA(sync_stream(s));
    if (incomplete_out) *incomplete_out = el.empty() ? 1 : 0;
  });
}

extern "C" int gim_apply_moves(const gim_graph* g, int32_t* assignment, int64_t* block_weights,
                               const uint8_t* to_move, const int32_t* dest, const gim_topology* t,
                               int64_t* delta_j_out, void* stream) {
  return guard([&] {
    GIM_CHECK(g && t, GIM_E_INVALID, "null argument");
    cudaStream_t s = (cudaStream_t)stream;
    Topo tp = get_topo(*t);
    RefineLevel L;
    L.g = view(*g);
    prepare_level(L, tp.k, s);
    RefineBuffers rb;
    alloc_refine_buffers(rb, g->n, tp.k, s);
    if (g->n) {
      GIM_CUDA(cudaMemcpyAsync(rb.to_move.get(), to_move, g->n, cudaMemcpyDeviceToDevice, s));
      GIM_CUDA(cudaMemcpyAsync(rb.dest.get(), dest, sizeof(int) * g->n, cudaMemcpyDeviceToDevice, s));
    }
    apply_moves(L, tp, assignment, reinterpret_cast<long long*>(block_weights), rb, s);
    long long dj = read_scalar(rb.dj, s);
    if (delta_j_out) *delta_j_out = dj;
  });
}

extern "C" int gim_refine(const gim_graph* g, const gim_topology* t, int32_t* assignment,
                          int64_t* block_weights, double phi, int32_t i_max, int32_t i_w_max,
                          double sigma_fraction, int32_t rho, int32_t jet, double jet_c,
                          uint64_t seed, double l_max, void* stream) {
  return guard([&] {
    GIM_CHECK(g && t, GIM_E_INVALID, "null argument");
    cudaStream_t s = (cudaStream_t)stream;
    Topo tp = get_topo(*t);
    RefineLevel L;
    L.g = view(*g);
    RefCfg c;
    c.phi = phi;
    c.i_max = i_max;
    c.i_w_max = i_w_max;
    c.sigma_fraction = sigma_fraction;
    c.rho = rho;
    c.jet = jet;
    c.jet_c = jet_c;
    c.seed = seed;
    RunStats st;
    RefineBuffers rb;
    refine(L, tp, assignment, reinterpret_cast<long long*>(block_weights), c, l_max, st, rb, s);
  });
}

extern "C" int gim_greedy_graph_growing(const gim_graph* g, int32_t k, int32_t* part,
                                        void* stream) {
  return guard([&] {
    GIM_CHECK(g && k >= 1, GIM_E_INVALID, "bad argument");
    GIM_CHECK(g->n > k || k == 1, GIM_E_INVALID, "greedy graph growing needs n > k");
    greedy_graph_growing(view(*g), k, part, (cudaStream_t)stream);
  });
}

extern "C" int gim_internal_partitioner(const gim_graph* g, int32_t k, double eps_local,
                                        uint64_t seed, int32_t* part, void* stream) {
  return guard([&] {
    GIM_CHECK(g && k >= 1, GIM_E_INVALID, "bad argument");
    cudaStream_t s = (cudaStream_t)stream;
    DevGraph dg = view(*g);
    long long total = total_vertex_weight(dg, s);
    RunStats st;
    internal_partitioner(dg, total, k, eps_local, seed, part, st, s);
    GIM_CUDA(sync_stream(s));
  });
}

extern "C" int gim_hierarchical_multisection(const gim_graph* g, const gim_topology* t, double eps,
                                             uint64_t seed, int32_t* assignment, void* stream) {
  return guard([&] {
    GIM_CHECK(g && t, GIM_E_INVALID, "null argument");
    cudaStream_t s = (cudaStream_t)stream;
    DevGraph dg = view(*g);
    GIM_CHECK(dg.n > 0, GIM_E_EMPTY, "cannot map an empty graph");
    (void)get_topo(*t);
    long long total = total_vertex_weight(dg, s);
    std::vector<long long> h(t->hierarchy, t->hierarchy + t->levels);
    RunStats st;
    RunCtx rc;
    rc.f = default_flags();
    CtxScope scope(&rc);
    hierarchical_multisection(dg, total, h, eps, seed, assignment, st, s);
    GIM_CUDA(sync_stream(s));
  });
}

// GPU-HM on host arrays (pipelines.py:49-110 as a standalone algorithm):
// upload as gim_integrated_map, multisection of the whole graph, int64 out
extern "C" int gim_hierarchical_multisection_host(int64_t n, const int64_t* offsets,
                                                  const int64_t* targets,
                                                  const int64_t* edge_weights,
                                                  const int64_t* vertex_weights,
                                                  const gim_topology* t, double eps,
                                                  uint64_t seed, int64_t* out_assignment,
                                                  int64_t* out_block_weights, void* stream) {
  return guard([&] {
    GIM_CHECK(t && offsets && out_assignment && out_block_weights, GIM_E_INVALID,
              "null argument");
    GIM_CHECK(n > 0, GIM_E_EMPTY, "cannot map an empty graph");
    cudaStream_t s = (cudaStream_t)stream;
    RunCtx rc;
    rc.f = default_flags();
    CtxScope scope(&rc);
    OwnedGraph G;
    upload_graph(n, offsets, targets, edge_weights, vertex_weights, G, s);
    Topo tp = get_topo(*t);
    std::vector<long long> h(t->hierarchy, t->hierarchy + t->levels);
    DBuf<int> part((size_t)n, s);
    DBuf<long long> bw((size_t)tp.k, s);
    RunStats st;
    reset_launches();
    hierarchical_multisection(G.view(), G.total_vw, h, eps, seed, part.get(), st, s);
    block_weights((int)n, G.vw.get(), part.get(), tp.k, bw.get(), s);
    int* h_part = static_cast<int*>(pinned_scratch(sizeof(int) * (size_t)n));
    GIM_CUDA(cudaMemcpyAsync(h_part, part.get(), sizeof(int) * n, cudaMemcpyDeviceToHost, s));
    GIM_CUDA(cudaMemcpyAsync(out_block_weights, bw.get(), sizeof(long long) * tp.k,
                             cudaMemcpyDeviceToHost, s));
    GIM_CUDA(sync_stream(s));
    for (long long i = 0; i < n; ++i) out_assignment[i] = h_part[i];
  });
}

extern "C" int gim_hierarchical_multisection_plugin(
    int64_t n, const int64_t* offsets, const int64_t* targets, const int64_t* edge_weights,
    const int64_t* vertex_weights, const gim_topology* t, double eps, uint64_t seed,
    gim_partition_fn partition, gim_trace_fn trace, void* user, int64_t* out_assignment,
    int64_t* out_block_weights, void* stream) {
  return guard([&] {
    GIM_CHECK(t && offsets && out_assignment && out_block_weights, GIM_E_INVALID,
              "null argument");
    GIM_CHECK(n > 0, GIM_E_EMPTY, "cannot map an empty graph");
    cudaStream_t s = (cudaStream_t)stream;
    RunCtx rc;
    rc.f = default_flags();
    CtxScope scope(&rc);
    OwnedGraph G;
    upload_graph(n, offsets, targets, edge_weights, vertex_weights, G, s);
    Topo tp = get_topo(*t);
    std::vector<long long> h(t->hierarchy, t->hierarchy + t->levels);
    DBuf<int> part((size_t)n, s);
    DBuf<long long> bw((size_t)tp.k, s);
    RunStats st;
    MsCtx C;
    C.h = h;
    C.k = tp.k;
    C.total = G.total_vw;
    C.eps = eps;
    C.assignment = part.get();
    C.st = &st;
    C.threads = false;
    GIM_CUDA(cudaGetDevice(&C.device));
    GIM_CUDA(cudaMemsetAsync(part.get(), 0, sizeof(int) * n, s));
    DBuf<int> ident_ids((size_t)n, s);
    k_iota<<<grid_for(n, 256), 256, 0, s>>>((int)n, ident_ids.get());
    count_launch();
    PluginCtx P{&C, partition, trace, user};
    std::vector<int> ident;
    descend_plugin(P, G.view(), G.total_vw, (int)h.size(), ident, ident_ids.get(), seed, s);
    block_weights((int)n, G.vw.get(), part.get(), tp.k, bw.get(), s);
    std::vector<int> hp((size_t)n);
    GIM_CUDA(cudaMemcpyAsync(hp.data(), part.get(), sizeof(int) * n, cudaMemcpyDeviceToHost, s));
    GIM_CUDA(cudaMemcpyAsync(out_block_weights, bw.get(), sizeof(long long) * tp.k,
                             cudaMemcpyDeviceToHost, s));
    GIM_CUDA(sync_stream(s));
    for (long long i = 0; i < n; ++i) out_assignment[i] = hp[(size_t)i];
  });
}

extern "C" int gim_integrated_map_device(const gim_graph* g, const gim_topology* t, double eps,
                                         uint64_t seed, const gim_im_params* params,
                                         int32_t* out_assignment, int64_t* out_block_weights,
                                         gim_im_stats* stats, void* stream) {
  return guard([&] {
    GIM_CHECK(g && t && out_assignment && out_block_weights, GIM_E_INVALID, "null argument");
    cudaStream_t s = (cudaStream_t)stream;
    DevGraph dg = view(*g);
    GIM_CHECK(dg.n > 0, GIM_E_EMPTY, "cannot map an empty graph");
    gim_im_params P = params ? *params : default_params();
    RunCtx rc;
    rc.f = flags_of(&P);
    CtxScope scope(&rc);
    long long total = total_vertex_weight(dg, s);
    (P.isolated == GIM_ISOLATED_STRIP ? integrated_map_strip : integrated_map_dispatch)(
        dg, total, *t, eps, seed, P, out_assignment,
                          reinterpret_cast<long long*>(out_block_weights), stats, s);
  });
}

extern "C" int gim_integrated_map(int64_t n, const int64_t* offsets, const int64_t* targets,
                                  const int64_t* edge_weights, const int64_t* vertex_weights,
                                  const gim_topology* t, double eps, uint64_t seed,
                                  const gim_im_params* params, int64_t* out_assignment,
                                  int64_t* out_block_weights, gim_im_stats* stats, void* stream) {
  return guard([&] {
    GIM_CHECK(t && offsets && out_assignment && out_block_weights, GIM_E_INVALID,
              "null argument");
    GIM_CHECK(n > 0, GIM_E_EMPTY, "cannot map an empty graph");
    cudaStream_t s = (cudaStream_t)stream;
    gim_im_params P = params ? *params : default_params();
    RunCtx rc;
    rc.f = flags_of(&P);
    CtxScope scope(&rc);
    OwnedGraph G;
    const auto t_up = std::chrono::steady_clock::now();
    const long long h2d = upload_graph(n, offsets, targets, edge_weights, vertex_weights, G, s);
    GIM_CUDA(sync_stream(s));
    const double ms_up =
        std::chrono::duration<double, std::milli>(std::chrono::steady_clock::now() - t_up).count();
    Topo tp = get_topo(*t);
    DBuf<int> part((size_t)n, s);
    DBuf<long long> bw((size_t)tp.k, s);
    (P.isolated == GIM_ISOLATED_STRIP ? integrated_map_strip : integrated_map_dispatch)(
        G.view(), G.total_vw, *t, eps, seed, P, part.get(), bw.get(), stats, s);
    const auto t_down = std::chrono::steady_clock::now();
    // int32 assignment -> pinned staging -> widened to int64 on the host by
    // worker threads (half the PCIe bytes, no pageable staging copy)
    int* h_part = static_cast<int*>(pinned_scratch(sizeof(int) * (size_t)n));
    GIM_CUDA(cudaMemcpyAsync(h_part, part.get(), sizeof(int) * n, cudaMemcpyDeviceToHost, s));
    GIM_CUDA(cudaMemcpyAsync(out_block_weights, bw.get(), sizeof(long long) * tp.k,
                             cudaMemcpyDeviceToHost, s));
    GIM_CUDA(sync_stream(s));
    {
      const int T = (int)std::max(1u, std::min(16u, std::thread::hardware_concurrency()));
      const long long per = (n + T - 1) / T;
      auto widen = [&](int t) {
        const long long a = std::min<long long>(n, t * per), b = std::min<long long>(n, a + per);
        for (long long i = a; i < b; ++i) out_assignment[i] = h_part[i];
      };
      std::vector<std::thread> pool;
      if (n >= (1ll << 20))
        for (int t = 1; t < T; ++t) pool.emplace_back(widen, t);
      else
        for (int t = 1; t < T; ++t) widen(t);
      widen(0);
      for (auto& th : pool) th.join();
    }
    if (stats) {
      stats->kernel_launches = launches();
      stats->ms_upload = ms_up;
      stats->bytes_h2d = h2d;
      stats->bytes_d2h = (long long)sizeof(int) * n + (long long)sizeof(long long) * tp.k;
      stats->ms_download = std::chrono::duration<double, std::milli>(
                               std::chrono::steady_clock::now() - t_down).count();
    }
  });
}

namespace gim {
bool metis_arrays(void* handle, long long* n, const long long** off, const long long** tgt,
                  const long long** w, const long long** vw);
void metis_free(void* handle);
}  // namespace gim

extern "C" int gim_metis_upload(void* handle, int32_t* offsets, int32_t* targets,
                                int32_t* weights, int32_t* vweights, int32_t* sources,
                                int64_t* total_vweight, void* stream) {
  return guard([&] {
    long long n = 0;
    const long long *off = nullptr, *tgt = nullptr, *w = nullptr, *vw = nullptr;
    GIM_CHECK(metis_arrays(handle, &n, &off, &tgt, &w, &vw), GIM_E_INVALID, "null handle");
    struct Free {
      void* h;
      ~Free() { metis_free(h); }
    } guard_free{handle};
    GIM_CHECK(offsets && total_vweight, GIM_E_INVALID, "null argument");
    cudaStream_t s = (cudaStream_t)stream;
    OwnedGraph G;
    upload_graph(n, reinterpret_cast<const int64_t*>(off), reinterpret_cast<const int64_t*>(tgt),
                 reinterpret_cast<const int64_t*>(w), reinterpret_cast<const int64_t*>(vw), G, s);
    const long long m2 = G.m2;
    GIM_CUDA(cudaMemcpyAsync(offsets, G.off.get(), sizeof(int) * (n + 1), cudaMemcpyDeviceToDevice, s));
    if (m2) {
      GIM_CUDA(cudaMemcpyAsync(targets, G.tgt.get(), sizeof(int) * m2, cudaMemcpyDeviceToDevice, s));
      GIM_CUDA(cudaMemcpyAsync(weights, G.w.get(), sizeof(int) * m2, cudaMemcpyDeviceToDevice, s));
      GIM_CUDA(cudaMemcpyAsync(sources, G.src.get(), sizeof(int) * m2, cudaMemcpyDeviceToDevice, s));
    }
    if (n) GIM_CUDA(cudaMemcpyAsync(vweights, G.vw.get(), sizeof(int) * n, cudaMemcpyDeviceToDevice, s));
    *total_vweight = G.total_vw;
    GIM_CUDA(sync_stream(s));
  });
}

extern "C" int gim_fill_sources(int32_t n, const int32_t* offsets, int32_t* sources, void* stream) {
  return guard([&] { fill_sources(n, offsets, sources, (cudaStream_t)stream); });
}

extern "C" int64_t gim_launch_count(void) { return launches(); }
extern "C" void gim_release_cached_memory(void) { gim::release_cached_memory(); }
extern "C" void gim_reset_launch_count(void) { reset_launches(); }

namespace gim {
template <class F>
static void update_defaults(F&& edit) {
  RunFlags f = default_flags();
  edit(f);
  set_default_flags(f);
}
}  // namespace gim

extern "C" void gim_set_fanout(int32_t on) {
  gim::update_defaults([&](gim::RunFlags& f) { f.fanout = on != 0; });
}
extern "C" void gim_set_fused(int32_t on) {
  gim::update_defaults([&](gim::RunFlags& f) { f.fused = on != 0; });
}
extern "C" void gim_set_batch(int32_t on) {
  gim::update_defaults([&](gim::RunFlags& f) { f.batch = on != 0; });
}
extern "C" void gim_set_rowwise_contraction(int32_t on) {
  gim::update_defaults([&](gim::RunFlags& f) { f.rowwise = on != 0; });
}
