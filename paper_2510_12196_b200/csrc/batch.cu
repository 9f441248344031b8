// Batched internal partitioner for the small subgraphs of the hierarchical
// multisection (pipelines.py:191-218, called from :49-110).
//
// The lower levels of the multisection tree hold dozens of independent
// subgraphs of a few hundred vertices (H = 4:8:6: 48 leaves' parents).
// Running each through the general path costs ~100 kernel launches and ~20
// host round trips per call, so the calls are host-latency bound.  Here
// all jobs of one tree level advance together, one CTA per job:
//
//   1. k_coarsen_small: the whole level stack of every job (matching
//      rounds, coarse ids, contraction) in ONE launch, one CTA per job,
//      levels written into a per-job arena (coarsening.py:164-295);
//   2. k_ggg on every job's coarsest graph in one launch;
//   3. per uncoarsening step: one projection/block-weight launch and one
//      shared-memory-resident Alg. 4 launch (k_refine_smem_batch) for all
//      jobs still refining.
//
// Results are identical to internal_partitioner(): every kernel computes the
// same values as the general path.  Jobs the fast path cannot take (two-hop
// matching needed, arena overflow, a level too large for shared memory, a
// strong rebalancing pass) fall back to the general code for that job.
#include <algorithm>
#include <vector>

#include "coarsen_dev.cuh"
#include "common.cuh"
#include "kernels.cuh"
#include "scan.cuh"

namespace gim {

constexpr int kBcBlock = 512;
constexpr int kBcMaxLevels = 24;

struct BcLevel {
  int n, m2;
  long long off, tgt, w, vw, cmap;  // word offsets into the job arena (-1: input level)
};

struct BcJob {
  int n, m2;
  const int* off;
  const int* tgt;
  const int* w;
  const int* vw;
  double l_max;
  unsigned long long seed;
  long long threshold;
  int* arena;
  long long cap;  // words
  int nl;
  int status;  // 0 ok, 1 level nl-1 needs two-hop matching, 2 out of room
  BcLevel lv[kBcMaxLevels];
};

// CTA-wide exclusive scan of in[0..N) into out (may alias); returns the total
__device__ int bc_scan(const int* in, int* out, int N) {
  __shared__ int tot;
  int carry = 0;
  for (int base = 0; base < N; base += kBcBlock) {
    const int i = base + threadIdx.x;
    const int x = i < N ? in[i] : 0;
    const int ex = block_excl_scan<int, kBcBlock>(x, &tot);
    if (i < N) out[i] = carry + ex;
    carry += tot;
    __syncthreads();
  }
  return carry;
}

__device__ long long bc_sum(long long v) {
  __shared__ long long red[kBcBlock / 32];
  v = warp_sum_ll(v);
  if (lane_id() == 0) red[threadIdx.x >> 5] = v;
  __syncthreads();
  long long r = 0;
  for (int i = 0; i < kBcBlock / 32; ++i) r += red[i];
  __syncthreads();
  return r;
}

__global__ void __launch_bounds__(kBcBlock) k_coarsen_small(BcJob* jobs) {
  BcJob& J = jobs[blockIdx.x];
  __shared__ long long s_top;
  __shared__ int s_stop;
  int* const A = J.arena;
  if (threadIdx.x == 0) {
    s_top = 0;
    J.status = 0;
    J.nl = 1;
    J.lv[0] = BcLevel{J.n, J.m2, -1, -1, -1, -1, -1};
  }
  __syncthreads();
  const int* off = J.off;
  const int* tgt = J.tgt;
  const int* w = J.w;
  const int* vw = J.vw;
  int n = J.n;
  long long m2 = J.m2;
  for (int lev = 0;; ++lev) {
    if ((long long)n < J.threshold) break;
    if (lev + 1 >= kBcMaxLevels) {
      if (threadIdx.x == 0) J.status = 2;
      break;
    }
    // this level needs <= 4n (partner, elig, pref, cmap) + 5 n_c + 2 (mem, L,
    // cnt, cvw) + 2 m2 (staged pairs) + 2 n_c + 1 + 2 m2 (the coarse level)
    if (s_top + 11ll * n + 4ll * m2 + 8 > J.cap) {
      if (threadIdx.x == 0) J.status = 2;
      break;
    }
    int* partner = A + s_top;
    int* elig = partner + n;
    int* pref = elig + n;
    int* cmap = pref + n;
    for (int v = threadIdx.x; v < n; v += kBcBlock) partner[v] = -1;
    __syncthreads();
    // ---- match_graph (coarsening.py:164-173): <= 2 HEM rounds, >= 40% stops
    const unsigned long long lseed = splitmix64(J.seed ^ (unsigned long long)lev);
    long long matched = 0;
    for (int r = 0; r < 2; ++r) {
      const double frac = n ? (double)matched / (double)n : 1.0;
      if (frac >= 0.40) break;
      const unsigned long long seed = splitmix64(lseed ^ (unsigned long long)(r + 1));
      for (int v = threadIdx.x; v < n; v += kBcBlock) elig[v] = partner[v] < 0 ? vw[v] : -1;
      __syncthreads();
      for (int v = threadIdx.x; v < n; v += kBcBlock) {
        const int cvv = elig[v];
        int best_u = -1;
        if (cvv >= 0) {
          HemCand best;
          best.u = -1;
          best.w = best.c = best.slot = 0;
          best.h = 0;
          const long long cv = cvv;
          for (int e = off[v]; e < off[v + 1]; ++e) {
            const int u = tgt[e];
            const int cu = elig[u];
            if (cu < 0 || (double)(cv + cu) > J.l_max) continue;
            HemCand c;
            c.w = w[e];
            c.c = cu;
            c.slot = e;
            c.u = u;
            c.h = hash2(seed, (unsigned long long)min(v, u), (unsigned long long)max(v, u));
            if (hem_better(c, best)) best = c;
          }
          best_u = best.u;
        }
        pref[v] = best_u;
      }
      __syncthreads();
      long long cnt = 0;
      for (int v = threadIdx.x; v < n; v += kBcBlock) {
        const int u = pref[v];
        if (u >= 0 && v < u && pref[u] == v) {
          partner[v] = u;
          partner[u] = v;
          cnt += 2;
        }
      }
      __syncthreads();
      matched += bc_sum(cnt);
    }
    {
      const double frac = n ? (double)matched / (double)n : 1.0;
      if (frac < 0.40) {  // two-hop matching: general path
        if (threadIdx.x == 0) J.status = 1;
        break;
      }
    }
    // ---- coarse ids (coarsening.py:176-188): roots in vertex order
    for (int v = threadIdx.x; v < n; v += kBcBlock) {
      const int p = partner[v];
      pref[v] = (p < 0 || v < p) ? 1 : 0;
    }
    __syncthreads();
    const int n_c = bc_scan(pref, pref, n);
    for (int v = threadIdx.x; v < n; v += kBcBlock) {
      const int p = partner[v];
      cmap[v] = (p >= 0 && p < v) ? pref[p] : pref[v];
    }
    __syncthreads();
    if ((double)n_c * 1.02 > (double)n) break;  // stall guard: level not added
    // ---- contraction of the matching (coarsening.py:191-249): rows sorted
    // by target, parallel edges summed, self loops dropped
    long long top = s_top + 4ll * n;  // keep partner/elig/pref/cmap (cmap persists)
    int* mem = A + top;               // [2 n_c]
    int* L = mem + 2ll * n_c;         // [n_c + 1] row bounds -> ub offsets
    int* cnt = L + n_c + 1;           // [n_c + 1] true degrees -> offsets
    int* cvw = cnt + n_c + 1;         // [n_c]
    for (int v = threadIdx.x; v < n; v += kBcBlock) {
      const int p = partner[v];
      if (p >= 0 && p < v) continue;
      const int c = cmap[v];
      mem[2 * c] = v;
      mem[2 * c + 1] = p;
      int len = off[v + 1] - off[v];
      int wsum = vw[v];
      if (p >= 0) {
        len += off[p + 1] - off[p];
        wsum += vw[p];
      }
      L[c] = len;
      cvw[c] = wsum;
    }
    __syncthreads();
    const int ubtot = bc_scan(L, L, n_c);
    int* tk = cvw + n_c;     // [ubtot] staged keys
    int* tw = tk + ubtot;    // [ubtot] staged weights
    long long after = (tw + ubtot) - A;
    if (after + 2ll * n_c + 1 + 2ll * ubtot + 8 > J.cap) {
      if (threadIdx.x == 0) J.status = 2;
      break;
    }
    for (int c = threadIdx.x; c < n_c; c += kBcBlock) {
      const int base = L[c];
      int m = 0;
      for (int h = 0; h < 2; ++h) {
        const int x = mem[2 * c + h];
        if (x < 0) break;
        for (int e = off[x]; e < off[x + 1]; ++e) {
          const int key = cmap[tgt[e]];
          if (key == c) continue;
          const int wt = w[e];
          int pos = m;
          while (pos > 0 && tk[base + pos - 1] > key) --pos;
          if (pos > 0 && tk[base + pos - 1] == key) {
            tw[base + pos - 1] += wt;
            continue;
          }
          for (int i = m; i > pos; --i) {
            tk[base + i] = tk[base + i - 1];
            tw[base + i] = tw[base + i - 1];
          }
          tk[base + pos] = key;
          tw[base + pos] = wt;
          ++m;
        }
      }
      cnt[c] = m;
    }
    __syncthreads();
    const int m2c = bc_scan(cnt, cnt, n_c);
    if (threadIdx.x == 0) cnt[n_c] = m2c;
    // the new level's arrays
    int* noff = A + after;
    int* ntgt = noff + n_c + 1;
    int* nw = ntgt + m2c;
    int* nvw = nw + m2c;
    __syncthreads();
    for (int c = threadIdx.x; c <= n_c; c += kBcBlock) noff[c] = cnt[c];
    for (int c = threadIdx.x; c < n_c; c += kBcBlock) {
      nvw[c] = cvw[c];
      const int b = L[c], o = cnt[c], d = cnt[c + 1] - o;
      for (int i = 0; i < d; ++i) {
        ntgt[o + i] = tk[b + i];
        nw[o + i] = tw[b + i];
      }
    }
    __syncthreads();
    if (threadIdx.x == 0) {
      J.lv[lev].cmap = cmap - A;
      J.lv[lev + 1] = BcLevel{n_c, m2c, noff - A, ntgt - A, nw - A, nvw - A, -1};
      J.nl = lev + 2;
      // keep cmap + the new level; everything after the new level is free
      s_top = (nvw + n_c) - A;
      // cmap lives inside the old scratch block below the new level: safe
    }
    __syncthreads();
    off = noff;
    tgt = ntgt;
    w = nw;
    vw = nvw;
    n = n_c;
    m2 = m2c;
  }
  (void)s_stop;
}

// ---- batched projection + block weights for one uncoarsening step

__global__ void __launch_bounds__(256) k_bproj_bw(const BpJob* jobs) {
  const BpJob J = jobs[blockIdx.x];
  __shared__ long long hist[1024];
  for (int b = threadIdx.x; b < J.k; b += blockDim.x) hist[b] = 0;
  __syncthreads();
  for (int v = threadIdx.x; v < J.n; v += blockDim.x) {
    const int p = J.cmap ? J.coarse[J.cmap[v]] : J.part[v];
    if (J.cmap) J.part[v] = p;
    atomicAdd(reinterpret_cast<unsigned long long*>(&hist[p]), (unsigned long long)J.vw[v]);
  }
  __syncthreads();
  for (int b = threadIdx.x; b < J.k; b += blockDim.x) J.bw[b] = hist[b];
}

// ---- batched subgraph extraction (graph.py:357-389) for one tree level:
// one CTA per node; children get local ids in vertex order, rows keep only
// slots inside the part in CSR order, plus the children's global ids.
// Child c of a node lives at the node's arena offset cbase[c]; every array
// starts 16-byte aligned (the edge-parallel kernels load int4):
// off[n_c + 1] | tgt[m2_c] | w[m2_c] | src[m2_c] | vw[n_c] | trans[n_c]

__host__ __device__ __forceinline__ long long ex_r4(long long x) { return (x + 3) & ~3ll; }

constexpr int kExBlock = 512;
constexpr int kExMaxParts = 64;

struct ExNode {
  int n, parts;
  const int* off;
  const int* tgt;
  const int* w;
  const int* vw;
  const int* part;
  const int* trans;    // global ids of the node's vertices
  int* arena;
  long long cap;       // words
  int* scratch;        // [2 n]: local ids, kept degrees / offsets
  // out
  int status;
  int cn[kExMaxParts], cm2[kExMaxParts];
  long long cbase[kExMaxParts];
  long long ctotal[kExMaxParts];
};

__global__ void __launch_bounds__(kExBlock) k_extract_batch(ExNode* nodes) {
  ExNode& X = nodes[blockIdx.x];
  const int n = X.n, P = X.parts;
  int* local = X.scratch;
  int* kdeg = X.scratch + n;
  __shared__ int s_cnt[kExMaxParts], s_m2[kExMaxParts];
  __shared__ long long s_tot[kExMaxParts];
  for (int c = threadIdx.x; c < P; c += kExBlock) {
    s_cnt[c] = 0;
    s_m2[c] = 0;
    s_tot[c] = 0;
  }
  __syncthreads();
  // per part: local ids (stable ranks) and kept-degree prefix sums, by CTA
  // scans over the vertex range (parts are few)
  for (int c = 0; c < P; ++c) {
    int carry = 0, carry2 = 0;
    long long tot = 0;
    __shared__ int t1, t2;
    for (int base = 0; base < n; base += kExBlock) {
      const int v = base + threadIdx.x;
      int in = 0, kd = 0;
      if (v < n && X.part[v] == c) {
        in = 1;
        for (int e = X.off[v]; e < X.off[v + 1]; ++e) kd += X.part[X.tgt[e]] == c;
        tot += X.vw[v];
      }
      const int ex = block_excl_scan<int, kExBlock>(in, &t1);
      const int ex2 = block_excl_scan<int, kExBlock>(kd, &t2);
      if (in) {
        local[v] = carry + ex;
        kdeg[v] = carry2 + ex2;  // row offset inside the child
      }
      carry += t1;
      carry2 += t2;
      __syncthreads();
    }
    tot = bc_sum(tot);
    if (threadIdx.x == 0) {
      s_cnt[c] = carry;
      s_m2[c] = carry2;
      s_tot[c] = tot;
    }
  }
  __syncthreads();
  // arena layout of the children
  __shared__ long long s_base[kExMaxParts];
  __shared__ int s_bad;
  if (threadIdx.x == 0) {
    long long at = 0;
    s_bad = 0;
    for (int c = 0; c < P; ++c) {
      s_base[c] = at;
      at += ex_r4(s_cnt[c] + 1ll) + 3 * ex_r4(s_m2[c]) + 2 * ex_r4(s_cnt[c]);
    }
    if (at > X.cap) s_bad = 1;
    X.status = s_bad;
    for (int c = 0; c < P; ++c) {
      X.cn[c] = s_cnt[c];
      X.cm2[c] = s_m2[c];
      X.cbase[c] = s_base[c];
      X.ctotal[c] = s_tot[c];
    }
  }
  __syncthreads();
  if (s_bad) return;
  for (int v = threadIdx.x; v < n; v += kExBlock) {
    const int c = X.part[v];
    const int nc = s_cnt[c], mc = s_m2[c];
    int* co = X.arena + s_base[c];
    int* ct = co + ex_r4(nc + 1ll);
    int* cw = ct + ex_r4(mc);
    int* cs = cw + ex_r4(mc);
    int* cv = cs + ex_r4(mc);
    int* cg = cv + ex_r4(nc);
    const int lv = local[v];
    int o = kdeg[v];
    co[lv] = o;
    if (lv == nc - 1) co[nc] = mc;
    cv[lv] = X.vw[v];
    cg[lv] = X.trans[v];
    for (int e = X.off[v]; e < X.off[v + 1]; ++e) {
      const int u = X.tgt[e];
      if (X.part[u] != c) continue;
      ct[o] = local[u];
      cw[o] = X.w[e];
      cs[o] = lv;
      ++o;
    }
  }
}

// ---------------------------------------------------------------------------
// host wrappers

void coarsen_small_batch(const std::vector<DevGraph>& gs, const std::vector<double>& l_max,
                         const std::vector<unsigned long long>& seeds, long long threshold,
                         std::vector<SmallStack>& out, DBuf<int>& arena, cudaStream_t s) {
  const int J = (int)gs.size();
  out.assign((size_t)J, SmallStack{});
  if (J == 0) return;
  std::vector<long long> base((size_t)J + 1, 0);
  for (int j = 0; j < J; ++j)
    base[(size_t)j + 1] = base[(size_t)j] + 32ll * (gs[(size_t)j].n + 1) + 16ll * gs[(size_t)j].m2 + 4096;
  arena = DBuf<int>((size_t)base[(size_t)J], s);
  BcJob* hj = static_cast<BcJob*>(pinned_scratch(sizeof(BcJob) * (size_t)J));
  for (int j = 0; j < J; ++j) {
    BcJob b{};
    const DevGraph& g = gs[(size_t)j];
    b.n = g.n;
    b.m2 = (int)g.m2;
    b.off = g.off;
    b.tgt = g.tgt;
    b.w = g.w;
    b.vw = g.vw;
    b.l_max = l_max[(size_t)j];
    b.seed = seeds[(size_t)j];
    b.threshold = threshold;
    b.arena = arena.get() + base[(size_t)j];
    b.cap = base[(size_t)j + 1] - base[(size_t)j];
    hj[j] = b;
  }
  DBuf<BcJob> dj((size_t)J, s);
  GIM_CUDA(cudaMemcpyAsync(dj.get(), hj, sizeof(BcJob) * (size_t)J, cudaMemcpyHostToDevice, s));
  k_coarsen_small<<<J, kBcBlock, 0, s>>>(dj.get());
  count_launch();
  GIM_LAUNCH_CHECK();
  GIM_CUDA(cudaMemcpyAsync(hj, dj.get(), sizeof(BcJob) * (size_t)J, cudaMemcpyDeviceToHost, s));
  GIM_CUDA(sync_stream(s));
  for (int j = 0; j < J; ++j) {
    const BcJob& b = hj[j];
    SmallStack& S = out[(size_t)j];
    S.status = b.status;
    S.nl = b.nl;
    if (b.status == 2) continue;
    int* A = arena.get() + base[(size_t)j];
    for (int l = 0; l < b.nl; ++l) {
      const BcLevel& L = b.lv[l];
      DevGraph d;
      if (l == 0) {
        d = gs[(size_t)j];
      } else {
        d.n = L.n;
        d.m2 = L.m2;
        d.off = A + L.off;
        d.tgt = A + L.tgt;
        d.w = A + L.w;
        d.vw = A + L.vw;
        d.src = nullptr;
      }
      S.levels.push_back(d);
      S.cmap.push_back(l + 1 < b.nl ? A + L.cmap : nullptr);
    }
  }
}

void extract_batch(const std::vector<DevGraph>& gs, const std::vector<const int*>& parts_of,
                   const std::vector<const int*>& trans, int parts, std::vector<ExChild>& out,
                   DBuf<int>& arena, cudaStream_t s) {
  const int N = (int)gs.size();
  out.clear();
  if (N == 0) return;
  GIM_CHECK(parts <= kExMaxParts, GIM_E_UNSUPPORTED, "too many parts for batched extraction");
  std::vector<long long> base((size_t)N + 1, 0), sbase((size_t)N + 1, 0);
  for (int j = 0; j < N; ++j) {
    const DevGraph& g = gs[(size_t)j];
    base[(size_t)j + 1] =
        base[(size_t)j] + ex_r4((g.n + 1ll) * 3 + 3 * g.m2 + 20ll * parts + 64);
    sbase[(size_t)j + 1] = sbase[(size_t)j] + 2ll * g.n + 4;
  }
  arena = DBuf<int>((size_t)base[(size_t)N], s);
  DBuf<int> scratch((size_t)sbase[(size_t)N], s);
  std::vector<ExNode> hn((size_t)N);
  for (int j = 0; j < N; ++j) {
    const DevGraph& g = gs[(size_t)j];
    ExNode x{};
    x.n = g.n;
    x.parts = parts;
    x.off = g.off;
    x.tgt = g.tgt;
    x.w = g.w;
    x.vw = g.vw;
    x.part = parts_of[(size_t)j];
    x.trans = trans[(size_t)j];
    x.arena = arena.get() + base[(size_t)j];
    x.cap = base[(size_t)j + 1] - base[(size_t)j];
    x.scratch = scratch.get() + sbase[(size_t)j];
    hn[(size_t)j] = x;
  }
  DBuf<ExNode> dn((size_t)N, s);
  GIM_CUDA(cudaMemcpyAsync(dn.get(), hn.data(), sizeof(ExNode) * (size_t)N,
                           cudaMemcpyHostToDevice, s));
  k_extract_batch<<<N, kExBlock, 0, s>>>(dn.get());
  count_launch();
  GIM_LAUNCH_CHECK();
  ExNode* hr = static_cast<ExNode*>(pinned_scratch(sizeof(ExNode) * (size_t)N));
  GIM_CUDA(cudaMemcpyAsync(hr, dn.get(), sizeof(ExNode) * (size_t)N, cudaMemcpyDeviceToHost, s));
  GIM_CUDA(sync_stream(s));
  for (int j = 0; j < N; ++j) {
    const ExNode& x = hr[j];
    GIM_CHECK(x.status == 0, GIM_E_INTERNAL, "batched extraction arena overflow");
    for (int c = 0; c < parts; ++c) {
      ExChild ch;
      ch.node = j;
      ch.part = c;
      ch.total = x.ctotal[c];
      int* co = arena.get() + base[(size_t)j] + x.cbase[c];
      const int nc = x.cn[c], mc = x.cm2[c];
      ch.g.n = nc;
      ch.g.m2 = mc;
      ch.g.off = co;
      ch.g.tgt = co + ex_r4(nc + 1ll);
      ch.g.w = ch.g.tgt + ex_r4(mc);
      ch.g.src = ch.g.w + ex_r4(mc);
      ch.g.vw = ch.g.src + ex_r4(mc);
      ch.trans = ch.g.vw + ex_r4(nc);
      out.push_back(ch);
    }
  }
}

void bproj_bw_batch(const std::vector<BpJob>& jobs, cudaStream_t s) {
  const int J = (int)jobs.size();
  if (J == 0) return;
  DBuf<BpJob> dj((size_t)J, s);  // pageable source: staged before the call returns
  GIM_CUDA(cudaMemcpyAsync(dj.get(), jobs.data(), sizeof(BpJob) * (size_t)J,
                           cudaMemcpyHostToDevice, s));
  k_bproj_bw<<<J, 256, 0, s>>>(dj.get());
  count_launch();
  GIM_LAUNCH_CHECK();
}

}  // namespace gim
