// K1 J evaluation and K2 block weights.
//
// J (mapping.py:76-91): sum over directed slots e of w_e * D[Pi(src_e), Pi(tgt_e)].
// Edge-parallel over the flat slot arrays (E_u form): the
// src/tgt/w streams are read fully coalesced with 128-bit vector loads, the
// two Pi gathers hit L2 (Pi is <= 64 MB at every config, L2 is 126 MB), and the
// int64 partial sums are reduced warp -> block -> one atomic per CTA.
#include "common.cuh"
#include "kernels.cuh"

namespace gim {

template <int BLOCK>
__global__ void __launch_bounds__(BLOCK) k_total_cost(long long m2, const int* __restrict__ src,
                                                      const int* __restrict__ tgt,
                                                      const int* __restrict__ w,
                                                      const int* __restrict__ part, Topo t,
                                                      long long* __restrict__ out) {
  long long acc = 0;
  const long long stride = (long long)gridDim.x * BLOCK * 4;
  long long base = ((long long)blockIdx.x * BLOCK + threadIdx.x) * 4;
  // vectorised body: 4 slots per thread per step (int4 loads; arrays are
  // cudaMalloc-aligned and m2 is split into a vector part and a tail)
  const long long m4 = m2 & ~3ll;
  for (long long e = base; e < m4; e += stride) {
    int4 s = *reinterpret_cast<const int4*>(src + e);
    int4 v = *reinterpret_cast<const int4*>(tgt + e);
    int4 ww = *reinterpret_cast<const int4*>(w + e);
    acc += (long long)ww.x * dist(t, __ldg(part + s.x), __ldg(part + v.x));
    acc += (long long)ww.y * dist(t, __ldg(part + s.y), __ldg(part + v.y));
    acc += (long long)ww.z * dist(t, __ldg(part + s.z), __ldg(part + v.z));
    acc += (long long)ww.w * dist(t, __ldg(part + s.w), __ldg(part + v.w));
  }
  for (long long e = m4 + (long long)blockIdx.x * BLOCK + threadIdx.x; e < m2;
       e += (long long)gridDim.x * BLOCK)
    acc += (long long)w[e] * dist(t, part[src[e]], part[tgt[e]]);
  block_sum_atomic<BLOCK>(acc, out);
}

void total_cost(const DevGraph& g, const int* part, const Topo& t, long long* j_out,
                cudaStream_t s) {
  GIM_CUDA(cudaMemsetAsync(j_out, 0, sizeof(long long), s));
  if (g.m2 == 0) return;
  // algorithmic bytes: offsets + Pi[v] per vertex, target +
  // weight + Pi[target] per slot
  ProfScope prof(P_JEVAL, 8.0 * g.n + 12.0 * g.m2, s);
  constexpr int B = 256;
  int grid = grid_for((g.m2 + 3) / 4, B, kSMs * 8);
  k_total_cost<B><<<grid, B, 0, s>>>(g.m2, g.src, g.tgt, g.w, part, t, j_out);
  GIM_LAUNCH_CHECK();
  count_launch();
}

// J with the caller's float distances (mapping.py:76-91, float path when
// Topology.integral_distances is false): per-slot w * d in float64, reduced
// warp -> block -> one double atomic per CTA
template <int BLOCK>
__global__ void __launch_bounds__(BLOCK) k_total_cost_f64(long long m2, const int* __restrict__ src,
                                                          const int* __restrict__ tgt,
                                                          const int* __restrict__ w,
                                                          const int* __restrict__ part, Topo t,
                                                          double* __restrict__ out) {
  __shared__ double red[BLOCK / 32];
  double acc = 0.0;
  for (long long e = (long long)blockIdx.x * BLOCK + threadIdx.x; e < m2;
       e += (long long)gridDim.x * BLOCK) {
    const unsigned long long c = __ldg(t.code + part[src[e]]) ^ __ldg(t.code + part[tgt[e]]);
    if (c) acc += (double)w[e] * __ldg(t.dbitf + (63 - __clzll(c)));
  }
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) acc += __shfl_xor_sync(0xffffffffu, acc, o);
  if (lane_id() == 0) red[threadIdx.x >> 5] = acc;
  __syncthreads();
  if (threadIdx.x == 0) {
    double x = 0.0;
    for (int i = 0; i < BLOCK / 32; ++i) x += red[i];
    if (x != 0.0) atomicAdd(out, x);
  }
}

void total_cost_f64(const DevGraph& g, const int* part, const Topo& t, double* j_out,
                    cudaStream_t s) {
  GIM_CUDA(cudaMemsetAsync(j_out, 0, sizeof(double), s));
  if (g.m2 == 0) return;
  ProfScope prof(P_JEVAL, 8.0 * g.n + 12.0 * g.m2, s);
  constexpr int B = 256;
  k_total_cost_f64<B><<<grid_for(g.m2, B, kSMs * 8), B, 0, s>>>(g.m2, g.src, g.tgt, g.w, part,
                                                                 t, j_out);
  GIM_LAUNCH_CHECK();
  count_launch();
}

// block weights: per-CTA shared histogram (k <= kSmemBins) with
// warp-aggregated shared atomics, one global atomic per (CTA, nonzero bin)
constexpr int kSmemBins = 8192;

template <int BLOCK>
__global__ void __launch_bounds__(BLOCK) k_block_weights(int n, const int* __restrict__ vw,
                                                         const int* __restrict__ part, int k,
                                                         long long* __restrict__ bw) {
  extern __shared__ long long hist[];
  for (int i = threadIdx.x; i < k; i += BLOCK) hist[i] = 0;
  __syncthreads();
  for (int v = blockIdx.x * BLOCK + threadIdx.x; v < n; v += gridDim.x * BLOCK) {
    int b = part[v];
    long long x = vw[v];
    unsigned peers = __match_any_sync(__activemask(), b);
    int leader = __ffs(peers) - 1;
    // sum of x over the peer group, lanes in ascending order
    long long sum = 0;
    unsigned m = peers;
    while (m) {
      int l = __ffs(m) - 1;
      m &= m - 1;
      sum += __shfl_sync(peers, x, l);
    }
    if ((int)lane_id() == leader) atomicAdd(reinterpret_cast<unsigned long long*>(&hist[b]),
                                            (unsigned long long)sum);
  }
  __syncthreads();
  for (int i = threadIdx.x; i < k; i += BLOCK)
    if (hist[i]) atomicAdd(reinterpret_cast<unsigned long long*>(&bw[i]),
                           (unsigned long long)hist[i]);
}

template <int BLOCK>
__global__ void __launch_bounds__(BLOCK) k_block_weights_global(int n, const int* __restrict__ vw,
                                                                const int* __restrict__ part,
                                                                long long* __restrict__ bw) {
  for (int v = blockIdx.x * BLOCK + threadIdx.x; v < n; v += gridDim.x * BLOCK)
    atomicAdd(reinterpret_cast<unsigned long long*>(&bw[part[v]]), (unsigned long long)vw[v]);
}

void block_weights(int n, const int* vw, const int* part, int k, long long* bw,
                   cudaStream_t s) {
  GIM_CUDA(cudaMemsetAsync(bw, 0, sizeof(long long) * k, s));
  if (n == 0) return;
  constexpr int B = 256;
  if (k <= kSmemBins) {
    int grid = grid_for(n, B, kSMs * 2);
    size_t smem = sizeof(long long) * k;
    if (smem > 48 * 1024)
      GIM_CUDA(cudaFuncSetAttribute(k_block_weights<B>,
                                    cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
    k_block_weights<B><<<grid, B, smem, s>>>(n, vw, part, k, bw);
  } else {
    k_block_weights_global<B><<<grid_for(n, B), B, 0, s>>>(n, vw, part, bw);
  }
  GIM_LAUNCH_CHECK();
  count_launch();
}

}  // namespace gim

using namespace gim;

extern "C" int gim_total_cost(const gim_graph* g, const int32_t* assignment,
                              const gim_topology* t, int64_t* j_out, void* stream) {
  return guard([&] {
    GIM_CHECK(g && t && j_out, GIM_E_INVALID, "null argument");
    Topo tp = get_topo(*t);
    total_cost(view(*g), assignment, tp, reinterpret_cast<long long*>(j_out),
               (cudaStream_t)stream);
  });
}

extern "C" int gim_total_cost_f64(const gim_graph* g, const int32_t* assignment,
                                  const gim_topology* t, double* j_out, void* stream) {
  return guard([&] {
    GIM_CHECK(g && t && j_out, GIM_E_INVALID, "null argument");
    Topo tp = get_topo(*t);
    total_cost_f64(view(*g), assignment, tp, j_out, (cudaStream_t)stream);
  });
}

extern "C" int gim_block_weights(const gim_graph* g, const int32_t* assignment, int32_t k,
                                 int64_t* bw_out, void* stream) {
  return guard([&] {
    GIM_CHECK(g && bw_out && k >= 1, GIM_E_INVALID, "bad argument");
    block_weights(g->n, g->vweights, assignment, k, reinterpret_cast<long long*>(bw_out),
                  (cudaStream_t)stream);
  });
}
