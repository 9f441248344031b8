// Hand-rolled stable LSD radix sort of (key, value) pairs, 8-bit digits.
//
// Per digit pass (reduce-then-scan form):
//   1. k_radix_hist   per-tile digit counts -> hist[digit * tiles + tile]
//   2. exclusive_scan over hist (digit-major) -> global bucket offsets
//   3. k_radix_scatter per-tile stable ranking + scatter
// Stable ranking: each warp owns a contiguous run of 32*ITEMS elements and
// walks it in 32-element steps; __match_any_sync groups equal digits, the
// rank inside a step is popc(peers & lanemask_lt), and a per-warp shared
// counter per digit carries ranks across steps.  Warp offsets inside the tile
// come from a per-digit prefix over warps, so element order is preserved.
// Only bits [0, end_bit) are sorted; keys must be < 2^end_bit.
#pragma once
#include "common.cuh"
#include "scan.cuh"

namespace gim {

constexpr int kRadixBlock = 256;
constexpr int kRadixItems = 8;
constexpr int kRadixWarps = kRadixBlock / 32;
constexpr int kRadixTile = kRadixBlock * kRadixItems;

template <class K>
__global__ void __launch_bounds__(kRadixBlock) k_radix_hist(long long n, const K* __restrict__ keys,
                                                            int shift, long long tiles,
                                                            int* __restrict__ hist) {
  __shared__ int cnt[256];
  for (int i = threadIdx.x; i < 256; i += kRadixBlock) cnt[i] = 0;
  __syncthreads();
  long long base = (long long)blockIdx.x * kRadixTile;
#pragma unroll
  for (int i = 0; i < kRadixItems; ++i) {
    long long idx = base + i * kRadixBlock + threadIdx.x;
    if (idx < n) atomicAdd(&cnt[(int)((keys[idx] >> shift) & 0xff)], 1);
  }
  __syncthreads();
  for (int d = threadIdx.x; d < 256; d += kRadixBlock)
    hist[(long long)d * tiles + blockIdx.x] = cnt[d];
}

template <class K, class V>
__global__ void __launch_bounds__(kRadixBlock) k_radix_scatter(
    long long n, const K* __restrict__ keys, const V* __restrict__ vals, K* __restrict__ okeys,
    V* __restrict__ ovals, int shift, long long tiles, const int* __restrict__ offs) {
  __shared__ int wcnt[kRadixWarps][256];
  __shared__ int gbase[256];
  const int warp = threadIdx.x >> 5;
  const unsigned lane = lane_id();
  for (int i = threadIdx.x; i < kRadixWarps * 256; i += kRadixBlock) (&wcnt[0][0])[i] = 0;
  for (int d = threadIdx.x; d < 256; d += kRadixBlock)
    gbase[d] = offs[(long long)d * tiles + blockIdx.x];
  __syncthreads();
  const long long wbase = (long long)blockIdx.x * kRadixTile + (long long)warp * 32 * kRadixItems;
  K k[kRadixItems];
  V v[kRadixItems];
  int rank[kRadixItems];
  const unsigned lt = (1u << lane) - 1u;
#pragma unroll
  for (int i = 0; i < kRadixItems; ++i) {
    long long idx = wbase + i * 32 + lane;
    bool ok = idx < n;
    unsigned act = __ballot_sync(0xffffffffu, ok);
    rank[i] = -1;
    if (ok) {
      k[i] = keys[idx];
      v[i] = vals[idx];
      int d = (int)((k[i] >> shift) & 0xff);
      unsigned peers = __match_any_sync(act, d);
      int leader = __ffs(peers) - 1;
      int old = 0;
      if ((int)lane == leader) {
        old = wcnt[warp][d];
        wcnt[warp][d] = old + __popc(peers);
      }
      old = __shfl_sync(peers, old, leader);
      rank[i] = old + __popc(peers & lt);
    }
    __syncwarp();
  }
  __syncthreads();
  // exclusive prefix over warps, per digit
  for (int d = threadIdx.x; d < 256; d += kRadixBlock) {
    int acc = 0;
#pragma unroll
    for (int w = 0; w < kRadixWarps; ++w) {
      int c = wcnt[w][d];
      wcnt[w][d] = acc;
      acc += c;
    }
  }
  __syncthreads();
#pragma unroll
  for (int i = 0; i < kRadixItems; ++i) {
    if (rank[i] >= 0) {
      int d = (int)((k[i] >> shift) & 0xff);
      long long pos = (long long)gbase[d] + wcnt[warp][d] + rank[i];
      okeys[pos] = k[i];
      ovals[pos] = v[i];
    }
  }
}

inline int bit_length(unsigned long long x) {
  int b = 0;
  while (x) {
    ++b;
    x >>= 1;
  }
  return b;
}

// Sort pairs in place (result ends in keys/vals; alt buffers are scratch of
// the same size).  Stable.  end_bit <= 8*sizeof(K).
template <class K, class V>
void radix_sort_pairs(long long n, K* keys, V* vals, K* alt_keys, V* alt_vals, int end_bit,
                      cudaStream_t s) {
  if (n <= 1 || end_bit <= 0) return;
  long long tiles = (n + kRadixTile - 1) / kRadixTile;
  DBuf<int> hist((size_t)(tiles * 256), s);
  K* ks = keys;
  V* vs = vals;
  K* kd = alt_keys;
  V* vd = alt_vals;
  int passes = (end_bit + 7) / 8;
  for (int p = 0; p < passes; ++p) {
    int shift = p * 8;
    k_radix_hist<K><<<(unsigned)tiles, kRadixBlock, 0, s>>>(n, ks, shift, tiles, hist.get());
    count_launch();
    exclusive_scan<int>(tiles * 256, LoadAs<int, int>{hist.get()}, StoreTo<int>{hist.get()},
                        (int*)nullptr, s);
    k_radix_scatter<K, V><<<(unsigned)tiles, kRadixBlock, 0, s>>>(n, ks, vs, kd, vd, shift,
                                                                   tiles, hist.get());
    count_launch();
    GIM_LAUNCH_CHECK();
    std::swap(ks, kd);
    std::swap(vs, vd);
  }
  if (ks != keys) {
    GIM_CUDA(cudaMemcpyAsync(keys, ks, sizeof(K) * n, cudaMemcpyDeviceToDevice, s));
    GIM_CUDA(cudaMemcpyAsync(vals, vs, sizeof(V) * n, cudaMemcpyDeviceToDevice, s));
  }
}

}  // namespace gim
