// Hand-written device-wide exclusive scan (reduce-then-scan, 3 launches).
//
// Input is a functor `in(i) -> T` so flags/counts can be scanned without
// materialising them; output is written through `out(i, prefix)`.
// Tile = BLOCK * ITEMS elements staged through padded shared memory so the
// global reads/writes are coalesced and the per-thread work is sequential.
#pragma once
#include "common.cuh"

namespace gim {

constexpr int kScanBlock = 256;
constexpr int kScanItems = 8;
constexpr int kScanTile = kScanBlock * kScanItems;

__host__ __device__ constexpr int scan_pad(int i) { return i + (i >> 5); }

template <class T>
__device__ __forceinline__ T warp_incl_scan(T v) {
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    T y = __shfl_up_sync(0xffffffffu, v, o);
    if ((int)lane_id() >= o) v += y;
  }
  return v;
}

// block-wide exclusive scan of one value per thread; returns the exclusive
// prefix, *total receives the block sum
template <class T, int BLOCK>
__device__ __forceinline__ T block_excl_scan(T v, T* total) {
  __shared__ T warp_tot[BLOCK / 32];
  T incl = warp_incl_scan(v);
  if (lane_id() == 31) warp_tot[threadIdx.x >> 5] = incl;
  __syncthreads();
  if (threadIdx.x < 32) {
    T x = threadIdx.x < BLOCK / 32 ? warp_tot[threadIdx.x] : T(0);
    T xi = warp_incl_scan(x);
    if (threadIdx.x < BLOCK / 32) warp_tot[threadIdx.x] = xi - x;
    if (threadIdx.x == 31) *total = xi;
  }
  __syncthreads();
  T r = warp_tot[threadIdx.x >> 5] + incl - v;
  __syncthreads();
  return r;
}

template <class T, class In>
__global__ void __launch_bounds__(kScanBlock) k_scan_reduce(long long n, In in, T* tile_sums) {
  long long base = (long long)blockIdx.x * kScanTile;
  T acc = 0;
#pragma unroll
  for (int i = 0; i < kScanItems; ++i) {
    long long idx = base + i * kScanBlock + threadIdx.x;
    if (idx < n) acc += in(idx);
  }
  __shared__ T tot;
  T dummy = block_excl_scan<T, kScanBlock>(acc, &tot);
  (void)dummy;
  if (threadIdx.x == 0) tile_sums[blockIdx.x] = tot;
}

// single-CTA scan of the tile sums (in place, exclusive), total -> *total
template <class T>
__global__ void __launch_bounds__(1024) k_scan_tiles(long long m, T* sums, T* total) {
  __shared__ T carry;
  if (threadIdx.x == 0) carry = 0;
  __syncthreads();
  for (long long b = 0; b < m; b += 1024) {
    long long i = b + threadIdx.x;
    T v = i < m ? sums[i] : T(0);
    __shared__ T tot;
    T ex = block_excl_scan<T, 1024>(v, &tot);
    if (i < m) sums[i] = ex + carry;
    __syncthreads();
    if (threadIdx.x == 0) carry += tot;
    __syncthreads();
  }
  if (threadIdx.x == 0 && total) *total = carry;
}

template <class T, class In, class Out>
__global__ void __launch_bounds__(kScanBlock) k_scan_down(long long n, In in, Out out,
                                                          const T* tile_sums) {
  __shared__ T buf[scan_pad(kScanTile) + 1];
  long long base = (long long)blockIdx.x * kScanTile;
#pragma unroll
  for (int i = 0; i < kScanItems; ++i) {
    int j = i * kScanBlock + threadIdx.x;
    long long idx = base + j;
    buf[scan_pad(j)] = idx < n ? in(idx) : T(0);
  }
  __syncthreads();
  T loc[kScanItems];
  T acc = 0;
#pragma unroll
  for (int i = 0; i < kScanItems; ++i) {
    loc[i] = buf[scan_pad(threadIdx.x * kScanItems + i)];
    acc += loc[i];
  }
  __shared__ T tot;
  T pre = block_excl_scan<T, kScanBlock>(acc, &tot) + tile_sums[blockIdx.x];
#pragma unroll
  for (int i = 0; i < kScanItems; ++i) {
    buf[scan_pad(threadIdx.x * kScanItems + i)] = pre;
    pre += loc[i];
  }
  __syncthreads();
#pragma unroll
  for (int i = 0; i < kScanItems; ++i) {
    int j = i * kScanBlock + threadIdx.x;
    long long idx = base + j;
    if (idx < n) out(idx, buf[scan_pad(j)]);
  }
}

// small inputs: one CTA walks the range in 1024-element chunks (one launch
// instead of three — the coarse levels are launch-latency bound)
constexpr long long kScanSmall = 8192;

template <class T, class In, class Out>
__global__ void __launch_bounds__(1024) k_scan_small(long long n, In in, Out out, T* total) {
  __shared__ T tot;
  T carry = 0;
  for (long long b = 0; b < n; b += 1024) {
    const long long i = b + threadIdx.x;
    const T v = i < n ? in(i) : T(0);
    const T ex = block_excl_scan<T, 1024>(v, &tot);
    if (i < n) out(i, carry + ex);
    carry += tot;
    __syncthreads();
  }
  if (threadIdx.x == 0 && total) *total = carry;
}

// exclusive scan of in(0..n-1); total (device pointer, may be null) gets the sum
template <class T, class In, class Out>
void exclusive_scan(long long n, In in, Out out, T* total, cudaStream_t s) {
  long long tiles = (n + kScanTile - 1) / kScanTile;
  if (tiles == 0) {
    if (total) GIM_CUDA(cudaMemsetAsync(total, 0, sizeof(T), s));
    return;
  }
  if (n <= kScanSmall) {
    k_scan_small<T, In, Out><<<1, 1024, 0, s>>>(n, in, out, total);
    GIM_LAUNCH_CHECK();
    count_launch(1);
    return;
  }
  DBuf<T> sums((size_t)tiles, s);
  k_scan_reduce<T, In><<<(unsigned)tiles, kScanBlock, 0, s>>>(n, in, sums.get());
  k_scan_tiles<T><<<1, 1024, 0, s>>>(tiles, sums.get(), total);
  k_scan_down<T, In, Out><<<(unsigned)tiles, kScanBlock, 0, s>>>(n, in, out, sums.get());
  GIM_LAUNCH_CHECK();
  count_launch(3);
}

// common functors
template <class T, class S>
struct LoadAs {
  const S* p;
  __device__ T operator()(long long i) const { return (T)p[i]; }
};
template <class T>
struct StoreTo {
  T* p;
  __device__ void operator()(long long i, T v) const { p[i] = v; }
};

}  // namespace gim
