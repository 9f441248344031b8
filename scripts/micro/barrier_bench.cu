// Microbenchmark: cost of one grid-wide barrier inside a persistent kernel
// (cooperative groups grid.sync vs a sense-reversing atomic barrier vs a
// hardware cluster barrier), per barrier, for grids of G CTAs x 256 threads.
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o barrier_bench barrier_bench.cu
#include <cooperative_groups.h>
#include <cstdio>
namespace cg = cooperative_groups;

__global__ void k_cg(int iters, int* sink) {
  auto g = cg::this_grid();
  int x = 0;
  for (int i = 0; i < iters; ++i) {
    x += threadIdx.x;
    g.sync();
  }
  if (x == -1) *sink = x;
}

// sense-reversing barrier: one arrival atomic per CTA, release/acquire at gpu scope
__device__ __forceinline__ void bar_flag(unsigned* count, volatile unsigned* gen, unsigned G,
                                         unsigned& mygen) {
  __syncthreads();
  if (threadIdx.x == 0) {
    mygen++;
    __threadfence();
    unsigned old = atomicAdd(count, 1u);
    if (old == G - 1) {
      *count = 0;
      __threadfence();
      *gen = mygen;
    } else {
      while (*gen != mygen) {}
    }
    __threadfence();
  }
  __syncthreads();
}

__global__ void k_flag(int iters, unsigned* count, unsigned* gen, int* sink) {
  unsigned mygen = 0;
  int x = 0;
  for (int i = 0; i < iters; ++i) {
    x += threadIdx.x;
    bar_flag(count, gen, gridDim.x, mygen);
  }
  if (x == -1) *sink = x;
}

__global__ void __cluster_dims__(16, 1, 1) k_cluster(int iters, int* sink) {
  auto c = cg::this_cluster();
  int x = 0;
  for (int i = 0; i < iters; ++i) {
    x += threadIdx.x;
    c.sync();
  }
  if (x == -1) *sink = x;
}

int main() {
  int* sink;
  unsigned *cnt, *gen;
  cudaMalloc(&sink, 4);
  cudaMalloc(&cnt, 4);
  cudaMalloc(&gen, 4);
  cudaEvent_t a, b;
  cudaEventCreate(&a);
  cudaEventCreate(&b);
  const int iters = 2000;
  int per = 0;
  cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per, k_cg, 256, 0);
  int sms = 0;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  for (int G : {16, 74, 148, 296, 444}) {
    if (G > per * sms) continue;
    int it = iters;
    void* args[] = {&it, &sink};
    cudaLaunchCooperativeKernel((void*)k_cg, G, 256, args, 0, 0);
    cudaDeviceSynchronize();
    cudaEventRecord(a);
    cudaLaunchCooperativeKernel((void*)k_cg, G, 256, args, 0, 0);
    cudaEventRecord(b);
    cudaEventSynchronize(b);
    float ms;
    cudaEventElapsedTime(&ms, a, b);
    cudaMemset(cnt, 0, 4);
    cudaMemset(gen, 0, 4);
    void* args2[] = {&it, &cnt, &gen, &sink};
    cudaLaunchCooperativeKernel((void*)k_flag, G, 256, args2, 0, 0);
    cudaDeviceSynchronize();
    cudaMemset(cnt, 0, 4);
    cudaMemset(gen, 0, 4);
    cudaEventRecord(a);
    cudaLaunchCooperativeKernel((void*)k_flag, G, 256, args2, 0, 0);
    cudaEventRecord(b);
    cudaEventSynchronize(b);
    float ms2;
    cudaEventElapsedTime(&ms2, a, b);
    printf("G=%d cg.grid.sync %.3f us/barrier | flag barrier %.3f us/barrier  (%s)\n", G,
           1000.0 * ms / iters, 1000.0 * ms2 / iters, cudaGetErrorString(cudaGetLastError()));
  }
  {
    int it = iters;
    k_cluster<<<16, 256>>>(it, sink);
    cudaDeviceSynchronize();
    cudaEventRecord(a);
    k_cluster<<<16, 256>>>(it, sink);
    cudaEventRecord(b);
    cudaEventSynchronize(b);
    float ms;
    cudaEventElapsedTime(&ms, a, b);
    printf("cluster(16).sync %.3f us/barrier (%s)\n", 1000.0 * ms / iters,
           cudaGetErrorString(cudaGetLastError()));
  }
  return 0;
}
