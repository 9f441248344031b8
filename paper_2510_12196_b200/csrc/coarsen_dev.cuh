// Device helpers shared by the coarsening kernels (coarsen.cu) and the
// batched small-graph partitioner (batch.cu): the heavy-edge rating order of
// coarsening.py:52-60 / 72-90.
#pragma once
#include "common.cuh"

namespace gim {

struct HemCand {
  int w, c, slot, u;
  unsigned long long h;
};

__device__ __forceinline__ bool hem_better(const HemCand& a, const HemCand& b) {
  if (a.u < 0) return false;
  if (b.u < 0) return true;
  unsigned long long aw2 = (unsigned long long)a.w * (unsigned long long)a.w;
  unsigned long long bw2 = (unsigned long long)b.w * (unsigned long long)b.w;
  unsigned __int128 lhs = (unsigned __int128)aw2 * (unsigned)b.c;
  unsigned __int128 rhs = (unsigned __int128)bw2 * (unsigned)a.c;
  if (lhs != rhs) return lhs > rhs;
  if (a.h != b.h) return a.h > b.h;
  return a.slot < b.slot;
}

__device__ __forceinline__ HemCand hem_shfl(const HemCand& x, int o) {
  HemCand y;
  y.w = __shfl_xor_sync(0xffffffffu, x.w, o);
  y.c = __shfl_xor_sync(0xffffffffu, x.c, o);
  y.slot = __shfl_xor_sync(0xffffffffu, x.slot, o);
  y.u = __shfl_xor_sync(0xffffffffu, x.u, o);
  y.h = __shfl_xor_sync(0xffffffffu, x.h, o);
  return y;
}

}  // namespace gim
