// Internal (C++) interface between the kernel translation units and the
// host driver.  Nothing here crosses the C ABI.
#pragma once
#include "common.cuh"

namespace gim {

// non-owning device view of one CSR level
struct DevGraph {
  int n = 0;
  long long m2 = 0;
  const int* off = nullptr;
  const int* tgt = nullptr;
  const int* w = nullptr;
  const int* vw = nullptr;
  const int* src = nullptr;
};

inline DevGraph view(const gim_graph& g) {
  DevGraph d;
  d.n = g.n;
  d.m2 = g.m2;
  d.off = g.offsets;
  d.tgt = g.targets;
  d.w = g.weights;
  d.vw = g.vweights;
  d.src = g.sources;
  return d;
}

// owning device CSR level
struct OwnedGraph {
  int n = 0;
  long long m2 = 0;
  long long total_vw = 0;  // exact c(V)
  DBuf<int> off, tgt, w, vw, src;
  DevGraph view() const {
    DevGraph d;
    d.n = n;
    d.m2 = m2;
    d.off = off.get();
    d.tgt = tgt.get();
    d.w = w.get();
    d.vw = vw.get();
    d.src = src.get();
    return d;
  }
};

// ---- jeval.cu
void total_cost(const DevGraph& g, const int* part, const Topo& t, long long* j_out,
                cudaStream_t s);
void block_weights(int n, const int* vw, const int* part, int k, long long* bw,
                   cudaStream_t s);

}  // namespace gim
