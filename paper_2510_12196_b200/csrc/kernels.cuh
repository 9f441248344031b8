// Internal (C++) interface between the kernel translation units and the
// host driver.  Nothing here crosses the C ABI.
#pragma once
#include <vector>

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
  int maxdeg = -1;  // an upper bound of the longest row, -1 = unknown
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
  int maxdeg = -1;         // an upper bound of the longest row, -1 = unknown
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
    d.maxdeg = maxdeg;
    return d;
  }
};

// ---- jeval.cu
void total_cost(const DevGraph& g, const int* part, const Topo& t, long long* j_out,
                cudaStream_t s);
void total_cost_f64(const DevGraph& g, const int* part, const Topo& t, double* j_out,
                    cudaStream_t s);
void block_weights(int n, const int* vw, const int* part, int k, long long* bw,
                   cudaStream_t s);

// ---- coarsen.cu
void hem_round(const DevGraph& g, int* partner, int* pref, double l_max,
               unsigned long long seed, long long* matched, cudaStream_t s,
               const long long* gate = nullptr);
long long two_hop(const DevGraph& g, int* partner, double l_max, long long matched_now,
                  long long* matched_d, cudaStream_t s);
int coarse_map(int n, const int* partner, int* cmap, cudaStream_t s);
long long contract_into(const DevGraph& g, const int* cmap, int n_c, int* c_off, int* c_tgt,
                        int* c_w, int* c_vw, int* c_src, cudaStream_t s);
void contract(const DevGraph& g, const int* cmap, int n_c, OwnedGraph& out, cudaStream_t s);
// contraction of a matching (<= 2 members per coarse vertex), row-wise
bool coarsen_level_fast(const DevGraph& g, double l_max, unsigned long long lseed, int* partner,
                        int* cmap, int* n_c_out, long long* matched_out, OwnedGraph& out,
                        int* m2c_dev, bool* stalled, const int* g_m2_dev, long long* g_m2_out,
                        cudaStream_t s);
void contract_matching(const DevGraph& g, const int* cmap, const int* partner, int n_c,
                       OwnedGraph& out, cudaStream_t s);
void project(int n, const int* cmap, const int* pc, int* pf, cudaStream_t s);

// ---- refine.cu
// one CSR level prepared for refinement: group width + heavy-vertex list
struct RefineLevel {
  DevGraph g;
  int vw = 32;       // lanes per vertex on the register path
  int n_heavy = 0;   // vertices with degree > vw (shared-memory path)
  DBuf<int> heavy;
};

// scratch of one refinement (sized for the finest level it serves)
struct RefineBuffers {
  DBuf<unsigned char> cand, to_move, locks;
  DBuf<int> dest, dest2;
  DBuf<long long> gkey;
  DBuf<unsigned int> rkeys, rkeys2;
  DBuf<int> rvals, rvals2;
  DBuf<long long> rexcl;
  DBuf<int> gstart, count;
  DBuf<long long> ctr;           // [movers, dJ] — zeroed by each candidate pass
  long long* movers = nullptr;   // ctr + 0
  long long* dj = nullptr;       // ctr + 1
  DBuf<unsigned char> masks;     // [ovl | elig] per block (rebalance)
  DBuf<int> elist;               // eligible block list (rebalance)
  DBuf<long long> jtmp;          // J scratch
  // device-resident loop (refine_fused.cu)
  DBuf<int> best;                // best mapping seen
  DBuf<long long> best_bw, fctr; // its block weights; [movers0, dj0, movers1, dj1, J]
  DBuf<unsigned char> rcell;     // weak-rebalance cell per vertex
  DBuf<unsigned char> fstate;    // FusedState (device)
  DBuf<int> bstamp, lists;       // boundary stamps; 5 work lists of n entries
  int cap_n = 0, cap_k = 0;      // sizes the buffers were allocated for
};

void prepare_level(RefineLevel& L, int k, cudaStream_t s);
// lane width only (the fused loop needs no heavy list until a host strong pass)
void prepare_level_vw(RefineLevel& L);
void alloc_refine_buffers(RefineBuffers& rb, int n, int k, cudaStream_t s);
void lp_pass(const RefineLevel& L, const Topo& t, const int* part, const unsigned char* locked,
             int jet, double jet_c, RefineBuffers& rb, cudaStream_t s);
void rebalance_pass(const RefineLevel& L, const Topo& t, const int* part, const long long* bw,
                    bool strong, double l_max, int rho, unsigned long long seed,
                    long long pass_counter, const unsigned char* ovl, const unsigned char* elig,
                    const int* elig_list, int n_elig, RefineBuffers& rb, cudaStream_t s);
void apply_moves(const RefineLevel& L, const Topo& t, int* part, long long* bw,
                 RefineBuffers& rb, cudaStream_t s);
long long conn_build(const DevGraph& g, const int* part, int k, int* c_off, int* c_blocks,
                     int* c_w, cudaStream_t s);

// ---- refine_fused.cu: device-resident Alg. 4
// control state shared between the persistent kernel and the host (which
// performs the rare strong passes between launches)
struct FusedState {
  long long J, best_j, best_maxw, maxw, pass_counter;
  long long iters, lp, weak;
  int i, i_w, best_balanced, locks_nonempty, lp_par, prev_n, stamp;
  int status;   // 0 = finished, 1 = strong pass due (host)
  int started;  // 0 = first launch of this refinement
  int reinit;   // 1 = re-establish the per-vertex list invariants on entry
  long long acct[16];  // Acct counters (common.cuh), summed over launches
};

struct FusedCfg {
  double l_max, sigma, phi, jet_c;
  int jet, rho, i_max, i_w_max;
  unsigned long long seed;
};

struct FusedBuffers {
  // aliases into RefineBuffers
  unsigned char *cand = nullptr, *tm0 = nullptr, *tm1 = nullptr, *rcell = nullptr;
  int *dest = nullptr, *rtgt = nullptr, *best = nullptr;
  long long *gkey = nullptr, *best_bw = nullptr, *ctr = nullptr;
  int *bstamp = nullptr, *wdeg = nullptr, *lsmall = nullptr, *lheavy = nullptr, *lcand = nullptr;
  int *lmov0 = nullptr, *lmov1 = nullptr;
  long long lp_seen = 0, weak_seen = 0;
  long long acct_seen[16] = {0};  // FusedState::acct already accounted
  // owned
  DBuf<long long> W, S;
  long long W_cap = 0, S_cap = 0;
  FusedState* state = nullptr;    // device
  FusedState* h_state = nullptr;  // pinned host mirror
};

bool fused_supported(int k, int rho);

// SURVEY §8(d) algorithmic bytes of refinement work described by Acct
// counter deltas `d` on a level of n vertices / m2 slots
double s8d_refine_bytes(const long long* d, long long n, long long m2, int k, int rho);

// batched small-graph partitioner pieces (batch.cu)
struct SmallStack {
  int status = 0;                 // 0 done; 1 the top level needs two-hop (continue); 2 general path
  int nl = 0;
  std::vector<DevGraph> levels;   // [0] = the input graph
  std::vector<const int*> cmap;   // level l -> l + 1 (null on the coarsest)
};
void coarsen_small_batch(const std::vector<DevGraph>& gs, const std::vector<double>& l_max,
                         const std::vector<unsigned long long>& seeds, long long threshold,
                         std::vector<SmallStack>& out, DBuf<int>& arena, cudaStream_t s);
struct BpJob {
  int n, k;
  const int* cmap;     // null: no projection (coarsest level)
  const int* coarse;   // coarse part (projection source)
  int* part;           // fine part (in when cmap is null, else out)
  const int* vw;
  long long* bw;
};
void bproj_bw_batch(const std::vector<BpJob>& jobs, cudaStream_t s);
struct ExChild {
  int node = 0, part = 0;
  long long total = 0;     // c(V) of the child
  DevGraph g;              // views into the extraction arena
  const int* trans = nullptr;  // global ids
};
void extract_batch(const std::vector<DevGraph>& gs, const std::vector<const int*>& parts_of,
                   const std::vector<const int*>& trans, int parts, std::vector<ExChild>& out,
                   DBuf<int>& arena, cudaStream_t s);
void ggg_batch(const std::vector<DevGraph>& gs, int k, const std::vector<int*>& parts,
               cudaStream_t s);

// batched shared-memory-resident refinement (refine_fused.cu)
struct SmemRefineJob {
  DevGraph g;
  int vw = 8;
  int* part = nullptr;
  long long* bw = nullptr;
  FusedCfg cfg{};
  int* best = nullptr;          // [n] scratch
  long long* best_bw = nullptr; // [k] scratch
  long long iters = 0, lp = 0, weak = 0;  // out
};
bool refine_smem_fits(long long n, long long m2, int k, int rho, int vw);
int refine_pick_vw(long long n, long long m2);
void refine_smem_batch(std::vector<SmemRefineJob>& jobs, const Topo& t, FusedState* states,
                       std::vector<char>& yielded, cudaStream_t s);
void refine_cluster_batch(std::vector<SmemRefineJob>& jobs, const Topo& t, FusedState* states,
                          std::vector<char>& yielded, cudaStream_t s);
bool refine_fused_run(const RefineLevel& L, const Topo& t, int* part, long long* bw,
                      const FusedCfg& cfg, FusedBuffers& fb, cudaStream_t s);

}  // namespace gim
