// Library-level plumbing: error state, memory pool, topology upload.
#include "common.cuh"
#include "kernels.cuh"

#include <sched.h>

#include <cmath>
#include <cstring>

#include <atomic>
#include <map>
#include <mutex>

namespace gim {

static thread_local std::string g_last_error;

void set_error(const std::string& msg) { g_last_error = msg; }
const char* last_error() { return g_last_error.c_str(); }

static void configure_pool_once();

cudaError_t sync_stream(cudaStream_t s) {
  for (int spin = 0;; ++spin) {
    cudaError_t e = cudaStreamQuery(s);
    if (e != cudaErrorNotReady) return e;
    if (spin >= 64) sched_yield();
  }
}

// ---- pinned scratch: process-wide free list, per-thread lease
namespace {
struct PinnedBlock {
  void* p = nullptr;
  size_t bytes = 0;
};
std::mutex g_pin_mu;
std::vector<PinnedBlock> g_pin_free;

struct PinnedLease {
  PinnedBlock b;
  ~PinnedLease() {
    if (!b.p) return;
    std::lock_guard<std::mutex> lk(g_pin_mu);
    g_pin_free.push_back(b);
  }
};
thread_local PinnedLease g_pin_lease;

std::mutex g_stream_mu;
std::map<int, std::vector<cudaStream_t>> g_stream_free;  // per device
}  // namespace

void* pinned_scratch(size_t bytes) {
  PinnedBlock& b = g_pin_lease.b;
  if (b.bytes >= bytes) return b.p;
  std::lock_guard<std::mutex> lk(g_pin_mu);
  if (b.p) g_pin_free.push_back(b);  // too small: back to the list
  b = PinnedBlock{};
  for (size_t i = 0; i < g_pin_free.size(); ++i) {
    if (g_pin_free[i].bytes >= bytes) {
      b = g_pin_free[i];
      g_pin_free.erase(g_pin_free.begin() + (long)i);
      return b.p;
    }
  }
  size_t sz = (size_t)1 << 16;
  while (sz < bytes) sz <<= 1;
  if (cudaMallocHost(&b.p, sz) != cudaSuccess) {
    b = PinnedBlock{};
    throw Error{GIM_E_CUDA, "cudaMallocHost failed"};
  }
  b.bytes = sz;
  return b.p;
}

cudaStream_t acquire_stream() {
  int dev = 0;
  GIM_CUDA(cudaGetDevice(&dev));
  {
    std::lock_guard<std::mutex> lk(g_stream_mu);
    auto& fl = g_stream_free[dev];
    if (!fl.empty()) {
      cudaStream_t s = fl.back();
      fl.pop_back();
      return s;
    }
  }
  cudaStream_t s = nullptr;
  GIM_CUDA(cudaStreamCreateWithFlags(&s, cudaStreamNonBlocking));
  return s;
}

void release_stream(cudaStream_t s) {
  if (!s) return;
  int dev = 0;
  cudaGetDevice(&dev);  // a worker releases on the device it acquired on
  std::lock_guard<std::mutex> lk(g_stream_mu);
  g_stream_free[dev].push_back(s);
}

// ---- stream-keyed caching allocator in front of the cudaMallocAsync pool.
// A mapping makes thousands of small allocations (per level, per
// multisection subtree, on many streams); cudaMallocAsync measured
// ~150 us per call here whenever the pool had to map memory, which
// dominated small-graph partitioner calls.  Blocks are cached per
// (stream, size class) for the life of the process and handed out again
// only on the stream they were released on (stream order = happens-before).
constexpr size_t kCacheMax = (size_t)16 << 30;  // larger buffers go to the pool
constexpr size_t kTrimClass = (size_t)16 << 20;  // "large" size classes

static size_t size_class(size_t b) {
  size_t c = 256;
  while (c < b) c <<= 1;
  return c;
}

namespace {
// keyed by device too: the legacy / per-thread default stream handles are
// the same value on every device
struct CacheKey {
  int dev;
  cudaStream_t s;
  size_t c;
  bool operator<(const CacheKey& o) const {
    if (dev != o.dev) return dev < o.dev;
    return s != o.s ? s < o.s : c < o.c;
  }
};
struct Owned {
  int dev;
  size_t c;
};
std::mutex g_cache_mu;
std::map<CacheKey, std::vector<void*>> g_cache_free;
std::unordered_map<void*, Owned> g_cache_owned;

int current_device() {
  int dev = 0;
  cudaGetDevice(&dev);
  return dev;
}
}  // namespace

static void* raw_alloc(size_t bytes, cudaStream_t s) {
  void* p = nullptr;
  cudaError_t e = cudaMallocAsync(&p, bytes, s);
  if (e != cudaSuccess)
    throw Error{GIM_E_CUDA, std::string("cudaMallocAsync(") + std::to_string(bytes) +
                                ") failed: " + cudaGetErrorString(e)};
  return p;
}

void* dmalloc(size_t bytes, cudaStream_t s) {
  if (bytes == 0) return nullptr;
  configure_pool_once();
  if (bytes > kCacheMax) return raw_alloc(bytes, s);
  const size_t c = size_class(bytes);
  const int dev = current_device();
  {
    std::lock_guard<std::mutex> lk(g_cache_mu);
    auto it = g_cache_free.find(CacheKey{dev, s, c});
    if (it != g_cache_free.end() && !it->second.empty()) {
      void* p = it->second.back();
      it->second.pop_back();
      g_cache_owned[p] = Owned{dev, c};
      return p;
    }
  }
  if (c >= kTrimClass) {
    // a large class this stream has none of: borrow a cached block one or two
    // classes up before mapping new memory (level sizes vary a little from
    // seed to seed and straddle class boundaries)
    std::lock_guard<std::mutex> lk(g_cache_mu);
    for (size_t up = c << 1; up <= (c << 2); up <<= 1) {
      auto it = g_cache_free.find(CacheKey{dev, s, up});
      if (it != g_cache_free.end() && !it->second.empty()) {
        void* p = it->second.back();
        it->second.pop_back();
        g_cache_owned[p] = Owned{dev, up};
        return p;
      }
    }
  }
  void* p = raw_alloc(c, s);
  std::lock_guard<std::mutex> lk(g_cache_mu);
  g_cache_owned[p] = Owned{dev, c};
  return p;
}

void dfree(void* p, cudaStream_t s) {
  if (!p) return;
  {
    std::lock_guard<std::mutex> lk(g_cache_mu);
    auto it = g_cache_owned.find(p);
    if (it != g_cache_owned.end()) {
      g_cache_free[CacheKey{it->second.dev, s, it->second.c}].push_back(p);
      g_cache_owned.erase(it);
      return;
    }
  }
  cudaFreeAsync(p, s);  // never throws from a destructor
}

// returns every cached block to its device's pool (stream-ordered on the
// stream that released it), then trims the pools
void release_cached_memory() {
  int cur = 0;
  cudaGetDevice(&cur);
  std::lock_guard<std::mutex> lk(g_cache_mu);
  std::map<int, bool> devs;
  for (auto& kv : g_cache_free) {
    cudaSetDevice(kv.first.dev);
    for (void* p : kv.second) cudaFreeAsync(p, kv.first.s);
    devs[kv.first.dev] = true;
  }
  g_cache_free.clear();
  for (auto& d : devs) {
    cudaSetDevice(d.first);
    cudaDeviceSynchronize();
    cudaMemPool_t pool;
    if (cudaDeviceGetDefaultMemPool(&pool, d.first) == cudaSuccess) cudaMemPoolTrimTo(pool, 0);
  }
  cudaSetDevice(cur);
}

static std::mutex g_topo_mu;
static std::map<std::vector<long long>, Topo> g_topo_cache;

// distance scale of a topology (gim_topology doc): the smallest shift s
// making every d * 2^s integral (dyadic distances: exact, the reference's
// float sums are exact too), else the largest s keeping d_max * 2^s < 2^31
// (J = sum w * d * 2^s < 2^62 for total edge weight < 2^31), d rounded
void topo_scale(int levels, const double* d, int* shift, int* exact) {
  double dmax = 0.0;
  for (int i = 0; i < levels; ++i) dmax = std::max(dmax, d[i]);
  for (int s = 0; s <= 40; ++s) {
    bool ok = true;
    for (int i = 0; i < levels && ok; ++i) {
      const double x = std::ldexp(d[i], s);
      ok = x == std::floor(x) && x < 9.0e15;
    }
    if (ok && (s == 0 || std::ldexp(dmax, s) < 2147483648.0)) {
      *shift = s;
      *exact = 1;
      return;
    }
  }
  int s = 0;
  while (s < 40 && std::ldexp(dmax, s + 1) < 2147483648.0) ++s;
  *shift = s;
  *exact = 0;
}

Topo get_topo(const gim_topology& tt) {
  const int levels = tt.levels;
  const int64_t* hierarchy = tt.hierarchy;
  const double* distances = tt.distances;
  GIM_CHECK(levels >= 1 && levels <= GIM_MAX_LEVELS, GIM_E_INVALID,
            "hierarchy must have 1.." + std::to_string(GIM_MAX_LEVELS) + " levels");
  std::vector<long long> key;
  long long k = 1;
  for (int i = 0; i < levels; ++i) {
    GIM_CHECK(hierarchy[i] >= 1, GIM_E_INVALID, "hierarchy factors must be >= 1");
    GIM_CHECK(distances[i] >= 0 && std::isfinite(distances[i]), GIM_E_INVALID,
              "distances must be nonnegative");
    if (i) GIM_CHECK(distances[i] >= distances[i - 1], GIM_E_INVALID,
                     "distances must be nondecreasing");
    k *= hierarchy[i];
    GIM_CHECK(k < (1ll << 30), GIM_E_OVERFLOW, "k too large for int32 block ids");
    long long dk;
    std::memcpy(&dk, &distances[i], sizeof(dk));
    key.push_back(hierarchy[i]);
    key.push_back(dk);
  }
  int dev = 0;
  GIM_CUDA(cudaGetDevice(&dev));
  key.push_back(-1 - dev);  // device tables: one copy per device
  std::lock_guard<std::mutex> lk(g_topo_mu);
  auto it = g_topo_cache.find(key);
  if (it != g_topo_cache.end()) return it->second;
  int dshift = 0, exact = 1;
  topo_scale(levels, distances, &dshift, &exact);
  // bit field layout: level 0 (least significant digit) in the low bits
  int shift[GIM_MAX_LEVELS];
  int bits = 0;
  std::vector<long long> dbit(64, 0);
  std::vector<double> dbitf(64, 0.0);
  for (int i = 0; i < levels; ++i) {
    int wdt = 0;
    while ((1ll << wdt) < hierarchy[i]) ++wdt;
    shift[i] = bits;
    const long long di = (long long)std::llround(std::ldexp(distances[i], dshift));
    for (int b = bits; b < bits + wdt && b < 64; ++b) {
      dbit[b] = di;
      dbitf[b] = distances[i];
    }
    bits += wdt;
  }
  GIM_CHECK(bits <= 64, GIM_E_UNSUPPORTED, "hierarchy digit codes exceed 64 bits");
  std::vector<unsigned long long> code((size_t)k);
  for (long long b = 0; b < k; ++b) {
    long long x = b;
    unsigned long long c = 0;
    for (int i = 0; i < levels; ++i) {
      c |= (unsigned long long)(x % hierarchy[i]) << shift[i];
      x /= hierarchy[i];
    }
    code[(size_t)b] = c;
  }
  std::vector<long long> lv(2 * (size_t)levels);
  {
    long long P = 1;
    for (int i = 0; i < levels; ++i) {
      P *= hierarchy[i];
      lv[(size_t)i] = P;
      lv[(size_t)(levels + i)] = (long long)std::llround(std::ldexp(distances[i], dshift));
    }
  }
  void* p = nullptr;
  const size_t cb = sizeof(unsigned long long) * (size_t)k;
  const size_t lvo = cb + sizeof(long long) * 64 + sizeof(double) * 64;
  size_t bytes = lvo + sizeof(long long) * lv.size();
  GIM_CUDA(cudaMalloc(&p, bytes));
  GIM_CUDA(cudaMemcpy(static_cast<char*>(p) + lvo, lv.data(), sizeof(long long) * lv.size(),
                      cudaMemcpyHostToDevice));
  GIM_CUDA(cudaMemcpy(p, code.data(), cb, cudaMemcpyHostToDevice));
  GIM_CUDA(cudaMemcpy(static_cast<char*>(p) + cb, dbit.data(), sizeof(long long) * 64,
                      cudaMemcpyHostToDevice));
  GIM_CUDA(cudaMemcpy(static_cast<char*>(p) + cb + sizeof(long long) * 64, dbitf.data(),
                      sizeof(double) * 64, cudaMemcpyHostToDevice));
  Topo t;
  t.L = levels;
  t.k = (int)k;
  t.dshift = dshift;
  t.exact = exact;
  t.code = static_cast<const unsigned long long*>(p);
  t.dbit = reinterpret_cast<const long long*>(static_cast<char*>(p) + cb);
  t.dbitf = reinterpret_cast<const double*>(static_cast<char*>(p) + cb + sizeof(long long) * 64);
  g_topo_cache.emplace(key, t);
  return t;
}

Topo get_flat_topo(int k) {
  gim_topology t{};
  t.levels = 1;
  t.hierarchy[0] = k;
  t.distances[0] = 1.0;
  return get_topo(t);
}

// one-time pool configuration: keep freed blocks cached (no OS round trips
// between refinement iterations / levels)
static void configure_pool_once() {
  static std::atomic<unsigned long long> done{0};  // bit per device
  int dev = 0;
  if (cudaGetDevice(&dev) != cudaSuccess || dev >= 64) return;
  const unsigned long long bit = 1ull << dev;
  if (done.load(std::memory_order_acquire) & bit) return;
  done.fetch_or(bit);
  cudaMemPool_t pool;
  if (cudaDeviceGetDefaultMemPool(&pool, dev) != cudaSuccess) return;
  uint64_t thr = UINT64_MAX;
  cudaMemPoolSetAttribute(pool, cudaMemPoolAttrReleaseThreshold, &thr);
}

// ---- run contexts (common.cuh)
static std::mutex g_flags_mu;
static RunFlags g_default_flags;
static RunCtx g_process_ctx;  // kernel-level calls outside integrated_map
static thread_local RunCtx* t_ctx = nullptr;

RunCtx& ctx() { return t_ctx ? *t_ctx : g_process_ctx; }

RunFlags default_flags() {
  std::lock_guard<std::mutex> lk(g_flags_mu);
  return g_default_flags;
}

void set_default_flags(const RunFlags& f) {
  std::lock_guard<std::mutex> lk(g_flags_mu);
  g_default_flags = f;
  g_process_ctx.f = f;
}

CtxScope::CtxScope(RunCtx* c) : prev(t_ctx) { t_ctx = c; }
CtxScope::~CtxScope() { t_ctx = prev; }

void count_launch(long long n) { ctx().launches.fetch_add(n, std::memory_order_relaxed); }
long long launches() { return ctx().launches.load(); }
void reset_launches() { ctx().launches.store(0); }

static thread_local bool t_concurrent = false;
ConcurrentScope::ConcurrentScope() : prev(t_concurrent) { t_concurrent = true; }
ConcurrentScope::~ConcurrentScope() { t_concurrent = prev; }
int coop_blocks_per_sm(int occ) {
  occ = std::max(occ, 1);
  return t_concurrent && occ > 1 ? occ - 1 : occ;
}

int device_sms() {
  static std::mutex mu;
  static std::map<int, int> cache;
  int dev = 0;
  GIM_CUDA(cudaGetDevice(&dev));
  std::lock_guard<std::mutex> lk(mu);
  auto it = cache.find(dev);
  if (it != cache.end()) return it->second;
  int sms = 0;
  GIM_CUDA(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev));
  cache[dev] = sms;
  return sms;
}

// ---- profiling records (per run context); CUDA events are pooled per device
static std::mutex g_ev_mu;
static std::map<int, std::vector<cudaEvent_t>> g_evpool;

static cudaEvent_t ev_get() {
  int dev = 0;
  GIM_CUDA(cudaGetDevice(&dev));
  {
    std::lock_guard<std::mutex> lk(g_ev_mu);
    auto& pool = g_evpool[dev];
    if (!pool.empty()) {
      cudaEvent_t e = pool.back();
      pool.pop_back();
      return e;
    }
  }
  cudaEvent_t e;
  GIM_CUDA(cudaEventCreate(&e));
  return e;
}

static void ev_put(cudaEvent_t a, cudaEvent_t b) {
  int dev = 0;
  cudaGetDevice(&dev);
  std::lock_guard<std::mutex> lk(g_ev_mu);
  g_evpool[dev].push_back(a);
  g_evpool[dev].push_back(b);
}

bool prof_on() { return ctx().f.prof; }

void prof_begin(int cls, double bytes, cudaStream_t s, void** token) {
  RunCtx& c = ctx();
  ProfRec r{cls, bytes, ev_get(), ev_get()};
  GIM_CUDA(cudaEventRecord(r.a, s));
  std::lock_guard<std::mutex> lk(c.mu);
  c.recs.push_back(r);
  *token = reinterpret_cast<void*>(c.recs.size());  // 1-based index
}

void prof_end(void* token, cudaStream_t s, double extra_bytes) {
  RunCtx& c = ctx();
  std::lock_guard<std::mutex> lk(c.mu);
  size_t i = reinterpret_cast<size_t>(token) - 1;
  if (i < c.recs.size()) {
    c.recs[i].bytes += extra_bytes;
    cudaEventRecord(c.recs[i].b, s);
  }
}

void prof_collect(double* ms, double* bytes, long long* count, int* top_cls, double* top_ms,
                  double* top_bytes) {
  RunCtx& c = ctx();
  std::lock_guard<std::mutex> lk(c.mu);
  *top_cls = -1;
  *top_ms = 0.0;
  *top_bytes = 0.0;
  for (auto& r : c.recs) {
    cudaEventSynchronize(r.b);
    float t = 0.f;
    cudaEventElapsedTime(&t, r.a, r.b);
    if (r.cls >= 0 && r.cls < P_COUNT) {
      ms[r.cls] += t;
      bytes[r.cls] += r.bytes;
      count[r.cls] += 1;
      if (r.bytes > *top_bytes) {
        *top_cls = r.cls;
        *top_ms = t;
        *top_bytes = r.bytes;
      }
    }
    ev_put(r.a, r.b);
  }
  c.recs.clear();
}

}  // namespace gim

extern "C" void gim_set_profiling(int32_t on) {
  gim::RunFlags f = gim::default_flags();
  f.prof = on != 0;
  gim::set_default_flags(f);
}

extern "C" int gim_version(void) {
  gim::configure_pool_once();
  return 1;
}

extern "C" const char* gim_last_error(void) { return gim::last_error(); }

extern "C" int gim_topology_scale(const gim_topology* t, int32_t* shift_out, int32_t* exact_out) {
  return gim::guard([&] {
    GIM_CHECK(t && shift_out && exact_out, GIM_E_INVALID, "null argument");
    GIM_CHECK(t->levels >= 1 && t->levels <= GIM_MAX_LEVELS, GIM_E_INVALID, "bad levels");
    int s = 0, e = 1;
    gim::topo_scale(t->levels, t->distances, &s, &e);
    *shift_out = s;
    *exact_out = e;
  });
}
