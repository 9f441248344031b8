// Native METIS-format reader (graph.py:170-294, `load_metis`): the same
// accepted language, the same CSR (file order within a vertex line kept) and
// the same MetisFormatError messages with 1-based line numbers, reported in
// the reference's order (parse errors in file order, then missing / unequal
// reverse edges in file order, then the header's edge count).
//
// The file is memory-mapped; line boundaries are found in one sequential
// sweep, then the vertex lines are parsed by worker threads over contiguous
// line ranges (per-line degree counts, a prefix sum, then the fill), and the
// reverse-edge check runs per row against sorted copies of the rows.
#include <fcntl.h>
#include <sys/mman.h>
#include <sys/stat.h>
#include <unistd.h>

#include <algorithm>
#include <atomic>
#include <cstring>
#include <string>
#include <thread>
#include <unordered_set>
#include <vector>

#include "common.cuh"

namespace gim {

namespace {

struct Line {
  long long b, e;  // byte range (without the newline)
  long long no;    // 1-based line number in the file
};

inline bool is_space(char c) {
  return c == ' ' || c == '\t' || c == '\r' || c == '\v' || c == '\f';
}

// Python int() on a whitespace-free token: [+-]?digits with single '_'
// between digits.  Returns false if not an integer.
bool py_int(const char* s, const char* e, long long* out) {
  if (s == e) return false;
  bool neg = false;
  if (*s == '+' || *s == '-') {
    neg = *s == '-';
    ++s;
  }
  if (s == e || *s < '0' || *s > '9') return false;
  unsigned long long v = 0;
  bool prev_us = false;
  for (; s < e; ++s) {
    if (*s == '_') {
      if (prev_us) return false;
      prev_us = true;
      continue;
    }
    if (*s < '0' || *s > '9') return false;
    prev_us = false;
    v = v * 10 + (unsigned long long)(*s - '0');
    if (v > (1ull << 62)) v = 1ull << 62;  // saturate (fails range checks later)
  }
  if (prev_us) return false;
  *out = neg ? -(long long)v : (long long)v;
  return true;
}

struct Tok {
  const char* s;
  const char* e;
};

void split(const char* b, const char* e, std::vector<Tok>& out) {
  out.clear();
  const char* p = b;
  while (p < e) {
    while (p < e && is_space(*p)) ++p;
    if (p >= e) break;
    const char* q = p;
    while (q < e && !is_space(*q)) ++q;
    out.push_back(Tok{p, q});
    p = q;
  }
}

std::string tok_repr(const Tok& t) { return "'" + std::string(t.s, t.e) + "'"; }

struct Err {
  long long line = -1;  // -1: none
  std::string msg;
};

}  // namespace

struct MetisGraph {
  long long n = 0, m2 = 0;
  std::vector<long long> off, tgt, w, vw, src;
};

// throws Error{GIM_E_FORMAT, "line N: ..."} on malformed input
static void parse_metis(const char* data, long long size, MetisGraph& G) {
  // ---- lines (a final line without '\n' counts), comment lines dropped
  std::vector<Line> lines;
  {
    long long b = 0, no = 1;
    for (long long i = 0; i <= size; ++i) {
      if (i == size || data[i] == '\n') {
        if (i == size && b == size) break;  // no trailing partial line
        long long s = b;
        while (s < i && (is_space(data[s]) || data[s] == '\n')) ++s;
        const bool comment = s < i && data[s] == '%';
        if (!comment) lines.push_back(Line{b, i, no});
        b = i + 1;
        ++no;
      }
    }
  }
  auto fail = [](long long line, const std::string& msg) {
    throw Error{GIM_E_FORMAT, "line " + std::to_string(line) + ": " + msg};
  };
  if (lines.empty()) fail(1, "empty graph file");
  std::vector<Tok> hdr;
  split(data + lines[0].b, data + lines[0].e, hdr);
  const long long hl = lines[0].no;
  if (hdr.size() != 2 && hdr.size() != 3) fail(hl, "header must be 'n m [fmt]'");
  long long n = 0, m = 0, fmtv = 0;
  if (!py_int(hdr[0].s, hdr[0].e, &n) || !py_int(hdr[1].s, hdr[1].e, &m) ||
      (hdr.size() == 3 && !py_int(hdr[2].s, hdr[2].e, &fmtv)))
    fail(hl, "malformed header");
  if (n < 0 || m < 0) fail(hl, "negative counts in header");
  std::string fmt = hdr.size() == 3 ? std::string(hdr[2].s, hdr[2].e) : "0";
  while (fmt.size() < 3) fmt = (fmt[0] == '-' || fmt[0] == '+')
                                   ? fmt.substr(0, 1) + "0" + fmt.substr(1)
                                   : "0" + fmt;  // str.zfill keeps the sign first
  if (fmt.size() != 3 || fmt[0] != '0')
    fail(hl, "unsupported format code " + (hdr.size() == 3 ? tok_repr(hdr[2]) : std::string("'0'")));
  const bool has_vw = fmt[1] == '1', has_ew = fmt[2] == '1';
  // ---- data lines: trailing blank lines beyond n are tolerated
  long long nd = (long long)lines.size() - 1;
  auto blank = [&](const Line& L) {
    for (long long i = L.b; i < L.e; ++i)
      if (!is_space(data[i])) return false;
    return true;
  };
  while (nd > n && blank(lines[(size_t)nd])) --nd;
  if (nd != n) {
    const long long last = nd > 0 ? lines[(size_t)nd].no : hl;
    fail(last, "expected " + std::to_string(n) + " vertex lines, found " + std::to_string(nd));
  }
  G.n = n;
  G.vw.assign((size_t)n, 1);
  G.off.assign((size_t)n + 1, 0);
  const int T = (int)std::max(1u, std::min(16u, std::thread::hardware_concurrency()));
  const long long per = (n + T - 1) / std::max(T, 1);
  std::vector<Err> errs((size_t)T);
  std::vector<long long> deg((size_t)std::max(n, 1ll), 0);
  // pass 1: validate tokens in file order (as the reference does, token by
  // token: parse, range, self loop, weight, duplicate), count entries
  auto pass1 = [&](int t) {
    std::vector<Tok> tk;
    std::vector<long long> seen;
    std::unordered_set<long long> seen_big;  // hub lines
    const long long v0 = std::min(n, t * per), v1 = std::min(n, v0 + per);
    for (long long v = v0; v < v1; ++v) {
      const Line& L = lines[(size_t)v + 1];
      split(data + L.b, data + L.e, tk);
      size_t pos = 0;
      auto err = [&](const std::string& m2) {
        errs[(size_t)t].line = L.no;
        errs[(size_t)t].msg = m2;
      };
      if (has_vw) {
        if (tk.empty()) return err("missing vertex weight");
        long long cv = 0;
        if (!py_int(tk[0].s, tk[0].e, &cv)) return err("bad vertex weight " + tok_repr(tk[0]));
        if (cv <= 0) return err("nonpositive vertex weight " + std::to_string(cv));
        G.vw[(size_t)v] = cv;
        pos = 1;
      }
      const size_t step = has_ew ? 2 : 1;
      if ((tk.size() - pos) % step) return err("dangling edge token");
      deg[(size_t)v] = (long long)((tk.size() - pos) / step);
      seen.clear();
      seen_big.clear();
      for (size_t j = pos; j < tk.size(); j += step) {
        long long u = 0, wt = 1;
        if (!py_int(tk[j].s, tk[j].e, &u) || (has_ew && !py_int(tk[j + 1].s, tk[j + 1].e, &wt)))
          return err("bad edge token");
        u -= 1;
        if (!(0 <= u && u < n))
          return err("neighbor " + std::to_string(u + 1) + " out of range [1," +
                     std::to_string(n) + "]");
        if (u == v) return err("self-loop at vertex " + std::to_string(v + 1));
        if (wt <= 0) return err("nonpositive edge weight " + std::to_string(wt));
        const bool dup = deg[(size_t)v] <= 64
                             ? std::find(seen.begin(), seen.end(), u) != seen.end()
                             : !seen_big.insert(u).second;
        if (dup)
          return err("duplicate neighbor " + std::to_string(u + 1) + " for vertex " +
                     std::to_string(v + 1));
        if (deg[(size_t)v] <= 64) seen.push_back(u);
      }
    }
  };
  {
    std::vector<std::thread> pool;
    for (int t = 1; t < T; ++t) pool.emplace_back(pass1, t);
    pass1(0);
    for (auto& th : pool) th.join();
  }
  for (const Err& e : errs)  // threads own increasing line ranges: first hit wins
    if (e.line >= 0) fail(e.line, e.msg);
  for (long long v = 0; v < n; ++v) G.off[(size_t)v + 1] = G.off[(size_t)v] + deg[(size_t)v];
  const long long m2 = G.off[(size_t)n];
  G.m2 = m2;
  G.tgt.resize((size_t)m2);
  G.w.resize((size_t)m2);
  G.src.resize((size_t)m2);
  // pass 2: fill (file order kept)
  auto pass2 = [&](int t) {
    std::vector<Tok> tk;
    const long long v0 = std::min(n, t * per), v1 = std::min(n, v0 + per);
    for (long long v = v0; v < v1; ++v) {
      const Line& L = lines[(size_t)v + 1];
      split(data + L.b, data + L.e, tk);
      const size_t pos = has_vw ? 1 : 0, step = has_ew ? 2 : 1;
      long long o = G.off[(size_t)v];
      for (size_t j = pos; j < tk.size(); j += step, ++o) {
        long long u = 0, wt = 1;
        py_int(tk[j].s, tk[j].e, &u);
        if (has_ew) py_int(tk[j + 1].s, tk[j + 1].e, &wt);
        G.tgt[(size_t)o] = u - 1;
        G.w[(size_t)o] = wt;
        G.src[(size_t)o] = v;
      }
    }
  };
  {
    std::vector<std::thread> pool;
    for (int t = 1; t < T; ++t) pool.emplace_back(pass2, t);
    pass2(0);
    for (auto& th : pool) th.join();
  }
  // reverse entries: rows sorted by target once, then a binary search per slot
  std::vector<long long> rk((size_t)m2), rw((size_t)m2);
  auto sort_rows = [&](int t) {
    std::vector<std::pair<long long, long long>> tmp;
    const long long v0 = std::min(n, t * per), v1 = std::min(n, v0 + per);
    for (long long v = v0; v < v1; ++v) {
      const long long b = G.off[(size_t)v], e = G.off[(size_t)v + 1];
      tmp.clear();
      for (long long i = b; i < e; ++i) tmp.emplace_back(G.tgt[(size_t)i], G.w[(size_t)i]);
      std::sort(tmp.begin(), tmp.end());
      for (long long i = b; i < e; ++i) {
        rk[(size_t)i] = tmp[(size_t)(i - b)].first;
        rw[(size_t)i] = tmp[(size_t)(i - b)].second;
      }
    }
  };
  {
    std::vector<std::thread> pool;
    for (int t = 1; t < T; ++t) pool.emplace_back(sort_rows, t);
    sort_rows(0);
    for (auto& th : pool) th.join();
  }
  for (auto& e : errs) e = Err{};
  auto check = [&](int t) {
    const long long v0 = std::min(n, t * per), v1 = std::min(n, v0 + per);
    for (long long v = v0; v < v1; ++v) {
      for (long long i = G.off[(size_t)v]; i < G.off[(size_t)v + 1]; ++i) {
        const long long u = G.tgt[(size_t)i], wt = G.w[(size_t)i];
        const long long b = G.off[(size_t)u], e = G.off[(size_t)u + 1];
        const auto it = std::lower_bound(rk.begin() + b, rk.begin() + e, v);
        const long long line = lines[(size_t)v + 1].no;
        if (it == rk.begin() + e || *it != v) {
          errs[(size_t)t].line = line;
          errs[(size_t)t].msg = "edge (" + std::to_string(v + 1) + "," + std::to_string(u + 1) +
                                ") has no reverse entry";
          return;
        }
        const long long back = rw[(size_t)(it - rk.begin())];
        if (back != wt) {
          errs[(size_t)t].line = line;
          errs[(size_t)t].msg = "edge (" + std::to_string(v + 1) + "," + std::to_string(u + 1) +
                                ") weight " + std::to_string(wt) + " != reverse weight " +
                                std::to_string(back);
          return;
        }
      }
    }
  };
  {
    std::vector<std::thread> pool;
    for (int t = 1; t < T; ++t) pool.emplace_back(check, t);
    check(0);
    for (auto& th : pool) th.join();
  }
  for (const Err& e : errs)
    if (e.line >= 0) fail(e.line, e.msg);
  if (m2 != 2 * m)
    fail(hl, "header claims " + std::to_string(m) + " edges, file has " + std::to_string(m2 / 2));
}

// the parsed CSR of a gim_metis_load handle (driver.cu uploads it)
bool metis_arrays(void* handle, long long* n, const long long** off, const long long** tgt,
                  const long long** w, const long long** vw) {
  auto* G = static_cast<MetisGraph*>(handle);
  if (!G) return false;
  *n = G->n;
  *off = G->off.data();
  *tgt = G->tgt.data();
  *w = G->w.data();
  *vw = G->vw.data();
  return true;
}

void metis_free(void* handle) { delete static_cast<MetisGraph*>(handle); }

}  // namespace gim

using namespace gim;

extern "C" int gim_metis_load(const char* path, void** handle, int64_t* n, int64_t* m2) {
  return guard([&] {
    GIM_CHECK(path && handle && n && m2, GIM_E_INVALID, "null argument");
    const int fd = ::open(path, O_RDONLY);
    GIM_CHECK(fd >= 0, GIM_E_IO, std::string("cannot open ") + path);
    struct stat st;
    if (fstat(fd, &st) != 0) {
      ::close(fd);
      throw Error{GIM_E_IO, std::string("cannot stat ") + path};
    }
    const long long size = (long long)st.st_size;
    const char* data = nullptr;
    void* map = nullptr;
    if (size > 0) {
      map = mmap(nullptr, (size_t)size, PROT_READ, MAP_PRIVATE, fd, 0);
      if (map == MAP_FAILED) {
        ::close(fd);
        throw Error{GIM_E_IO, std::string("cannot map ") + path};
      }
      data = static_cast<const char*>(map);
    }
    auto* G = new MetisGraph();
    try {
      static const char empty = '\0';
      parse_metis(data ? data : &empty, size, *G);
    } catch (...) {
      delete G;
      if (map) munmap(map, (size_t)size);
      ::close(fd);
      throw;
    }
    if (map) munmap(map, (size_t)size);
    ::close(fd);
    *handle = G;
    *n = G->n;
    *m2 = G->m2;
  });
}

extern "C" int gim_metis_fetch(void* handle, int64_t* offsets, int64_t* targets,
                               int64_t* eweights, int64_t* vweights, int64_t* sources) {
  return guard([&] {
    GIM_CHECK(handle, GIM_E_INVALID, "null handle");
    auto* G = static_cast<MetisGraph*>(handle);
    auto put = [](const std::vector<long long>& v, int64_t* out) {
      if (out && !v.empty()) std::memcpy(out, v.data(), sizeof(long long) * v.size());
    };
    put(G->off, offsets);
    put(G->tgt, targets);
    put(G->w, eweights);
    put(G->vw, vweights);
    put(G->src, sources);
    delete G;
  });
}
