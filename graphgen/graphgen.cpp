// graphgen/graphgen.cpp -- seeded synthetic CSR graph generator (host C++).
//
// Shared INPUT infrastructure: it feeds both the CUDA path and the oracle and holds none of
// the method's arithmetic (no BFS, no scan of frontier degrees, no partitioning).  It builds
// the five BASELINE.json workloads (ER, 2-D grid, R-MAT 20/24, R-MAT 22 + path tail) and the
// tiny test graphs, as int32 CSR (row_offsets[n+1], col_indices[nnz]).
//
// Randomness: a counter-based generator, rng(seed, stream, index) = SplitMix64 finaliser of a
// (seed, stream, index) mix, so every draw is independent of thread count and order
// (DESIGN.md "input recipe").  Bounded draws use the 32x32 multiply-shift (bias < 2^-32 * n).
#include <algorithm>
#include <atomic>
#include <cstdint>
#include <cstdlib>
#include <cstring>
#include <new>
#include <numeric>
#include <string>
#include <thread>
#include <vector>
#include <chrono>
#include <cstdio>

namespace {

thread_local std::string g_err;
double now_s() { return std::chrono::duration<double>(std::chrono::steady_clock::now().time_since_epoch()).count(); }
void phase(const char *what, double &t0) {
  static const bool verbose = std::getenv("GG_VERBOSE") != nullptr;
  double t = now_s();
  if (verbose) std::fprintf(stderr, "[graphgen] %-10s %.3f s\n", what, t - t0);
  t0 = t;
}

enum : uint64_t {
  STREAM_EDGES = 0x45444745ull,   // "EDGE"
  STREAM_PERM = 0x5045524dull,    // "PERM"
  STREAM_EXTRA = 0x45585452ull,   // "EXTR"
  STREAM_ANCHOR = 0x414e4348ull,  // "ANCH"
  STREAM_SOURCES = 0x53524353ull, // "SRCS"
};

inline uint64_t mix64(uint64_t z) {
  z += 0x9e3779b97f4a7c15ull;
  z = (z ^ (z >> 30)) * 0xbf58476d1ce4e5b9ull;
  z = (z ^ (z >> 27)) * 0x94d049bb133111ebull;
  return z ^ (z >> 31);
}
inline uint64_t rng_key(uint64_t seed, uint64_t stream) {
  return mix64(seed * 0x632be59bd9b4e019ull + stream);
}
inline uint64_t rng_at(uint64_t key, uint64_t i) { return mix64(key ^ (i * 0x9e3779b97f4a7c15ull)); }
inline uint64_t rng(uint64_t seed, uint64_t stream, uint64_t i) { return rng_at(rng_key(seed, stream), i); }
inline uint32_t bounded32(uint32_t r, uint32_t bound) {
  return (uint32_t)(((uint64_t)r * (uint64_t)bound) >> 32);
}

int num_threads(int t) {
  if (t > 0) return t;
  unsigned h = std::thread::hardware_concurrency();
  return h ? (int)h : 4;
}

template <class F>
void parallel_for(int64_t n, int threads, F f) {  // f(begin, end, tid)
  threads = (int)std::min<int64_t>(threads, std::max<int64_t>(n, 1));
  if (threads <= 1) { f(0, n, 0); return; }
  std::vector<std::thread> ts;
  for (int t = 0; t < threads; ++t) {
    int64_t b = n * t / threads, e = n * (t + 1) / threads;
    ts.emplace_back([=] { f(b, e, t); });
  }
  for (auto &th : ts) th.join();
}

struct Graph {
  int32_t n = 0;
  std::vector<int32_t> ro, col;
  int64_t meta[8] = {0, 0, 0, 0, 0, 0, 0, 0};
};

struct Edges {
  std::vector<int32_t> u, v;
};

// CSR from an edge list: drop self-loops (optional), symmetrise (optional), sort each row,
// and remove duplicates (optional).  Edges are radix-partitioned by source into buckets of
// consecutive rows (thread-local histograms, no atomics), each bucket is sorted as packed
// (u << 32 | v) keys, so the result is independent of thread count and scatter order.
bool build_csr(int32_t n, Edges &E, bool symmetrize, bool dedup, bool drop_self, int threads,
               Graph &g) {
  const int64_t m = (int64_t)E.u.size();
  double t0 = now_s();
  for (int64_t i = 0; i < m; ++i) {
    if (E.u[i] < 0 || E.u[i] >= n || E.v[i] < 0 || E.v[i] >= n) {
      g_err = "edge " + std::to_string(i) + " (" + std::to_string(E.u[i]) + "," +
              std::to_string(E.v[i]) + ") out of range";
      return false;
    }
  }
  const int T = std::max(1, (int)std::min<int64_t>(num_threads(threads), std::max<int64_t>(m, 1)));
  int shift = 0;
  while (((int64_t)(n - 1) >> shift) >= 4096) ++shift;
  const int64_t B = ((int64_t)(n - 1) >> shift) + 1;
  std::vector<int64_t> hist((size_t)T * B, 0);
  auto range = [&](int t, int64_t &b, int64_t &e) { b = m * t / T; e = m * (t + 1) / T; };
  {
    std::vector<std::thread> ts;
    for (int t = 0; t < T; ++t)
      ts.emplace_back([&, t] {
        int64_t b, e;
        range(t, b, e);
        int64_t *h = hist.data() + (size_t)t * B;
        for (int64_t i = b; i < e; ++i) {
          int32_t u = E.u[i], v = E.v[i];
          if (drop_self && u == v) continue;
          h[u >> shift]++;
          if (symmetrize) h[v >> shift]++;
        }
      });
    for (auto &th : ts) th.join();
  }
  std::vector<int64_t> bstart((size_t)B + 1, 0);
  for (int64_t b = 0; b < B; ++b) {
    int64_t s = 0;
    for (int t = 0; t < T; ++t) s += hist[(size_t)t * B + b];
    bstart[b + 1] = bstart[b] + s;
  }
  for (int64_t b = 0; b < B; ++b) {  // per-thread write cursors
    int64_t run = bstart[b];
    for (int t = 0; t < T; ++t) {
      int64_t c = hist[(size_t)t * B + b];
      hist[(size_t)t * B + b] = run;
      run += c;
    }
  }
  const int64_t raw = bstart[B];
  std::vector<uint64_t> pairs;
  try { pairs.resize((size_t)std::max<int64_t>(raw, 1)); } catch (...) { g_err = "oom"; return false; }
  {
    std::vector<std::thread> ts;
    for (int t = 0; t < T; ++t)
      ts.emplace_back([&, t] {
        int64_t b, e;
        range(t, b, e);
        int64_t *cur = hist.data() + (size_t)t * B;
        uint64_t *p = pairs.data();
        for (int64_t i = b; i < e; ++i) {
          uint32_t u = (uint32_t)E.u[i], v = (uint32_t)E.v[i];
          if (drop_self && u == v) continue;
          p[cur[u >> shift]++] = ((uint64_t)u << 32) | v;
          if (symmetrize) p[cur[v >> shift]++] = ((uint64_t)v << 32) | u;
        }
      });
    for (auto &th : ts) th.join();
  }
  phase("partition", t0);
  std::vector<int32_t>().swap(E.u);
  std::vector<int32_t>().swap(E.v);
  std::vector<int64_t> bkeep((size_t)B, 0);
  std::vector<int32_t> deg((size_t)n, 0);
  {
    std::atomic<int64_t> next{0};
    std::vector<std::thread> ts;
    for (int t = 0; t < T; ++t)
      ts.emplace_back([&] {
        for (;;) {
          int64_t b = next.fetch_add(1);
          if (b >= B) break;
          uint64_t *pb = pairs.data() + bstart[b], *pe = pairs.data() + bstart[b + 1];
          std::sort(pb, pe);
          uint64_t *ke = dedup ? std::unique(pb, pe) : pe;
          bkeep[b] = ke - pb;
          for (uint64_t *q = pb; q < ke; ++q) deg[*q >> 32]++;  // rows of bucket b only
        }
      });
    for (auto &th : ts) th.join();
  }
  phase("sort", t0);
  int64_t total = 0;
  for (int64_t b = 0; b < B; ++b) total += bkeep[b];
  if (total > INT32_MAX) { g_err = "nnz exceeds int32"; return false; }
  g.n = n;
  g.ro.assign((size_t)n + 1, 0);
  for (int32_t u = 0; u < n; ++u) g.ro[u + 1] = g.ro[u] + deg[u];
  try { g.col.resize((size_t)total); } catch (...) { g_err = "oom"; return false; }
  parallel_for(B, T, [&](int64_t lo, int64_t hi, int) {
    for (int64_t b = lo; b < hi; ++b) {
      int32_t *dst = g.col.data() + g.ro[(int64_t)b << shift];
      const uint64_t *pb = pairs.data() + bstart[b];
      for (int64_t k = 0; k < bkeep[b]; ++k) dst[k] = (int32_t)(uint32_t)pb[k];
    }
  });
  phase("compact", t0);
  return true;
}

void rmat_edges(int scale, int64_t m, double a, double b, double c, uint64_t seed, int threads,
                Edges &E) {
  E.u.resize((size_t)m);
  E.v.resize((size_t)m);
  const uint64_t ta = (uint64_t)(a * 4294967296.0);
  const uint64_t tab = (uint64_t)((a + b) * 4294967296.0);
  const uint64_t tabc = (uint64_t)((a + b + c) * 4294967296.0);
  const int words = (scale + 1) / 2;  // two 32-bit draws per 64-bit word
  const uint64_t key = rng_key(seed, STREAM_EDGES);
  parallel_for(m, threads, [&](int64_t lo, int64_t hi, int) {
    for (int64_t i = lo; i < hi; ++i) {
      uint32_t u = 0, v = 0;
      uint64_t h = 0;
      for (int bit = 0; bit < scale; ++bit) {
        if ((bit & 1) == 0) h = rng_at(key, (uint64_t)i * words + bit / 2);
        uint64_t r = (bit & 1) ? (h >> 32) : (h & 0xffffffffull);
        // quadrant a=(0,0), b=(0,1), c=(1,0), d=(1,1) for (src bit, dst bit), MSB first
        // (branch-free) src bit = r >= a+b (quadrants c, d); dst bit = b or d
        uint32_t su = (uint32_t)(r >= tab);
        uint32_t sv = (uint32_t)(r >= ta) ^ su ^ (uint32_t)(r >= tabc);
        u = (u << 1) | su;
        v = (v << 1) | sv;
      }
      E.u[i] = (int32_t)u;
      E.v[i] = (int32_t)v;
    }
  });
}

std::vector<int32_t> permutation(int32_t n, uint64_t seed) {  // seeded Fisher-Yates
  std::vector<int32_t> p((size_t)n);
  std::iota(p.begin(), p.end(), 0);
  for (int64_t i = (int64_t)n - 1; i > 0; --i) {
    uint32_t j = bounded32((uint32_t)(rng(seed, STREAM_PERM, (uint64_t)i) >> 32), (uint32_t)(i + 1));
    std::swap(p[i], p[j]);
  }
  return p;
}

struct DSU {
  std::vector<int32_t> p;
  explicit DSU(int32_t n) : p((size_t)n) { std::iota(p.begin(), p.end(), 0); }
  int32_t find(int32_t x) {
    while (p[x] != x) { p[x] = p[p[x]]; x = p[x]; }
    return x;
  }
  void unite(int32_t a, int32_t b) {
    a = find(a); b = find(b);
    if (a == b) return;
    if (a < b) std::swap(a, b);
    p[a] = b;  // smaller id is the root: deterministic
  }
};

// component label per vertex (root id) and the largest component's root (ties: smaller root)
int32_t largest_component(int32_t n, const int32_t *ro, const int32_t *col, std::vector<int32_t> &lab) {
  DSU d(n);
  for (int32_t u = 0; u < n; ++u)
    for (int64_t k = ro[u]; k < ro[u + 1]; ++k) d.unite(u, col[k]);
  lab.resize((size_t)n);
  std::vector<int32_t> sz((size_t)n, 0);
  for (int32_t u = 0; u < n; ++u) { lab[u] = d.find(u); sz[lab[u]]++; }
  int32_t best = 0;
  for (int32_t u = 0; u < n; ++u) if (sz[u] > sz[best]) best = u;
  return best;
}

}  // namespace

extern "C" {

typedef Graph gg_graph;

const char *gg_last_error() { return g_err.c_str(); }
int32_t gg_n(const gg_graph *g) { return g->n; }
int64_t gg_nnz(const gg_graph *g) { return (int64_t)g->col.size(); }
int64_t gg_meta(const gg_graph *g, int k) { return (k >= 0 && k < 8) ? g->meta[k] : -1; }
void gg_copy(const gg_graph *g, int32_t *ro, int32_t *col) {
  std::memcpy(ro, g->ro.data(), sizeof(int32_t) * g->ro.size());
  if (!g->col.empty()) std::memcpy(col, g->col.data(), sizeof(int32_t) * g->col.size());
}
void gg_free(gg_graph *g) { delete g; }

// Tiny / test graphs from an explicit edge list.
gg_graph *gg_from_edges(int32_t n, int64_t m, const int32_t *u, const int32_t *v, int symmetrize,
                        int dedup, int drop_self_loops) {
  if (n < 1 || m < 0) { g_err = "invalid n/m"; return nullptr; }
  Edges E;
  E.u.assign(u, u + m);
  E.v.assign(v, v + m);
  auto *g = new (std::nothrow) Graph;
  if (!g || !build_csr(n, E, symmetrize, dedup, drop_self_loops, 1, *g)) { delete g; return nullptr; }
  return g;
}

// Erdos-Renyi G(n, m): m uniform (u,v) draws, self-loops and duplicates removed, symmetrised
// (BASELINE.json configs[0]; reading R24).
gg_graph *gg_er(int32_t n, int64_t m, uint64_t seed, int threads) {
  if (n < 1 || m < 0) { g_err = "invalid n/m"; return nullptr; }
  threads = num_threads(threads);
  Edges E;
  E.u.resize((size_t)m);
  E.v.resize((size_t)m);
  parallel_for(m, threads, [&](int64_t b, int64_t e, int) {
    for (int64_t i = b; i < e; ++i) {
      uint64_t h = rng(seed, STREAM_EDGES, (uint64_t)i);
      E.u[i] = (int32_t)bounded32((uint32_t)(h >> 32), (uint32_t)n);
      E.v[i] = (int32_t)bounded32((uint32_t)h, (uint32_t)n);
    }
  });
  auto *g = new (std::nothrow) Graph;
  if (!g || !build_csr(n, E, true, true, true, threads, *g)) { delete g; return nullptr; }
  return g;
}

// rows x cols 4-neighbour grid, id = r*cols + c (BASELINE.json configs[1]); rows sorted.
gg_graph *gg_grid(int32_t rows, int32_t cols) {
  if (rows < 1 || cols < 1 || (int64_t)rows * cols > INT32_MAX) { g_err = "invalid grid"; return nullptr; }
  auto *g = new (std::nothrow) Graph;
  if (!g) return nullptr;
  int32_t n = rows * cols;
  g->n = n;
  g->ro.assign((size_t)n + 1, 0);
  g->col.reserve((size_t)4 * n);
  for (int32_t r = 0; r < rows; ++r)
    for (int32_t c = 0; c < cols; ++c) {
      int32_t id = r * cols + c;
      if (r > 0) g->col.push_back(id - cols);
      if (c > 0) g->col.push_back(id - 1);
      if (c + 1 < cols) g->col.push_back(id + 1);
      if (r + 1 < rows) g->col.push_back(id + cols);
      g->ro[id + 1] = (int32_t)g->col.size();
    }
  return g;
}

// R-MAT(scale, edge factor): ef*2^scale recursive-quadrant draws, seeded id permutation,
// self-loops dropped, symmetrised, duplicates removed (configs[2], configs[3]; reading R19).
gg_graph *gg_rmat(int scale, int ef, double a, double b, double c, uint64_t seed, int permute,
                  int threads) {
  if (scale < 0 || scale > 30 || ef < 0 || a < 0 || b < 0 || c < 0 || a + b + c > 1.0) {
    g_err = "invalid rmat parameters";
    return nullptr;
  }
  threads = num_threads(threads);
  int32_t n = (int32_t)1 << scale;
  int64_t m = (int64_t)ef << scale;
  Edges E;
  double t0 = now_s();
  rmat_edges(scale, m, a, b, c, seed, threads, E);
  phase("draw", t0);
  if (permute) {
    auto p = permutation(n, seed);
    parallel_for(m, threads, [&](int64_t lo, int64_t hi, int) {
      for (int64_t i = lo; i < hi; ++i) { E.u[i] = p[E.u[i]]; E.v[i] = p[E.v[i]]; }
    });
  }
  phase("permute", t0);
  auto *g = new (std::nothrow) Graph;
  if (!g || !build_csr(n, E, true, true, true, threads, *g)) { delete g; return nullptr; }
  return g;
}

// R-MAT + 1% uniform extra edges among the R-MAT ids + a simple path of path_len NEW vertices
// attached to a uniform vertex of the giant component (configs[4]; reading R20).
// meta: [0] anchor, [1] first path vertex, [2] far end, [3] giant-component size (R-MAT part).
gg_graph *gg_rmat_tail(int scale, int ef, double a, double b, double c, uint64_t seed,
                       double extra_frac, int32_t path_len, int threads) {
  if (scale < 1 || scale > 28 || path_len < 1 || extra_frac < 0) { g_err = "invalid tail parameters"; return nullptr; }
  threads = num_threads(threads);
  int32_t n0 = (int32_t)1 << scale;
  int64_t m = (int64_t)ef << scale;
  int64_t extra = (int64_t)(extra_frac * (double)ef * (double)n0);
  Edges E;
  rmat_edges(scale, m, a, b, c, seed, threads, E);
  auto p = permutation(n0, seed);
  parallel_for(m, threads, [&](int64_t lo, int64_t hi, int) {
    for (int64_t i = lo; i < hi; ++i) { E.u[i] = p[E.u[i]]; E.v[i] = p[E.v[i]]; }
  });
  E.u.resize((size_t)(m + extra));
  E.v.resize((size_t)(m + extra));
  for (int64_t i = 0; i < extra; ++i) {
    uint64_t h = rng(seed, STREAM_EXTRA, (uint64_t)i);
    E.u[m + i] = (int32_t)bounded32((uint32_t)(h >> 32), (uint32_t)n0);
    E.v[m + i] = (int32_t)bounded32((uint32_t)h, (uint32_t)n0);
  }
  // giant component of the R-MAT + extra part (union-find over the edge list)
  DSU d(n0);
  for (int64_t i = 0; i < m + extra; ++i) if (E.u[i] != E.v[i]) d.unite(E.u[i], E.v[i]);
  std::vector<int32_t> sz((size_t)n0, 0);
  for (int32_t u = 0; u < n0; ++u) sz[d.find(u)]++;
  int32_t best = 0;
  for (int32_t u = 0; u < n0; ++u) if (sz[u] > sz[best]) best = u;
  int32_t giant = sz[best];
  uint32_t pick = bounded32((uint32_t)(rng(seed, STREAM_ANCHOR, 0) >> 32), (uint32_t)giant);
  int32_t anchor = -1;
  for (int32_t u = 0, k = 0; u < n0; ++u)
    if (d.find(u) == best) { if ((uint32_t)k == pick) { anchor = u; break; } ++k; }
  int32_t n = n0 + path_len;
  E.u.push_back(anchor);
  E.v.push_back(n0);
  for (int32_t i = 0; i + 1 < path_len; ++i) { E.u.push_back(n0 + i); E.v.push_back(n0 + i + 1); }
  auto *g = new (std::nothrow) Graph;
  if (!g || !build_csr(n, E, true, true, true, threads, *g)) { delete g; return nullptr; }
  g->meta[0] = anchor;
  g->meta[1] = n0;
  g->meta[2] = n0 + path_len - 1;
  g->meta[3] = giant;
  return g;
}

// Seeded distinct sources.  mode 0: uniform among non-isolated vertices (Graph500 style);
// mode 1: uniform in the largest connected component.  Returns the number written.
int gg_pick_sources(int32_t n, const int32_t *ro, const int32_t *col, int mode, int count,
                    uint64_t seed, int32_t *out) {
  if (n < 1 || count < 0 || (mode != 0 && mode != 1)) { g_err = "invalid source request"; return -1; }
  std::vector<int32_t> lab;
  int32_t best = -1;
  if (mode == 1) best = largest_component(n, ro, col, lab);
  int got = 0;
  for (uint64_t i = 0; got < count && i < (uint64_t)count * 100000ull; ++i) {
    int32_t v = (int32_t)bounded32((uint32_t)(rng(seed, STREAM_SOURCES, i) >> 32), (uint32_t)n);
    bool ok = mode == 0 ? (ro[v + 1] > ro[v]) : (lab[v] == best);
    for (int k = 0; ok && k < got; ++k) if (out[k] == v) ok = false;
    if (ok) out[got++] = v;
  }
  return got;
}

// Size of the connected component containing v (for GTEPS bookkeeping of tiny graphs).
int64_t gg_component_size(int32_t n, const int32_t *ro, const int32_t *col, int32_t v) {
  std::vector<int32_t> lab;
  largest_component(n, ro, col, lab);
  int64_t c = 0;
  for (int32_t u = 0; u < n; ++u) c += lab[u] == lab[v];
  return c;
}

}  // extern "C"
