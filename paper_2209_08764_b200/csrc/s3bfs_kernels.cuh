// paper_2209_08764_b200/csrc/s3bfs_kernels.cuh -- sm_100a kernels of the S3BFS hot path.
//
// "P:n" = /root/reference/PAPER.md line n; "Fig1 Lk" = item k of Figure 1;
// "R<k>" = reading k in DESIGN.md.  This file shares nothing with oracle/ (test-only code).
//
// Kernels (one level = one pass of (a)-(e)):
//   k_init     Fig1 L1-L8   level/parent <- -1, level[s] = 0, parent[s] = s, frontier = [s]
//   k_explore  (c)+(d)      Fig1 L17-L18: equal edge chunks per CTA ("(almost) equal
//                           division"), start vertex by a 32-ary warp search of the degree
//                           scan (R8), tile-wise edge->vertex map, coalesced col streaming,
//                           plain-store labelling with the benign race -- no
//                           atomic instruction anywhere in this kernel.
//   k_compact  (e)+(a)+(b)  Fig1 L19-L29 + L12-L15 of the NEXT level: keep cand[k] iff
//                           Owner[cand[k]] == k, decoupled look-back scan of (kept, degree-sum)
//                           pairs across CTAs, write f_next / row starts / degree scan.
//   k_small    tier 0 (f)   one CTA runs whole levels (a)-(e) in shared memory while the level
//                           stays tiny (P:22 -- "never use more cores than necessary").
//   k_dispatch (f)          graph mode: selects the tier of the next WHILE iteration.
//   k_scan_u32 (b) alone    test entry: the same look-back scan over a plain int32 array.
//   k_find_start (c) alone  test entry: the same warp search, one warp per worker.
#pragma once
#include <cuda_runtime.h>
#include <stdint.h>

#include "../../include/s3bfs.h"

namespace s3bfs {

// ---- compile-time geometry --------------------------------------------------------------
constexpr int KD_THREADS = 512;                 // k_explore / k_compact CTA size
constexpr int KD_WARPS = KD_THREADS / 32;
constexpr int KD_TILE = 4096;                   // candidate-buffer slack per CTA (edges)
constexpr int KS_THREADS = 1024;                // k_small CTA size
constexpr int KS_ECAP = 8192;                   // T0 maximum (edges per tier-0 level)
constexpr int KS_NCAP = KS_ECAP;                // frontier capacity of tier 0 (kept <= e_l)
constexpr int KS_IPT = KS_ECAP / KS_THREADS;    // dedup items per thread
constexpr int SCAN_THREADS = 512;
constexpr int SCAN_ITEMS = 8;
constexpr int SCAN_TILE = SCAN_THREADS * SCAN_ITEMS;

constexpr int TIER_SMALL = 0, TIER_LARGE = 1, TIER_DONE = 2;

// Device control block: the paper's loop state (Fig1 L8-L11, L15-L16) kept on the device so
// the level loop needs no host round trip.
struct Ctl {
  int32_t level;      // l: level of the current frontier (Fig1 L8, L10)
  int32_t n_l;        // |CurLevelVertices| (Fig1 L9)
  int32_t e_l;        // EdgeSum[n_l - 1] (Fig1 L15)
  int32_t cur;        // which frontier buffer holds CurLevelVertices
  int32_t tier;       // TIER_SMALL / TIER_LARGE / TIER_DONE
  int32_t p_l;        // P_l = CTAs of this level (Fig1 L16)
  int32_t chunk;      // edges per CTA (ceil(e_l / P_l))
  int32_t wcap;       // candidate capacity per warp
  int32_t n_next, e_next;   // written by the last k_compact CTA in tile order
  uint32_t done_ctr;        // last-CTA election in k_compact (not the discovery path)
  int32_t num_levels;       // stats records written
  int32_t cand_acc;         // stats: candidates of the level (incl. duplicates)
  int32_t source;
  int32_t pad0, pad1;
  int32_t *level_out, *parent_out;
  unsigned long long t_prev;
  unsigned long long t_kx_begin, t_kx_end;  // k_explore CTA 0 start, k_compact CTA 0 start
};

struct Params {
  const int32_t *ro, *col;
  int32_t n;
  Ctl *ctl;
  int32_t *owner;
  int32_t *f[2], *frs[2], *fex[2];  // frontier ids, their row starts, exclusive degree scan
  int32_t *cand;
  int2 *cand_rd;          // (row start, degree) of kept candidates, pass 1 -> pass 2 of k_compact
  uint32_t *bm;           // visited bitmap: bit v set => level[v] != -1 (a filter; level[] rules)
  int32_t *wcnt;
  unsigned long long *status;
  s3bfs_level_stat *stats;
  int32_t stats_cap;
  int32_t p_max, grain, t0, variant, collect_stats;
  int32_t use_graph;
  unsigned long long h_while, h_t0, h_t1;  // cudaGraphConditionalHandle values
};

// ---- PTX helpers ------------------------------------------------------------------------
__device__ __forceinline__ unsigned long long globaltimer() {
  unsigned long long t;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
  return t;
}
// Status reads of the racing arrays (level[], owner[]): weak loads, L1-cacheable.  Within one
// kernel launch a stale -1 only re-discovers v at the SAME level (benign, R18); L1 is
// invalidated at every launch, so staleness never crosses a level boundary.
__device__ __forceinline__ int ld_weak(const int32_t *p) {
  int v;
  asm volatile("ld.global.s32 %0, [%1];" : "=r"(v) : "l"(p));
  return v;
}
// L2 eviction policies (createpolicy): the adjacency is streamed once per level and must not
// evict the status array, which every arc probes at random.
__device__ __forceinline__ unsigned long long policy_evict_first() {
  unsigned long long p;
  asm volatile("createpolicy.fractional.L2::evict_first.b64 %0, 1.0;" : "=l"(p));
  return p;
}
__device__ __forceinline__ unsigned long long policy_evict_last() {
  unsigned long long p;
  asm volatile("createpolicy.fractional.L2::evict_last.b64 %0, 1.0;" : "=l"(p));
  return p;
}
// read-only stream (col_indices): non-coherent, no L1 allocation, L2 evict-first
__device__ __forceinline__ int ldg_stream(const int32_t *p, unsigned long long pol) {
  int v;
  asm volatile("ld.global.nc.L1::no_allocate.L2::cache_hint.s32 %0, [%1], %2;"
               : "=r"(v) : "l"(p), "l"(pol));
  return v;
}
// status probe of level[] (racing array, weak load) with an L2 evict-last hint
__device__ __forceinline__ int ld_status(const int32_t *p, unsigned long long pol) {
  int v;
  asm volatile("ld.global.L2::cache_hint.s32 %0, [%1], %2;" : "=r"(v) : "l"(p), "l"(pol));
  return v;
}
__device__ __forceinline__ uint32_t ld_status_u32(const uint32_t *p, unsigned long long pol) {
  uint32_t v;
  asm volatile("ld.global.L2::cache_hint.u32 %0, [%1], %2;" : "=r"(v) : "l"(p), "l"(pol));
  return v;
}
__device__ __forceinline__ void st_weak(int32_t *p, int v) {
  asm volatile("st.global.s32 [%0], %1;" ::"l"(p), "r"(v) : "memory");
}
__device__ __forceinline__ unsigned long long ld_relaxed_u64(const unsigned long long *p) {
  unsigned long long v;
  asm volatile("ld.relaxed.gpu.global.u64 %0, [%1];" : "=l"(v) : "l"(p) : "memory");
  return v;
}
__device__ __forceinline__ void st_relaxed_u64(unsigned long long *p, unsigned long long v) {
  asm volatile("st.relaxed.gpu.global.u64 [%0], %1;" ::"l"(p), "l"(v) : "memory");
}
__device__ __forceinline__ int ld_volatile(const int32_t *p) {
  return *(const volatile int32_t *)p;
}
__device__ __forceinline__ unsigned lanemask_lt() {
  unsigned m;
  asm("mov.u32 %0, %%lanemask_lt;" : "=r"(m));
  return m;
}

__device__ __forceinline__ int warp_incl_scan(int x) {
  const int lane = threadIdx.x & 31;
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    int y = __shfl_up_sync(0xffffffffu, x, o);
    if (lane >= o) x += y;
  }
  return x;
}
__device__ __forceinline__ int warp_sum(int x) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) x += __shfl_xor_sync(0xffffffffu, x, o);
  return x;
}

// (c) Find-StartExpPoint (Fig1 L17; R8): the largest u in [0, n_l) with excl[u] <= t,
// i.e. the unique frontier vertex whose edge range [excl[u], excl[u+1]) holds global edge t
// (t < excl[n_l]).  32-ary search by one full warp: ceil(log32(n_l)) dependent probes.
__device__ __forceinline__ int warp_search(const int32_t *__restrict__ excl, int n_l, int t) {
  const int lane = threadIdx.x & 31;
  int lo = 0, hi = n_l;  // answer in [lo, hi), excl[lo] <= t
  while (hi - lo > 1) {
    const int step = (hi - lo + 31) >> 5;
    const int p = lo + lane * step;
    const bool ok = (p < hi) && (__ldg(excl + p) <= t);
    const unsigned m = __ballot_sync(0xffffffffu, ok);  // a prefix of lanes (excl sorted)
    const int k = 31 - __clz(m);
    lo += k * step;
    hi = min(hi, lo + step);
  }
  return lo;
}

// ---- decoupled look-back (Merrill & Garland single-pass scan; the (b) step) ----------
// Status word: [63:62] flag (0 invalid, 1 aggregate, 2 inclusive prefix) | payload.
// PAIR payload: [61:31] kept count, [30:0] degree sum (both < 2^31 by create-time checks).
// U32 payload:  [31:0] value (two's-complement wrap, the test-only plain scan).
constexpr unsigned long long FLAG_A = 1ull << 62, FLAG_P = 2ull << 62;
struct Pair { uint32_t a, b; };
template <bool PAIR>
__device__ __forceinline__ unsigned long long pack(Pair v) {
  return PAIR ? (((unsigned long long)v.a << 31) | v.b) : (unsigned long long)v.a;
}
template <bool PAIR>
__device__ __forceinline__ Pair unpack(unsigned long long s) {
  Pair v;
  if (PAIR) { v.a = (uint32_t)((s >> 31) & 0x7fffffffu); v.b = (uint32_t)(s & 0x7fffffffu); }
  else { v.a = (uint32_t)s; v.b = 0; }
  return v;
}
// Called by ONE full warp of tile `tile`; returns the exclusive prefix of the tile (to all
// lanes) after publishing the tile's inclusive prefix.  `status` entries < tile are written
// by the tiles before it; the caller guarantees they were reset before this pass.
template <bool PAIR>
__device__ Pair lookback(unsigned long long *status, int tile, Pair agg) {
  const int lane = threadIdx.x & 31;
  if (tile == 0) {
    if (lane == 0) st_relaxed_u64(status, FLAG_P | pack<PAIR>(agg));
    return Pair{0, 0};
  }
  if (lane == 0) st_relaxed_u64(status + tile, FLAG_A | pack<PAIR>(agg));
  Pair excl{0, 0};
  int pred = tile - 1;
  unsigned ns = 32;
  for (;;) {
    const int idx = pred - lane;
    unsigned long long s = idx >= 0 ? ld_relaxed_u64(status + idx) : FLAG_P;
    const unsigned flag = (unsigned)(s >> 62);
    const unsigned mP = __ballot_sync(0xffffffffu, flag == 2);
    const unsigned mI = __ballot_sync(0xffffffffu, flag == 0);
    const int firstP = mP ? __ffs(mP) - 1 : 32;
    const unsigned need = firstP >= 31 ? 0xffffffffu : ((2u << firstP) - 1u);
    if (mI & need) {  // a predecessor has not published yet
      __nanosleep(ns);
      if (ns < 1024) ns <<= 1;
      continue;
    }
    Pair v = (lane <= firstP) ? unpack<PAIR>(s) : Pair{0, 0};
    excl.a += (uint32_t)warp_sum((int)v.a);
    excl.b += (uint32_t)warp_sum((int)v.b);
    if (firstP < 32) break;
    pred -= 32;
  }
  if (lane == 0) {
    Pair inc{excl.a + agg.a, excl.b + agg.b};
    st_relaxed_u64(status + tile, FLAG_P | pack<PAIR>(inc));
  }
  return excl;
}

// ---- (f) level-adaptive sizing: the tier and P_l of the level held in ctl ------------------
// P_l = min(P_max, ceil(e_l / grain)) -- the GPU form of P_l <- Min(P, e_l) (Fig1 L16):
// a "core" here is a CTA that streams >= grain edges.  variant 1 = work-insensitive.
__device__ void record_stat(const Params &P, Ctl *c, int32_t level, int32_t n_l, int32_t e_l,
                            int32_t tier, int32_t grid, int32_t cand, int32_t kept,
                            unsigned long long t0, unsigned long long t1,
                            unsigned long long tx0 = 0, unsigned long long tx1 = 0) {
  if (!P.collect_stats) return;
  const int k = c->num_levels;
  if (k < P.stats_cap) {
    s3bfs_level_stat r;
    r.level = level; r.n_l = n_l; r.e_l = e_l; r.tier = tier; r.grid = grid;
    r.candidates = cand; r.kept = kept; r.pad = 0; r.t_begin_ns = t0; r.t_end_ns = t1;
    r.t_explore_begin_ns = tx0; r.t_explore_end_ns = tx1;
    P.stats[k] = r;
  }
  c->num_levels = k + 1;
}

__device__ void decide(const Params &P, Ctl *c, int32_t n_l, int32_t e_l) {
  c->n_l = n_l;
  c->e_l = e_l;
  if (n_l == 0 || e_l == 0) {  // C10: nothing to explore, the loop ends (Fig1 L9)
    if (n_l > 0) {
      const unsigned long long t = globaltimer();
      record_stat(P, c, c->level, n_l, 0, TIER_DONE, 0, 0, 0, t, t);
    }
    c->tier = TIER_DONE;
    c->p_l = 0;
    return;
  }
  if (P.variant == 0 && P.t0 >= 0 && e_l <= P.t0 && n_l <= KS_NCAP) {
    c->tier = TIER_SMALL;
    c->p_l = 1;
    return;
  }
  long long pt = P.variant ? (long long)P.p_max
                           : min((long long)P.p_max, ((long long)e_l + P.grain - 1) / P.grain);
  if (pt < 1) pt = 1;
  const long long chunk = ((long long)e_l + pt - 1) / pt;
  const long long p_l = ((long long)e_l + chunk - 1) / chunk;
  c->tier = TIER_LARGE;
  c->p_l = (int32_t)p_l;
  c->chunk = (int32_t)chunk;
  c->wcap = (int32_t)((chunk + KD_WARPS - 1) / KD_WARPS);  // edges (and candidates) per warp
}

// ---- init (Fig1 L1-L8) ----------------------------------------------------------------------
// level[v] <- -1 (d <- infinity, R1), parent[v] <- -1; level[s] = 0, parent[s] = s (R2).
// Owner is NOT initialised (R3: every read of Owner[v] follows a write in the same level).
__global__ void k_init(Params P, int32_t s, int32_t *level, int32_t *parent) {
  const int n = P.n;
  const long long gtid = (long long)blockIdx.x * blockDim.x + threadIdx.x;
  const long long gstride = (long long)gridDim.x * blockDim.x;
  const bool vec = ((((uintptr_t)level) | ((uintptr_t)parent)) & 15) == 0;
  long long done = 0;
  if (vec) {
    const long long n4 = n >> 2;
    for (long long i = gtid; i < n4; i += gstride) {
      int4 lv = make_int4(-1, -1, -1, -1), pv = lv;
      const long long b = i << 2;
      if (s >= b && s < b + 4) {
        const int j = (int)(s - b);
        (&lv.x)[j] = 0;
        (&pv.x)[j] = s;
      }
      reinterpret_cast<int4 *>(level)[i] = lv;
      reinterpret_cast<int4 *>(parent)[i] = pv;
    }
    done = n4 << 2;
  }
  for (long long i = done + gtid; i < n; i += gstride) {
    level[i] = (i == s) ? 0 : -1;
    parent[i] = (i == s) ? s : -1;
  }
  const long long nw = ((long long)n + 31) >> 5;  // visited bitmap: only the source
  for (long long i = gtid; i < nw; i += gstride)
    P.bm[i] = (i == (s >> 5)) ? (1u << (s & 31)) : 0u;
  if (blockIdx.x == 0 && threadIdx.x == 0) {
    Ctl *c = P.ctl;
    const int r0 = P.ro[s], r1 = P.ro[s + 1];
    P.f[0][0] = s;        // Fig1 L7: CurLevelVertices <- [s]
    P.frs[0][0] = r0;
    P.fex[0][0] = 0;      // exclusive degree scan of the frontier (R5)
    P.fex[0][1] = r1 - r0;
    c->level = 0;         // Fig1 L8
    c->cur = 0;
    c->source = s;
    c->level_out = level;
    c->parent_out = parent;
    c->num_levels = 0;
    c->done_ctr = 0;
    c->cand_acc = 0;
    c->t_prev = globaltimer();
    decide(P, c, 1, r1 - r0);
  }
}

// Graph mode: one thread selects what the next WHILE iteration runs (f).
__global__ void k_dispatch(Params P) {
  const int t = P.ctl->tier;
  cudaGraphSetConditional((cudaGraphConditionalHandle)P.h_t0, t == TIER_SMALL ? 1u : 0u);
  cudaGraphSetConditional((cudaGraphConditionalHandle)P.h_t1, t == TIER_LARGE ? 1u : 0u);
  if (t == TIER_DONE) cudaGraphSetConditional((cudaGraphConditionalHandle)P.h_while, 0u);
}

// ---- (c)+(d): k_explore ----------------------------------------------------------------------
// CTA b < P_l owns global edges [b*chunk, min((b+1)*chunk, e_l)) of the level, split evenly
// over its warps: each warp is one of the paper's workers with an (almost) equal share of the
// level's edges (Fig1 L16-L17).  A warp finds its start vertex with the 32-ary search
// (c), then walks its edges in groups of 32 -- lane i takes edge e+i, so a group reads 32
// consecutive col entries (coalesced streaming, Fig1 L18).  Edge -> frontier vertex mapping
// uses a register window of 32 consecutive frontier vertices (their degree-scan entries,
// ids and row starts): a 5-step shuffle search per lane, no shared memory, no CTA barrier,
// so warps progress independently and keep KX_GROUPS groups of loads in flight.
// Discovery (EXPLORE-VERTEX): if level[v] == -1 then level[v] = l+1, parent[v] = x,
// Owner[v] = slot, cand[slot] = v -- plain stores, the paper's benign race, no atomics.
// The candidate slot is a unique id (R4), so Owner dedup keeps exactly one copy even when
// two lanes of one warp discover v together.
constexpr int KX_GROUPS = 8;
constexpr int KX_MIN_BLOCKS = 2;
__global__ void __launch_bounds__(KD_THREADS, KX_MIN_BLOCKS) k_explore(Params P) {
  Ctl *c = P.ctl;
  if (c->tier != TIER_LARGE) return;
  const int b = blockIdx.x;
  const int p_l = c->p_l;
  if (b >= p_l) return;
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int n_l = c->n_l, e_l = c->e_l, chunk = c->chunk, cur = c->cur, wcap = c->wcap;
  const int new_level = c->level + 1;  // Fig1 L10: discoveries get l+1 (R11)
  int32_t *__restrict__ level = c->level_out;
  int32_t *__restrict__ parent = c->parent_out;
  const int32_t *__restrict__ fx = P.f[cur];
  const int32_t *__restrict__ frs = P.frs[cur];
  const int32_t *__restrict__ fex = P.fex[cur];
  const int32_t *__restrict__ col = P.col;
  int32_t *__restrict__ owner = P.owner;
  int32_t *__restrict__ cand = P.cand;
  const uint32_t *__restrict__ bm = P.bm;

  if (tid == 0) {
    P.status[b] = 0ull;  // reset k_compact's look-back word for this level
    if (b == 0) c->t_kx_begin = globaltimer();
  }
  const int E0 = b * chunk;
  const int E1 = min(E0 + chunk, e_l);
  const int e_begin = min(E0 + warp * wcap, E1);
  const int e_end = min(e_begin + wcap, E1);
  const int segbase = (b * KD_WARPS + warp) * wcap;
  const unsigned long long pol_stream = policy_evict_first();
  const unsigned long long pol_status = policy_evict_last();
  int wcount = 0;
  if (e_begin < e_end) {
    int u0 = warp_search(fex, n_l, e_begin);  // Find-StartExpPoint (c)
    int wex, wx, wb, lim;
    auto load_window = [&](int base) {
      const int u = base + lane;
      wex = (u < n_l) ? __ldg(fex + u) : 0x7fffffff;
      wx = (u < n_l) ? __ldg(fx + u) : 0;
      wb = (u < n_l) ? __ldg(frs + u) - wex : 0;
      lim = __ldg(fex + min(base + 32, n_l));
    };
    load_window(u0);
    int e = e_begin;
    while (e < e_end) {
      while (lim <= e) {  // window exhausted (also skips runs of zero-degree vertices, C9)
        u0 += 32;
        load_window(u0);
      }
      const int bend = min(e_end, lim);
      int v[KX_GROUPS], xv[KX_GROUPS];
#pragma unroll
      for (int g = 0; g < KX_GROUPS; ++g) {
        const int my_e = e + g * 32 + lane;
        int j = 0;  // largest window slot with excl <= my_e
#pragma unroll
        for (int s = 16; s >= 1; s >>= 1) {
          const int cj = __shfl_sync(0xffffffffu, wex, j + s);
          if (cj <= my_e) j += s;
        }
        xv[g] = __shfl_sync(0xffffffffu, wx, j);
        const int pos = __shfl_sync(0xffffffffu, wb, j) + my_e;
        v[g] = (my_e < bend) ? ldg_stream(col + pos, pol_stream) : -1;
      }
      // status: the visited bitmap first (2 MB at scale 24: stays in L2), level[] only when the
      // bit is clear (unvisited, or discovered earlier in this same level)
      uint32_t bw[KX_GROUPS];
#pragma unroll
      for (int g = 0; g < KX_GROUPS; ++g)
        bw[g] = (v[g] >= 0) ? ld_status_u32(bm + (v[g] >> 5), pol_status) : 0xffffffffu;
      int lv[KX_GROUPS];
#pragma unroll
      for (int g = 0; g < KX_GROUPS; ++g)
        lv[g] = ((bw[g] >> (v[g] & 31)) & 1u) ? 0 : ld_status(level + v[g], pol_status);
#pragma unroll
      for (int g = 0; g < KX_GROUPS; ++g) {
        const bool disc = lv[g] == -1;
        const unsigned m = __ballot_sync(0xffffffffu, disc);
        if (disc) {
          const int slot = segbase + wcount + __popc(m & lanemask_lt());
          st_weak(level + v[g], new_level);
          st_weak(parent + v[g], xv[g]);
          st_weak(owner + v[g], slot);
          cand[slot] = v[g];
        }
        wcount += __popc(m);
      }
      e = min(e + KX_GROUPS * 32, bend);
    }
  }
  if (lane == 0) P.wcnt[b * KD_WARPS + warp] = wcount;
}

// ---- (e)+(a)+(b): k_compact -------------------------------------------------------------------
// CTA b handles the candidate segments its k_explore twin wrote (one per warp).
// Pass 1 (Fig1 L20-L23): keep cand[k] iff Owner[cand[k]] == k, compacting in place, and sum
// the kept vertices' degrees (Fig1 L13 for the next level).  Then a decoupled look-back over
// CTAs scans the (kept, degree-sum) pairs (Fig1 L24 and L14 of the next level in one pass).
// Pass 2 (Fig1 L25-L29): write the next frontier, its row starts and its exclusive degree
// scan.  The last CTA to finish advances the control block (Fig1 L9-L10, L15-L16).
__global__ void __launch_bounds__(KD_THREADS, 2) k_compact(Params P) {
  Ctl *c = P.ctl;
  if (c->tier != TIER_LARGE) return;
  const int b = blockIdx.x;
  const int p_l = c->p_l;
  if (b >= p_l) return;
  __shared__ int32_t s_k[KD_WARPS], s_d[KD_WARPS];
  __shared__ int s_last;
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int nxt = c->cur ^ 1;
  const int32_t *__restrict__ ro = P.ro;
  const int32_t *__restrict__ owner = P.owner;
  int32_t *__restrict__ cand = P.cand;
  const int seg = (b * KD_WARPS + warp) * c->wcap;
  const int cnt = P.wcnt[b * KD_WARPS + warp];
  if (b == 0 && tid == 0) c->t_kx_end = globaltimer();

  int2 *__restrict__ crd = P.cand_rd;
  int kept = 0, dsum = 0;
  for (int k0 = 0; k0 < cnt; k0 += 32) {
    const int k = k0 + lane;
    bool keep = false;
    int v = 0, r0 = 0, d = 0;
    if (k < cnt) {
      v = cand[seg + k];
      keep = ld_weak(owner + v) == seg + k;  // Fig1 L22: "if Owner[v] = i"
      if (keep) {
        r0 = __ldg(ro + v);
        d = __ldg(ro + v + 1) - r0;
        atomicOr(P.bm + (v >> 5), 1u << (v & 31));  // publish "visited" (filter only, R17)
      }
    }
    const unsigned m = __ballot_sync(0xffffffffu, keep);
    if (keep) {
      const int q = seg + kept + __popc(m & lanemask_lt());
      cand[q] = v;
      crd[q] = make_int2(r0, d);
    }
    kept += __popc(m);
    dsum += d;
  }
  dsum = warp_sum(dsum);
  if (lane == 0) { s_k[warp] = kept; s_d[warp] = dsum; }
  if (P.collect_stats) {
    const int tot = warp_sum(lane == 0 ? cnt : 0);
    if (lane == 0 && tot) atomicAdd(&c->cand_acc, tot);  // statistics only
  }
  __syncthreads();
  if (warp == 0) {
    const int kk = lane < KD_WARPS ? s_k[lane] : 0;
    const int dd = lane < KD_WARPS ? s_d[lane] : 0;
    const int ik = warp_incl_scan(kk), id = warp_incl_scan(dd);
    const Pair agg{(uint32_t)__shfl_sync(0xffffffffu, ik, 31),
                   (uint32_t)__shfl_sync(0xffffffffu, id, 31)};
    const Pair ex = lookback<true>(P.status, b, agg);
    if (lane < KD_WARPS) { s_k[lane] = (int)ex.a + ik - kk; s_d[lane] = (int)ex.b + id - dd; }
    if (b == p_l - 1 && lane == 0) {  // the level's totals: n_{l+1}, e_{l+1} (Fig1 L15)
      const int n_next = (int)(ex.a + agg.a), e_next = (int)(ex.b + agg.b);
      c->n_next = n_next;
      c->e_next = e_next;
      P.fex[nxt][n_next] = e_next;
    }
  }
  __syncthreads();
  int koff = s_k[warp], doff = s_d[warp];
  int32_t *__restrict__ fn = P.f[nxt];
  int32_t *__restrict__ frsn = P.frs[nxt];
  int32_t *__restrict__ fexn = P.fex[nxt];
  for (int k0 = 0; k0 < kept; k0 += 32) {
    const int k = k0 + lane;
    int v = 0, r0 = 0, d = 0;
    if (k < kept) {
      v = cand[seg + k];
      const int2 rd = crd[seg + k];
      r0 = rd.x;
      d = rd.y;
    }
    const int inc = warp_incl_scan(d);
    if (k < kept) {
      fn[koff + k] = v;
      frsn[koff + k] = r0;
      fexn[koff + k] = doff + inc - d;
    }
    doff += __shfl_sync(0xffffffffu, inc, 31);
  }
  // last-CTA election (one atomic per CTA; not on the discovery path, R17)
  __threadfence();
  __syncthreads();
  if (tid == 0) s_last = atomicAdd(&c->done_ctr, 1u) == (unsigned)(p_l - 1);
  __syncthreads();
  if (s_last && tid == 0) {
    __threadfence();
    const int n_next = ld_volatile(&c->n_next), e_next = ld_volatile(&c->e_next);
    const unsigned long long t = globaltimer();
    record_stat(P, c, c->level, c->n_l, c->e_l, TIER_LARGE, p_l, ld_volatile(&c->cand_acc),
                n_next, c->t_prev, t, *(volatile unsigned long long *)&c->t_kx_begin,
                *(volatile unsigned long long *)&c->t_kx_end);
    c->cand_acc = 0;
    c->done_ctr = 0;
    c->t_prev = t;
    c->level = c->level + 1;  // Fig1 L10
    c->cur = nxt;
    decide(P, c, n_next, e_next);
  }
}

// ---- tier 0: k_small -------------------------------------------------------------------------
// One CTA runs consecutive tiny levels (e_l <= T0) with __syncthreads between the steps: the
// paper's "use only as many cores as there is work" at CTA granularity.  Same
// per-level contract as k_explore + k_compact; the owner label is the level-local edge
// index e (unique, R4); frontier, degree scan and candidates live in shared memory.
// Global level/parent/owner writes of this CTA are ordered for its own later reads by the
// CTA barrier (one SM), so multi-level operation is safe.
__global__ void __launch_bounds__(KS_THREADS, 1) k_small(Params P) {
  Ctl *c = P.ctl;
  if (c->tier != TIER_SMALL) return;
  extern __shared__ int32_t smem[];
  int32_t *sf = smem;                 // CurLevelVertices
  int32_t *srs = sf + KS_NCAP;        // row starts
  int32_t *sex = srs + KS_NCAP;       // exclusive degree scan, KS_NCAP + 1 entries
  int32_t *cv = sex + KS_NCAP + 4;    // candidate per level-local edge (or -1)
  __shared__ int32_t s_wk[KS_THREADS / 32], s_wd[KS_THREADS / 32], s_wc[KS_THREADS / 32];
  __shared__ int32_t s_tot[3];

  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int32_t *__restrict__ ro = P.ro;
  const int32_t *__restrict__ col = P.col;
  int32_t *__restrict__ level = c->level_out;
  int32_t *__restrict__ parent = c->parent_out;
  int32_t *__restrict__ owner = P.owner;
  int n_l = c->n_l, e_l = c->e_l, L = c->level;
  const int cur = c->cur;
  unsigned long long t_prev = c->t_prev;
  for (int i = tid; i < n_l; i += KS_THREADS) {
    sf[i] = P.f[cur][i];
    srs[i] = P.frs[cur][i];
    sex[i] = P.fex[cur][i];
  }
  if (tid == 0) sex[n_l] = e_l;
  __syncthreads();

  for (;;) {
    // (c)+(d): explore, edge e -> vertex u by binary search of the smem degree scan
    int ncand = 0;
    for (int e = tid; e < e_l; e += KS_THREADS) {
      int lo = 0, hi = n_l;
      while (hi - lo > 1) {
        const int mid = (lo + hi) >> 1;
        if (sex[mid] <= e) lo = mid; else hi = mid;
      }
      const int x = sf[lo];
      const int v = __ldg(col + srs[lo] + (e - sex[lo]));
      int w = -1;
      if (ld_weak(level + v) == -1) {
        st_weak(level + v, L + 1);
        st_weak(parent + v, x);
        st_weak(owner + v, e);
        w = v;
        ++ncand;
      }
      cv[e] = w;
    }
    __syncthreads();
    // (e): owner check + next-level degree, blocked items for the scan
    const int ipt = (e_l + KS_THREADS - 1) / KS_THREADS;
    const int e0 = tid * ipt;
    int kv[KS_IPT], kr[KS_IPT], kd[KS_IPT];
    int cnt = 0, dsum = 0;
#pragma unroll
    for (int i = 0; i < KS_IPT; ++i) {
      kv[i] = -1;
      kr[i] = 0;
      kd[i] = 0;
      const int e = e0 + i;
      if (i < ipt && e < e_l) {
        const int v = cv[e];
        if (v >= 0) {
          const int ow = ld_weak(owner + v);
          const int r0 = __ldg(ro + v), r1 = __ldg(ro + v + 1);
          if (ow == e) { kv[i] = v; kr[i] = r0; kd[i] = r1 - r0; }
        }
      }
    }
#pragma unroll
    for (int i = 0; i < KS_IPT; ++i) {
      cnt += kv[i] >= 0;
      dsum += kd[i];
    }
    // block exclusive scan of (cnt, dsum)
    const int ik = warp_incl_scan(cnt), id = warp_incl_scan(dsum);
    const int wc = P.collect_stats ? warp_sum(ncand) : 0;
    if (lane == 31) { s_wk[warp] = ik; s_wd[warp] = id; }
    if (lane == 0) s_wc[warp] = wc;
    __syncthreads();
    if (warp == 0) {
      const int a = s_wk[lane], d = s_wd[lane];
      const int ia = warp_incl_scan(a), idd = warp_incl_scan(d);
      const int ctot = warp_sum(s_wc[lane]);
      s_wk[lane] = ia - a;
      s_wd[lane] = idd - d;
      if (lane == 31) { s_tot[0] = ia; s_tot[1] = idd; s_tot[2] = ctot; }
    }
    __syncthreads();
    int kpos = s_wk[warp] + ik - cnt, dpos = s_wd[warp] + id - dsum;
    const int n_next = s_tot[0], e_next = s_tot[1];
#pragma unroll
    for (int i = 0; i < KS_IPT; ++i) {
      if (kv[i] >= 0) {
        // visited bit: plain read-modify-write, no atomic -- a racing update can only lose a
        // bit (the filter then falls back to level[]), never set one wrongly
        uint32_t *wp = P.bm + (kv[i] >> 5);
        *(volatile uint32_t *)wp = *(volatile uint32_t *)wp | (1u << (kv[i] & 31));
        sf[kpos] = kv[i];
        srs[kpos] = kr[i];
        sex[kpos] = dpos;
        ++kpos;
        dpos += kd[i];
      }
    }
    if (tid == 0) {
      sex[n_next] = e_next;
      const unsigned long long t = globaltimer();
      record_stat(P, c, L, n_l, e_l, TIER_SMALL, 1, s_tot[2], n_next, t_prev, t);
      t_prev = t;
    }
    __syncthreads();
    ++L;
    n_l = n_next;
    e_l = e_next;
    if (n_l == 0 || e_l == 0 || P.t0 < 0 || e_l > P.t0 || n_l > KS_NCAP) break;
  }
  // leave tier 0: spill the frontier (if any work remains) and hand over the control block
  if (n_l > 0 && e_l > 0) {
    for (int i = tid; i < n_l; i += KS_THREADS) {
      P.f[cur][i] = sf[i];
      P.frs[cur][i] = srs[i];
      P.fex[cur][i] = sex[i];
    }
    if (tid == 0) P.fex[cur][n_l] = e_l;
  }
  if (tid == 0) {
    c->level = L;
    c->t_prev = t_prev;
    decide(P, c, n_l, e_l);
  }
}

// ---- test entry kernels ---------------------------------------------------------------------
// (b) alone: tiles of SCAN_TILE int32 in blocked order, block scan + decoupled look-back.
__global__ void __launch_bounds__(SCAN_THREADS) k_scan_u32(const int32_t *__restrict__ in,
                                                           int32_t *__restrict__ out, int n,
                                                           unsigned long long *status) {
  __shared__ int32_t s_w[SCAN_THREADS / 32];
  __shared__ uint32_t s_ex;
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const long long base = (long long)blockIdx.x * SCAN_TILE + (long long)tid * SCAN_ITEMS;
  int x[SCAN_ITEMS];
  int sum = 0;
#pragma unroll
  for (int i = 0; i < SCAN_ITEMS; ++i) {
    x[i] = (base + i < n) ? __ldg(in + base + i) : 0;
    sum += x[i];
  }
  const int inc = warp_incl_scan(sum);
  if (lane == 31) s_w[warp] = inc;
  __syncthreads();
  if (warp == 0) {
    const int a = lane < SCAN_THREADS / 32 ? s_w[lane] : 0;
    const int ia = warp_incl_scan(a);
    if (lane < SCAN_THREADS / 32) s_w[lane] = ia - a;
    const Pair agg{(uint32_t)__shfl_sync(0xffffffffu, ia, 31), 0};
    const Pair ex = lookback<false>(status, blockIdx.x, agg);
    if (lane == 0) s_ex = ex.a;
    if (lane == 0 && blockIdx.x == gridDim.x - 1) out[n] = (int)(ex.a + agg.a);
  }
  __syncthreads();
  int run = (int)(s_ex + (uint32_t)s_w[warp] + (uint32_t)(inc - sum));
#pragma unroll
  for (int i = 0; i < SCAN_ITEMS; ++i) {
    if (base + i < n) out[base + i] = run;
    run += x[i];
  }
}

// (c) alone: worker w (one warp each) finds its start vertex and offset by warp_search.
__global__ void k_find_start(const int32_t *__restrict__ excl, int n_l, int chunk, int p_l,
                             int32_t *out_u, int32_t *out_off) {
  const int w = (blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  if (w >= p_l) return;
  const int lane = threadIdx.x & 31;
  const int e_l = __ldg(excl + n_l);
  const long long s = (long long)w * chunk;
  if (s >= e_l) {
    if (lane == 0) { out_u[w] = -1; out_off[w] = -1; }
    return;
  }
  const int u = warp_search(excl, n_l, (int)s);
  if (lane == 0) { out_u[w] = u; out_off[w] = (int)(s - __ldg(excl + u)); }
}

// create-time CSR validation: err bit 1 row_offsets[0] != 0, 2 decreasing,
// 4 row_offsets[n] != nnz, 8 a column out of range.
__global__ void k_validate(const int32_t *ro, const int32_t *col, int n, long long nnz,
                           int *err) {
  const long long gs = (long long)gridDim.x * blockDim.x;
  const long long g = (long long)blockIdx.x * blockDim.x + threadIdx.x;
  if (g == 0) {
    if (ro[0] != 0) atomicOr(err, 1);
    if ((long long)ro[n] != nnz) atomicOr(err, 4);
  }
  for (long long i = g; i < n; i += gs)
    if (ro[i] > ro[i + 1]) atomicOr(err, 2);
  for (long long i = g; i < nnz; i += gs)
    if (col[i] < 0 || col[i] >= n) atomicOr(err, 8);
}

// debug: fill Owner with values that look like live candidate slots (R3 pin).
__global__ void k_poison(int32_t *owner, int n, int range) {
  const long long gs = (long long)gridDim.x * blockDim.x;
  for (long long i = (long long)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += gs)
    owner[i] = (int32_t)(((unsigned)i * 2654435761u) % (unsigned)max(range, 1));
}

}  // namespace s3bfs
