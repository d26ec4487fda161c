// paper_2209_08764_b200/csrc/s3bfs_kernels.cuh -- sm_100a kernels of the S3BFS hot path.
//
// "P:n" = /root/reference/PAPER.md line n; "Fig1 Lk" = item k of Figure 1;
// "R<k>" = reading k in DESIGN.md.  This file shares nothing with oracle/ (test-only code).
//
// Vertex ids.  s3bfs_create builds an internal copy of the graph whose vertices are relabelled
// by descending degree (DESIGN.md s.7): the hottest vertices get the smallest internal ids, so
// their visited bits share a few L1-resident lines of the bitmap.  Every traversal kernel works
// in internal ids; k_finalize writes the caller's level[]/parent[] in caller ids at the end.
// With reordering off (opts.reorder < 0) n2o/o2n are NULL and the two id spaces coincide.
//
// Kernels (one level = one pass of (a)-(e)):
//   k_init     Fig1 L1-L8   visited bitmap <- {s}, claim tags <- 0, frontier = [s], d[s] = 0
//   k_explore  (c)+(d)      Fig1 L17-L18: equal edge slices per warp, start vertex by a
//                           32-ary warp search of the degree scan (R8), coalesced col stream,
//                           visited test (bitmap, then a per-level claim tag at a hashed
//                           slot, R26), d/parent/Owner
//                           labelling with plain stores -- the benign race, no atomic
//                           instruction.
//   k_compact  (e)+(a)+(b)  Fig1 L19-L29 + L12-L15 of the NEXT level: keep cand[k] iff
//                           Owner[cand[k]] == k, decoupled look-back scan of (kept, degree-sum)
//                           pairs across CTAs, write f_next / row starts / degree scan.
//   k_small    tier 0 (f)   one CTA runs whole levels (a)-(e) in shared memory while the level
//                           stays tiny (P:22 -- "never use more cores than necessary");
//                           its warp 0 alone runs levels of <= 32 edges (tiny_levels).
//   k_cluster  (f) middle   one 8-CTA thread-block cluster runs consecutive mid-size levels,
//                           frontier replicated through distributed shared memory.
//   k_fb_clear/k_fb_set/k_bottom_up   NEXT-3 bottom-up levels (direction-optimising option).
//   k_dist_init/k_dist_keep/k_dist_advance/k_dist_finalize   NEXT-4: one traversal over G ranks
//                           (1-D vertex partition; k_explore<true> routes candidates to owners).
//   k_finalize              d[0:n-1] and parent in caller ids ("Returns d[0:n-1]").
//   k_scan_u32 (b) alone    test entry: the same look-back scan over a plain int32 array.
//   k_find_start (c) alone  test entry: the same warp search, one warp per worker.
#pragma once
#include <cuda_runtime.h>
#include <cooperative_groups.h>
#include <stdint.h>

#include <type_traits>

#include "../../include/s3bfs.h"

namespace s3bfs {

// Bounds-checked build (S3BFS_CHECK=1, tests/check_suite.py): compute-sanitizer is not
// available on the GPU pool, so every index the traversal kernels derive from data (frontier
// slots, col positions, vertex ids, bitmap words, claim slots, candidate slots, shared-memory
// slots) is checked against its buffer; a violation prints the site and traps.
#if S3BFS_CHECK
#define S3_CHK(i, lim) do { if (!((long long)(i) >= 0 && (long long)(i) < (long long)(lim))) { \
    printf("S3BFS_CHECK %s:%d: %s = %lld not in [0, %lld)\n", __FILE__, __LINE__, #i,      \
           (long long)(i), (long long)(lim)); __trap(); } } while (0)
#else
#define S3_CHK(i, lim) ((void)0)
#endif

// ---- compile-time geometry (the -D switches exist for scripts/kx_micro.py experiments) -----
#ifndef S3BFS_KD_THREADS
#define S3BFS_KD_THREADS 1024
#endif
#ifndef S3BFS_KD_MINB
#define S3BFS_KD_MINB (1024 / S3BFS_KD_THREADS)
#endif
#ifndef S3BFS_KX_GROUPS
#define S3BFS_KX_GROUPS 8
#endif
#ifndef S3BFS_KS_SCAN1
#define S3BFS_KS_SCAN1 1  // k_small: one-barrier block scan (0: warp-0 scan + 2nd barrier)
#endif
#ifndef S3BFS_KC_FENCE
#define S3BFS_KC_FENCE 0  // k_cluster: extra __threadfence before the owner-check barrier
#endif
#ifndef S3BFS_KC_PUSH
#define S3BFS_KC_PUSH 1  // k_cluster: CTA totals pushed into every CTA's table (0: 8 DSMEM reads)
#endif
#ifndef S3BFS_KX_FAST
#define S3BFS_KX_FAST 1   // uniform-row fast path
#endif
#ifndef S3BFS_KX_RANK
#define S3BFS_KX_RANK 1   // rank (REDUX + POPC) edge->row mapping for multi-row batches
#endif
#ifndef S3BFS_KX_VEC
#define S3BFS_KX_VEC 1    // 16-byte col loads in the uniform-row fast path
#endif
#ifndef S3BFS_CLAIM_SCATTER
#define S3BFS_CLAIM_SCATTER 1  // claim tag of v at a multiplicative-hash slot (see claim_slot)
#endif
#ifndef S3BFS_BM_AGG
#define S3BFS_BM_AGG 1  // k_compact: one atomicOr per run of same-word kept candidates
#endif
#ifndef S3BFS_COL_HINT
#define S3BFS_COL_HINT 1  // col loads carry the L2 evict-first policy
#endif
#ifndef S3BFS_T0_WITH_CLUSTER
#define S3BFS_T0_WITH_CLUSTER 2048  // default T0 when the cluster tier is on (measured crossover)
#endif
#ifndef S3BFS_CLAIM_MIN_BYTES
#define S3BFS_CLAIM_MIN_BYTES (8u << 20)  // claim array floor (measured, DESIGN R26)
#endif
#ifndef S3BFS_TAG_MODE_PCT
#define S3BFS_TAG_MODE_PCT 80  // default of opts.tag_mode_pct
#endif
#ifndef S3BFS_KX_QUEUE
#define S3BFS_KX_QUEUE 1  // k_explore: claim checks + discoveries via a warp-private queue
#endif
#ifndef S3BFS_KX_TAG2
#define S3BFS_KX_TAG2 1   // k_explore tag mode: hub rechecks as a second in-batch probe round
#endif
#ifndef S3BFS_KX_TAG2_MIN_WCAP
#define S3BFS_KX_TAG2_MIN_WCAP 8192  // ... on levels with at least this many edges per warp
#endif
#ifndef S3BFS_KC_REVERSE
#define S3BFS_KC_REVERSE 1  // k_compact walks every candidate segment newest entry first
#endif
#ifndef S3BFS_SPLIT_MIN_EDGES
#define S3BFS_SPLIT_MIN_EDGES (32 << 20)  // level passes: default of opts.split_min_edges
#endif
#ifndef S3BFS_SPLIT_FIRST_PCT
#define S3BFS_SPLIT_FIRST_PCT 6           // default of opts.split_first_pct
#endif
#ifndef S3BFS_SPLIT_PASSES
#define S3BFS_SPLIT_PASSES 2              // default of opts.split_passes
#endif
#ifndef S3BFS_KX_TRANSPOSE
#define S3BFS_KX_TRANSPOSE 1  // k_explore: a CTA's warps take slices spread over the whole range
#endif
#ifndef S3BFS_KX_PIECES
#define S3BFS_KX_PIECES 4  // k_explore: pieces per worker's share (with S3BFS_KX_TRANSPOSE)
#endif
#ifndef S3BFS_KX_PIECES_MIN_EDGES
#define S3BFS_KX_PIECES_MIN_EDGES 4096  // ... on shares of at least this many edges
#endif
#ifndef S3BFS_KS_ONCHIP
#define S3BFS_KS_ONCHIP 1  // k_small: Owner race in a shared-memory table (no L2 round trip)
#endif
#ifndef S3BFS_LB_WIDE
#define S3BFS_LB_WIDE 1  // k_compact: CTA-wide one-round-trip prefix over all predecessors
#endif
#ifndef S3BFS_CHECK
#define S3BFS_CHECK 0  // 1: bounds-checked build (every traversal index checked; trap + message)
#endif
#ifndef S3BFS_BU_W
#define S3BFS_BU_W 4
#endif
#ifndef S3BFS_BU_P
#define S3BFS_BU_P 2
#endif
#ifndef S3BFS_KC_GROUPS
#define S3BFS_KC_GROUPS 4
#endif
#ifndef S3BFS_BU_TILES_PER_CTA
#define S3BFS_BU_TILES_PER_CTA 4  // bottom-up: about this many tiles per resident CTA
#endif
#ifndef S3BFS_LB_MAX_NS
#define S3BFS_LB_MAX_NS 128  // look-back backoff cap (ns; 1024 measured 0.2-0.6 % slower)
#endif
#ifndef S3BFS_BM_NC
#define S3BFS_BM_NC 1     // bitmap probes through the non-coherent (read-only) path
#endif
constexpr int KD_THREADS = S3BFS_KD_THREADS;    // k_explore / k_compact CTA size
constexpr int KD_MIN_BLOCKS = S3BFS_KD_MINB;    // CTAs per SM the register budget targets
constexpr int KD_WARPS = KD_THREADS / 32;
constexpr int KD_SLACK = 64;                    // candidate-buffer slack per CTA
constexpr int KX_GROUPS = S3BFS_KX_GROUPS;      // 32-edge groups per batch and warp
constexpr int KC_GROUPS = S3BFS_KC_GROUPS;      // 32-candidate groups per k_compact round
constexpr int DIST_MAX = 8;                     // NEXT-4: ranks per traversal (one node)
#ifndef S3BFS_KQ_GROUPS
#define S3BFS_KQ_GROUPS 2  // k_explore queue: flush check after this many groups
#endif
constexpr int KQ_CAP = 32 + S3BFS_KQ_GROUPS * 32;  // k_explore warp queue (< 32 kept + groups)
#ifndef S3BFS_KS_THREADS
#define S3BFS_KS_THREADS 1024
#endif
constexpr int KS_THREADS = S3BFS_KS_THREADS;    // k_small CTA size (<= 1024, a multiple of 32)
constexpr int KS_ECAP = S3BFS_KS_ONCHIP ? 4096 : 8192;  // T0 maximum (edges per tier-0 level)
constexpr int KS_TAB_BITS = 14;                 // k_small on-chip Owner table: 2^14 entries
constexpr int KS_TAB = 1 << KS_TAB_BITS;
static_assert(KS_ECAP <= KS_TAB, "k_small Owner-table entries hold a level-local edge index");
constexpr int KS_NCAP = KS_ECAP;                // frontier capacity of tier 0 (kept <= e_l)
constexpr int KS_IPT = KS_ECAP / KS_THREADS;    // dedup items per thread
constexpr int SCAN_THREADS = 512;
constexpr int SCAN_ITEMS = 8;
constexpr int SCAN_TILE = SCAN_THREADS * SCAN_ITEMS;

constexpr int TIER_SMALL = 0, TIER_LARGE = 1, TIER_DONE = 2, TIER_BU = 3, TIER_CLUSTER = 4;
// cluster tier (f, SURVEY 8(a) "optional middle tier"): one cluster of KC_CL CTAs
constexpr int KC_CL = 8;                         // CTAs per cluster (portable size)
constexpr int KC_THREADS = 1024;
constexpr int KC_ECTA = 4096;                    // level edges per CTA (e_l <= 32,768)
constexpr int KC_FCAP = 8192;                    // replicated frontier capacity
constexpr int KC_IPT = KC_ECTA / KC_THREADS;
// k_small / k_cluster scan their per-warp totals with warp 0 reading one entry per lane
static_assert(KC_THREADS == 1024, "cluster CTAs must have 32 warps (warp totals: one per lane)");
static_assert(KS_THREADS % 32 == 0 && KS_THREADS <= 1024, "k_small: whole warps, <= 32");
static_assert(KX_GROUPS % 4 == 0, "k_explore packs 4 window slots per register");
constexpr int BU_W = S3BFS_BU_W;   // bottom-up: bitmap words per warp round
constexpr int BU_P = S3BFS_BU_P;   // bottom-up: in-neighbours probed per vertex per round

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
  int32_t wcap;       // edges (= candidate capacity) per warp
  int32_t e_lo, e_hi; // the edge range [e_lo, e_hi) of the level this pass explores: the
                      // whole level, or one of its passes (see plan_pass)
  int32_t pieces;     // pieces per worker's share of the pass (k_explore)
  int32_t pass;       // passes of the current level already done
  int32_t n_acc, e_acc;  // next frontier entries / degree sum the level's earlier passes wrote
  unsigned long long t_kx_first, kx_ns;  // stats: first pass's k_explore start, summed k_explore ns
  int32_t g_n_next, g_e_next;  // NEXT-4: the next level's frontier size / edges over all ranks
  int32_t n_next, e_next;   // written by the last k_compact CTA in tile order
  uint32_t done_ctr;        // last-CTA election in k_compact (not the discovery path)
  uint32_t tile_ctr;        // look-back tile ids in start order (forward progress under any
                            // CTA dispatch order, e.g. concurrent traversals; not discovery)
  int32_t num_levels;       // stats records written
  int32_t cand_acc;         // stats: candidates of the level (incl. duplicates)
  int32_t source;
  int32_t bu;               // NEXT-3: the current level runs bottom-up
  int32_t fb_valid;         // fb[cur] already holds the current frontier (a bottom-up product)
  int32_t probe_tags;       // k_explore's visited test of this level: tag mode (1) or bitmap
                            // mode (0), see k_explore; set by decide_tier
  long long m_visited;      // sum of the degrees of all visited vertices (Beamer's m_u = m - it)
  int32_t *level_out, *parent_out;
  unsigned long long t_prev;
  unsigned long long t_kx_begin, t_kx_end;  // k_explore CTA 0 start, k_compact CTA 0 start
  unsigned long long t_dbg[4];  // first-level timeline: init start, dispatch, k_small start/end
};

struct Params {
  const int32_t *col;           // internal adjacency (degree-ordered copy, or the caller's)
  int4 *vinfo;                  // vertex records, 32 B (one sector) per internal vertex v:
                                //  vinfo[2v]   = {row start, degree, caller id, 0} (static)
                                //  vinfo[2v+1] = {d, parent (caller id), Owner, 0}: d/parent
                                //  valid where the visited bit is set; Owner (Fig1 L3) never
                                //  initialised (R3).  A discovery is ONE 16-byte store into
                                //  the sector k_compact's Owner check reads (see vdyn)
  const int4 *vs16;             // dense copy of the records' static halves, 16 B per vertex
                                //  ({row start, degree, caller id, 0}, read-only): the small
                                //  tiers and the bottom-up step read it -- frontiers of
                                //  near-consecutive ids (paths, grid diagonals, the bottom-up
                                //  sweep over id order) share its sectors
  const int32_t *n2o, *o2n;     // internal -> caller ids and back (NULL: identity)
  int32_t n;
  Ctl *ctl;
  int32_t *f[2], *frs[2], *fex[2];  // frontier: caller ids (parents of the next level's
                                    // discoveries), internal row starts, degree scan
  int32_t *cand;                // candidate per slot (k_explore), compacted by k_compact
  int2 *cand_rd;                // (row start, degree) of kept candidates, pass 1 -> pass 2
  uint32_t *bm;                 // visited bitmap: bit set => visited (exact at level start),
                                //  plus one always-set 16 B sentinel block after the padded end
  unsigned long long pol_first, pol_last;  // L2 createpolicy descriptors (evict-first for the
                                //  col stream, evict-last for the bitmap), made once at create:
                                //  as kernel parameters they are uniform (no per-load R2UR)
  int32_t v_sent;               // sentinel vertex id (first bit of that block): k_explore's
                                //  masked lanes probe it and need no validity test
  uint8_t *claim;               // per-vertex discovery tag: nonzero once v was discovered (in
                                //  any level, by any kernel), at slot claim_slot(v) (scattered)
  uint32_t claim_mask;          // claim array size - 1 (a power of two >= n)
  int32_t hub;                  // k_explore tag mode: ids < hub are tested in the bitmap
                                //  first, the others by their discovery tag alone (one probe)
  int32_t tag_pct;              // tag mode while m_visited < tag_pct % of nnz (< 0: never)
  int32_t split_min, split_pct, split_passes;  // level passes (plan_pass): levels of at least
                                //  split_min edges in tag mode run in up to split_passes passes,
                                //  the first over split_pct % of the level's edges (<= 0: off)
  uint32_t *fb[2];              // NEXT-3: frontier bitmaps (bottom-up levels only)
  int2 *lpd;                    // NEXT-3: {d, parent} of the vertices a bottom-up level found,
  uint32_t *bub;                //  dense (8 B per id), and the bitmap of those vertices: the
                                //  sweep owns 32 consecutive ids per warp, so its labels
                                //  coalesce here (into the 32-byte records they are 32 partial
                                //  sectors); k_finalize reads them where bub's bit is set
                                //  (NULL without direction optimisation)
  const int32_t *tro, *tcol;    // NEXT-3: in-adjacency (internal ids) the bottom-up step scans
  int32_t *wcnt;
  unsigned long long *status;
  s3bfs_level_stat *stats;
  int32_t stats_cap;
  int32_t p_max, grain, t0, variant, collect_stats;
  int32_t tc_max;               // cluster tier: levels with t0 < e_l <= tc_max (< 0: off)
  int32_t direction, do_alpha, do_beta;  // NEXT-3 switch rule (Beamer): alpha, beta
  int32_t n_scan;               // bottom-up scans internal ids [0, n_scan): the ones with deg > 0
  unsigned long long *bu_status;  // NEXT-3: look-back words of the bottom-up tiles
  int32_t bu_tiles, bu_tile_w;  // NEXT-3: bottom-up tiles and their width (bitmap words)
  // NEXT-4, 1-D vertex partition over G = dist_size ranks: internal id v is
  // owned by rank (v / 32) mod G (block-cyclic 32-id blocks: one visited-bitmap word per owner,
  // hubs spread over the ranks); its local slot is (v / 32 / G) * 32 + v mod 32.  vinfo / lp /
  // the frontier / col are the rank's own (local slots, local CSR rows); bm and claim stay
  // over global ids (the bitmap is replicated: every owner publishes its words to its peers).
  int32_t dist_size, dist_rank; // 1, 0 on a single GPU
  int32_t nloc;                 // local vertex slots of this rank
  int2 *recv;                   // this rank's receive segments {v, parent}: source s's block
                                //  at rofs[s], its warp g's segment at rofs[s] + g * wcap_s
  int32_t *rcnt;                // per (source rank, source warp): candidates in that segment
  int2 *rmeta;                  // per source rank: {wcap, p_l} of the level
  int2 *rtot;                   // per source rank: {n_next, e_next} of the level
  int32_t rofs[DIST_MAX + 1];   // receive block offsets (identical on every rank)
  int2 *p_recv[DIST_MAX];       // peers' (and this rank's) arrays, mapped into this process
  int32_t *p_rcnt[DIST_MAX];
  int2 *p_rmeta[DIST_MAX];
  int2 *p_rtot[DIST_MAX];
  uint32_t *p_bm[DIST_MAX];
  int4 *p_vinfo[DIST_MAX];      // peers' vertex records (the sender stores the Owner label)
  long long nnz;
  long long cand_cap;           // candidate buffer entries (bounds-checked build)
  long long nnz_all;            // arcs of the whole graph (= nnz on one GPU; NEXT-4: all ranks')
  int32_t col_vec;              // col is 16-byte aligned: vectorised loads allowed
  int32_t use_graph;
  unsigned long long h_while, h_tier;  // cudaGraphConditionalHandle values (WHILE; SWITCH on
                                       // the tier: body 0 tier 0, 1 top-down, 2 bottom-up)
};

// ---- PTX helpers ------------------------------------------------------------------------
__device__ __forceinline__ unsigned long long globaltimer() {
  unsigned long long t;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
  return t;
}
// L2 eviction policies (createpolicy): the adjacency is streamed once per level and must not
// evict the visited bitmap / claim tags, which every arc probes at random.
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
// read-only stream (col_indices): non-coherent, L1-allocating (neighbouring 32-edge groups of
// one warp share a boundary line), L2 evict-first
__device__ __forceinline__ int ldg_stream(const int32_t *p, unsigned long long pol) {
  int v;
#if S3BFS_COL_HINT
  asm("ld.global.nc.L2::cache_hint.s32 %0, [%1], %2;" : "=r"(v) : "l"(p), "l"(pol));
#else
  v = __ldg(p);
#endif
  return v;
}
__device__ __forceinline__ int4 ldg_stream4(const int32_t *p, unsigned long long pol) {
  int4 v;
#if S3BFS_COL_HINT
  asm("ld.global.nc.L2::cache_hint.v4.s32 {%0, %1, %2, %3}, [%4], %5;"
               : "=r"(v.x), "=r"(v.y), "=r"(v.z), "=r"(v.w) : "l"(p), "l"(pol));
#else
  v = __ldg(reinterpret_cast<const int4 *>(p));
#endif
  return v;
}
// 1 << k for 0 <= k < 32, else 0 (PTX shl clamps shift amounts >= 32; k < 0 is a huge
// unsigned amount)
__device__ __forceinline__ unsigned shl1(int k) {
  unsigned r;
  asm("shl.b32 %0, 1, %1;" : "=r"(r) : "r"(k));
  return r;
}
// rotate right by (k mod 32): bit 0 of the result is bit (k mod 32) of w (one SHF.WRAP)
__device__ __forceinline__ uint32_t rotr32(uint32_t w, int k) {
  uint32_t r;
  asm("shf.r.wrap.b32 %0, %1, %1, %2;" : "=r"(r) : "r"(w), "r"(k));
  return r;
}
// the visited bitmap inside k_explore: read-only there (written by earlier kernels only); the
// hot vertices' words stay L1-resident thanks to the degree order
__device__ __forceinline__ uint32_t ldg_status_u32(const uint32_t *p, unsigned long long pol) {
  uint32_t v;
  asm("ld.global.nc.L2::cache_hint.u32 %0, [%1], %2;" : "=r"(v) : "l"(p), "l"(pol));
  return v;
}
__device__ __forceinline__ uint32_t ld_status_u32(const uint32_t *p, unsigned long long pol) {
  uint32_t v;
  asm volatile("ld.global.L2::cache_hint.u32 %0, [%1], %2;" : "=r"(v) : "l"(p), "l"(pol));
  return v;
}
// Claim tag slot of internal vertex v: (v * golden) mod 2^k, a bijection on [0, 2^k).  The
// degree-ordered relabel packs the targets a discovery-heavy level hits hardest into a narrow
// id band; with claim[v] at slot v, every SM's probe and store of that band lands on a few
// L2 lines (measured: R-MAT 20's discovery level 317 us relabelled vs 123 us unrelabelled).
// Scattering the tags spreads them over all L2 lines/slices; the bitmap keeps the relabel's
// locality (the heavy level's hub bits stay in few, L1-resident words).
__device__ __forceinline__ uint32_t claim_slot(const Params &P, int v) {
  return S3BFS_CLAIM_SCATTER ? ((uint32_t)v * 0x9E3779B1u) & P.claim_mask : (uint32_t)v;
}
// claim tags: L2-coherent byte loads/stores (no stale L1 line hides another SM's claim)
__device__ __forceinline__ int ld_cg_u8(const uint8_t *p) {
  unsigned v;
  asm volatile("ld.global.cg.u8 %0, [%1];" : "=r"(v) : "l"(p));
  return (int)v;
}
// k_explore's one probe per arc (Fig1 L18 "if d[v] = infinity"): a hub id (or the sentinel)
// reads its visited-bitmap word through the read-only path (L1-resident for the hottest ids),
// any other id reads its discovery tag at L2 (evict-last: the tags must outlive the col
// stream).  The caller decodes: a bit of the word, or tag == 0 ("not discovered yet").
__device__ __forceinline__ int ld_cg_u8_hint(const uint8_t *p, unsigned long long pol) {
  unsigned v;
  asm volatile("ld.global.cg.L2::cache_hint.u8 %0, [%1], %2;" : "=r"(v) : "l"(p), "l"(pol));
  return (int)v;
}
__device__ __forceinline__ void st_u8(uint8_t *p, int v) {
  asm volatile("st.global.u8 [%0], %1;" ::"l"(p), "r"(v) : "memory");
}
// a vertex kept by a kernel other than k_explore (tier 0, cluster tier, bottom-up, NEXT-4
// merge) gets its discovery tag too: k_explore tests non-hub ids by the tag alone
__device__ __forceinline__ void mark_tag(const Params &P, int v) {
  st_u8(P.claim + claim_slot(P, v), 1);
}
__device__ __forceinline__ void st_weak(int32_t *p, int v) {
  asm volatile("st.global.s32 [%0], %1;" ::"l"(p), "r"(v) : "memory");
}
__device__ __forceinline__ void st_weak_v2(int2 *p, int a, int b) {
  asm volatile("st.global.v2.s32 [%0], {%1, %2};" ::"l"(p), "r"(a), "r"(b) : "memory");
}
__device__ __forceinline__ int4 ld_weak_v4(const int4 *p) {
  int4 r;
  asm volatile("ld.global.v4.s32 {%0, %1, %2, %3}, [%4];"
               : "=r"(r.x), "=r"(r.y), "=r"(r.z), "=r"(r.w) : "l"(p));
  return r;
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
// vertex record accessors (layout: Params::vinfo)
__device__ __forceinline__ const int4 *vstat(const int4 *vinfo, int v) {
  return vinfo + 2 * (long long)v;
}
__device__ __forceinline__ int4 *vdyn(int4 *vinfo, int v) { return vinfo + 2 * (long long)v + 1; }
__device__ __forceinline__ int2 *lp_of(int4 *vinfo, int v) {
  return reinterpret_cast<int2 *>(vdyn(vinfo, v));
}
__device__ __forceinline__ int32_t *owner_of(int4 *vinfo, int v) {
  return reinterpret_cast<int32_t *>(vdyn(vinfo, v)) + 2;
}
// {row start, degree, caller id, Owner} of v: the static half plus the Owner word of the
// dynamic half -- both in v's one sector (nc: a kernel that does not write the records;
// cg: L2-coherent; weak: plain loads, the same SM wrote the Owner)
__device__ __forceinline__ int4 ld_vrec_nc(const int4 *vinfo, int v) {
  int4 r = __ldg(vstat(vinfo, v));
  r.w = __ldg(reinterpret_cast<const int32_t *>(vstat(vinfo, v)) + 6);
  return r;
}
// the same through one 256-bit load (k_compact: one request per candidate)
__device__ __forceinline__ int4 ld_vrec256_nc(const int4 *vinfo, int v) {
  int4 r;
  int d0, d1, d2, d3;
  asm("ld.global.nc.v8.s32 {%0, %1, %2, %3, %4, %5, %6, %7}, [%8];"
      : "=r"(r.x), "=r"(r.y), "=r"(r.z), "=r"(d0), "=r"(d1), "=r"(d2), "=r"(r.w), "=r"(d3)
      : "l"(vstat(vinfo, v)));
  return r;
}
__device__ __forceinline__ int4 ld_vrec_cg(const int4 *vs16, const int4 *vinfo, int v) {
  int4 r = __ldcg(vs16 + v);  // static half from the dense copy
  r.w = __ldcg(reinterpret_cast<const int32_t *>(vstat(vinfo, v)) + 6);
  return r;
}
__device__ __forceinline__ int4 ld_vrec_weak(const int4 *vinfo, int v) {
  int4 r;
  asm volatile("ld.global.v4.s32 {%0, %1, %2, %3}, [%4];"
               : "=r"(r.x), "=r"(r.y), "=r"(r.z), "=r"(r.w) : "l"(vstat(vinfo, v)));
  asm volatile("ld.global.s32 %0, [%1];"
               : "=r"(r.w) : "l"(reinterpret_cast<const int32_t *>(vstat(vinfo, v)) + 6));
  return r;
}
// EXPLORE-VERTEX's labelling (Fig1 L18, L22) in one plain 16-byte store: {d, parent, Owner}
__device__ __forceinline__ void st_discovery(int4 *vinfo, int v, int d, int parent, int owner) {
  asm volatile("st.global.v4.s32 [%0], {%1, %2, %3, %4};" ::"l"(vdyn(vinfo, v)), "r"(d),
               "r"(parent), "r"(owner), "r"(0) : "memory");
}

// k_small's on-chip Owner table: round r's bijection of the 32-bit ids (odd multiplies,
// xor-shifts and an added constant are each invertible)
__device__ __forceinline__ uint32_t ks_hash(uint32_t v, int r) {
  uint32_t x = v * 0x9E3779B1u + (uint32_t)r * 0x7F4A7C15u;
  x ^= x >> 16;
  x *= 0x85EBCA6Bu;
  x ^= x >> 13;
  return x;
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
      if (ns < S3BFS_LB_MAX_NS) ns <<= 1;
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
// Tier 0 keeps the record counter in a register across its levels (a global read-after-write
// of num_levels per level sat on the critical path of every one-vertex level).
__device__ __forceinline__ void record_stat_at(const Params &P, int &k, int32_t level, int32_t n_l,
                                               int32_t e_l, int32_t tier, int32_t cand,
                                               int32_t kept, unsigned long long t0,
                                               unsigned long long t1) {
  if (!P.collect_stats) return;
  if (k < P.stats_cap) {
    s3bfs_level_stat r;
    r.level = level; r.n_l = n_l; r.e_l = e_l; r.tier = tier;
    r.grid = tier == TIER_CLUSTER ? KC_CL : 1;
    r.candidates = cand; r.kept = kept; r.pad = 0; r.t_begin_ns = t0; r.t_end_ns = t1;
    r.t_explore_begin_ns = 0; r.t_explore_end_ns = 0;
    P.stats[k] = r;
  }
  ++k;
}
__device__ void record_stat(const Params &P, Ctl *c, int32_t level, int32_t n_l, int32_t e_l,
                            int32_t tier, int32_t grid, int32_t cand, int32_t kept,
                            unsigned long long t0, unsigned long long t1,
                            unsigned long long tx0 = 0, unsigned long long tx1 = 0,
                            int32_t passes = 0) {
  if (!P.collect_stats) return;
  const int k = c->num_levels;
  if (k < P.stats_cap) {
    s3bfs_level_stat r;
    r.level = level; r.n_l = n_l; r.e_l = e_l; r.tier = tier; r.grid = grid;
    r.candidates = cand; r.kept = kept; r.pad = passes; r.t_begin_ns = t0; r.t_end_ns = t1;
    r.t_explore_begin_ns = tx0; r.t_explore_end_ns = tx1;
    P.stats[k] = r;
  }
  c->num_levels = k + 1;
}

// Graph mode: the thread that decides the next level's tier also steers the captured loop --
// WHILE (more levels) and one SWITCH node inside a WHILE iteration that runs the tier's body
// (tier 0 / top-down / bottom-up; one conditional evaluation per level).  No dispatch kernel.
__device__ void steer(const Params &P, int tier) {
  if (!P.use_graph) return;
  const unsigned body = tier == TIER_SMALL ? 0u : tier == TIER_LARGE ? 1u : tier == TIER_BU ? 2u
                      : tier == TIER_CLUSTER ? 3u : 7u;
  cudaGraphSetConditional((cudaGraphConditionalHandle)P.h_tier, body);
  cudaGraphSetConditional((cudaGraphConditionalHandle)P.h_while, tier != TIER_DONE ? 1u : 0u);
}

__device__ void decide_tier(const Params &P, Ctl *c, int32_t n_l, int32_t e_l);
__device__ void plan_pass(const Params &P, Ctl *c);
__device__ void decide(const Params &P, Ctl *c, int32_t n_l, int32_t e_l) {
  decide_tier(P, c, n_l, e_l);
  steer(P, c->tier);
}
__device__ void decide_tier(const Params &P, Ctl *c, int32_t n_l, int32_t e_l) {
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
  if (P.direction) {  // NEXT-3: Beamer's direction-optimising switch
    const long long m_u = P.nnz - c->m_visited;  // arcs of still-unvisited vertices
    if (!c->bu) {
      if ((long long)e_l * P.do_alpha > m_u) c->bu = 1;
    } else if (P.do_beta > 0 && (long long)n_l * P.do_beta < (long long)P.n) {
      c->bu = 0;
    }
    if (c->bu) {
      c->tier = TIER_BU;
      c->p_l = P.p_max;
      return;
    }
  }
  if (P.variant == 0 && P.t0 >= 0 && e_l <= P.t0 && n_l <= KS_NCAP) {
    c->tier = TIER_SMALL;
    c->p_l = 1;
    return;
  }
  if (P.variant == 0 && e_l <= P.tc_max && n_l <= KC_FCAP) {
    c->tier = TIER_CLUSTER;
    c->p_l = KC_CL;
    return;
  }
  c->tier = TIER_LARGE;
  c->pass = 0;
  c->n_acc = 0;
  c->e_acc = 0;
  c->kx_ns = 0;
  plan_pass(P, c);
}
// The next pass of the tier-1 level in ctl: its edge range, visited-test mode and grid.
// Level passes.  A discovery-heavy level reaches each new vertex many times (R-MAT 24: ~16
// arcs per discovered vertex on the mixed levels, ~90 per hub on the first discovery level);
// only the first is a discovery, every later one must ask L2 for the claim tag because the
// visited bitmap is exact at level START only (measured 4.5 us per 10^6 such re-checks
// against 1.46 us per 10^6 plain arcs: the largest term of those levels).  Such a level runs
// as passes over consecutive edge ranges [e_lo, e_hi) of the same frontier and degree scan:
// every pass is a complete k_explore + k_compact (Owner dedup, visited bits published,
// survivors APPENDED to the next frontier), so the later passes find the vertices of the
// earlier ones in the bitmap.  Same level number, same result: a pass boundary is just a point
// where the level's "d[v] = infinity" state is refreshed; P_l is sized per pass (Fig1 L16).
// A small first pass pays most: after 1/8 of the edges ~88 % of the level's new vertices
// (those with many arcs) are already found.
__device__ void plan_pass(const Params &P, Ctl *c) {
  const long long e_l = c->e_l;
  const long long e_lo = c->pass == 0 ? 0 : c->e_hi;
  // k_explore's visited test: tag mode while few arcs end at visited vertices (m_visited =
  // degrees of all visited vertices, the frontier included; arc ends for a symmetric graph)
  c->probe_tags = P.tag_pct >= 0 &&
                  (double)c->m_visited * 100.0 < (double)P.nnz_all * (double)P.tag_pct;
  long long e_hi = e_l;
  if (P.variant == 0 && P.dist_size == 1 && P.split_passes > 1 && P.split_min > 0 &&
      e_l >= P.split_min && c->probe_tags && c->pass + 1 < P.split_passes) {
    const long long first = max(e_l * P.split_pct / 100, 1LL);
    const long long rest = (e_l - first + P.split_passes - 2) / (P.split_passes - 1);
    e_hi = min(e_l, c->pass == 0 ? first : e_lo + max(rest, 1LL));
  }
  const long long es = e_hi - e_lo;
  long long pt = P.variant ? (long long)P.p_max
                           : min((long long)P.p_max, (es + P.grain - 1) / P.grain);
  if (pt < 1) pt = 1;
  const long long chunk = es > 0 ? (es + pt - 1) / pt : 1;
  long long p_l = (es + chunk - 1) / chunk;
  if (p_l < 1) p_l = 1;  // an empty slice still runs one (idle) CTA: k_compact reports 0
  c->e_lo = (int32_t)e_lo;
  c->e_hi = (int32_t)e_hi;
  c->p_l = (int32_t)p_l;
  c->chunk = (int32_t)chunk;
#if S3BFS_KX_TRANSPOSE
  {  // edges (= candidate capacity) per worker: `pieces` pieces of equal length
    const long long w = max((es + p_l * KD_WARPS - 1) / (p_l * KD_WARPS), 1LL);
    const int pieces = w >= S3BFS_KX_PIECES_MIN_EDGES ? S3BFS_KX_PIECES : 1;
    const long long plen = (w + pieces - 1) / pieces;
    c->pieces = pieces;
    c->wcap = (int32_t)(plen * pieces);
  }
#else
  c->pieces = 1;
  c->wcap = (int32_t)((chunk + KD_WARPS - 1) / KD_WARPS);  // edges (and candidates) per warp
#endif
}

// ---- init (Fig1 L1-L8) ----------------------------------------------------------------------
// d <- infinity is the cleared visited bitmap (R1): only the source's bit is set, with
// {d, parent} = {0, s} (R2).  Claim tags <- 0.  Owner is NOT initialised (R3).  The caller's
// level/parent arrays are written once, by k_finalize.
__global__ void k_init(Params P, int32_t s, int32_t *level, int32_t *parent) {
  const int n = P.n;
  const long long gtid = (long long)blockIdx.x * blockDim.x + threadIdx.x;
  const long long gstride = (long long)gridDim.x * blockDim.x;
  const int si = P.o2n ? __ldg(P.o2n + s) : s;  // the source's internal id
  const long long nw4 = ((long long)n + 127) >> 7;  // bitmap as uint4 (16 B padded)
  for (long long i = gtid; i <= nw4; i += gstride) {  // block nw4: the all-ones sentinel
    uint4 w = i == nw4 ? make_uint4(~0u, ~0u, ~0u, ~0u) : make_uint4(0, 0, 0, 0);
    if (i == (si >> 7)) (&w.x)[(si >> 5) & 3] = 1u << (si & 31);
    reinterpret_cast<uint4 *>(P.bm)[i] = w;
    if (P.bub && i < nw4) reinterpret_cast<uint4 *>(P.bub)[i] = make_uint4(0, 0, 0, 0);
  }
  const long long nc = ((long long)P.claim_mask + 16) >> 4;  // claim tags <- 0 (all slots),
  const uint32_t ss = claim_slot(P, si);                       // but the source's (discovered)
  for (long long i = gtid; i < nc; i += gstride) {
    uint4 z = make_uint4(0, 0, 0, 0);
    if (i == (long long)(ss >> 4)) (&z.x)[(ss >> 2) & 3] = 1u << (8 * (ss & 3));
    reinterpret_cast<uint4 *>(P.claim)[i] = z;
  }
  if (blockIdx.x == 0 && threadIdx.x == 0) {
    Ctl *c = P.ctl;
    const int4 vs = *vstat(P.vinfo, si);
    *lp_of(P.vinfo, si) = make_int2(0, s);
    P.f[0][0] = s;        // Fig1 L7: CurLevelVertices <- [s]
    P.frs[0][0] = vs.x;
    P.fex[0][0] = 0;      // exclusive degree scan of the frontier (R5)
    P.fex[0][1] = vs.y;
    c->level = 0;         // Fig1 L8
    c->cur = 0;
    c->source = s;
    c->level_out = level;
    c->parent_out = parent;
    c->num_levels = 0;
    c->done_ctr = 0;
    c->tile_ctr = 0;
    c->cand_acc = 0;
    c->t_prev = globaltimer();
    c->t_dbg[0] = c->t_prev;
    c->t_dbg[1] = 0;
    c->bu = 0;
    c->fb_valid = 0;
    c->m_visited = vs.y;
    decide(P, c, 1, vs.y);
  }
}

// create time: the two L2 cache-policy descriptors k_explore passes with its loads
__global__ void k_policies(unsigned long long *out) {
  out[0] = policy_evict_first();
  out[1] = policy_evict_last();
}

// ---- (c)+(d): k_explore ----------------------------------------------------------------------
// CTA b < P_l owns global edges [b*chunk, min((b+1)*chunk, e_l)) of the level, split evenly
// over its warps: each warp is one of the paper's workers with an (almost) equal share of the
// level's edges (Fig1 L16-L17).  A warp finds its start vertex with the 32-ary search
// (c), then walks its edges in batches of KX_GROUPS groups of 32 -- lane i takes edge e+i, so
// a group reads 32 consecutive col entries (coalesced streaming, Fig1 L18).  Edge -> frontier
// vertex mapping uses a register window of 32 consecutive frontier vertices (their
// degree-scan entries, ids and row starts): one warp-uniform shuffle search per batch, and a
// per-lane search only when the batch spans several rows.  No shared memory, no CTA barrier,
// so warps progress independently.
// Visited test (the paper's "d[v] = infinity", R1): the visited bitmap (exact at level start,
// read-only here) and, for a clear bit, the vertex's 1-byte claim tag, which equals this
// level's tag once some worker discovered v in this level.
// Discovery (EXPLORE-VERTEX): claim[v] = tag, {d, parent}[v] = {l+1, x}, Owner[v] =
// slot, cand[slot] = v -- plain stores, the paper's benign race, no atomics.  Racing
// discoverers that all saw an old tag store the same d and a valid parent and enqueue
// duplicates; the Owner check keeps exactly one (R4).
// DIST = NEXT-4's rank kernel (candidates routed to owners); the single-GPU kernel is
// k_explore<false> and carries none of that code
template <bool DIST>
__global__ void __launch_bounds__(KD_THREADS, KD_MIN_BLOCKS) k_explore(Params P) {
  Ctl *c = P.ctl;
  if (c->tier != TIER_LARGE) return;
  const int b = blockIdx.x;
  const int p_l = c->p_l;
  if (DIST && threadIdx.x == 0)  // NEXT-4: k_dist_keep's look-back word of tile b
    P.status[b] = 0ull;                      // (gridDim = P_max in dist mode)
  if (b >= p_l) return;
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int n_l = c->n_l, chunk = c->chunk, cur = c->cur, wcap = c->wcap;
  const int new_level = c->level + 1;     // Fig1 L10: discoveries get l+1 (R11)
  const int tag = 1 + (c->level % 255);   // never 0, the per-run initial value
  const int32_t *__restrict__ fx = P.f[cur];
  const int32_t *__restrict__ frs = P.frs[cur];
  const int32_t *__restrict__ fex = P.fex[cur];
  const int32_t *__restrict__ col = P.col;
  int4 *__restrict__ vinfo = P.vinfo;
  int32_t *__restrict__ cand = P.cand;
  const uint32_t *__restrict__ bm = P.bm;
  uint8_t *__restrict__ claim = P.claim;
  const int vs = P.v_sent;  // masked lanes' target: its visited bit is always set
  // tag mode's second probe round pays on long slices (R-MAT 24: +1.6 %); on short ones the
  // extra dependent round trip per batch costs more than the queue it spares (R-MAT 20: -1.7 %)
  const bool tag2 = S3BFS_KX_TAG2 && wcap >= S3BFS_KX_TAG2_MIN_WCAP;
  const int hub = P.hub;                              // ids < hub: bitmap first
  const uint32_t tag_span = (uint32_t)(P.n - P.hub);  // ids in [hub, n): tag only

  if (tid == 0) {
    if (!DIST) P.status[b] = 0ull;  // reset k_compact's look-back word
    if (b == 0) c->t_kx_begin = globaltimer();
  }
#if S3BFS_KX_TRANSPOSE
  // Worker (b, warp) takes slice warp * P_l + b of the pass's P_l * KD_WARPS equal slices: a
  // CTA's warps sample the whole edge range, so every CTA sees the same mix of long and short
  // rows whatever the order of the frontier (a frontier whose first part holds the
  // high-degree vertices -- the survivors of an earlier pass -- left the CTAs of the
  // short-row part 20 % behind the others with contiguous chunks)
  // ... and each worker's share is `pieces` equal pieces spread over the range the same way
  // (piece j of worker t = piece j * P_l * KD_WARPS + t): every WARP then walks the same mix,
  // and the kernel does not end on the warps whose one slice held only short rows
  (void)chunk;
  const int pieces = c->pieces, plen = wcap / pieces;
  int e_begin = 0, e_end = 0;
  auto set_piece = [&](int j) {
    const long long es0 = (long long)c->e_lo +
                          ((long long)j * p_l * KD_WARPS + (warp * p_l + b)) * plen;
    e_begin = (int)min(es0, (long long)c->e_hi);
    e_end = (int)min((long long)e_begin + plen, (long long)c->e_hi);
  };
  set_piece(0);
#else
  const int pieces = 1;
  auto set_piece = [&](int) {};
  const int E0 = c->e_lo + b * chunk;
  const int E1 = min(E0 + chunk, c->e_hi);
  const int e_begin = min(E0 + warp * wcap, E1);
  const int e_end = min(e_begin + wcap, E1);
#endif
  const int segbase = (b * KD_WARPS + warp) * wcap;
  const unsigned long long pol_stream = P.pol_first;
  const unsigned long long pol_status = P.pol_last;
  int wcount = 0;
  int u0 = 0, wex = 0, wx = 0, wb = 0, lim = 0;
  bool wzero = false;  // the window holds an empty row (two equal row starts)
  auto load_window = [&](int base) {
    const int u = base + lane;
    wex = (u < n_l) ? __ldg(fex + u) : 0x7fffffff;
    wx = (u < n_l) ? __ldg(fx + u) : 0;
    wb = (u < n_l) ? __ldg(frs + u) - wex : 0;
    lim = __ldg(fex + min(base + 32, n_l));
    const int down = __shfl_down_sync(0xffffffffu, wex, 1);  // all lanes shuffle
    const int nxt_start = (lane < 31) ? down : lim;
    wzero = __any_sync(0xffffffffu, u < n_l && nxt_start == wex);
  };
  if (e_begin < e_end) {
    u0 = warp_search(fex, n_l, e_begin);  // Find-StartExpPoint (c)
    load_window(u0);
  }
  // Map the batch of edges [e, e_next) onto lanes and load their targets: v[g] = col entry of
  // edge e + 32g + lane (-1 outside the batch), byte g of xs = its frontier vertex's window slot
  // (the caller id is shuffled only on discovery).
  auto map_load = [&](int e, int (&v)[KX_GROUPS], uint32_t (&xs)[KX_GROUPS / 4]) -> int {
    while (lim <= e) {  // window exhausted (also skips runs of zero-degree vertices, C9)
      u0 += 32;
      load_window(u0);
    }
    const int bend = min(e_end, lim);
    // window slot of the batch's first edge (warp-uniform): the window's row starts are
    // non-decreasing and wex_0 <= e, so it is the count of row starts <= e, minus one
    const int j0 = __popc(__ballot_sync(0xffffffffu, wex <= e)) - 1;
    const int row_end = (j0 < 31) ? __shfl_sync(0xffffffffu, wex, min(j0 + 1, 31)) : lim;
    int e_next = min(e + KX_GROUPS * 32, bend);
    if (S3BFS_KX_FAST && row_end >= e_next) {
      // the whole batch lies in one frontier row (most R-MAT arcs): uniform x and base
      const int x = j0;
      const int base = __shfl_sync(0xffffffffu, wb, j0);
      const int start = base + e;  // col index of the batch's first edge
      const int a0 = start & ~3;   // 16-byte aligned
#pragma unroll
      for (int k = 0; k < KX_GROUPS / 4; ++k) xs[k] = (uint32_t)x * 0x01010101u;
      if (S3BFS_KX_VEC && P.col_vec && (long long)a0 + KX_GROUPS * 32 <= P.nnz) {
        // vectorised streaming: lane i loads 16 B at a0 + 4*(i + 32k), i.e. each warp
        // instruction fetches 512 contiguous bytes of the row; edges outside
        // [start, row/slice end) are masked.  Next batch starts 16-byte aligned.
        const int lim_idx = base + bend;
        if (a0 == start && a0 + KX_GROUPS * 32 <= lim_idx) {
          // interior batch (aligned, whole): no masking
#pragma unroll
          for (int k = 0; k < KX_GROUPS / 4; ++k) {
            S3_CHK(a0 + 4 * (lane + 32 * k) + 3, P.nnz);
            const int4 q = ldg_stream4(col + a0 + 4 * (lane + 32 * k), pol_stream);
            v[4 * k + 0] = q.x;
            v[4 * k + 1] = q.y;
            v[4 * k + 2] = q.z;
            v[4 * k + 3] = q.w;
          }
        } else {
#pragma unroll
          for (int k = 0; k < KX_GROUPS / 4; ++k) {
            const int i0 = a0 + 4 * (lane + 32 * k);
            S3_CHK(i0 + 3, P.nnz);
            const int4 q = ldg_stream4(col + i0, pol_stream);  // in bounds: a0 + 256 <= nnz
            v[4 * k + 0] = (i0 + 0 >= start && i0 + 0 < lim_idx) ? q.x : vs;
            v[4 * k + 1] = (i0 + 1 >= start && i0 + 1 < lim_idx) ? q.y : vs;
            v[4 * k + 2] = (i0 + 2 >= start && i0 + 2 < lim_idx) ? q.z : vs;
            v[4 * k + 3] = (i0 + 3 >= start && i0 + 3 < lim_idx) ? q.w : vs;
          }
        }
        e_next = min(bend, a0 + KX_GROUPS * 32 - base);
      } else {
#pragma unroll
        for (int g = 0; g < KX_GROUPS; ++g) {  // masked lanes re-load the batch's first edge
          const int my_e = e + g * 32 + lane;
          S3_CHK(base + (my_e < bend ? my_e : e), P.nnz);
          const int t = ldg_stream(col + base + (my_e < bend ? my_e : e), pol_stream);
          v[g] = (my_e < bend) ? t : vs;
        }
      }
    } else if (S3BFS_KX_RANK && !wzero) {
      // several rows in the batch: rank mapping.  Window lane j's row starts at edge wex_j;
      // for group g (edges eg .. eg+31) the row starts strictly inside the group form a
      // 32-bit mask (one REDUX), and lane i's row is the group's first row plus the number
      // of row starts at or below edge eg+i (exact while no row of the window is empty)
      // (row starts in [eg, eg+31] -> mask bit rel; r = row of edge eg-1, so lane i's row is
      // r + popc(mask & bits 0..i); the batch's first edge lies in row j0)
      const unsigned le = 0xffffffffu >> (31 - lane);  // bits 0 .. lane
      const int pfirst = __shfl_sync(0xffffffffu, wb, j0) + e;  // col index of edge e (valid)
      const int lb = bend - e - lane;  // group g's lane is inside the batch iff 32 g < lb
      int r = j0;
#pragma unroll
      for (int g = 0; g < KX_GROUPS; ++g) {
        const int eg = e + g * 32;
        const int rel = wex - eg;  // this window lane's row start relative to the group
        const unsigned m = __reduce_or_sync(0xffffffffu, shl1(rel));  // starts in [eg, eg+31]
        if (g == 0) r -= (int)(m & 1u);  // a row starting exactly at e is row j0 itself
        const int j = r + __popc(m & le);
        xs[g >> 2] |= (uint32_t)j << (8 * (g & 3));
        const int pos = __shfl_sync(0xffffffffu, wb, j) + eg + lane;
        const bool ok = g * 32 < lb;
        S3_CHK(ok ? pos : pfirst, P.nnz);
        const int t = ldg_stream(col + (ok ? pos : pfirst), pol_stream);  // unconditional
        v[g] = ok ? t : vs;
        r += __popc(m);
      }
    } else {
#pragma unroll
      for (int g = 0; g < KX_GROUPS; ++g) {
        const int my_e = e + g * 32 + lane;
        int j = j0;  // largest window slot with excl <= my_e (>= j0)
#pragma unroll
        for (int s = 16; s >= 1; s >>= 1) {
          const int cj = __shfl_sync(0xffffffffu, wex, min(j + s, 31));
          if (j + s <= 31 && cj <= my_e) j += s;
        }
        xs[g >> 2] |= (uint32_t)j << (8 * (g & 3));
        const int pos = __shfl_sync(0xffffffffu, wb, j) + my_e;
        const int pf = __shfl_sync(0xffffffffu, wb, j0) + e;
        S3_CHK(my_e < bend ? pos : pf, P.nnz);
        const int t = ldg_stream(col + (my_e < bend ? pos : pf), pol_stream);
        v[g] = (my_e < bend) ? t : vs;
      }
    }
    return e_next;
  };
#if !S3BFS_KX_QUEUE
  // Discovery of the batch's groups flagged in discm (Fig1 L18-L22): plain stores -- the tag,
  // {d, parent}, Owner = the candidate slot, and the candidate itself (benign race, R4).
  auto discover = [&](const int (&v)[KX_GROUPS], const uint32_t (&xs)[KX_GROUPS / 4],
                      uint32_t discm) {
    const unsigned wdisc = __reduce_or_sync(0xffffffffu, discm);
    if (!wdisc) return;  // warp-uniform skip: most batches of the heavy levels find nothing
#pragma unroll
    for (int g = 0; g < KX_GROUPS; ++g) {
      if (!((wdisc >> g) & 1u)) continue;
      // parent: the window slot's caller id (the window is unchanged since map_load)
      const int par = __shfl_sync(0xffffffffu, wx, (xs[g >> 2] >> (8 * (g & 3))) & 31u);
      const bool disc = (discm >> g) & 1u;
      const unsigned m = __ballot_sync(0xffffffffu, disc);
      if (disc) {
        const int slot = segbase + wcount + __popc(m & lanemask_lt());
        st_u8(claim + claim_slot(P, v[g]), tag);
        st_discovery(vinfo, v[g], new_level, par, slot);  // d[v] <- l, parent, Owner[v] <- i
        cand[slot] = v[g];                         // Q[i].Enqueue(v)
      }
      wcount += __popc(m);
    }
  };
#endif
  // The level's visited test (Fig1 L18 "if d[v] = infinity"), chosen per level by
  // decide_tier from the share of arcs that end at visited vertices:
  //  bitmap mode (most targets visited, the heavy levels): every target's visited bit (exact
  //    at level start; hub words L1-resident), then the discovery tag of the few clear ones;
  //  tag mode (most targets new, the discovery-heavy levels): a hub id (< P.hub) reads its
  //    bit first, any other id only its discovery tag (nonzero once discovered) -- one probe
  //    instead of two for the arcs that reach new vertices.
  // Masked slots probe the sentinel (its bit is always set), so the tests are branch-free.
#if S3BFS_KX_QUEUE
  // Warp-private queue of the batch's rare items -- targets whose claim tag must be read
  // (bitmap clear) or that were found undiscovered (tag mode) -- with their parents.  The
  // items of many batches are resolved 32 at a time, one per lane (claim tag, then the
  // discovery stores), instead of per group under predication: a heavy level flags about
  // 2 % of its targets, which otherwise cost every lane the claim and discovery code of
  // every flagged group (ncu: 45 % of the heavy level's instructions, profiles/).
  __shared__ int2 s_q[KD_WARPS][KQ_CAP];
  __shared__ int32_t s_dc[DIST ? KD_WARPS : 1][DIST_MAX];  // NEXT-4: per destination rank
  if (DIST) {
    if (lane < DIST_MAX) s_dc[warp][lane] = 0;
    __syncwarp();
  }
  int2 *const q = s_q[warp];
  int qn = 0;  // warp-uniform queue length
  // resolve the first cnt (<= 32) items; the rest (qn - cnt) move to the front
  auto flush = [&](int cnt) {
    __syncwarp();
    const bool valid = lane < cnt;
    const int2 it = valid ? q[lane] : make_int2(0, 0);
    const int v = it.x & 0x7fffffff;
    const uint32_t cs = claim_slot(P, v);
    int cl = 0;
    if (valid && it.x < 0) cl = ld_cg_u8(claim + cs);  // Fig1 L18: already claimed this level?
    const bool disc = valid && cl == 0;
    const unsigned m = __ballot_sync(0xffffffffu, disc);
    if (!DIST) {
      if (disc) {  // EXPLORE-VERTEX's discovery: plain stores, the benign race (R4)
        const int slot = segbase + wcount + __popc(m & lanemask_lt());
        S3_CHK(v, P.n);
        S3_CHK(slot, (long long)(b * KD_WARPS + warp + 1) * wcap);
        st_u8(claim + cs, tag);
        st_discovery(vinfo, v, new_level, it.y, slot);  // d[v] <- l, parent (Fig1 L18),
                                                        // Owner[v] <- i (benign race)
        cand[slot] = v;                        // Q[i].Enqueue(v)
      }
      wcount += __popc(m);
    } else {
      // NEXT-4: the candidate {v, parent} goes straight into the receive segment of this warp
      // in v's owner rank (a peer store over NVLink, or this rank's own buffer); the owner
      // runs the Owner check (e).  The tag only filters this rank's repeats.
      if (disc) st_u8(claim + cs, tag);
      const int d = disc ? (v >> 5) % P.dist_size : -1;
      for (int dd = 0; dd < P.dist_size; ++dd) {
        const unsigned md = __ballot_sync(0xffffffffu, d == dd);
        if (!md) continue;  // warp-uniform
        if (d == dd) {
          const int k = s_dc[warp][dd] + __popc(md & lanemask_lt());
          S3_CHK(k, wcap);
          const int slot = P.rofs[P.dist_rank] + segbase + k;
          P.p_recv[dd][slot] = make_int2(v, it.y);
          // Owner[v] <- slot in the owner's records (Fig1 L22; the benign race, plain stores
          // from every rank that sends v: one label survives, the owner keeps that copy)
          st_weak(owner_of(P.p_vinfo[dd], ((v >> 5) / P.dist_size) * 32 + (v & 31)), slot);
        }
        __syncwarp();
        if (lane == 0) s_dc[warp][dd] += __popc(md);
        __syncwarp();
      }
    }
    const int rest = qn - cnt;
    for (int i = 0; i < rest; i += 32) {  // in order: chunk i never reads a slot written before
      const int2 t = i + lane < rest ? q[cnt + i + lane] : make_int2(0, 0);
      __syncwarp();
      if (i + lane < rest) q[i + lane] = t;
    }
    __syncwarp();
    qn = rest;
  };
  // enqueue group g's flagged lanes (chk: the claim tag decides)
  auto enqueue = [&](int g, bool flag, bool chk, int vg, const uint32_t (&xs)[KX_GROUPS / 4]) {
    const unsigned m = __ballot_sync(0xffffffffu, flag);
    const int par = __shfl_sync(0xffffffffu, wx, (xs[g >> 2] >> (8 * (g & 3))) & 31u);
    if (flag) q[qn + __popc(m & lanemask_lt())] = make_int2(vg | (chk ? (int)0x80000000u : 0), par);
    qn += __popc(m);
  };
#endif
  auto run = [&](auto tag_mode) {
    constexpr bool TAGS = decltype(tag_mode)::value;
    int e = e_begin;
    while (e < e_end) {
      int v[KX_GROUPS];
      uint32_t xs[KX_GROUPS / 4];  // window slots of the groups' frontier vertices, a byte each
#pragma unroll
      for (int k = 0; k < KX_GROUPS / 4; ++k) xs[k] = 0;
      e = map_load(e, v, xs);
      uint32_t needm = 0;  // targets whose discovery tag decides (bit clear at level start)
      uint32_t discm = 0;  // targets found undiscovered: candidates (Fig1 L19-L22)
      if constexpr (TAGS) {
#pragma unroll
        for (int g = 0; g < KX_GROUPS; ++g) {
          const bool via_tag = (uint32_t)(v[g] - hub) < tag_span;
          S3_CHK(v[g] >> 5, (P.v_sent >> 5) + 4);
          uint32_t r;
          if (via_tag) r = (uint32_t)ld_cg_u8_hint(claim + claim_slot(P, v[g]), pol_status);
          else r = ldg_status_u32(bm + (v[g] >> 5), pol_status);
          needm |= (via_tag ? 0u : (~rotr32(r, v[g]) & 1u)) << g;
          discm |= (via_tag ? (uint32_t)(r == 0u) : 0u) << g;
        }
#if S3BFS_KX_TAG2
        // Second probe round of tag mode: a hub whose bit is clear at level start is, in a
        // discovery-heavy level, most often already claimed by an earlier arc of this level
        // (ncu: 72 % of the level's arcs, each a queue item whose claim load stalled its flush:
        // 5.8 serial flushes per batch).  Their tags are read here, all groups' loads in flight
        // at once, and only true discoveries reach the queue (220 M -> 146 M warp instructions
        // on R-MAT 24's first discovery level; the big mixed levels gain 4-5 %).
        if (tag2 && __reduce_or_sync(0xffffffffu, needm)) {  // warp-uniform
          int cl[KX_GROUPS];
#pragma unroll
          for (int g = 0; g < KX_GROUPS; ++g)
            cl[g] = ((needm >> g) & 1u) ? ld_cg_u8_hint(claim + claim_slot(P, v[g]), pol_status) : 1;
#pragma unroll
          for (int g = 0; g < KX_GROUPS; ++g) discm |= (uint32_t)(cl[g] == 0) << g;
          needm = 0;
        }
#endif
      } else {
#pragma unroll
        for (int g = 0; g < KX_GROUPS; ++g) {
          S3_CHK(v[g] >> 5, (P.v_sent >> 5) + 4);
          const uint32_t w = ldg_status_u32(bm + (v[g] >> 5), pol_status);
          needm |= (~rotr32(w, v[g]) & 1u) << g;  // bit (v mod 32) of w, inverted
        }
      }
#if S3BFS_KX_QUEUE
      const uint32_t itm = needm | discm;
      const unsigned witm = __reduce_or_sync(0xffffffffu, itm);
      if (witm) {  // warp-uniform skip; then only the flagged groups
#pragma unroll
        for (int g = 0; g < KX_GROUPS; ++g) {
          if ((witm >> g) & 1u) enqueue(g, (itm >> g) & 1u, (needm >> g) & 1u, v[g], xs);
          if ((g % S3BFS_KQ_GROUPS) == S3BFS_KQ_GROUPS - 1) {  // at most 32 + KQ_GROUPS * 32 queued
            while (qn >= 32) flush(32);
          }
        }
      }
    }
  };
#else
      const unsigned wneed = __reduce_or_sync(0xffffffffu, needm);
      if (wneed) {  // warp-uniform skip
#pragma unroll
        for (int h = 0; h < KX_GROUPS; h += 4) {  // 4 tag loads in flight (register budget)
          int cl[4];
#pragma unroll
          for (int g = 0; g < 4; ++g)
            cl[g] = ((needm >> (h + g)) & 1u) ? ld_cg_u8(claim + claim_slot(P, v[h + g])) : 1;
#pragma unroll
          for (int g = 0; g < 4; ++g) discm |= (uint32_t)(cl[g] == 0) << (h + g);
        }
      }
      discover(v, xs, discm);
    }
  };
#endif
  for (int j = 0;;) {
    if (c->probe_tags) run(std::true_type{});
    else run(std::false_type{});
    if (++j >= pieces) break;
    set_piece(j);
    if (e_begin < e_end) {
      u0 = warp_search(fex, n_l, e_begin);
      load_window(u0);
    }
  }
#if S3BFS_KX_QUEUE
  if (qn > 0) flush(qn);  // warp-uniform: the slice's remaining items
#endif
  S3_CHK(segbase + wcount, P.cand_cap);
  if (lane == 0) P.wcnt[b * KD_WARPS + warp] = wcount;
  if (DIST) {  // NEXT-4: segment counts and the level's {wcap, p_l} to every owner
    __syncwarp();
    const int gw = b * KD_WARPS + warp;
    if (lane < P.dist_size)
      P.p_rcnt[lane][(long long)P.dist_rank * P.p_max * KD_WARPS + gw] = s_dc[warp][lane];
    if (b == 0 && tid == 0)
      for (int d = 0; d < P.dist_size; ++d) P.p_rmeta[d][P.dist_rank] = make_int2(wcap, p_l);
    __threadfence_system();  // the peer stores are visible before this grid completes
  }
}

// Publish the visited bits of a warp's kept candidates: lanes holding the same bitmap word in
// a run of consecutive lanes OR their bits together (segmented shuffle scan) and the run's
// last lane issues one atomicOr -- same-word atomics from one instruction would serialise in
// the L2 atomic unit.  Same-word lanes in different runs still issue separate (correct) ORs.
__device__ __forceinline__ void bm_publish(uint32_t *bm, bool keep, int v, int lane) {
#if S3BFS_BM_AGG
  const int wd = keep ? (v >> 5) : -1;
  uint32_t acc = keep ? 1u << (v & 31) : 0u;
  const int prev = __shfl_up_sync(0xffffffffu, wd, 1);
  const unsigned heads = __ballot_sync(0xffffffffu, lane == 0 || prev != wd);
  const int run0 = 31 - __clz(heads & ((2u << lane) - 1u));  // first lane of my run
#pragma unroll
  for (int s = 1; s < 32; s <<= 1) {
    const uint32_t o = __shfl_up_sync(0xffffffffu, acc, s);
    if (lane - s >= run0) acc |= o;
  }
  const bool last = lane == 31 || ((heads >> (lane + 1)) & 1u);
  if (keep && last) atomicOr(bm + wd, acc);
#else
  if (keep) atomicOr(bm + (v >> 5), 1u << (v & 31));
#endif
}

// ---- (e)+(a)+(b): k_compact -------------------------------------------------------------------
// CTA b handles the candidate segments its k_explore twin wrote (one per warp).
// Pass 1 (Fig1 L20-L23): keep cand[k] iff Owner[cand[k]] == k (one 16-byte vertex-record
// probe gives Owner, row start and degree); publish the kept vertex's visited bit and
// compact (id, row start, degree) in place -- the degree is Fig1 L13 of the next level.
// The next frontier holds caller ids (from the same record), the parents k_explore records.
// A decoupled look-back over CTAs scans the (kept, degree-sum) pairs (Fig1 L24 and L14 of
// the next level in one pass).  Pass 2 (Fig1 L25-L29): write the next frontier, its row
// starts and its exclusive degree scan.  The last CTA to finish advances the control block
// (Fig1 L9-L10, L15-L16).
__global__ void __launch_bounds__(KD_THREADS, KD_MIN_BLOCKS) k_compact(Params P) {
  Ctl *c = P.ctl;
  if (c->tier != TIER_LARGE) return;
  const int p_l = c->p_l;
  __shared__ int32_t s_k[KD_WARPS], s_d[KD_WARPS];
  __shared__ int32_t s_la[KD_WARPS], s_ld[KD_WARPS];  // S3BFS_LB_WIDE: predecessor sums
  __shared__ int s_last, s_tile;
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  // Surplus CTAs (blockIdx >= P_l) do no work but are still counted by the last-CTA
  // election below: the control block is rewritten only after EVERY CTA of this launch has
  // read it (a late-starting surplus CTA would otherwise see the next level's state).
  const int nxt = c->cur ^ 1;
  if ((int)blockIdx.x < p_l) {
  if (tid == 0) s_tile = (int)atomicAdd(&c->tile_ctr, 1u);  // look-back order = start order
  __syncthreads();
  const int b = s_tile;  // this CTA handles tile b: the segments of k_explore's CTA b
  const int4 *__restrict__ vinfo = P.vinfo;
  int32_t *__restrict__ cand = P.cand;
  int2 *__restrict__ crd = P.cand_rd;
  const int seg = (b * KD_WARPS + warp) * c->wcap;
  const int cnt = P.wcnt[b * KD_WARPS + warp];
  const int n_acc = c->n_acc, e_acc = c->e_acc;  // written by the level's earlier passes
  if (b == 0 && tid == 0) c->t_kx_end = globaltimer();

  int kept = 0, dsum = 0;
  // S3BFS_KC_REVERSE: newest candidates first -- their records are the ones k_explore's
  // discovery stores left in L2; walking oldest first, the gathers that miss push exactly
  // those out before they are read.  The kept entries are then compacted towards the
  // segment's end (write position >= every unread entry), pass 2 reads them from there.
#if S3BFS_KC_REVERSE
  for (int k0 = cnt > 0 ? ((cnt - 1) / (32 * KC_GROUPS)) * (32 * KC_GROUPS) : -1; k0 >= 0;
       k0 -= 32 * KC_GROUPS) {
#else
  for (int k0 = 0; k0 < cnt; k0 += 32 * KC_GROUPS) {
#endif
    int v[KC_GROUPS];
#pragma unroll
    for (int g = 0; g < KC_GROUPS; ++g) {
      const int k = k0 + g * 32 + lane;
      if (k < cnt) S3_CHK(seg + k, P.cand_cap);
      v[g] = (k < cnt) ? cand[seg + k] : -1;
      if (k < cnt) S3_CHK(v[g], P.n);
    }
    int4 vi[KC_GROUPS];  // {row start, degree, caller id, Owner}: one sector per candidate
#pragma unroll
    for (int g = 0; g < KC_GROUPS; ++g)
      vi[g] = (v[g] >= 0) ? ld_vrec256_nc(vinfo, v[g]) : make_int4(0, 0, 0, -1);
#pragma unroll
    for (int g = 0; g < KC_GROUPS; ++g) {
      const int k = k0 + g * 32 + lane;
      const bool keep = v[g] >= 0 && vi[g].w == seg + k;  // Fig1 L22: "if Owner[v] = i"
      const int d = keep ? vi[g].y : 0;
      bm_publish(P.bm, keep, v[g], lane);  // exact visited bit (R17)
      const unsigned m = __ballot_sync(0xffffffffu, keep);
      if (keep) {
#if S3BFS_KC_REVERSE
        const int q = seg + cnt - 1 - kept - __popc(m & lanemask_lt());
#else
        const int q = seg + kept + __popc(m & lanemask_lt());
#endif
        S3_CHK(q, P.cand_cap);
        cand[q] = vi[g].z;
        crd[q] = make_int2(vi[g].x, d);
      }
      kept += __popc(m);
      dsum += d;
    }
  }
  dsum = warp_sum(dsum);
  if (lane == 0) { s_k[warp] = kept; s_d[warp] = dsum; }
  if (P.collect_stats) {
    const int tot = warp_sum(lane == 0 ? cnt : 0);
    if (lane == 0 && tot) atomicAdd(&c->cand_acc, tot);  // statistics only
  }
  __syncthreads();
#if S3BFS_LB_WIDE
  // (b) across CTAs in one round trip: CTA b publishes its (kept, degree-sum) aggregate and
  // every thread reads one predecessor's (P_l <= P_max <= 512 = the CTA size): the exclusive
  // prefix is their sum, complete once every predecessor has published (tiles are numbered in
  // start order, so each has started).  A chained look-back needs ~P_l / 32 dependent round
  // trips for the last tiles; this needs one, plus a CTA reduction.
  int koff, doff;
  {
    const int kk = lane < KD_WARPS ? s_k[lane] : 0;  // every warp scans the warp totals
    const int dd = lane < KD_WARPS ? s_d[lane] : 0;
    const int ik = warp_incl_scan(kk), id = warp_incl_scan(dd);
    const Pair agg{(uint32_t)__shfl_sync(0xffffffffu, ik, 31),
                   (uint32_t)__shfl_sync(0xffffffffu, id, 31)};
    if (tid == 0) st_relaxed_u64(P.status + b, FLAG_A | pack<true>(agg));
    Pair ex{0, 0};
    for (unsigned ns = 32;;) {
      const unsigned long long sv = tid < b ? ld_relaxed_u64(P.status + tid) : FLAG_A;
      const Pair v = unpack<true>(sv);
      const int sa = warp_sum((int)v.a), sd = warp_sum((int)v.b);
      if (lane == 0) { s_la[warp] = sa; s_ld[warp] = sd; }
      if (!__syncthreads_or((sv >> 62) == 0)) {  // (also the barrier before the reads below)
        ex.a = (uint32_t)warp_sum(lane < KD_WARPS ? s_la[lane] : 0);
        ex.b = (uint32_t)warp_sum(lane < KD_WARPS ? s_ld[lane] : 0);
        break;
      }
      __nanosleep(ns);
      if (ns < S3BFS_LB_MAX_NS) ns <<= 1;
    }
    // (the level's earlier passes already wrote n_acc entries with degree sum e_acc)
    koff = n_acc + (int)ex.a + __shfl_sync(0xffffffffu, ik - kk, warp);
    doff = e_acc + (int)ex.b + __shfl_sync(0xffffffffu, id - dd, warp);
    if (b == p_l - 1 && tid == 0) {  // the pass's totals -> n_{l+1}, e_{l+1} (Fig1 L15)
      const int n_next = (int)(ex.a + agg.a), e_next = (int)(ex.b + agg.b);
      c->n_next = n_next;
      c->e_next = e_next;
      P.fex[nxt][n_acc + n_next] = e_acc + e_next;
    }
  }
#else
  if (warp == 0) {
    const int kk = lane < KD_WARPS ? s_k[lane] : 0;
    const int dd = lane < KD_WARPS ? s_d[lane] : 0;
    const int ik = warp_incl_scan(kk), id = warp_incl_scan(dd);
    const Pair agg{(uint32_t)__shfl_sync(0xffffffffu, ik, 31),
                   (uint32_t)__shfl_sync(0xffffffffu, id, 31)};
    const Pair ex = lookback<true>(P.status, b, agg);
    if (lane < KD_WARPS) {
      s_k[lane] = n_acc + (int)ex.a + ik - kk;
      s_d[lane] = e_acc + (int)ex.b + id - dd;
    }
    if (b == p_l - 1 && lane == 0) {  // the pass's totals -> n_{l+1}, e_{l+1} (Fig1 L15)
      const int n_next = (int)(ex.a + agg.a), e_next = (int)(ex.b + agg.b);
      c->n_next = n_next;
      c->e_next = e_next;
      P.fex[nxt][n_acc + n_next] = e_acc + e_next;
    }
  }
  __syncthreads();
  int koff = s_k[warp], doff = s_d[warp];
#endif
  int32_t *__restrict__ fn = P.f[nxt];
  int32_t *__restrict__ frsn = P.frs[nxt];
  int32_t *__restrict__ fexn = P.fex[nxt];
  for (int k0 = 0; k0 < kept; k0 += 32) {
    const int k = k0 + lane;
    int v = 0, r0 = 0, d = 0;
    if (k < kept) {
      const int kk = S3BFS_KC_REVERSE ? cnt - kept + k : k;  // kept entries: the segment's end
      v = cand[seg + kk];
      const int2 rd = crd[seg + kk];
      r0 = rd.x;
      d = rd.y;
    }
    const int inc = warp_incl_scan(d);
    if (k < kept) {
      S3_CHK(koff + k, P.n);
      fn[koff + k] = v;
      frsn[koff + k] = r0;
      fexn[koff + k] = doff + inc - d;
    }
    doff += __shfl_sync(0xffffffffu, inc, 31);
  }
  }  // active CTA
  // last-CTA election over the whole grid (one atomic per CTA; not the discovery path, R17)
  __threadfence();
  __syncthreads();
  if (tid == 0) s_last = atomicAdd(&c->done_ctr, 1u) == gridDim.x - 1;
  __syncthreads();
  if (s_last && tid == 0) {
    __threadfence();
    const int n_pass = ld_volatile(&c->n_next), e_pass = ld_volatile(&c->e_next);
    const unsigned long long t = globaltimer();
    const unsigned long long kb = *(volatile unsigned long long *)&c->t_kx_begin;
    const unsigned long long ke = *(volatile unsigned long long *)&c->t_kx_end;
    if (c->pass == 0) c->t_kx_first = kb;
    c->kx_ns += ke - kb;
    c->done_ctr = 0;
    c->tile_ctr = 0;
    c->m_visited += e_pass;
    c->n_acc += n_pass;
    c->e_acc += e_pass;
    c->pass += 1;
    if (c->e_hi < c->e_l) {  // the level's next pass (plan_pass): same frontier, next edges
      plan_pass(P, c);
      steer(P, TIER_LARGE);
    } else {
      const int n_next = c->n_acc, e_next = c->e_acc;
      // one record per level: candidates and kept summed over its passes, k_explore's time
      // as [first pass's start, + the passes' summed durations], passes in `pad`
      record_stat(P, c, c->level, c->n_l, c->e_l, TIER_LARGE, p_l, ld_volatile(&c->cand_acc),
                  n_next, c->t_prev, t, c->t_kx_first, c->t_kx_first + c->kx_ns, c->pass);
      c->cand_acc = 0;
      c->t_prev = t;
      c->level = c->level + 1;  // Fig1 L10
      c->cur = nxt;
      c->fb_valid = 0;
      decide(P, c, n_next, e_next);
    }
  }
}

// ---- NEXT-4: one traversal over G ranks, 1-D vertex partition ------------
// Rank r owns the internal ids v with (v / 32) mod G == r, their CSR rows (a local CSR whose
// targets stay global ids), and their state (vinfo / lp / Owner in local slots).  Per level:
//   k_explore (dist mode)  the local frontier's arcs; a target whose visited bit (replicated
//                          bitmap, exact at level start) is clear goes as {v, parent} straight
//                          into the receive segment of its owner, and the segment slot into
//                          the owner's Owner[v] (peer stores over NVLink; Fig1 L22's benign race
//                          now spans the senders: plain stores, one label survives)
//   k_dist_keep            keep a received candidate iff Owner[v] is its slot; d/parent, the
//                          owner's bitmap words (atomicOr into its own and every peer's replica,
//                          off the discovery path), and the next local frontier by the
//                          (kept, degree-sum) look-back scan over (source rank, CTA) tiles
//                          (Fig1 L23-L29, L12-L15)
//   k_dist_advance         the level's totals over all ranks (each rank published its own into
//                          every peer's rtot) decide the loop (Fig1 L9) and the local P_l
// The exchange is peer memory (no collective carries data); the driver only orders the phases
// across ranks (stream-ordered barriers).
__device__ __forceinline__ int dist_local(const Params &P, int v) {
  return ((v >> 5) / P.dist_size) * 32 + (v & 31);
}
__device__ __forceinline__ int dist_global(const Params &P, int lv) {
  return (((lv >> 5) * P.dist_size + P.dist_rank) << 5) + (lv & 31);
}

__global__ void k_dist_init(Params P, int32_t s) {
  const long long gtid = (long long)blockIdx.x * blockDim.x + threadIdx.x;
  const long long gstride = (long long)gridDim.x * blockDim.x;
  const int si = P.o2n ? __ldg(P.o2n + s) : s;
  const long long nw4 = ((long long)P.n + 127) >> 7;
  for (long long i = gtid; i <= nw4; i += gstride) {  // every replica: visited = {s} + sentinel
    uint4 w = i == nw4 ? make_uint4(~0u, ~0u, ~0u, ~0u) : make_uint4(0, 0, 0, 0);
    if (i == (si >> 7)) (&w.x)[(si >> 5) & 3] = 1u << (si & 31);
    reinterpret_cast<uint4 *>(P.bm)[i] = w;
  }
  const long long nc = ((long long)P.claim_mask + 16) >> 4;
  for (long long i = gtid; i < nc; i += gstride)
    reinterpret_cast<uint4 *>(P.claim)[i] = make_uint4(0, 0, 0, 0);
  if (blockIdx.x == 0 && threadIdx.x == 0) {
    Ctl *c = P.ctl;
    int n_l = 0, e_l = 0;
    if ((si >> 5) % P.dist_size == P.dist_rank) {  // the source's owner seeds its frontier
      const int ls = dist_local(P, si);
      const int4 vs = *vstat(P.vinfo, ls);
      *lp_of(P.vinfo, ls) = make_int2(0, s);
      P.f[0][0] = s;
      P.frs[0][0] = vs.x;
      P.fex[0][0] = 0;
      P.fex[0][1] = vs.y;
      n_l = 1;
      e_l = vs.y;
    } else {
      P.fex[0][0] = 0;
    }
    c->level = 0;
    c->cur = 0;
    c->source = s;
    c->num_levels = 0;
    c->done_ctr = 0;
    c->tile_ctr = 0;
    c->cand_acc = 0;
    c->t_prev = globaltimer();
    c->bu = 0;
    c->fb_valid = 0;
    c->m_visited = 0;
    c->g_n_next = 1;
    c->g_e_next = 0;
    decide_tier(P, c, n_l, e_l);
    if (c->tier == TIER_DONE) {  // an empty local frontier still explores (one idle CTA)
      c->tier = TIER_LARGE;
      c->p_l = 1;
      c->chunk = 1;
      c->wcap = 1;
      c->pieces = 1;
      c->e_lo = 0;
      c->e_hi = 0;
    }
  }
}

// keep iff Owner[v] == slot (Fig1 L22-L23).  Tile b (start order) = the segments of every source
// rank's CTA b: warp w handles segment b * 16 + w of each source in turn
__global__ void __launch_bounds__(KD_THREADS, KD_MIN_BLOCKS) k_dist_keep(Params P) {
  Ctl *c = P.ctl;
  if (c->tier != TIER_LARGE) return;  // a level enqueued past the end of the traversal
  __shared__ int32_t s_k[KD_WARPS], s_d[KD_WARPS];
  __shared__ int32_t s_kc[KD_WARPS][DIST_MAX];  // kept per (warp, source), pass 1 -> pass 2
  __shared__ int s_last, s_tile;
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int nxt = c->cur ^ 1, new_level = c->level + 1;
  const int nt = P.p_max;
  const int nwmax = P.p_max * KD_WARPS;
  if (tid == 0) s_tile = (int)atomicAdd(&c->tile_ctr, 1u);  // look-back order = start order
  __syncthreads();
  const int t = s_tile;
  if (t < nt) {
    const int gseg = t * KD_WARPS + warp;
    int kept = 0, dsum = 0;
    for (int src = 0; src < P.dist_size; ++src) {
      const int2 m = P.rmeta[src];
      const int cnt = t < m.y ? P.rcnt[(long long)src * nwmax + gseg] : 0;
      const long long base = P.rofs[src] + (long long)gseg * m.x;
      int ks = 0;
      for (int k0 = 0; k0 < cnt; k0 += 32) {
        const int k = k0 + lane;
        int2 it = make_int2(-1, 0);
        int4 vi = make_int4(0, 0, 0, -1);
        int lv = 0;
        if (k < cnt) {
          it = P.recv[base + k];
          lv = dist_local(P, it.x);
          vi = ld_vrec_weak(P.vinfo, lv);  // Owner written by the senders' k_explore
        }
        // the surviving label's copy, unless v was visited in an earlier level: a sender's tag
        // mode knows only its own sends, so it may send a vertex another rank found before
        const bool keep = k < cnt && vi.w == (int)(base + k) &&
                          !((__ldcg(P.bm + (it.x >> 5)) >> (it.x & 31)) & 1u);
        if (keep) *lp_of(P.vinfo, lv) = make_int2(new_level, it.y);  // d[v] <- l, parent (Fig1 L18)
        for (int d = 0; d < P.dist_size; ++d)             // the owner's bitmap words, in its own
          bm_publish(P.p_bm[d], keep, it.x, lane);         // replica and every peer's
        const unsigned mk = __ballot_sync(0xffffffffu, keep);
        if (keep) P.recv[base + ks + __popc(mk & lanemask_lt())].x = it.x;  // in place
        ks += __popc(mk);
        dsum += keep ? vi.y : 0;
      }
      if (lane == 0) s_kc[warp][src] = ks;
      kept += ks;
    }
    dsum = warp_sum(dsum);
    if (lane == 0) { s_k[warp] = kept; s_d[warp] = dsum; }
    __syncthreads();
    if (warp == 0) {
      const int kk = s_k[lane & (KD_WARPS - 1)] * (lane < KD_WARPS);
      const int dd = s_d[lane & (KD_WARPS - 1)] * (lane < KD_WARPS);
      const int ik = warp_incl_scan(kk), id = warp_incl_scan(dd);
      const Pair agg{(uint32_t)__shfl_sync(0xffffffffu, ik, 31),
                     (uint32_t)__shfl_sync(0xffffffffu, id, 31)};
      const Pair ex = lookback<true>(P.status, t, agg);
      if (lane < KD_WARPS) {
        s_k[lane] = (int)ex.a + ik - kk;
        s_d[lane] = (int)ex.b + id - dd;
      }
      if (t == nt - 1 && lane == 0) {
        c->n_next = (int)(ex.a + agg.a);
        c->e_next = (int)(ex.b + agg.b);
        P.fex[nxt][c->n_next] = c->e_next;
      }
    }
    __syncthreads();
    int koff = s_k[warp], doff = s_d[warp];
    for (int src = 0; src < P.dist_size; ++src) {  // pass 2: the next local frontier (L25-L29)
      const int ks = s_kc[warp][src];
      const long long base = P.rofs[src] + (long long)gseg * P.rmeta[src].x;
      for (int k0 = 0; k0 < ks; k0 += 32) {
        const int k = k0 + lane;
        int v = 0;
        int4 vi = make_int4(0, 0, 0, 0);
        if (k < ks) {
          v = P.recv[base + k].x;
          vi = __ldg(vstat(P.vinfo, dist_local(P, v)));
        }
        const int d = k < ks ? vi.y : 0;
        const int inc = warp_incl_scan(d);
        if (k < ks) {
          S3_CHK(koff + k, P.nloc);
          P.f[nxt][koff + k] = vi.z;
          P.frs[nxt][koff + k] = vi.x;
          P.fex[nxt][koff + k] = doff + inc - d;
        }
        doff += __shfl_sync(0xffffffffu, inc, 31);
      }
      koff += ks;
    }
  }
  __threadfence();
  __syncthreads();
  if (tid == 0) s_last = atomicAdd(&c->done_ctr, 1u) == gridDim.x - 1;
  __syncthreads();
  if (s_last && tid == 0) {  // every tile is done: this rank's totals to every rank
    __threadfence();
    const int n_next = ld_volatile(&c->n_next), e_next = ld_volatile(&c->e_next);
    for (int d = 0; d < P.dist_size; ++d) P.p_rtot[d][P.dist_rank] = make_int2(n_next, e_next);
    c->done_ctr = 0;
    c->tile_ctr = 0;
    __threadfence_system();
  }
}

// Fig1 L9-L11, L15-L16 over all ranks: the global totals end the loop; the local ones size P_l
// flag (optional, e.g. mapped pinned host memory): -1 once the traversal is done, else the
// next frontier's size over all ranks -- the driver reads it a few levels late, so levels are
// enqueued without a host round trip (levels enqueued past the end are no-ops)
__global__ void k_dist_advance(Params P, long long *flag) {
  if (threadIdx.x != 0) return;
  Ctl *c = P.ctl;
  if (c->tier == TIER_DONE) {
    if (flag) *(volatile long long *)flag = -1;
    return;
  }
  long long gn = 0, ge = 0;
  for (int s = 0; s < P.dist_size; ++s) {
    const int32_t *t = reinterpret_cast<const int32_t *>(P.rtot + s);
    gn += ld_volatile(t);
    ge += ld_volatile(t + 1);
  }
  const unsigned long long tt = globaltimer();
  record_stat(P, c, c->level, c->n_l, c->e_l, TIER_LARGE, c->p_l, 0, c->n_next, c->t_prev, tt);
  c->t_prev = tt;
  c->g_n_next = (int32_t)gn;
  c->g_e_next = (int32_t)(ge < 0x7fffffff ? ge : 0x7fffffff);
  c->m_visited += ge;  // arcs of all visited vertices (all ranks): k_explore's tag-mode rule
  c->level = c->level + 1;
  c->cur ^= 1;
  if (gn == 0) {
    c->n_l = 0;
    c->e_l = 0;
    c->tier = TIER_DONE;
    if (flag) *(volatile long long *)flag = -1;
    return;
  }
  if (flag) *(volatile long long *)flag = gn;
  decide_tier(P, c, c->n_next, c->e_next);
  if (c->tier == TIER_DONE) {  // no local work this level: one idle CTA keeps the protocol
    c->tier = TIER_LARGE;
    c->p_l = 1;
    c->chunk = 1;
    c->wcap = 1;
    c->pieces = 1;
    c->e_lo = 0;
    c->e_hi = 0;
  }
}

// level/parent (caller ids) of this rank's vertices; the others stay as the caller set them
__global__ void k_dist_finalize(Params P, int32_t *level, int32_t *parent) {
  for (long long lv = (long long)blockIdx.x * blockDim.x + threadIdx.x; lv < P.nloc;
       lv += (long long)gridDim.x * blockDim.x) {
    const int v = dist_global(P, (int)lv);
    if (v >= P.n) continue;
    if ((__ldg(P.bm + (v >> 5)) >> (v & 31)) & 1u) {
      const int o = P.n2o ? __ldg(P.n2o + v) : v;
      const int2 r = *lp_of(P.vinfo, lv);
      level[o] = r.x;
      parent[o] = r.y;
    }
  }
}

// create time: arcs per owner rank (receive block sizes), the local CSR (rows of this rank's
// vertices, global target ids) and its vertex records
__global__ void k_dist_rank_arcs(const int32_t *ro, int n, int G, unsigned long long *cnt) {
  unsigned long long acc[DIST_MAX] = {};
  for (long long v = (long long)blockIdx.x * blockDim.x + threadIdx.x; v < n;
       v += (long long)gridDim.x * blockDim.x)
    acc[(v >> 5) % G] += (unsigned long long)(ro[v + 1] - ro[v]);
  for (int d = 0; d < G; ++d)
    if (acc[d]) atomicAdd(cnt + d, acc[d]);
}
__global__ void k_dist_local_deg(Params P, const int32_t *ro, int32_t *deg_l) {
  for (long long lv = (long long)blockIdx.x * blockDim.x + threadIdx.x; lv < P.nloc;
       lv += (long long)gridDim.x * blockDim.x) {
    const int v = dist_global(P, (int)lv);
    deg_l[lv] = v < P.n ? ro[v + 1] - ro[v] : 0;
  }
}
__global__ void k_dist_copy_rows(Params P, const int32_t *ro, const int32_t *col,
                                 const int32_t *ro_l, int32_t *col_l) {
  const int lane = threadIdx.x & 31;
  const long long w0 = ((long long)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  const long long nw = ((long long)gridDim.x * blockDim.x) >> 5;
  for (long long lv = w0; lv < P.nloc; lv += nw) {
    const int v = dist_global(P, (int)lv);
    if (v >= P.n) continue;
    const int a = ro[v], d = ro[v + 1] - a, o = ro_l[lv];
    for (int k = lane; k < d; k += 32) col_l[o + k] = col[a + k];
  }
}
__global__ void k_dist_build_vinfo(Params P, const int32_t *ro_l, const int32_t *n2o,
                                   int4 *vinfo_l) {
  for (long long lv = (long long)blockIdx.x * blockDim.x + threadIdx.x; lv < P.nloc;
       lv += (long long)gridDim.x * blockDim.x) {
    const int v = dist_global(P, (int)lv);
    const int cid = v < P.n ? (n2o ? n2o[v] : v) : -1;
    vinfo_l[2 * lv] = make_int4(ro_l[lv], ro_l[lv + 1] - ro_l[lv], cid, 0);
    vinfo_l[2 * lv + 1] = make_int4(-1, -1, -1, 0);
  }
}

// ---- tier 0, warp path: consecutive tiny levels (n_l <= 32, e_l <= 32) ---------------------------
// Run by warp 0 of k_small alone, frontier in registers (lane u holds frontier vertex u), no
// CTA barrier: lane i takes edge i (its vertex by a 5-step shuffle search of the degree
// scan), loads col, then the visited word and the vertex record together.  Duplicates among
// the warp's lanes are removed by __match_any_sync -- the same "one copy survives" rule as
// the Owner check (R4), without the Owner round trip.  Returns when the next level is not
// tiny (or empty), leaving that frontier in shared memory and its (n, e, level) in st[].
__device__ void tiny_levels(const Params &P, Ctl *c, int32_t *sf, int32_t *srs, int32_t *sex,
                            int32_t *st, unsigned long long &t_prev, long long &m_add, int &nrec) {
  const int lane = threadIdx.x & 31;
  const int32_t *__restrict__ col = P.col;
  int n_l = st[0], e_l = st[1], L = st[2];
  const int lim_e = (P.t0 >= 0 && P.t0 < 32) ? P.t0 : 32;
  int fx = lane < n_l ? sf[lane] : 0;
  int frs = lane < n_l ? srs[lane] : 0;
  int fex = lane < n_l ? sex[lane] : 0x7fffffff;
  for (;;) {
    int u = 0;  // this lane's frontier slot (a one-vertex frontier, e.g. a path: slot 0)
    if (n_l > 1) {
#pragma unroll
      for (int s = 16; s >= 1; s >>= 1) {
        const int cu = __shfl_sync(0xffffffffu, fex, u + s);
        if (cu <= lane) u += s;
      }
    }
    const int px = __shfl_sync(0xffffffffu, fx, u);
    const int pr = __shfl_sync(0xffffffffu, frs, u);
    const int pe = __shfl_sync(0xffffffffu, fex, u);
    const bool has = lane < e_l;
    if (has) S3_CHK(pr + (lane - pe), P.nnz);
    const int v = has ? __ldg(col + pr + (lane - pe)) : 0;
    S3_CHK(v, P.n);
    const uint32_t w = __ldcg(P.bm + (v >> 5));      // published by atomicOr at L2
    // issued together with the bitmap word; through L2 (ld.global.cg), never the read-only
    // path: k_small's block levels store Owner into the same 16-byte record in this launch
    const int4 vi = __ldcg(P.vs16 + v);
    const bool fresh = has && !((w >> (v & 31)) & 1u);
    const unsigned fm = __ballot_sync(0xffffffffu, fresh);
    const int ncand = __popc(fm);
    bool keep = fresh;  // at most one fresh lane (a path level): nothing to deduplicate
    if (ncand > 1) {
      const unsigned mm = __match_any_sync(0xffffffffu, fresh ? v : -1 - lane);
      keep = fresh && lane == __ffs(mm) - 1;
    }
    const unsigned km = ncand > 1 ? __ballot_sync(0xffffffffu, keep) : fm;
    if (keep) {
      *lp_of(P.vinfo, v) = make_int2(L + 1, px);      // d[v] <- l, parent (Fig1 L18)
      atomicOr(P.bm + (v >> 5), 1u << (v & 31));      // exact visited bit
      mark_tag(P, v);
    }
    const int d = keep ? vi.y : 0;
    const int n_next = __popc(km);
    int e_next, nfx, nfr, nfe;
    if (n_next == 1) {  // one kept vertex (a path): no scan, one source lane
      const int src = __ffs(km) - 1;
      e_next = __shfl_sync(0xffffffffu, d, src);
      nfx = __shfl_sync(0xffffffffu, vi.z, src);
      nfr = __shfl_sync(0xffffffffu, vi.x, src);
      nfe = 0;
    } else {
      const int inc = warp_incl_scan(d);
      e_next = __shfl_sync(0xffffffffu, inc, 31);
      const int src = lane < n_next ? (int)__fns(km, 0, lane + 1) : 0;
      nfx = __shfl_sync(0xffffffffu, vi.z, src);
      nfr = __shfl_sync(0xffffffffu, vi.x, src);
      nfe = __shfl_sync(0xffffffffu, inc - d, src);
    }
    if (lane == 0) {
      const unsigned long long t = globaltimer();
      record_stat_at(P, nrec, L, n_l, e_l, TIER_SMALL, ncand, n_next, t_prev, t);
      t_prev = t;
      m_add += e_next;
    }
    fx = lane < n_next ? nfx : 0;
    frs = lane < n_next ? nfr : 0;
    fex = lane < n_next ? nfe : 0x7fffffff;
    ++L;
    n_l = n_next;
    e_l = e_next;
    // orders this level's bitmap atomics / tag and record stores before the next level's
    // probes by the other lanes (shuffles and votes do not order memory, PTX model)
    __syncwarp();
    if (n_l == 0 || e_l == 0 || n_l > 32 || e_l > lim_e) break;
  }
  if (lane < n_l) {
    sf[lane] = fx;
    srs[lane] = frs;
    sex[lane] = fex;
  }
  if (lane == 0) {
    sex[n_l] = e_l;
    st[0] = n_l;
    st[1] = e_l;
    st[2] = L;
  }
}

// ---- tier 0: k_small -------------------------------------------------------------------------
// One CTA runs consecutive tiny levels (e_l <= T0) with __syncthreads between the steps: the
// paper's "use only as many cores as there is work" at CTA granularity.  Same
// per-level contract as k_explore + k_compact; the owner label is the level-local edge
// index e (unique, R4); frontier, degree scan and candidates live in shared memory.
// The visited bitmap is exact at every level start (bits of kept vertices are published with
// atomicOr in the compaction step, after the discovery step), and this CTA's global writes
// are ordered for its own later reads by the CTA barrier (one SM), so multi-level operation
// is safe.
__global__ void __launch_bounds__(KS_THREADS, 1) k_small(Params P) {
  Ctl *c = P.ctl;
  if (c->tier != TIER_SMALL) return;
  extern __shared__ int32_t smem[];
  int32_t *sf = smem;                 // CurLevelVertices (caller ids)
  int32_t *srs = sf + KS_NCAP;        // internal row starts
  int32_t *sex = srs + KS_NCAP;       // exclusive degree scan, KS_NCAP + 1 entries
#if !S3BFS_KS_ONCHIP
  int32_t *cv = sex + KS_NCAP + 4;    // candidate per level-local edge (or -1)
  int32_t *cpv = cv + KS_ECAP;        // its discoverer
#endif                                // (S3BFS_KS_ONCHIP: this space is the Owner table)
  __shared__ int32_t s_wk[32], s_wd[32], s_wc[32];  // warp totals (entries past the warps: 0)
  __shared__ int32_t s_tot[3];
  __shared__ int32_t s_tiny[3];

  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int32_t *__restrict__ col = P.col;
  int4 *__restrict__ vinfo = P.vinfo;
  const uint32_t *__restrict__ bm = P.bm;
  int n_l = c->n_l, e_l = c->e_l, L = c->level;
  const int cur = c->cur;
  unsigned long long t_prev = c->t_prev;
  if (tid == 0 && L == 0) c->t_dbg[2] = globaltimer();
  long long m_add = 0;  // degrees of the frontiers created here (thread 0)
  int nrec = c->num_levels;  // stats records (thread 0), written back before decide()
  for (int i = tid; i < n_l; i += KS_THREADS) {
    sf[i] = P.f[cur][i];
    srs[i] = P.frs[cur][i];
    sex[i] = P.fex[cur][i];
  }
  if (tid == 0) sex[n_l] = e_l;
  if (KS_THREADS < 1024 && tid < 32 - KS_THREADS / 32) {
    s_wk[KS_THREADS / 32 + tid] = 0;
    s_wd[KS_THREADS / 32 + tid] = 0;
    s_wc[KS_THREADS / 32 + tid] = 0;
  }
  __syncthreads();

  for (;;) {
    if (n_l <= 32 && e_l <= 32) {  // tiny levels: warp 0 alone, no CTA barrier per level
      if (tid == 0) { s_tiny[0] = n_l; s_tiny[1] = e_l; s_tiny[2] = L; }
      __syncwarp();
      if (warp == 0) tiny_levels(P, c, sf, srs, sex, s_tiny, t_prev, m_add, nrec);
      __syncthreads();
      n_l = s_tiny[0];
      e_l = s_tiny[1];
      L = s_tiny[2];
      if (n_l == 0 || e_l == 0 || P.t0 < 0 || e_l > P.t0 || n_l > KS_NCAP) break;
      continue;
    }
    // (c)+(d): explore, edge e -> vertex u by binary search of the smem degree scan; a
    // thread's (<= KS_IPT) edges issue their col loads together, then their visited probes
    int ncand = 0;
    int ev[KS_IPT], ux[KS_IPT], lo[KS_IPT], hi[KS_IPT];
#pragma unroll
    for (int i = 0; i < KS_IPT; ++i) { lo[i] = 0; hi[i] = n_l; }
#pragma unroll
    for (int i = 0; i < KS_IPT; ++i) {
      const int e = tid + i * KS_THREADS;
      if (e < e_l) {
        while (hi[i] - lo[i] > 1) {
          const int mid = (lo[i] + hi[i]) >> 1;
          if (sex[mid] <= e) lo[i] = mid; else hi[i] = mid;
        }
      }
    }
#pragma unroll
    for (int i = 0; i < KS_IPT; ++i) {
      const int e = tid + i * KS_THREADS;
      ev[i] = -1;
      ux[i] = 0;
      if (e < e_l) {
        S3_CHK(lo[i], n_l);
        ux[i] = sf[lo[i]];
        S3_CHK(srs[lo[i]] + (e - sex[lo[i]]), P.nnz);
        ev[i] = __ldg(col + srs[lo[i]] + (e - sex[lo[i]]));
        S3_CHK(ev[i], P.n);
      }
    }
#if S3BFS_KS_ONCHIP
    // The visited word and the vertex record of every target in one round trip (both depend
    // only on the col entry; L1-bypassing: bits are published by atomicOr at L2, H2).
    uint32_t wv[KS_IPT];
    int4 rv[KS_IPT];
#pragma unroll
    for (int i = 0; i < KS_IPT; ++i) {
      wv[i] = ev[i] >= 0 ? __ldcg(bm + (ev[i] >> 5)) : 0xffffffffu;
      rv[i] = ev[i] >= 0 ? __ldcg(P.vs16 + ev[i]) : make_int4(0, 0, 0, 0);
    }
    uint32_t open = 0;  // this thread's candidates (visited bit clear) not yet decided
#pragma unroll
    for (int i = 0; i < KS_IPT; ++i)
      open |= (uint32_t)(ev[i] >= 0 && !((wv[i] >> (ev[i] & 31)) & 1u)) << i;
    ncand = __popc(open);
    // (e) Owner race on chip (Fig1 L20-L22; DESIGN R27): the Owner label of v lives in a
    // 2^14-entry shared table at slot h(v) & (2^14 - 1), stored as {h(v) >> 14, edge index} --
    // h a bijection of the 32-bit ids, so (slot, tag) names exactly one vertex.  Every copy
    // of v stores its label (plain stores, the benign race), then reads the slot back: the tag
    // of v means the race for v is decided (keep iff the label is this copy's); another tag
    // means another vertex took the slot, and v's copies race again with the next round's
    // hash.  Every copy of v sees the same slot state, so exactly one copy is kept.
    int32_t *tab = sex + KS_NCAP + 4;
    uint32_t km = 0;
    for (int r = 0;; ++r) {
#pragma unroll
      for (int i = 0; i < KS_IPT; ++i)
        if ((open >> i) & 1u) {
          const uint32_t h = ks_hash((uint32_t)ev[i], r);
          tab[h & (KS_TAB - 1)] = (int32_t)((h & ~(uint32_t)(KS_TAB - 1)) | (tid + i * KS_THREADS));
        }
      __syncthreads();
#pragma unroll
      for (int i = 0; i < KS_IPT; ++i)
        if ((open >> i) & 1u) {
          const uint32_t h = ks_hash((uint32_t)ev[i], r);
          const uint32_t t = (uint32_t)tab[h & (KS_TAB - 1)];
          if (((t ^ h) & ~(uint32_t)(KS_TAB - 1)) == 0) {  // v's own slot state: decided
            open &= ~(1u << i);
            if ((t & (KS_TAB - 1)) == (uint32_t)(tid + i * KS_THREADS)) km |= 1u << i;
          }
        }
      if (!__syncthreads_or(open != 0)) break;  // also orders this round's reads before the
    }                                            // next round's stores
    int kv[KS_IPT], kr[KS_IPT], kd[KS_IPT];
    int cnt = 0, dsum = 0;
#pragma unroll
    for (int i = 0; i < KS_IPT; ++i) {
      kv[i] = -1;
      kr[i] = 0;
      kd[i] = 0;
      if ((km >> i) & 1u) {
        const int v = ev[i];
        kv[i] = rv[i].z; kr[i] = rv[i].x; kd[i] = rv[i].y;
        *lp_of(vinfo, v) = make_int2(L + 1, ux[i]);  // d[v] <- l, parent (Fig1 L18)
        atomicOr(P.bm + (v >> 5), 1u << (v & 31));  // exact visited bit (not discovery)
        mark_tag(P, v);
      }
      cnt += kv[i] >= 0;
      dsum += kd[i];
    }
#else
    uint32_t wv[KS_IPT];
#pragma unroll
    for (int i = 0; i < KS_IPT; ++i)  // L1-bypassing: bits are published by atomicOr at L2 in
      wv[i] = ev[i] >= 0 ? __ldcg(bm + (ev[i] >> 5)) : 0xffffffffu;  // earlier levels (H2)
#pragma unroll
    for (int i = 0; i < KS_IPT; ++i) {
      const int e = tid + i * KS_THREADS;
      if (e < e_l) {
        const int v = ev[i];
        int w = -1;
        if (!((wv[i] >> (v & 31)) & 1u)) {
          st_weak(owner_of(vinfo, v), e);  // Owner[v] <- e (benign race)
          w = v;
          ++ncand;
        }
        S3_CHK(e, KS_ECAP);
        cv[e] = w;
        cpv[e] = ux[i];
      }
    }
    __syncthreads();
    // (e): owner check + next-level degree, blocked items for the scan
    const int ipt = (e_l + KS_THREADS - 1) / KS_THREADS;
    const int e0 = tid * ipt;
    int kv[KS_IPT], kr[KS_IPT], kd[KS_IPT];
    int cnt = 0, dsum = 0;
    int4 vis[KS_IPT];  // all record loads first (one round trip for the thread's items)
#pragma unroll
    for (int i = 0; i < KS_IPT; ++i) {
      const int e = e0 + i;
      const int v = (i < ipt && e < e_l) ? cv[e] : -1;
      kv[i] = v;
      vis[i] = v >= 0 ? ld_vrec_weak(vinfo, v) : make_int4(0, 0, 0, -1);  // same-SM: coherent
    }
#pragma unroll
    for (int i = 0; i < KS_IPT; ++i) {
      const int e = e0 + i;
      const int v = kv[i];
      kv[i] = -1;
      kr[i] = 0;
      kd[i] = 0;
      if (v >= 0 && vis[i].w == e) {
        kv[i] = vis[i].z; kr[i] = vis[i].x; kd[i] = vis[i].y;
        *lp_of(vinfo, v) = make_int2(L + 1, cpv[e]);  // d[v] <- l, parent (Fig1 L18)
        atomicOr(P.bm + (v >> 5), 1u << (v & 31));  // exact visited bit (not discovery)
        mark_tag(P, v);
      }
    }
#pragma unroll
    for (int i = 0; i < KS_IPT; ++i) {
      cnt += kv[i] >= 0;
      dsum += kd[i];
    }
#endif
    // block exclusive scan of (cnt, dsum)
    const int ik = warp_incl_scan(cnt), id = warp_incl_scan(dsum);
    const int wc = P.collect_stats ? warp_sum(ncand) : 0;
    if (lane == 31) { s_wk[warp] = ik; s_wd[warp] = id; }
    if (lane == 0) s_wc[warp] = wc;
    __syncthreads();
#if S3BFS_KS_SCAN1
    // every warp scans the 32 warp totals itself (one CTA barrier per scan instead of two; the
    // totals are rewritten only after the level's closing barrier)
    int kpos, dpos, n_next, e_next;
    {
      const int a = s_wk[lane], d = s_wd[lane];
      const int ia = warp_incl_scan(a), idd = warp_incl_scan(d);
      kpos = __shfl_sync(0xffffffffu, ia - a, warp) + ik - cnt;
      dpos = __shfl_sync(0xffffffffu, idd - d, warp) + id - dsum;
      n_next = __shfl_sync(0xffffffffu, ia, 31);
      e_next = __shfl_sync(0xffffffffu, idd, 31);
      if (warp == 0 && P.collect_stats) {
        const int ctot = warp_sum(s_wc[lane]);
        if (lane == 0) s_tot[2] = ctot;
      }
    }
#else
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
#endif
#pragma unroll
    for (int i = 0; i < KS_IPT; ++i) {
      if (kv[i] >= 0) {
        S3_CHK(kpos, KS_NCAP);
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
      record_stat_at(P, nrec, L, n_l, e_l, TIER_SMALL, s_tot[2], n_next, t_prev, t);
      t_prev = t;
      m_add += e_next;
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
    c->num_levels = nrec;
    c->level = L;
    c->t_prev = t_prev;
    c->m_visited += m_add;
    c->fb_valid = 0;
    c->bu = 0;
    decide(P, c, n_l, e_l);
  }
}

// ---- cluster tier: k_cluster ------------------------------------------------------------------
// SURVEY 8(a)/(f)'s optional middle tier: one thread-block cluster of KC_CL CTAs runs
// consecutive mid-size levels (T0 < e_l <= tc_max, n_l <= KC_FCAP) inside one launch -- no
// kernel launch and no captured-loop iteration per level, and KC_CL SMs instead of tier 0's
// one.  Every CTA holds the whole frontier in its shared memory (replicated through
// distributed shared memory); CTA r explores edges [r e_l / KC_CL, (r+1) e_l / KC_CL) with the
// k_small step (search of the degree scan, col, visited word, Owner = global edge index);
// after a cluster barrier it checks Owner through L2 (another SM wrote it), keeps its
// vertices, and the CTAs exchange their (kept, degree-sum) totals through DSMEM; each CTA then
// writes its kept vertices into every CTA's frontier (continuing) or into the global frontier
// (the level that leaves the tier).  Same per-level contract as k_small / k_explore+k_compact.
__global__ void __cluster_dims__(KC_CL, 1, 1) __launch_bounds__(KC_THREADS, 1) k_cluster(Params P) {
  namespace cg = cooperative_groups;
  cg::cluster_group cl = cg::this_cluster();
  Ctl *c = P.ctl;
  if (c->tier != TIER_CLUSTER) return;  // read before any CTA of the cluster can change it
  extern __shared__ int32_t smem[];
  int32_t *sf = smem;                 // frontier caller ids (replicated)
  int32_t *srs = sf + KC_FCAP;        // internal row starts
  int32_t *sex = srs + KC_FCAP;       // exclusive degree scan, KC_FCAP + 1 entries
  int32_t *cv = sex + KC_FCAP + 4;    // candidate per local edge (or -1)
  int32_t *cpv = cv + KC_ECTA;        // its discoverer (caller id)
  __shared__ int32_t s_wk[KC_THREADS / 32], s_wd[KC_THREADS / 32], s_wc[KC_THREADS / 32];
#if S3BFS_KC_PUSH
  __shared__ int32_t s_all[KC_CL][3];  // every CTA's (kept, degree sum, candidates), pushed here
#else
  __shared__ int32_t s_tot[3];        // this CTA's kept, degree sum, candidates
#endif
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int rank = (int)cl.block_rank();
  const int32_t *__restrict__ col = P.col;
  int4 *__restrict__ vinfo = P.vinfo;
  const uint32_t *__restrict__ bm = P.bm;
  int n_l = c->n_l, e_l = c->e_l, L = c->level;
  const int cur = c->cur, nxt = cur ^ 1;
  unsigned long long t_prev = c->t_prev;
  int nrec = c->num_levels;
  long long m_add = 0;
  for (int i = tid; i < n_l; i += KC_THREADS) {
    sf[i] = P.f[cur][i];
    srs[i] = P.frs[cur][i];
    sex[i] = P.fex[cur][i];
  }
  if (tid == 0) sex[n_l] = e_l;
  cl.sync();  // every CTA has read the control block and its frontier copy
  for (;;) {
    const int lo = (int)((long long)e_l * rank / KC_CL);
    const int ne = (int)((long long)e_l * (rank + 1) / KC_CL) - lo;  // <= KC_ECTA
    // (c)+(d): local edge k -> global edge lo + k -> frontier slot by binary search
    int ncand = 0;
    int ev[KC_IPT], ux[KC_IPT];
#pragma unroll
    for (int i = 0; i < KC_IPT; ++i) {
      const int k = tid + i * KC_THREADS;
      ev[i] = -1;
      ux[i] = 0;
      if (k < ne) {
        const int e = lo + k;
        int a = 0, z = n_l;
        while (z - a > 1) {
          const int mid = (a + z) >> 1;
          if (sex[mid] <= e) a = mid; else z = mid;
        }
        S3_CHK(a, n_l);
        ux[i] = sf[a];
        S3_CHK(srs[a] + (e - sex[a]), P.nnz);
        ev[i] = __ldg(col + srs[a] + (e - sex[a]));
        S3_CHK(ev[i], P.n);
      }
    }
    uint32_t wv[KC_IPT];
#pragma unroll
    for (int i = 0; i < KC_IPT; ++i) wv[i] = ev[i] >= 0 ? __ldcg(bm + (ev[i] >> 5)) : 0xffffffffu;
#pragma unroll
    for (int i = 0; i < KC_IPT; ++i) {
      const int k = tid + i * KC_THREADS;
      if (k < ne) {
        const int v = ev[i];
        int w = -1;
        if (!((wv[i] >> (v & 31)) & 1u)) {
          st_weak(owner_of(vinfo, v), lo + k);  // Owner[v] <- global edge index (benign race)
          w = v;
          ++ncand;
        }
        S3_CHK(k, KC_ECTA);
        cv[k] = w;
        cpv[k] = ux[i];
      }
    }
#if S3BFS_KC_FENCE
    __threadfence();
#endif
    cl.sync();  // its arrive is a release (MEMBAR.ALL.GPU in SASS): the Owner stores reach L2
                // before any CTA of the cluster checks them
    // (e): owner check through L2 (the winner may sit on another SM), blocked items
    const int ipt = (ne + KC_THREADS - 1) / KC_THREADS;
    const int k0 = tid * ipt;
    int kv[KC_IPT], kr[KC_IPT], kd[KC_IPT];
    int4 vis[KC_IPT];
#pragma unroll
    for (int i = 0; i < KC_IPT; ++i) {
      const int k = k0 + i;
      const int v = (i < ipt && k < ne) ? cv[k] : -1;
      kv[i] = v;
      vis[i] = v >= 0 ? ld_vrec_cg(P.vs16, vinfo, v) : make_int4(0, 0, 0, -1);
    }
    int cnt = 0, dsum = 0;
#pragma unroll
    for (int i = 0; i < KC_IPT; ++i) {
      const int k = k0 + i;
      const int v = kv[i];
      kv[i] = -1;
      kr[i] = 0;
      kd[i] = 0;
      if (v >= 0 && vis[i].w == lo + k) {
        kv[i] = vis[i].z; kr[i] = vis[i].x; kd[i] = vis[i].y;
        *lp_of(vinfo, v) = make_int2(L + 1, cpv[k]);  // d[v] <- l, parent (Fig1 L18)
        atomicOr(P.bm + (v >> 5), 1u << (v & 31));   // exact visited bit (not discovery)
        mark_tag(P, v);
        ++cnt;
        dsum += kd[i];
      }
    }
    // CTA scan of (cnt, dsum)
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
#if S3BFS_KC_PUSH
      const int tk = __shfl_sync(0xffffffffu, ia, 31), td = __shfl_sync(0xffffffffu, idd, 31);
      if (lane < KC_CL) {  // lane r pushes the totals into CTA r's table (DSMEM stores)
        int32_t *t = cl.map_shared_rank(&s_all[rank][0], lane);
        t[0] = tk; t[1] = td; t[2] = ctot;
      }
#else
      if (lane == 31) { s_tot[0] = ia; s_tot[1] = idd; s_tot[2] = ctot; }
#endif
    }
    cl.sync();  // every CTA's totals are published (DSMEM)
    int koff = 0, doff = 0, n_next = 0, e_next = 0, c_all = 0;
#pragma unroll
    for (int r = 0; r < KC_CL; ++r) {  // the cluster's exclusive scan over CTA totals
#if S3BFS_KC_PUSH
      const int32_t *t = &s_all[r][0];
#else
      const int32_t *t = cl.map_shared_rank(s_tot, r);
#endif
      const int k = t[0], d = t[1];
      if (r < rank) { koff += k; doff += d; }
      n_next += k;
      e_next += d;
      c_all += t[2];
    }
    const bool stay = n_next > 0 && e_next > 0 && e_next > P.t0 && e_next <= P.tc_max &&
                      n_next <= KC_FCAP;
    int kpos = koff + s_wk[warp] + ik - cnt, dpos = doff + s_wd[warp] + id - dsum;
#pragma unroll
    for (int i = 0; i < KC_IPT; ++i) {
      if (kv[i] >= 0) {
        S3_CHK(kpos, stay ? KC_FCAP : P.n);
        if (stay) {  // the next level stays here: write every CTA's frontier copy
#pragma unroll
          for (int r = 0; r < KC_CL; ++r) {
            cl.map_shared_rank(sf, r)[kpos] = kv[i];
            cl.map_shared_rank(srs, r)[kpos] = kr[i];
            cl.map_shared_rank(sex, r)[kpos] = dpos;
          }
        } else {     // the level leaves the tier: the global frontier for the next tier
          P.f[nxt][kpos] = kv[i];
          P.frs[nxt][kpos] = kr[i];
          P.fex[nxt][kpos] = dpos;
        }
        ++kpos;
        dpos += kd[i];
      }
    }
    if (tid == 0) {
      if (stay) sex[n_next] = e_next;
      else if (rank == 0) P.fex[nxt][n_next] = e_next;
    }
    if (rank == 0 && tid == 0) {
      const unsigned long long t = globaltimer();
      record_stat_at(P, nrec, L, n_l, e_l, TIER_CLUSTER, c_all, n_next, t_prev, t);
      t_prev = t;
      m_add += e_next;
    }
    cl.sync();  // frontier copies complete (and every CTA done with the old ones)
    ++L;
    n_l = n_next;
    e_l = e_next;
    if (!stay) break;
  }
  if (rank == 0 && tid == 0) {  // leave the tier: hand over the control block
    __threadfence();
    c->num_levels = nrec;
    c->level = L;
    c->cur = nxt;
    c->t_prev = t_prev;
    c->m_visited += m_add;
    c->fb_valid = 0;
    c->bu = 0;
    decide(P, c, n_l, e_l);
  }
}

// ---- NEXT-3: direction-optimising bottom-up level (P:131 names it as compatible) --------------
// Beamer's bottom-up step over the same state: every vertex not yet visited looks for a
// neighbour in the current frontier (a bitmap), stopping at the first one.  The frontier
// bitmap is built from the frontier list when the previous level was top-down.
__global__ void k_fb_clear(Params P) {
  Ctl *c = P.ctl;
  if (c->tier != TIER_BU) return;
  const long long gs = (long long)gridDim.x * blockDim.x;
  const long long g = (long long)blockIdx.x * blockDim.x + threadIdx.x;
  for (long long i = g; i < P.bu_tiles; i += gs) P.bu_status[i] = 0ull;  // k_bottom_up's look-back
  if (c->fb_valid) return;
  const long long nw4 = ((long long)P.n + 127) >> 7;
  uint4 *fb = reinterpret_cast<uint4 *>(P.fb[c->cur]);
  for (long long i = g; i < nw4; i += gs) fb[i] = make_uint4(0, 0, 0, 0);
}
__global__ void k_fb_set(Params P) {
  Ctl *c = P.ctl;
  if (c->tier != TIER_BU || c->fb_valid) return;
  const int n_l = c->n_l;
  const int32_t *f = P.f[c->cur];
  uint32_t *fb = P.fb[c->cur];
  for (long long u = (long long)blockIdx.x * blockDim.x + threadIdx.x; u < n_l;
       u += (long long)gridDim.x * blockDim.x) {
    const int o = f[u];
    S3_CHK(o, P.n);
    const int i = P.o2n ? __ldg(P.o2n + o) : o;
    S3_CHK(i, P.n);
    atomicOr(fb + (i >> 5), 1u << (i & 31));  // frontier membership (not the discovery path)
  }
}
// One warp per visited-bitmap word (32 consecutive internal ids); the warp owns the word, so
// the visited word and the next frontier's bitmap word are written with plain stores and no
// vertex can be found twice (no Owner dedup needed).  CTA b takes a contiguous range of
// words; found vertices are compacted into the next frontier list with the same decoupled
// look-back (kept, degree-sum) scan as k_compact.
__global__ void __launch_bounds__(KD_THREADS, KD_MIN_BLOCKS) k_bottom_up(Params P) {
  Ctl *c = P.ctl;
  if (c->tier != TIER_BU) return;
  __shared__ int32_t s_k[KD_WARPS], s_d[KD_WARPS];
  __shared__ int s_last, s_tile;
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int nb = gridDim.x, nt = P.bu_tiles;
  const int cur = c->cur, nxt = cur ^ 1;
  const int new_level = c->level + 1;
  const int4 *__restrict__ vinfo = P.vinfo;
  const uint32_t *__restrict__ fbc = P.fb[cur];
  uint32_t *__restrict__ fbn = P.fb[nxt];
  uint32_t *__restrict__ bm = P.bm;
  const int nwords = (int)((((long long)P.n + 127) >> 7) << 2);
  const int nscan = P.n_scan;
  // Tiles of bu_tile_w bitmap words (about S3BFS_BU_TILES_PER_CTA per resident CTA, >= 64),
  // taken in start order by the resident CTAs until none is
  // left: a tile of long fruitless scans (vertices with no frontier in-neighbour read their
  // whole row) holds up one CTA, not the grid (CTA-sized fixed ranges left most warps waiting
  // at the look-back barrier).
  for (;;) {
  if (tid == 0) s_tile = (int)atomicAdd(&c->tile_ctr, 1u);  // look-back order = start order
  __syncthreads();
  const int b = s_tile;
  if (b >= nt) break;
  const int w0 = min(b * P.bu_tile_w, nwords), w1 = min(w0 + P.bu_tile_w, nwords);
  if (b == 0 && tid == 0) c->t_kx_begin = globaltimer();
  // pass 1: BU_W words per warp round (BU_W independent probe chains per lane); every round
  // probes the next BU_P in-neighbours of each unresolved vertex, loads issued together
  int kept = 0, dsum = 0;
  for (int wb = w0 + warp * BU_W; wb < w1; wb += KD_WARPS * BU_W) {
    uint32_t bw[BU_W];
    int r0[BU_W], r1[BU_W], dg[BU_W], pu[BU_W];
#pragma unroll
    for (int i = 0; i < BU_W; ++i) {
      const int w = wb + i;
      const int v = (w << 5) + lane;
      bw[i] = (w < w1) ? bm[w] : 0xffffffffu;
      const bool act = w < w1 && v < nscan && !((bw[i] >> lane) & 1u);
      r0[i] = act ? __ldg(P.tro + v) : 0;
      r1[i] = act ? __ldg(P.tro + v + 1) : 0;
      dg[i] = act ? __ldg(P.vs16 + v).y : 0;  // out-degree: the next level's e_l (Fig1 L13)
      pu[i] = -1;
    }
    for (;;) {  // rounds until every vertex found a frontier in-neighbour or ran out of them
      bool more = false;
#pragma unroll
      for (int i = 0; i < BU_W; ++i) more |= r0[i] < r1[i];
      if (!__any_sync(0xffffffffu, more)) break;
      int u[BU_W][BU_P];
#pragma unroll
      for (int i = 0; i < BU_W; ++i)
#pragma unroll
        for (int j = 0; j < BU_P; ++j)
          u[i][j] = (r0[i] + j < r1[i]) ? __ldg(P.tcol + r0[i] + j) : -1;
#if S3BFS_CHECK
#pragma unroll
      for (int i = 0; i < BU_W; ++i)
#pragma unroll
        for (int j = 0; j < BU_P; ++j) {
          if (r0[i] + j < r1[i]) S3_CHK(r0[i] + j, P.nnz);
          if (u[i][j] >= 0) S3_CHK(u[i][j], P.n);
        }
#endif
      uint32_t fw[BU_W][BU_P];
#pragma unroll
      for (int i = 0; i < BU_W; ++i)
#pragma unroll
        for (int j = 0; j < BU_P; ++j)
          fw[i][j] = (u[i][j] >= 0) ? __ldg(fbc + (u[i][j] >> 5)) : 0u;
#pragma unroll
      for (int i = 0; i < BU_W; ++i) {
#pragma unroll
        for (int j = BU_P - 1; j >= 0; --j)  // the first hit in row order wins
          if (u[i][j] >= 0 && ((fw[i][j] >> (u[i][j] & 31)) & 1u)) pu[i] = u[i][j];
        r0[i] = (pu[i] >= 0) ? r1[i] : r0[i] + BU_P;
      }
    }
#pragma unroll
    for (int i = 0; i < BU_W; ++i) {
      const int w = wb + i;
      const int v = (w << 5) + lane;
      const bool found = pu[i] >= 0;
      if (found) {
        P.lpd[v] = make_int2(new_level, __ldg(P.vs16 + pu[i]).z);  // d, parent (caller id)
        mark_tag(P, v);
      }
      const unsigned m = __ballot_sync(0xffffffffu, found);
      if (lane == 0 && w < w1) {
        if (m) {
          bm[w] = bw[i] | m;        // this warp owns word w
          atomicOr(P.bub + w, m);   // these vertices' labels are in lpd (fire-and-forget OR:
                                    // earlier bottom-up levels' bits stay; no discovery race
                                    // exists in this step, R17 concerns the top-down path)
        }
        fbn[w] = m;
      }
      kept += __popc(m);
      dsum += found ? dg[i] : 0;
    }
  }
  dsum = warp_sum(dsum);
  if (lane == 0) { s_k[warp] = kept; s_d[warp] = dsum; }
  __syncthreads();
  if (warp == 0) {
    const int kk = lane < KD_WARPS ? s_k[lane] : 0;
    const int dd = lane < KD_WARPS ? s_d[lane] : 0;
    const int ik = warp_incl_scan(kk), id = warp_incl_scan(dd);
    const Pair agg{(uint32_t)__shfl_sync(0xffffffffu, ik, 31),
                   (uint32_t)__shfl_sync(0xffffffffu, id, 31)};
    const Pair ex = lookback<true>(P.bu_status, b, agg);
    if (lane < KD_WARPS) {
      s_k[lane] = (int)ex.a + ik - kk;
      s_d[lane] = (int)ex.b + id - dd;
    }
    if (b == nt - 1 && lane == 0) {
      const int n_next = (int)(ex.a + agg.a), e_next = (int)(ex.b + agg.b);
      c->n_next = n_next;
      c->e_next = e_next;
      P.fex[nxt][n_next] = e_next;
    }
  }
  __syncthreads();
  // pass 2: the warp's found vertices (its own fbn words) into the next frontier list
  int koff = s_k[warp], doff = s_d[warp];
  for (int wb = w0 + warp * BU_W; wb < w1; wb += KD_WARPS * BU_W)
  for (int w = wb; w < min(wb + BU_W, w1); ++w) {
    const uint32_t m = fbn[w];
    if (!m) continue;
    const bool mine = (m >> lane) & 1u;
    const int4 vi = mine ? __ldg(P.vs16 + (w << 5) + lane) : make_int4(0, 0, 0, 0);
    const int d = mine ? vi.y : 0;
    const int inc = warp_incl_scan(d);
    const int pos = koff + __popc(m & lanemask_lt());
    if (mine) {
      S3_CHK(pos, P.n);
      P.f[nxt][pos] = vi.z;
      P.frs[nxt][pos] = vi.x;
      P.fex[nxt][pos] = doff + inc - d;
    }
    koff += __popc(m);
    doff += __shfl_sync(0xffffffffu, inc, 31);
  }
  __syncthreads();  // s_tile, s_k, s_d are reused by the next tile
  }  // tiles
  __threadfence();
  __syncthreads();
  if (tid == 0) s_last = atomicAdd(&c->done_ctr, 1u) == (unsigned)(nb - 1);
  __syncthreads();
  if (s_last && tid == 0) {
    __threadfence();
    const int n_next = ld_volatile(&c->n_next), e_next = ld_volatile(&c->e_next);
    const unsigned long long t = globaltimer();
    record_stat(P, c, c->level, c->n_l, c->e_l, TIER_BU, nb, n_next, n_next, c->t_prev, t,
                *(volatile unsigned long long *)&c->t_kx_begin, t);
    c->done_ctr = 0;
    c->tile_ctr = 0;
    c->t_prev = t;
    c->level = c->level + 1;
    c->cur = nxt;
    c->m_visited += e_next;
    c->fb_valid = 1;
    decide(P, c, n_next, e_next);
  }
}

// ---- d[0:n-1] in caller ids --------------------------------------------------------------
// level[o] = d of internal vertex o2n[o] if its visited bit is set, else -1 (unreachable, R1);
// parent[o] = its recorded parent (a caller id, R2).  Reads the internal records in caller
// order; the caller's arrays are written exactly once, coalesced.
// BU = the direction-optimising handle's instance (NEXT-3: vertices a bottom-up level found
// carry their labels in the dense lpd array, bub says which); the top-down handle's instance
// has none of it
template <bool BU>
__global__ void k_finalize(Params P) {
  const Ctl *c = P.ctl;
  int32_t *__restrict__ level = c->level_out;
  int32_t *__restrict__ parent = c->parent_out;
  const int n = P.n;
  for (long long o = (long long)blockIdx.x * blockDim.x + threadIdx.x; o < n;
       o += (long long)gridDim.x * blockDim.x) {
    const int i = P.o2n ? __ldg(P.o2n + o) : (int)o;
    S3_CHK(i, P.n);
    int lv = -1, pa = -1;
    if ((__ldg(P.bm + (i >> 5)) >> (i & 31)) & 1u) {
      const bool bu = BU && ((__ldg(P.bub + (i >> 5)) >> (i & 31)) & 1u);  // NEXT-3 label
      const int2 r = bu ? __ldg(P.lpd + i)
                        : __ldg(reinterpret_cast<const int2 *>(vstat(P.vinfo, i) + 1));
      lv = r.x;
      pa = r.y;
    }
    level[o] = lv;
    parent[o] = pa;
  }
}

// ---- create-time graph preparation (not on the traversal path) --------------------------------
__global__ void k_degrees(const int32_t *ro, int n, int32_t *deg, int32_t *iota) {
  for (long long i = (long long)blockIdx.x * blockDim.x + threadIdx.x; i < n;
       i += (long long)gridDim.x * blockDim.x) {
    deg[i] = ro[i + 1] - ro[i];
    iota[i] = (int32_t)i;
  }
}
__global__ void k_inverse_perm(const int32_t *n2o, int n, int32_t *o2n, const int32_t *ro,
                               int32_t *deg2) {
  for (long long i = (long long)blockIdx.x * blockDim.x + threadIdx.x; i < n;
       i += (long long)gridDim.x * blockDim.x) {
    const int o = n2o[i];
    o2n[o] = (int32_t)i;
    deg2[i] = ro[o + 1] - ro[o];
  }
}
// one warp per internal row: col2[ro2[i] + j] = o2n[col[ro[n2o[i]] + j]]
__global__ void k_relabel_rows(const int32_t *ro, const int32_t *col, const int32_t *n2o,
                               const int32_t *o2n, const int32_t *ro2, int n, int32_t *col2) {
  const int lane = threadIdx.x & 31;
  const long long w0 = ((long long)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  const long long ws = ((long long)gridDim.x * blockDim.x) >> 5;
  for (long long i = w0; i < n; i += ws) {
    const int o = n2o[i];
    const int s = ro[o], len = ro[o + 1] - s, d = ro2[i];
    for (int j = lane; j < len; j += 32) col2[d + j] = o2n[col[s + j]];
  }
}
// symmetry test of the arc multiset (create time, NEXT-3): sums of a 64-bit hash of (u, v)
// and of (v, u) over all arcs -- equal iff the multiset is symmetric (with prob. 1 - 2^-64)
__device__ __forceinline__ unsigned long long mix64(unsigned long long z) {
  z += 0x9e3779b97f4a7c15ull;
  z = (z ^ (z >> 30)) * 0xbf58476d1ce4e5b9ull;
  z = (z ^ (z >> 27)) * 0x94d049bb133111ebull;
  return z ^ (z >> 31);
}
__global__ void k_sym_hash(const int32_t *ro, const int32_t *col, int n,
                           unsigned long long *out) {
  const int lane = threadIdx.x & 31;
  unsigned long long a = 0, b = 0;
  for (long long u = ((long long)blockIdx.x * blockDim.x + threadIdx.x) >> 5; u < n;
       u += ((long long)gridDim.x * blockDim.x) >> 5) {
    for (int k = ro[u] + lane; k < ro[u + 1]; k += 32) {
      const unsigned long long v = (unsigned)col[k];
      a += mix64(((unsigned long long)u << 32) | v);
      b += mix64((v << 32) | (unsigned long long)u);
    }
  }
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) {
    a += __shfl_xor_sync(0xffffffffu, a, o);
    b += __shfl_xor_sync(0xffffffffu, b, o);
  }
  if (lane == 0) { atomicAdd(out, a); atomicAdd(out + 1, b); }
}
// transpose (in-adjacency): in-degree count, then scatter (create time, order irrelevant)
__global__ void k_in_degree(const int32_t *ro, const int32_t *col, int n, int32_t *tdeg) {
  const int lane = threadIdx.x & 31;
  for (long long u = ((long long)blockIdx.x * blockDim.x + threadIdx.x) >> 5; u < n;
       u += ((long long)gridDim.x * blockDim.x) >> 5)
    for (int k = ro[u] + lane; k < ro[u + 1]; k += 32) atomicAdd(tdeg + col[k], 1);
}
__global__ void k_transpose(const int32_t *ro, const int32_t *col, int n, int32_t *cursor,
                            int32_t *tcol) {
  const int lane = threadIdx.x & 31;
  for (long long u = ((long long)blockIdx.x * blockDim.x + threadIdx.x) >> 5; u < n;
       u += ((long long)gridDim.x * blockDim.x) >> 5)
    for (int k = ro[u] + lane; k < ro[u + 1]; k += 32) tcol[atomicAdd(cursor + col[k], 1)] = (int)u;
}
// number of vertices with degree > 0 (create time; with the degree order they are a prefix)
__global__ void k_count_nonzero(const int32_t *deg, int n, int *out) {
  int c = 0;
  for (long long i = (long long)blockIdx.x * blockDim.x + threadIdx.x; i < n;
       i += (long long)gridDim.x * blockDim.x)
    c += deg[i] > 0;
  c = warp_sum(c);
  if ((threadIdx.x & 31) == 0 && c) atomicAdd(out, c);
}
// the vertex records (Params::vinfo) over a CSR's row offsets: static half, dynamic half reset
__global__ void k_build_vinfo(const int32_t *ro, const int32_t *n2o, int n, int4 *vinfo,
                              int4 *vs16) {
  for (long long i = (long long)blockIdx.x * blockDim.x + threadIdx.x; i < n;
       i += (long long)gridDim.x * blockDim.x) {
    const int4 st = make_int4(ro[i], ro[i + 1] - ro[i], n2o ? n2o[i] : (int)i, 0);
    vinfo[2 * i] = st;
    vinfo[2 * i + 1] = make_int4(-1, -1, 0, 0);
    vs16[i] = st;
  }
}

// ---- test entry kernels ---------------------------------------------------------------------
// (b) alone: tiles of SCAN_TILE int32 in blocked order, block scan + decoupled look-back.
__global__ void __launch_bounds__(SCAN_THREADS) k_scan_u32(const int32_t *__restrict__ in,
                                                           int32_t *__restrict__ out, int n,
                                                           unsigned long long *status) {
  // status[0, gridDim.x) = look-back words, status[gridDim.x] = tile counter (all zeroed by
  // the caller): tiles are numbered in CTA start order, so a spinning CTA only ever waits for
  // CTAs that already started (forward progress next to concurrent traversals, as k_compact)
  __shared__ int32_t s_w[SCAN_THREADS / 32];
  __shared__ uint32_t s_ex;
  __shared__ int s_tile;
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  if (tid == 0)
    s_tile = (int)atomicAdd(reinterpret_cast<unsigned int *>(status + gridDim.x), 1u);
  __syncthreads();
  const int tile = s_tile;
  const long long base = (long long)tile * SCAN_TILE + (long long)tid * SCAN_ITEMS;
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
    const Pair ex = lookback<false>(status, tile, agg);
    if (lane == 0) s_ex = ex.a;
    if (lane == 0 && tile == (int)gridDim.x - 1) out[n] = (int)(ex.a + agg.a);
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
__global__ void k_poison(int4 *vinfo, int n, int range) {
  const long long gs = (long long)gridDim.x * blockDim.x;
  for (long long i = (long long)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += gs)
    vinfo[2 * i + 1] = make_int4(0x5a5a5a5a, 0x5a5a5a5a,  // {d, parent} garbage until written
                                 (int32_t)(((unsigned)i * 2654435761u) % (unsigned)max(range, 1)), 0);
}

}  // namespace s3bfs
