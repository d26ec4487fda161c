/*
 * include/s3bfs.h -- C ABI of the B200-native S3BFS frontier-expansion path.
 *
 * The library (paper_2209_08764_b200/libs3bfs.so, sources in paper_2209_08764_b200/csrc/)
 * runs the level-synchronous BFS of PAPER.md Figure 1, "Parallel-BFS(s, P) ... Returns
 * d[0:n-1]", on one B200 (sm_100a).  "P:n" below = /root/reference/PAPER.md line n;
 * "Fig1 Lk" = item k of the Figure 1 enumerate (SURVEY.md section 0 maps items to lines);
 * "S:n" = /root/reference/SPEC.md line n (interfaces only).  DESIGN.md lists every reading.
 *
 * Per level the path runs, entirely on the device:
 *   (a) frontier degree gather            Fig1 L12-L13
 *   (b) exclusive prefix sum of degrees   Fig1 L14-L15, Blelloch
 *   (c) equal-work edge split (search)    Fig1 L17
 *   (d) explore + level/parent/owner      Fig1 L18, benign race, no atomics
 *   (e) owner dedup + compaction          Fig1 L19-L29
 *   (f) level-adaptive launch sizing      P_l = min(P, W) (Fig1 L11, L16)
 * (a)+(b) are fused into (e)'s write-out of the next frontier; (c) is fused into (d).
 *
 * Conventions (all entry points):
 *   - Graph: int32 CSR out-adjacency, row_offsets[n+1], col_indices[nnz].  Every
 *     arc (u, v) is explored from u.  Multigraphs and self-loops are allowed (DESIGN R14).
 *   - Output: level[v] = hop distance d(s, v), -1 if unreachable (DESIGN R1, the paper's
 *     d <- infinity, Fig1 L3); parent[s] = s, parent[v] = some u with (u, v) an arc and
 *     level[u] = level[v] - 1, parent[v] = -1 if unreachable (DESIGN R2; not in the paper).
 *   - Errors: every call returns an s3bfs_status; nothing throws or aborts across the ABI.
 *     s3bfs_last_error() gives the detail of the last failure on a handle.
 *   - Asynchrony: s3bfs_run only ENQUEUES work on `stream`; results are valid once the caller
 *     synchronises that stream.  One traversal at a time per handle.
 */
#ifndef S3BFS_H_
#define S3BFS_H_

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

/* CUDA stream handle as an opaque pointer (identical to cudaStream_t; NULL = legacy stream).
 * Declared here so this header needs no CUDA include. */
typedef void *s3bfs_stream_t;

typedef struct s3bfs_ctx *s3bfs_handle; /* opaque */

typedef enum {
  S3BFS_OK = 0,
  S3BFS_ERR_INVALID_ARGUMENT = 1, /* null / non-device pointer, n <= 0, nnz out of range,
                                     source not in [0, n) */
  S3BFS_ERR_UNSUPPORTED = 2,      /* device is not compute capability 10.x, or a size the
                                     int32 index words cannot address */
  S3BFS_ERR_OUT_OF_MEMORY = 3,    /* workspace allocation failed */
  S3BFS_ERR_CUDA = 4,             /* a CUDA runtime/driver error; detail in s3bfs_last_error */
  S3BFS_ERR_INVALID_GRAPH = 5     /* validate_csr found a CSR invariant violated */
} s3bfs_status;

/* Options.  A zero-initialised struct (or NULL) selects every default.  Mirrors the
 * paper's tunables: P (max cores) and GRAINSIZE, and the work-insensitive
 * comparison variant. */
typedef struct {
  int32_t edges_per_cta;   /* grain of (f): P_l = min(P_max, ceil(e_l / grain)).  0 -> 1024 */
  int32_t tier0_max_edges; /* T0: a level with e_l <= T0 (and n_l <= 8192) runs in the
                              single-CTA tier.  0 -> 8192 (the maximum); < 0 -> tier 0 off */
  int32_t loop_mode;       /* 0/1: level loop captured in a CUDA graph (WHILE + SWITCH nodes);
                              2: host-driven loop (one device->host read per level; run then
                              blocks until the traversal ends) */
  int32_t collect_stats;   /* 0/1: per-level statistics on; -1: off */
  int32_t validate_csr;    /* 1: s3bfs_create checks row_offsets/col_indices on the device */
  int32_t variant;         /* 0: work-sensitive (paper's S3BFS); 1: work-insensitive -- every
                              level uses the full grid P_max and tier 0 is off */
  int32_t max_ctas;        /* cap on P_max (the paper's P); 0 -> SMs x resident CTAs/SM */
  int32_t debug_poison;    /* 1: fill the internal Owner array with garbage at create, to
                              prove it is never read before written (DESIGN R3) */
  int32_t time_kernels;    /* 1 (host-loop mode only): bracket every kernel launch with CUDA
                              events on the run's stream; read by s3bfs_get_kernel_times */
  int32_t reorder;         /* 0/1: create builds an internal copy of the graph relabelled by
                              descending degree (outputs stay in caller ids); -1: traverse the
                              caller's arrays directly (no copy) */
  int32_t direction;       /* NEXT-3: 1 = direction-optimising -- a level runs
                              bottom-up when e_l * alpha > arcs of unvisited vertices, and returns
                              top-down when n_l * beta < n (Beamer); 0 = top-down S3BFS only */
  int32_t do_alpha;        /* 0 -> 14 */
  int32_t do_beta;         /* 0 -> 24; < 0 -> never switch back */
  int32_t dist_size;       /* NEXT-4: 0/1 single GPU; G in [2, 8]: this handle is rank dist_rank
                              of a 1-D vertex partition over G ranks: it owns the
                              internal ids v with (v / 32) mod G == dist_rank, their CSR rows and
                              their state; driven by the s3bfs_dist_* calls below, not s3bfs_run.
                              Every level runs on tier 1; direction must be 0; no clones */
  int32_t dist_rank;       /* NEXT-4: 0 <= dist_rank < dist_size */
  int32_t cluster_max_edges; /* cluster tier (one 8-CTA thread-block cluster running
                              consecutive levels with T0 < e_l <= this and n_l <= 8192 in one
                              launch).  0 -> 32768 (the maximum); < 0 -> off.  With it on, the
                              default T0 (tier0_max_edges = 0) is 2048 */
  int32_t hub_vertices;    /* visited test of k_explore (Fig1 L18 "if d[v] = infinity"): internal
                              ids below this count (the highest-degree vertices, whose visited
                              bits stay L1-resident) are tested in the visited bitmap first, all
                              others directly by their 1-byte discovery tag (one probe).  0 ->
                              the default (2^19); < 0 -> every vertex through the bitmap first */
  int32_t tag_mode_pct;    /* that split ("tag mode") is used on a level while fewer than this
                              percentage of all arcs end at visited vertices (the discovery-heavy
                              levels); other levels test every target's visited bit first.
                              0 -> the default (80); > 100 -> every level; < 0 -> never */
  int32_t split_min_edges; /* level passes (Fig1 L18's "d[v] = infinity" state refreshed inside a
                              level): a tier-1 level of at least this many edges whose visited
                              test is in tag mode runs as consecutive passes over its edge range,
                              each a complete explore + dedup that publishes its discoveries'
                              visited bits and appends its survivors to the next frontier; the
                              level's result is the same.  0 -> the default; < 0 -> never */
  int32_t split_first_pct; /* the first pass's share of the level's edges, percent (0 -> default) */
  int32_t split_passes;    /* passes per such level (the rest of the edges is divided evenly
                              over the later passes).  0 -> the default; 1 -> never split */
} s3bfs_options;

/* One record per BFS level (the SPEC LevelStats analogue).  n_l = |frontier|
 * (Fig1 L9), e_l = sum of its degrees (Fig1 L15), tier 0 = single CTA, 1 = full kernels,
 * 2 = a last level with e_l = 0 (nothing explored), 3 = bottom-up (NEXT-3), grid = CTAs used
 * (P_l; tier 4 = the cluster tier, grid = its CTAs), candidates =
 * discoveries incl. benign-race duplicates, kept = n_{l+1} after owner dedup.  Times are
 * %globaltimer ns: level start (= previous level's end, so launch gaps count) and end; for
 * tier 1 also k_explore's start (its CTA 0) and k_compact's start (its CTA 0), whose
 * difference is the exploration kernel's duration inside the captured loop (0 for tier 0).
 * A tier-1 level that ran as several passes (s3bfs_options.split_*) is still ONE record:
 * candidates and kept summed over the passes, grid = the last pass's P_l, pad = the number of
 * passes, t_explore_end_ns - t_explore_begin_ns = the passes' summed k_explore durations. */
typedef struct {
  int32_t level, n_l, e_l, tier, grid, candidates, kept, pad;
  uint64_t t_begin_ns, t_end_ns;
  uint64_t t_explore_begin_ns, t_explore_end_ns;
} s3bfs_level_stat;

/* Create a traversal context over a CSR graph already resident in device memory.
 * row_offsets: device, n+1 int32, BORROWED (caller keeps it alive and unmodified until
 * destroy).  col_indices: device, nnz int32, borrowed (may be NULL iff nnz == 0).
 * Requires 1 <= n <= INT32_MAX - 256, 0 <= nnz <= INT32_MAX - workspace slack.  The handle owns its
 * workspace (per-vertex records, two frontier buffers, candidate buffer, visited bitmap, claim
 * tags, control block, stats) and, unless opts->reorder < 0, a degree-ordered internal copy
 * of the graph (4 nnz + 8 n more bytes), built here on `stream`.
 * May synchronise `stream`.  On failure *out is set to NULL. */
s3bfs_status s3bfs_create(s3bfs_handle *out, int32_t n, int64_t nnz, const int32_t *row_offsets,
                          const int32_t *col_indices, const s3bfs_options *opts,
                          s3bfs_stream_t stream);

/* NEXT-2 (multi-source throughput): a new handle over src's prepared graph (the internal
 * degree-ordered copy and in-adjacency are shared, reference-counted; the workspace is the
 * clone's own), so K handles can run K traversals concurrently on K streams.  Same options
 * as src.  src may be destroyed before its clones.  May synchronise `stream`. */
s3bfs_status s3bfs_clone(s3bfs_handle src, s3bfs_handle *out, s3bfs_stream_t stream);

/* Parallel-BFS(s, P): enqueue one traversal from `source` on `stream`.
 * level, parent: device, n int32 each, caller-owned, FULLY overwritten.
 * Errors: INVALID_ARGUMENT for source outside [0, n) or null/non-device outputs. */
s3bfs_status s3bfs_run(s3bfs_handle h, int32_t source, int32_t *level, int32_t *parent,
                       s3bfs_stream_t stream);

/* Free the handle and its workspace (synchronises the last run's stream).  NULL is a no-op. */
s3bfs_status s3bfs_destroy(s3bfs_handle h);

/* Static description of a status code. */
const char *s3bfs_status_string(s3bfs_status s);

/* Detail string of the last error on h (valid until the next call on h). */
s3bfs_status s3bfs_last_error(s3bfs_handle h, const char **msg);

/* Copy the last run's per-level records (synchronises the stream of that run).
 * Writes min(cap, levels) records to out (host memory) and the level count to *num_levels. */
s3bfs_status s3bfs_get_level_stats(s3bfs_handle h, s3bfs_level_stat *out, int32_t cap,
                                   int32_t *num_levels);

/* Device-side tunables the handle resolved (for reports): P_max, grain, T0, CTA sizes, and
 * td_chain / bu_chain = the (k_explore, k_compact) pairs / (k_fb_clear, k_fb_set,
 * k_bottom_up) triples the captured loop runs per entry into the top-down / bottom-up body
 * (consecutive levels of one direction; surplus ones return at once); universal_body = 1:
 * every body continues with the kernels of the tiers that usually follow (S C T^td [B^bu
 * T^td] C S from its own tier on, S = k_small, C = k_cluster, T = pair, B = triple);
 * prologue = 1 (top-down handles): that whole sequence also runs once between k_init and the
 * WHILE node, so a typical traversal needs no conditional round trip at all. */
typedef struct {
  int32_t num_sms, p_max, edges_per_cta, tier0_max_edges;
  int32_t kd_threads, kd_tile_edges, ksmall_threads, ksmall_max_frontier;
  int32_t td_chain, bu_chain, universal_body, prologue;
  int64_t workspace_bytes;
} s3bfs_info;
s3bfs_status s3bfs_get_info(s3bfs_handle h, s3bfs_info *out);

/* CUDA-event kernel times of the last run (options.time_kernels = 1 and loop_mode = 2;
 * otherwise all zero).  Synchronises the run's stream. */
typedef struct {
  double explore_ms, compact_ms, small_ms, bottom_up_ms;  /* summed over launches */
  int32_t explore_launches, compact_launches, small_launches, bottom_up_launches;
} s3bfs_kernel_times;
s3bfs_status s3bfs_get_kernel_times(s3bfs_handle h, s3bfs_kernel_times *out);

/* Test-only: %globaltimer stamps of the last run's first level (ns): out[0] k_init start,
 * out[1] first k_dispatch, out[2] k_small start (0 when not reached).  Synchronises. */
s3bfs_status s3bfs_debug_timeline(s3bfs_handle h, uint64_t out[4]);

/* ---- NEXT-4: one traversal over G ranks, 1-D vertex partition -------
 * Rank r (a handle created with dist_size = G, dist_rank = r, typically one per GPU of a node)
 * owns the internal ids v with (v / 32) mod G == r (block-cyclic 32-id blocks of the degree
 * order: one visited-bitmap word per owner, the hubs spread over the ranks), their CSR rows
 * (a local CSR built at create from the caller's global CSR) and their state (d, parent,
 * Owner).  The visited bitmap is replicated.  Per level, on every rank:
 *   s3bfs_dist_explore   (c)(d) over the local frontier; a target with a clear visited bit goes
 *                        as {v, parent} straight into v's owner's receive segment for this warp
 *                        (stores into the peer's memory over NVLink / NVSwitch: the exchange
 *                        is fused into the exploration kernel, no collective carries data)
 *   -- every rank's explore complete (a stream-ordered barrier across ranks) --
 *   s3bfs_dist_dedup     (e)(a)(b) on the owner: Owner[v] <- slot for every received
 *                        candidate, keep iff Owner[v] == slot (the benign race stays on one
 *                        GPU), d/parent, the next local frontier by the look-back scan; the
 *                        owner's updated bitmap words and its {n_next, e_next} into every peer
 *   -- every rank's dedup complete --
 *   s3bfs_dist_advance   the level's totals over all ranks (Fig1 L9): *done = 1 ends the loop
 * then s3bfs_dist_end writes level/parent of the rank's own vertices (caller ids); the other
 * entries keep the -1 s3bfs_dist_begin wrote, so an element-wise max over the ranks' arrays
 * is the full answer.  Connection: every rank exports its exchange record, the records are
 * shared (any host channel, e.g. torch.distributed), and every rank connects to all of them:
 * use_ipc = 1 opens peers' allocations through CUDA IPC (one process per GPU); use_ipc = 0
 * takes the addresses as they are (several ranks in one process, e.g. a one-GPU loopback).
 * All calls need a handle created with dist_size > 1 (else UNSUPPORTED). */
typedef struct {
  uint64_t base;            /* the rank's exchange allocation (device address in its process) */
  uint64_t recv, rcnt, rmeta, rtot, bm, vinfo;  /* arrays inside it (same layout on every
                                               rank): receive segments, their counts, per-source
                                               {wcap, P_l} and totals, the visited-bitmap
                                               replica, the vertex records (Owner) */
  uint8_t ipc[64];          /* cudaIpcMemHandle_t of the allocation (valid if ipc_valid) */
  int32_t ipc_valid;
  int32_t rank, size;
  int32_t pad;
} s3bfs_dist_peer;

/* This rank's exchange record (host struct, caller-owned). */
s3bfs_status s3bfs_dist_export(s3bfs_handle h, s3bfs_dist_peer *out);

/* peers: `count` = G records in rank order (this rank's included).  Call once after create
 * (again to reconnect).  INVALID_ARGUMENT for a wrong count/order; CUDA if an IPC open fails. */
s3bfs_status s3bfs_dist_connect(s3bfs_handle h, const s3bfs_dist_peer *peers, int32_t count,
                                int32_t use_ipc);

/* Start a traversal from `source` (caller id, the same on every rank).  level/parent: device,
 * n int32 each, caller-owned; set to -1 here (enqueued on `stream`) and written for this
 * rank's vertices by s3bfs_dist_end. */
s3bfs_status s3bfs_dist_begin(s3bfs_handle h, int32_t source, int32_t *level, int32_t *parent,
                              s3bfs_stream_t stream);

/* Explore this rank's part of the current level (enqueued on `stream`). */
s3bfs_status s3bfs_dist_explore(s3bfs_handle h, s3bfs_stream_t stream);

/* Deduplicate the candidates received this level (keep the copy whose slot is Owner[v]);
 * publish bitmap words (atomicOr into every replica) and totals (enqueued on `stream`; every
 * rank's explore of this level must have completed before it runs). */
s3bfs_status s3bfs_dist_dedup(s3bfs_handle h, s3bfs_stream_t stream);

/* Advance the level from the totals of all ranks (every rank's dedup of this level must have
 * completed).  With done / n_next non-NULL it synchronises `stream` and returns *done = 1 when
 * no rank has a next frontier, *n_next = the next frontier's size over all ranks. */
s3bfs_status s3bfs_dist_advance(s3bfs_handle h, s3bfs_stream_t stream, int32_t *done,
                                int64_t *n_next);

/* Advance without a host round trip: enqueued on `stream`, and the advance writes -1 into
 * *flag once no rank has a next frontier, else the next frontier's size over all ranks.  flag:
 * int64 the device can write, e.g. pinned host memory (read it after an event recorded behind
 * this call).  Calls after the end are no-ops (every s3bfs_dist_* kernel checks the level's
 * state), so a driver may enqueue a few levels ahead and check the flags late. */
s3bfs_status s3bfs_dist_advance_flag(s3bfs_handle h, s3bfs_stream_t stream, int64_t *flag);

/* Synchronise `stream` and read the last advance: *done = 1 when no rank has a next frontier,
 * *n_next = the next frontier's size over all ranks (either may be NULL, not both). */
s3bfs_status s3bfs_dist_status(s3bfs_handle h, s3bfs_stream_t stream, int32_t *done,
                               int64_t *n_next);

/* Write level/parent (caller ids) of this rank's vertices for the traversal begun by
 * s3bfs_dist_begin (enqueued on `stream`). */
s3bfs_status s3bfs_dist_end(s3bfs_handle h, s3bfs_stream_t stream);

/* ---- test-only entry points (same kernels the traversal uses) ------------------------ */

/* (b) alone: single-pass decoupled-look-back exclusive scan (Fig1 L14; DESIGN R5).
 * in: device, n int32; out: device, n+1 int32 with out[0] = 0, out[i+1] = out[i] + in[i]
 * (two's-complement wrap).  n == 0 writes out[0] = 0.  Enqueued on `stream`. */
s3bfs_status s3bfs_debug_exclusive_scan(const int32_t *in, int32_t *out, int32_t n,
                                        s3bfs_stream_t stream);

/* (c) alone: Find-StartExpPoint (Fig1 L17) by the device search (DESIGN R8).
 * excl: device, n_l+1 int32 exclusive degree scan (excl[n_l] = e_l > 0).  For worker
 * w < p_l with s_w = w*chunk < e_l: out_u[w] = the u with excl[u] <= s_w < excl[u+1],
 * out_off[w] = s_w - excl[u]; workers with s_w >= e_l get -1.  out_*: device, p_l int32. */
s3bfs_status s3bfs_debug_find_start_points(const int32_t *excl, int32_t n_l, int32_t chunk,
                                           int32_t p_l, int32_t *out_u, int32_t *out_off,
                                           s3bfs_stream_t stream);

#ifdef __cplusplus
}
#endif
#endif /* S3BFS_H_ */
