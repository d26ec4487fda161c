/*
 * oracle/s3bfs_oracle.c -- the CPU ORACLE for the S3BFS hot path.
 *
 * TEST INFRASTRUCTURE ONLY.  Only tests/, __graft_entry__.smoke() and bench.py's
 * cpu_baseline / --impl reference legs may load or call this file's library.  The
 * product path (paper_2209_08764_b200/) never links, imports or executes it, and the
 * two share no code, headers, tables or helpers.
 *
 * Everything here is plain, serial, obviously-correct C written from the paper
 * (/root/reference/PAPER.md, "P:n" = line n) in the paper's order and notation:
 *
 *   oracle_bfs                -- the plain definition: level[v] = hop distance d(s,v),
 *                                a FIFO-queue BFS, Theta(m+n) ("T_s = Theta(m+n)",
 *                                Fig.1 header P:62 "Returns d[0:n-1]").
 *   oracle_inclusive_scan     -- Parallel-Prefix-Sum of Fig.1 L14, plain running sum.
 *   oracle_exclusive_scan     -- the exclusive form used by the GPU path (R5):
 *                                excl[0]=0, excl[i+1]=excl[i]+in[i]; excl[n] = e_l (Fig.1 L15).
 *   oracle_find_start_points  -- Find-StartExpPoint, Fig.1 L17, by the paper's own
 *                                range-marking rule, NOT binary search.
 *   oracle_dedup_linearize    -- Fig.1 L19-L29: keep v in Q[i] iff Owner[v]=i,
 *                                Sizes, Parallel-Prefix-Sum(Sizes), linearisation.
 *   oracle_s3bfs_fig1         -- Figure 1 end to end (L1-L29), its P workers simulated one
 *                                after another (a legal serialisation of each parallel for).
 *   oracle_level_profile      -- n_l, e_l per level, m_c, n_c from a level array (the
 *                                quantities of Fig.1 L9/L15 and the P:37-41 accounting).
 *   oracle_check_bfs          -- Graph500-style level/parent certificate (R2).
 *
 * Unreached is -1 (reading R1: the paper's d <- infinity, Fig.1 L3).
 * Parity pins for every function live in tests/test_oracle_pins.py.
 */
#include <stdint.h>
#include <stdlib.h>
#include <string.h>

#define OR_OK 0
#define OR_EINVAL 1
#define OR_EOVERFLOW 2
#define OR_ENOMEM 3

/* ------------------------------------------------------------------------------------ */
/* Plain definition of the output: serial FIFO-queue BFS.             */
/* level[v] = d(s,v) or -1; parent[s] = s; parent[v] = the first discoverer; -1 if none. */
/* ------------------------------------------------------------------------------------ */
int oracle_bfs(int32_t n, const int32_t *row_offsets, const int32_t *col_indices,
               int32_t source, int32_t *level, int32_t *parent) {
  if (n <= 0 || !row_offsets || !level || !parent) return OR_EINVAL;
  if (source < 0 || source >= n) return OR_EINVAL; /* "source out of range -> rejection" */
  int32_t *queue = (int32_t *)malloc(sizeof(int32_t) * (size_t)n);
  if (!queue) return OR_ENOMEM;
  for (int32_t v = 0; v < n; ++v) { level[v] = -1; parent[v] = -1; }
  level[source] = 0;
  parent[source] = source;
  int64_t head = 0, tail = 0;
  queue[tail++] = source;
  while (head < tail) {
    int32_t u = queue[head++];
    for (int64_t k = row_offsets[u]; k < row_offsets[u + 1]; ++k) {
      int32_t v = col_indices[k];
      if (level[v] == -1) {
        level[v] = level[u] + 1;
        parent[v] = u;
        queue[tail++] = v;
      }
    }
  }
  free(queue);
  return OR_OK;
}

/* Parallel-Prefix-Sum (Fig.1 L14; Blelloch, cited at P:31) -- the result it reaches is
 * the inclusive running sum; written out serially.  Returns OR_EOVERFLOW if a prefix does
 * not fit int32 (the index word of the CSR). */
int oracle_inclusive_scan(const int32_t *in, int64_t n, int32_t *out) {
  if (n < 0 || (n > 0 && (!in || !out))) return OR_EINVAL;
  int64_t run = 0;
  for (int64_t i = 0; i < n; ++i) {
    run += in[i];
    if (run > INT32_MAX || run < INT32_MIN) return OR_EOVERFLOW;
    out[i] = (int32_t)run;
  }
  return OR_OK;
}

/* Exclusive form with the total appended (R5): out has n+1 entries,
 * out[0] = 0, out[i+1] = out[i] + in[i], so out[n] = e_l of Fig.1 L15. */
int oracle_exclusive_scan(const int32_t *in, int64_t n, int32_t *out) {
  if (n < 0 || !out || (n > 0 && !in)) return OR_EINVAL;
  int64_t run = 0;
  out[0] = 0;
  for (int64_t i = 0; i < n; ++i) {
    run += in[i];
    if (run > INT32_MAX || run < INT32_MIN) return OR_EOVERFLOW;
    out[i + 1] = (int32_t)run;
  }
  return OR_OK;
}

/* Find-StartExpPoint (Fig.1 L17) by the paper's range rule:
 * "For each entry of the EdgeSum array, in parallel we first determine a thread id t_s that
 * can start at that location ... and a thread id t_e that could possibly end at that node.
 * ... For each nonempty range, we write this node's position as the corresponding thread's
 * start location."
 * edge_sum is the INCLUSIVE scan of the frontier degrees (Fig.1 L14).  Worker t starts at
 * global edge t*chunk (SPEC S:96 reading; R6).  For frontier entry u with
 * exclusive start s_u = edge_sum[u-1] (0 for u=0) and end edge_sum[u], the workers starting
 * inside it are t in [ceil(s_u/chunk), ceil(edge_sum[u]/chunk) - 1] (clipped to < p_l).
 * out_u[t] = u, out_off[t] = t*chunk - s_u.  Entries never written stay -1. */
int oracle_find_start_points(const int32_t *edge_sum, int32_t n_l, int64_t chunk, int32_t p_l,
                             int32_t *out_u, int32_t *out_off) {
  if (n_l < 0 || p_l < 0 || chunk <= 0 || (p_l > 0 && (!out_u || !out_off))) return OR_EINVAL;
  for (int32_t t = 0; t < p_l; ++t) { out_u[t] = -1; out_off[t] = -1; }
  for (int32_t u = 0; u < n_l; ++u) {             /* "for each entry of the EdgeSum array" */
    int64_t s_u = (u == 0) ? 0 : edge_sum[u - 1];
    int64_t e_u = edge_sum[u];
    int64_t t_s = (s_u + chunk - 1) / chunk;       /* first worker starting at or after s_u */
    int64_t t_e = (e_u + chunk - 1) / chunk - 1;   /* last worker starting before e_u */
    for (int64_t t = t_s; t <= t_e && t < p_l; ++t) {
      out_u[t] = u;
      out_off[t] = (int32_t)(t * chunk - s_u);
    }
  }
  return OR_OK;
}

/* Deduplication + linearisation, Fig.1 L19-L29, over P_l private queues given
 * flat: queue i holds items[q_begin[i] .. q_begin[i+1]).  Keeps v in Q[i] iff Owner[v] = i
 * (L22), Sizes[i] = |Q[i]| (L23), Parallel-Prefix-Sum(Sizes) inclusive (L24), then copies Q[i]
 * to CurLevelVertices at offset 0 (i=0) or Sizes[i-1] (L27-L29).
 * out_sizes (p_l, inclusive scan) and out_frontier (capacity = total items) are written;
 * *out_count = Sizes[P_l-1]. */
int oracle_dedup_linearize(int32_t p_l, const int64_t *q_begin, const int32_t *items,
                           const int32_t *owner, int32_t *out_sizes, int32_t *out_frontier,
                           int64_t *out_count) {
  if (p_l < 0 || !out_count || (p_l > 0 && (!q_begin || !out_sizes))) return OR_EINVAL;
  /* L20-L23: per-worker filter, preserving order */
  int64_t total_in = p_l > 0 ? q_begin[p_l] : 0;
  int32_t *kept = (int32_t *)malloc(sizeof(int32_t) * (size_t)(total_in > 0 ? total_in : 1));
  int64_t *kbeg = (int64_t *)malloc(sizeof(int64_t) * (size_t)(p_l + 1));
  if (!kept || !kbeg) { free(kept); free(kbeg); return OR_ENOMEM; }
  int64_t w = 0;
  for (int32_t i = 0; i < p_l; ++i) {
    kbeg[i] = w;
    for (int64_t j = q_begin[i]; j < q_begin[i + 1]; ++j) {
      int32_t v = items[j];
      if (owner[v] == i) kept[w++] = v;   /* "if Owner[v] = i then Q-New.Enqueue(v)" */
    }
    out_sizes[i] = (int32_t)(w - kbeg[i]); /* "Sizes[i] <- |Q[i]|" */
  }
  kbeg[p_l] = w;
  /* L24: Parallel-Prefix-Sum(Sizes) */
  int rc = oracle_inclusive_scan(out_sizes, p_l, out_sizes);
  if (rc != OR_OK) { free(kept); free(kbeg); return rc; }
  /* L25-L29: linearisation */
  for (int32_t i = 0; i < p_l; ++i) {
    int64_t offset = (i == 0) ? 0 : out_sizes[i - 1];
    for (int64_t j = kbeg[i]; j < kbeg[i + 1]; ++j) out_frontier[offset + (j - kbeg[i])] = kept[j];
  }
  *out_count = p_l > 0 ? out_sizes[p_l - 1] : 0;
  free(kept);
  free(kbeg);
  return OR_OK;
}

/* Figure 1 end to end (L1-L29), with P workers simulated one after the other.  Each parallel
 * for is executed as a sequential loop over its workers, which is one legal serialisation of
 * the paper's benign race.  Returns d (as level[], -1 = infinity) and, per level l
 * (the frontier CurLevelVertices at distance l), n_l, e_l and P_l = Min(P, e_l) of Fig.1 L16.
 * stats arrays have capacity max_levels; *num_levels counts every level with n_l > 0. */
int oracle_s3bfs_fig1(int32_t n, const int32_t *row_offsets, const int32_t *col_indices,
                      int32_t s, int32_t P, int32_t *level, int32_t max_levels,
                      int64_t *out_nl, int64_t *out_el, int64_t *out_pl, int32_t *num_levels) {
  if (n <= 0 || P < 1 || s < 0 || s >= n || !level || !num_levels) return OR_EINVAL;
  int32_t *owner = (int32_t *)malloc(sizeof(int32_t) * (size_t)n);
  int32_t *cur = (int32_t *)malloc(sizeof(int32_t) * (size_t)n);   /* CurLevelVertices */
  int32_t *edge_sum = (int32_t *)malloc(sizeof(int32_t) * (size_t)n);
  int32_t *q_items = (int32_t *)malloc(sizeof(int32_t) * (size_t)n); /* all Q[i] back to back */
  int64_t *q_begin = (int64_t *)malloc(sizeof(int64_t) * ((size_t)P + 1));
  int32_t *su = (int32_t *)malloc(sizeof(int32_t) * (size_t)P);
  int32_t *soff = (int32_t *)malloc(sizeof(int32_t) * (size_t)P);
  int32_t *sizes = (int32_t *)malloc(sizeof(int32_t) * (size_t)P);
  int rc = OR_OK;
  if (!owner || !cur || !edge_sum || !q_items || !q_begin || !su || !soff || !sizes) {
    rc = OR_ENOMEM;
    goto done;
  }
  /* L1-L3: d[u] <- inf, Owner[u] <- P */
  for (int32_t u = 0; u < n; ++u) { level[u] = -1; owner[u] = P; }
  level[s] = 0; owner[s] = 0;                 /* L4 */
  cur[0] = s;                                 /* L7 */
  int64_t n_l = 1;
  int32_t l = 0;                              /* L8 */
  *num_levels = 0;
  while (n_l > 0) {                           /* L9 */
    /* L12-L13: EdgeSum[u] <- Degree[CurLevelVertices[u]] */
    for (int64_t u = 0; u < n_l; ++u)
      edge_sum[u] = row_offsets[cur[u] + 1] - row_offsets[cur[u]];
    rc = oracle_inclusive_scan(edge_sum, n_l, edge_sum); /* L14 */
    if (rc != OR_OK) goto done;
    int64_t e_l = edge_sum[n_l - 1];          /* L15 */
    int64_t p_l = e_l < P ? e_l : P;          /* L16: P_l <- Min(P, e_l) */
    if (*num_levels < max_levels) {
      out_nl[*num_levels] = n_l; out_el[*num_levels] = e_l; out_pl[*num_levels] = p_l;
    }
    (*num_levels)++;
    l = l + 1;                                /* L10: discoveries get the new l */
    int64_t total_q = 0;
    if (p_l > 0) {
      int64_t chunk = (e_l + p_l - 1) / p_l;  /* "(almost) equal division", DESIGN R6 */
      rc = oracle_find_start_points(edge_sum, (int32_t)n_l, chunk, (int32_t)p_l, su, soff); /* L17 */
      if (rc != OR_OK) goto done;
      /* L18: EXPLORE-VERTEX.  Worker i scans global edges [i*chunk, min((i+1)*chunk, e_l)),
       * walking CurLevelVertices from its start point; every unvisited endpoint gets d = l,
       * Owner = i and is appended to Q[i]. */
      for (int64_t i = 0; i < p_l; ++i) {
        q_begin[i] = total_q;
        int64_t e_begin = i * chunk;
        int64_t e_end = e_begin + chunk < e_l ? e_begin + chunk : e_l;
        int64_t u = su[i];
        int64_t off = soff[i];
        for (int64_t e = e_begin; e < e_end; ++e) {
          int64_t s_u = (u == 0) ? 0 : edge_sum[u - 1];
          while (e >= edge_sum[u]) { ++u; s_u = edge_sum[u - 1]; off = 0; }
          off = e - s_u;
          int32_t x = cur[u];
          int32_t v = col_indices[row_offsets[x] + off];
          if (level[v] == -1) {
            level[v] = l;
            owner[v] = (int32_t)i;
            q_items[total_q++] = v;
          }
        }
      }
      q_begin[p_l] = total_q;
      /* L19-L29: dedup by final owner, Sizes scan, linearise into CurLevelVertices */
      int64_t count = 0;
      rc = oracle_dedup_linearize((int32_t)p_l, q_begin, q_items, owner, sizes, cur, &count);
      if (rc != OR_OK) goto done;
      n_l = count;
    } else {
      n_l = 0;                                /* e_l = 0: nothing to explore (DESIGN R10) */
    }
  }
done:
  free(owner); free(cur); free(edge_sum); free(q_items); free(q_begin);
  free(su); free(soff); free(sizes);
  return rc;
}

/* Per-level profile of a level array: n_l = |{v : level[v] = l}|, e_l = sum of Degree over
 * them (Fig.1 L13-L15), m_c = sum_l e_l (arcs reachable from the source), n_c = sum_l n_l.
 * Returns the number of levels (max level + 1) in *num_levels. */
int oracle_level_profile(int32_t n, const int32_t *row_offsets, const int32_t *level,
                         int32_t max_levels, int64_t *out_nl, int64_t *out_el,
                         int32_t *num_levels, int64_t *m_c, int64_t *n_c) {
  if (n <= 0 || !row_offsets || !level || !num_levels || !m_c || !n_c) return OR_EINVAL;
  int32_t L = 0;
  for (int32_t v = 0; v < n; ++v) {
    if (level[v] < -1) return OR_EINVAL;
    if (level[v] + 1 > L) L = level[v] + 1;
  }
  for (int32_t l = 0; l < max_levels; ++l) { out_nl[l] = 0; out_el[l] = 0; }
  *m_c = 0; *n_c = 0;
  for (int32_t v = 0; v < n; ++v) {
    int32_t l = level[v];
    if (l < 0) continue;
    int64_t deg = (int64_t)row_offsets[v + 1] - row_offsets[v];
    if (l < max_levels) { out_nl[l] += 1; out_el[l] += deg; }
    *m_c += deg;
    *n_c += 1;
  }
  *num_levels = L;
  return OR_OK;
}

/* Is (p, v) an arc?  Binary search when every row is sorted, else a linear scan. */
static int has_arc(const int32_t *ro, const int32_t *col, int32_t p, int32_t v, int sorted) {
  int64_t lo = ro[p], hi = ro[p + 1];
  if (!sorted) {
    for (int64_t k = lo; k < hi; ++k) if (col[k] == v) return 1;
    return 0;
  }
  while (lo < hi) {
    int64_t mid = lo + (hi - lo) / 2;
    if (col[mid] < v) lo = mid + 1; else hi = mid;
  }
  return lo < ro[p + 1] && col[lo] == v;
}

/* Certificate (R2; Graph500 validation style).  Codes:
 *   0 ok; 1 source entry wrong (level[s] != 0 or parent[s] != s);
 *   2 reached v != s whose parent is out of range; 3 level[parent[v]] != level[v]-1;
 *   4 (parent[v], v) is not an arc; 5 an arc (u,v) with level[u] >= 0 and
 *   (level[v] == -1 or level[v] > level[u]+1); 6 unreached v with parent[v] != -1 or
 *   level[v] < -1.   *bad_vertex names the first offending vertex (v; for code 5 the head v).
 * These conditions pin level = d(s, .) exactly: the parent chain gives level[v] >= d(s,v),
 * arc-closure along a shortest path gives level[v] <= d(s,v). */
int oracle_check_bfs(int32_t n, const int32_t *ro, const int32_t *col, int32_t s,
                     const int32_t *level, const int32_t *parent, int64_t *bad_vertex) {
  if (n <= 0 || !ro || !level || !parent || !bad_vertex || s < 0 || s >= n) return -1;
  *bad_vertex = -1;
  int sorted = 1;
  for (int32_t u = 0; u < n && sorted; ++u)
    for (int64_t k = ro[u] + 1; k < ro[u + 1]; ++k)
      if (col[k - 1] > col[k]) { sorted = 0; break; }
  if (level[s] != 0 || parent[s] != s) { *bad_vertex = s; return 1; }
  for (int32_t v = 0; v < n; ++v) {
    if (level[v] < -1) { *bad_vertex = v; return 6; }
    if (level[v] == -1) {
      if (parent[v] != -1) { *bad_vertex = v; return 6; }
      continue;
    }
    if (v == s) continue;
    int32_t p = parent[v];
    if (p < 0 || p >= n) { *bad_vertex = v; return 2; }
    if (level[p] != level[v] - 1) { *bad_vertex = v; return 3; }
    if (!has_arc(ro, col, p, v, sorted)) { *bad_vertex = v; return 4; }
  }
  for (int32_t u = 0; u < n; ++u) {
    if (level[u] < 0) continue;
    for (int64_t k = ro[u]; k < ro[u + 1]; ++k) {
      int32_t v = col[k];
      if (level[v] == -1 || level[v] > level[u] + 1) { *bad_vertex = v; return 5; }
    }
  }
  return 0;
}
