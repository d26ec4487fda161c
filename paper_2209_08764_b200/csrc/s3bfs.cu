// paper_2209_08764_b200/csrc/s3bfs.cu -- host side of the C ABI declared in include/s3bfs.h.
//
// Owns the workspace, resolves the (f) tunables (P_max from the occupancy of the level
// kernels on this device, the grain, T0), and builds the captured level loop:
//
//   s3bfs_run:  graph { k_init (Fig1 L1-L8);
//                       WHILE(n_l > 0) {                                   Fig1 L9
//                         SWITCH(tier): 0 { k_small }                      (f) tier 0
//                                       1 { (k_explore; k_compact) x 4 }   (c)(d) / (e)(a)(b)
//                                       2 { (k_fb_clear; k_fb_set; k_bottom_up) x 3 } NEXT-3
//                                       3 { k_cluster: consecutive mid-size levels }  (f)
//                       }
//                       k_finalize }
//   The kernel that decides a level's successor sets the conditional handles (no dispatch
//   kernel); k_init's per-run arguments are patched into the executable graph per run.
//   Bodies 1 and 2 chain S3BFS_TD_CHAIN pairs / S3BFS_BU_CHAIN triples so consecutive levels
//   of one direction skip a conditional round trip; kernels of another tier return at once.
//
// The host crosses the host/device boundary once per traversal (enqueue); the level loop,
// P_l and every per-level decision stay on the device (SURVEY.md s.8(a) row f, H6).
#include <cuda_runtime.h>

#include <atomic>
#include <cstdio>
#include <cstring>
#include <new>
#include <string>

#include <cub/device/device_radix_sort.cuh>
#include <cub/device/device_scan.cuh>
#include <cub/device/device_segmented_sort.cuh>

#include "s3bfs_kernels.cuh"

using namespace s3bfs;

// Device memory of the prepared graph (degree-ordered CSR, id maps, in-adjacency), shared by a
// handle and its clones (NEXT-2: concurrent traversals); freed with the last of them.
struct GraphStore {
  void *g2 = nullptr, *g3 = nullptr;
  size_t b2 = 0, b3 = 0;
  std::atomic<int> refs{1};
  ~GraphStore() {
    if (g2) cudaFree(g2);
    if (g3) cudaFree(g3);
  }
};

struct s3bfs_ctx {
  int dev = 0, num_sms = 0;
  int32_t n = 0;
  int64_t nnz = 0;
  const int32_t *ro = nullptr, *col = nullptr;
  s3bfs_options opt{};
  Params P{};
  void *ws = nullptr;
  GraphStore *gs = nullptr;         // shared prepared graph (see GraphStore)
  const int32_t *ro_int = nullptr;  // row offsets of the internal CSR
  size_t ws_bytes = 0;
  int64_t cand_cap = 0;
  size_t ks_smem = 0, kc_smem = 0;
  int loop_graph = 1;
  cudaGraph_t graph = nullptr;
  cudaGraphExec_t exec = nullptr;
  cudaGraphNode_t init_node = nullptr;
  cudaStream_t last_stream = nullptr;
  bool ran = false;
  Ctl *h_ctl = nullptr;  // pinned, host-loop mode
  bool time_kernels = false;
  cudaEvent_t ev[4] = {nullptr, nullptr, nullptr, nullptr};
  s3bfs_kernel_times kt{};
  // NEXT-4 (dist_size > 1): the rank's local CSR, the exchange allocation peers write into,
  // and the peers' exchange allocations opened through CUDA IPC (other processes)
  void *dgraph = nullptr;
  void *xws = nullptr;
  size_t xws_bytes = 0;
  void *ipc_open[DIST_MAX] = {};
  int32_t *d_level = nullptr, *d_parent = nullptr;
  std::string err;
};

namespace {

thread_local std::string g_err;

s3bfs_status fail(s3bfs_ctx *h, s3bfs_status s, const std::string &msg) {
  if (h) h->err = msg;
  g_err = msg;
  return s;
}

s3bfs_status cuda_fail(s3bfs_ctx *h, cudaError_t e, const char *what) {
  std::string m = std::string(what) + ": " + cudaGetErrorName(e) + " (" + cudaGetErrorString(e) + ")";
  return fail(h, e == cudaErrorMemoryAllocation ? S3BFS_ERR_OUT_OF_MEMORY : S3BFS_ERR_CUDA, m);
}

#define CK(h, call)                                      \
  do {                                                   \
    cudaError_t e_ = (call);                             \
    if (e_ != cudaSuccess) return cuda_fail(h, e_, #call); \
  } while (0)

bool is_device_ptr(const void *p) {
  cudaPointerAttributes a;
  if (cudaPointerGetAttributes(&a, p) != cudaSuccess) {
    cudaGetLastError();
    return false;
  }
  return a.type == cudaMemoryTypeDevice || a.type == cudaMemoryTypeManaged;
}

size_t align256(size_t x) { return (x + 255) & ~(size_t)255; }

// A stream-ordered temporary freed (cudaFreeAsync on its stream) when it leaves scope, so an
// early error return cannot leak it.
struct AsyncTmp {
  void *p = nullptr;
  cudaStream_t st;
  explicit AsyncTmp(cudaStream_t s) : st(s) {}
  AsyncTmp(const AsyncTmp &) = delete;
  AsyncTmp &operator=(const AsyncTmp &) = delete;
  ~AsyncTmp() {
    if (p) cudaFreeAsync(p, st);
  }
  cudaError_t alloc(size_t bytes) { return cudaMallocAsync(&p, bytes, st); }
  template <class T> T *as() const { return static_cast<T *>(p); }
};

int init_grid(const s3bfs_ctx *h) {
  long long want = ((long long)h->n / 4 + 255) / 256;
  long long cap = (long long)h->num_sms * 8;
  if (want < 1) want = 1;
  return (int)(want < cap ? want : cap);
}

int finalize_grid(const s3bfs_ctx *h) {
  long long want = ((long long)h->n + 255) / 256;
  long long cap = (long long)h->num_sms * 8;
  return (int)(want < cap ? (want < 1 ? 1 : want) : cap);
}

// Degree-ordered internal copy (DESIGN.md s.7): internal id i = rank of the vertex in a stable
// sort by descending degree, so the hottest vertices get the smallest ids and their visited
// bits share a few L1-resident bitmap lines.  Create-time preprocessing, off the traversal
// path (CUB's radix sort is the library primitive for the sort).
s3bfs_status build_reordered(s3bfs_ctx *h, cudaStream_t st) {
  const int n = h->n;
  const long long nnz = h->nnz;
  size_t off = 0;
  auto take = [&](size_t bytes) { size_t o = off; off += align256(bytes); return o; };
  const size_t o_col2 = take((size_t)nnz * 4 + 16);
  const size_t o_n2o = take((size_t)n * 4), o_o2n = take((size_t)n * 4);
  const size_t o_ro2 = take((size_t)(n + 1) * 4);
  h->gs->b2 = off;
  CK(h, cudaMalloc(&h->gs->g2, off));
  char *g = (char *)h->gs->g2;
  int32_t *col2 = (int32_t *)(g + o_col2);
  int32_t *n2o = (int32_t *)(g + o_n2o), *o2n = (int32_t *)(g + o_o2n);
  int32_t *ro2 = (int32_t *)(g + o_ro2);
  AsyncTmp deg_b(st), degs_b(st), iota_b(st), tmp_b(st), status_b(st), nz_b(st);
  size_t tmp_bytes = 0;
  CK(h, cub::DeviceRadixSort::SortPairsDescending(nullptr, tmp_bytes, (int32_t *)nullptr,
                                                  (int32_t *)nullptr, (int32_t *)nullptr, n2o,
                                                  n, 0, 32, st));
  CK(h, deg_b.alloc((size_t)n * 4));
  CK(h, degs_b.alloc((size_t)n * 4));
  CK(h, iota_b.alloc((size_t)n * 4));
  CK(h, tmp_b.alloc(tmp_bytes));
  int32_t *deg = deg_b.as<int32_t>(), *deg_sorted = degs_b.as<int32_t>(), *iota = iota_b.as<int32_t>();
  void *tmp = tmp_b.p;
  const int grid = h->num_sms * 8;
  k_degrees<<<grid, 256, 0, st>>>(h->ro, n, deg, iota);
  CK(h, cub::DeviceRadixSort::SortPairsDescending(tmp, tmp_bytes, deg, deg_sorted, iota, n2o, n,
                                                  0, 32, st));
  k_inverse_perm<<<grid, 256, 0, st>>>(n2o, n, o2n, h->ro, deg);  // deg <- internal degrees
  // ro2 = exclusive scan of the internal degrees: the look-back scan kernel (b)
  const int tiles = (int)(((long long)n + SCAN_TILE - 1) / SCAN_TILE);
  CK(h, status_b.alloc((size_t)(tiles + 1) * 8));  // + the tile counter
  unsigned long long *status = status_b.as<unsigned long long>();
  CK(h, cudaMemsetAsync(status, 0, (size_t)(tiles + 1) * 8, st));
  k_scan_u32<<<tiles, SCAN_THREADS, 0, st>>>(deg, ro2, n, status);
  k_relabel_rows<<<h->num_sms * 16, 256, 0, st>>>(h->ro, h->col, n2o, o2n, ro2, n, col2);
  k_build_vinfo<<<grid, 256, 0, st>>>(ro2, n2o, n, h->P.vinfo, const_cast<int4 *>(h->P.vs16));
  int h_nz = 0;
  CK(h, nz_b.alloc(4));
  int *d_nz = nz_b.as<int>();
  CK(h, cudaMemsetAsync(d_nz, 0, 4, st));
  k_count_nonzero<<<grid, 256, 0, st>>>(deg, n, d_nz);  // internal degrees, descending
  CK(h, cudaMemcpyAsync(&h_nz, d_nz, 4, cudaMemcpyDeviceToHost, st));
  CK(h, cudaGetLastError());
  CK(h, cudaStreamSynchronize(st));
  h->P.col = col2;
  h->P.n2o = n2o;
  h->P.o2n = o2n;
  h->P.n_scan = h_nz;  // internal ids >= h_nz have degree 0: bottom-up never scans them
  h->ro_int = ro2;
  return S3BFS_OK;
}

// NEXT-4 (dist_size > 1): this rank's local CSR (the rows of its block-cyclic vertex slots,
// targets in global internal ids) and vertex records, and the exchange allocation its peers
// write into (receive segments, segment counts, per-source {wcap, p_l} and totals, and the
// replicated visited bitmap).  Every rank computes the same receive layout (block offsets
// from the arcs each rank owns), so a sender writes at the same offsets on every peer.
s3bfs_status build_dist(s3bfs_ctx *h, cudaStream_t st, int nloc) {
  Params &P = h->P;
  const int G = P.dist_size, r = P.dist_rank, n = h->n;
  P.nloc = nloc;
  const int32_t *ro = h->ro_int, *col = P.col;
  const int grid = h->num_sms * 8;
  AsyncTmp cnt_b(st), deg_b(st), tmp_b(st);
  CK(h, cnt_b.alloc(8 * DIST_MAX));
  unsigned long long *d_cnt = cnt_b.as<unsigned long long>();
  CK(h, cudaMemsetAsync(d_cnt, 0, 8 * DIST_MAX, st));
  k_dist_rank_arcs<<<grid, 256, 0, st>>>(ro, n, G, d_cnt);
  unsigned long long h_cnt[DIST_MAX] = {};
  CK(h, cudaMemcpyAsync(h_cnt, d_cnt, 8 * DIST_MAX, cudaMemcpyDeviceToHost, st));
  CK(h, cudaStreamSynchronize(st));
  const long long nnz_l = (long long)h_cnt[r];
  // local CSR: degrees of the local slots, their exclusive scan, the copied rows
  size_t off = 0;
  auto take = [&](size_t bytes) { size_t o = off; off += align256(bytes); return o; };
  const size_t o_ro = take((size_t)(nloc + 1) * 4), o_col = take((size_t)nnz_l * 4 + 16);
  CK(h, cudaMalloc(&h->dgraph, off));
  int32_t *ro_l = (int32_t *)((char *)h->dgraph + o_ro);
  int32_t *col_l = (int32_t *)((char *)h->dgraph + o_col);
  CK(h, deg_b.alloc((size_t)(nloc + 1) * 4));
  int32_t *deg_l = deg_b.as<int32_t>();
  CK(h, cudaMemsetAsync(deg_l + nloc, 0, 4, st));
  k_dist_local_deg<<<grid, 256, 0, st>>>(P, ro, deg_l);
  size_t tmp_bytes = 0;
  CK(h, cub::DeviceScan::ExclusiveSum(nullptr, tmp_bytes, deg_l, ro_l, nloc + 1, st));
  CK(h, tmp_b.alloc(tmp_bytes));
  CK(h, cub::DeviceScan::ExclusiveSum(tmp_b.p, tmp_bytes, deg_l, ro_l, nloc + 1, st));
  k_dist_copy_rows<<<grid, 256, 0, st>>>(P, ro, col, ro_l, col_l);
  CK(h, cudaGetLastError());
  P.col = col_l;
  P.nnz = nnz_l;
  // receive layout (identical on every rank) and the exchange allocation
  long long ofs = 0;
  for (int t = 0; t < G; ++t) {
    P.rofs[t] = (int32_t)ofs;
    ofs += (long long)h_cnt[t] + (long long)P.p_max * (KD_WARPS + 1 + KD_SLACK) + 64;
    if (ofs >= INT32_MAX)
      return fail(h, S3BFS_ERR_UNSUPPORTED, "NEXT-4 receive buffer exceeds int32 slots");
  }
  P.rofs[G] = (int32_t)ofs;
  const size_t bm_bytes = ((size_t)n + 127) / 128 * 16;
  const long long nwmax = (long long)P.p_max * KD_WARPS;
  off = 0;
  const size_t o_recv = take((size_t)ofs * 8), o_rcnt = take((size_t)G * nwmax * 4);
  const size_t o_rmeta = take((size_t)G * 8), o_rtot = take((size_t)G * 8);
  const size_t o_bm = take(bm_bytes + 16);
  const size_t o_vinfo = take((size_t)(nloc + 32) * 32);  // the records senders write Owner into
  h->xws_bytes = off;
  CK(h, cudaMalloc(&h->xws, off));
  char *x = (char *)h->xws;
  CK(h, cudaMemsetAsync(x + o_rcnt, 0, o_bm - o_rcnt, st));
  P.recv = (int2 *)(x + o_recv);
  P.rcnt = (int32_t *)(x + o_rcnt);
  P.rmeta = (int2 *)(x + o_rmeta);
  P.rtot = (int2 *)(x + o_rtot);
  P.bm = (uint32_t *)(x + o_bm);
  P.vinfo = (int4 *)(x + o_vinfo);
  k_dist_build_vinfo<<<grid, 256, 0, st>>>(P, ro_l, P.n2o, P.vinfo);
  CK(h, cudaGetLastError());
  for (int d = 0; d < DIST_MAX; ++d) {  // until s3bfs_dist_connect: every rank is this one
    P.p_recv[d] = P.recv;
    P.p_rcnt[d] = P.rcnt;
    P.p_rmeta[d] = P.rmeta;
    P.p_rtot[d] = P.rtot;
    P.p_bm[d] = P.bm;
    P.p_vinfo[d] = P.vinfo;
  }
  CK(h, cudaStreamSynchronize(st));
  return S3BFS_OK;
}

// Sort every row of a CSR by (internal) id, out of place: with degree-ordered ids the
// highest-degree neighbours come first, where the bottom-up step finds its frontier parents.
s3bfs_status sort_rows(s3bfs_ctx *h, const int32_t *ro, const int32_t *in, int32_t *out,
                       cudaStream_t st) {
  if (h->nnz == 0) return S3BFS_OK;
  AsyncTmp tmp(st);
  size_t bytes = 0;
  CK(h, cub::DeviceSegmentedSort::SortKeys(nullptr, bytes, in, out, (int)h->nnz, h->n, ro,
                                           ro + 1, st));
  CK(h, tmp.alloc(bytes));
  CK(h, cub::DeviceSegmentedSort::SortKeys(tmp.p, bytes, in, out, (int)h->nnz, h->n, ro, ro + 1,
                                           st));
  CK(h, cudaStreamSynchronize(st));  // the sort has consumed tmp before it is released
  return S3BFS_OK;
}

// NEXT-3: the in-adjacency the bottom-up step scans, rows sorted by internal id.  For a
// symmetric graph (every BASELINE config) it is a row-sorted copy of the internal CSR;
// otherwise the row-sorted transpose.  (The top-down adjacency stays in input order: sorted
// rows make k_compact's visited-bit publication contend on shared words -- measured.)
s3bfs_status build_in_adjacency(s3bfs_ctx *h, cudaStream_t st) {
  const int n = h->n;
  const long long nnz = h->nnz;
  const int32_t *ro = h->ro_int, *col = h->P.col;
  unsigned long long hh[2] = {0, 0};
  AsyncTmp dh_b(st), tuns_b(st), tdeg_b(st), status_b(st);
  CK(h, dh_b.alloc(16));
  unsigned long long *d_h = dh_b.as<unsigned long long>();
  CK(h, cudaMemsetAsync(d_h, 0, 16, st));
  k_sym_hash<<<h->num_sms * 16, 256, 0, st>>>(ro, col, n, d_h);
  CK(h, cudaMemcpyAsync(hh, d_h, 16, cudaMemcpyDeviceToHost, st));
  CK(h, cudaStreamSynchronize(st));
  size_t off = 0;
  auto take = [&](size_t bytes) { size_t o = off; off += align256(bytes); return o; };
  const size_t o_tro = take((size_t)(n + 1) * 4), o_tcol = take((size_t)nnz * 4 + 16);
  CK(h, cudaMalloc(&h->gs->g3, off));
  h->gs->b3 = off;
  int32_t *tro = (int32_t *)((char *)h->gs->g3 + o_tro);
  int32_t *tcol = (int32_t *)((char *)h->gs->g3 + o_tcol);
  if (hh[0] == hh[1]) {
    s3bfs_status ss = sort_rows(h, ro, col, tcol, st);
    if (ss != S3BFS_OK) return ss;
    CK(h, cudaStreamSynchronize(st));
    h->P.tro = ro;
    h->P.tcol = tcol;
    return S3BFS_OK;
  }
  CK(h, tuns_b.alloc((size_t)nnz * 4 + 16));
  CK(h, tdeg_b.alloc((size_t)n * 4));
  int32_t *tunsorted = tuns_b.as<int32_t>(), *tdeg = tdeg_b.as<int32_t>();
  CK(h, cudaMemsetAsync(tdeg, 0, (size_t)n * 4, st));
  k_in_degree<<<h->num_sms * 16, 256, 0, st>>>(ro, col, n, tdeg);
  const int tiles = (int)(((long long)n + SCAN_TILE - 1) / SCAN_TILE);
  CK(h, status_b.alloc((size_t)(tiles + 1) * 8));  // + the tile counter
  unsigned long long *status = status_b.as<unsigned long long>();
  CK(h, cudaMemsetAsync(status, 0, (size_t)(tiles + 1) * 8, st));
  k_scan_u32<<<tiles, SCAN_THREADS, 0, st>>>(tdeg, tro, n, status);
  CK(h, cudaMemcpyAsync(tdeg, tro, (size_t)n * 4, cudaMemcpyDeviceToDevice, st));  // cursors
  k_transpose<<<h->num_sms * 16, 256, 0, st>>>(ro, col, n, tdeg, tunsorted);
  CK(h, cudaGetLastError());
  s3bfs_status ss = sort_rows(h, tro, tunsorted, tcol, st);
  if (ss != S3BFS_OK) return ss;
  CK(h, cudaStreamSynchronize(st));
  h->P.tro = tro;
  h->P.tcol = tcol;
  h->P.n_scan = n;  // the degree-order prefix is by out-degree; in-degrees differ here
  return S3BFS_OK;
}

#ifndef S3BFS_TD_CHAIN
#define S3BFS_TD_CHAIN 4  // top-down (k_explore, k_compact) pairs per SWITCH body
#endif
#ifndef S3BFS_UNIVERSAL_BODY
#define S3BFS_UNIVERSAL_BODY 1  // every SWITCH body chains the rest of a traversal's tiers
#endif
#ifndef S3BFS_GRAPH_PROLOGUE
#define S3BFS_GRAPH_PROLOGUE 1  // the canonical tier sequence once before the WHILE node
#endif
#ifndef S3BFS_BU_CHAIN
#define S3BFS_BU_CHAIN 3  // bottom-up (k_fb_clear, k_fb_set, k_bottom_up) triples per body
#endif
bool graph_prologue(const s3bfs_ctx *h) { return S3BFS_GRAPH_PROLOGUE && !h->P.direction; }
s3bfs_status build_graph(s3bfs_ctx *h) {
  cudaGraph_t g = nullptr;
  CK(h, cudaGraphCreate(&g, 0));
  h->graph = g;
  cudaGraphConditionalHandle hw, ht;
  CK(h, cudaGraphConditionalHandleCreate(&hw, g, 1, cudaGraphCondAssignDefault));
  CK(h, cudaGraphConditionalHandleCreate(&ht, g, 7, cudaGraphCondAssignDefault));
  h->P.h_while = hw;
  h->P.h_tier = ht;
  h->P.use_graph = 1;

  cudaGraphNodeParams wp = {};
  wp.type = cudaGraphNodeTypeConditional;
  wp.conditional.handle = hw;
  wp.conditional.type = cudaGraphCondTypeWhile;
  wp.conditional.size = 1;
  void *args[] = {&h->P};
  {  // first node: k_init (its source / output pointers are patched per run)
    int32_t s0 = 0;
    int32_t *l0 = nullptr, *p0 = nullptr;
    void *iargs[] = {&h->P, &s0, &l0, &p0};
    cudaKernelNodeParams ki = {};
    ki.func = (void *)k_init;
    ki.gridDim = dim3(init_grid(h));
    ki.blockDim = dim3(256);
    ki.kernelParams = iargs;
    CK(h, cudaGraphAddKernelNode(&h->init_node, g, nullptr, 0, &ki));
  }
  auto kparams = [&](void *fn, int grid, int block, size_t smem) {
    cudaKernelNodeParams k = {};
    k.func = fn;
    k.gridDim = dim3(grid);
    k.blockDim = dim3(block);
    k.sharedMemBytes = (unsigned)smem;
    k.kernelParams = args;
    return k;
  };
  // A chain of tier kernels: every kernel returns at once unless the current level is of its
  // tier, so a chain runs consecutive levels of changing tiers kernel to kernel, without a
  // conditional round trip (k_small / k_cluster run a whole run of their levels per launch,
  // a (k_explore, k_compact) pair or a bottom-up triple one level).  S = k_small, C =
  // k_cluster, T = top-down pair, B = bottom-up triple.  The canonical sequence of a
  // traversal is S C T^td C S (top-down) or S C T^td B^bu T^td C S (direction-optimising).
  const std::string seq = std::string("SC") + std::string(S3BFS_TD_CHAIN, 'T') +
      (h->P.direction ? std::string(S3BFS_BU_CHAIN, 'B') + std::string(S3BFS_TD_CHAIN, 'T')
                      : std::string()) + "CS";
  auto add_chain = [&](cudaGraph_t bg, const std::string &chain, cudaGraphNode_t prev,
                       cudaGraphNode_t *last) -> s3bfs_status {
    auto add = [&](void *fn, int grid, int block, size_t smem) -> s3bfs_status {
      cudaGraphNode_t nd;
      cudaKernelNodeParams kp = kparams(fn, grid, block, smem);
      CK(h, cudaGraphAddKernelNode(&nd, bg, prev ? &prev : nullptr, prev ? 1 : 0, &kp));
      prev = nd;
      return S3BFS_OK;
    };
    for (const char k : chain) {
      s3bfs_status r = S3BFS_OK;
      if (k == 'S') {
        r = add((void *)k_small, 1, KS_THREADS, h->ks_smem);
      } else if (k == 'C') {
        r = add((void *)k_cluster, KC_CL, KC_THREADS, h->kc_smem);
      } else if (k == 'T') {
        r = add((void *)k_explore<false>, h->P.p_max, KD_THREADS, 0);
        if (r == S3BFS_OK) r = add((void *)k_compact, h->P.p_max, KD_THREADS, 0);
      } else {  // 'B'
        r = add((void *)k_fb_clear, h->num_sms * 4, 256, 0);
        if (r == S3BFS_OK) r = add((void *)k_fb_set, h->num_sms * 4, 256, 0);
        if (r == S3BFS_OK) r = add((void *)k_bottom_up, h->P.p_max, KD_THREADS, 0);
      }
      if (r != S3BFS_OK) return r;
    }
    if (last) *last = prev;
    return S3BFS_OK;
  };
  // S3BFS_GRAPH_PROLOGUE (top-down handles): the canonical sequence runs once straight after
  // k_init, so a typical traversal never enters the WHILE body (the WHILE only evaluates its
  // condition).  Not with direction optimisation: its 29-launch sequence costs more idle
  // launches than the round trips it saves (R-MAT 20 -3 %, ER -2 %).
  cudaGraphNode_t pre = h->init_node;
  if (graph_prologue(h)) {
    s3bfs_status r = add_chain(g, seq, h->init_node, &pre);
    if (r != S3BFS_OK) return r;
  }
  cudaGraphNode_t wnode;
  CK(h, cudaGraphAddNode(&wnode, g, &pre, 1, &wp));
  cudaGraph_t body = wp.conditional.phGraph_out[0];

  {  // after the loop: d[0:n-1] and parent in caller ids
    cudaKernelNodeParams kf = {};
    kf.func = h->P.bub ? (void *)k_finalize<true> : (void *)k_finalize<false>;
    kf.gridDim = dim3(finalize_grid(h));
    kf.blockDim = dim3(256);
    kf.kernelParams = args;
    cudaGraphNode_t fnode;
    CK(h, cudaGraphAddKernelNode(&fnode, g, &wnode, 1, &kf));
  }
  // One SWITCH per WHILE iteration selects the body of the tier the next level runs in:
  // body 0 tier 0, body 1 top-down, body 2 bottom-up (NEXT-3), body 3 the cluster tier.
  // S3BFS_UNIVERSAL_BODY: body t is the canonical sequence from tier t on; otherwise body t
  // = its own tier only (S, T^td, B^bu, C).
  const char body_tier[4] = {'S', 'T', 'B', 'C'};
  cudaGraphNodeParams sp = {};
  sp.type = cudaGraphNodeTypeConditional;
  sp.conditional.handle = ht;
  sp.conditional.type = cudaGraphCondTypeSwitch;
  sp.conditional.size = 4;  // body 2 stays empty without NEXT-3
  cudaGraphNode_t snode;
  CK(h, cudaGraphAddNode(&snode, body, nullptr, 0, &sp));
  for (int bi = 0; bi < 4; ++bi) {
    if (bi == 2 && !h->P.direction) continue;
    const char t = body_tier[bi];
    const std::string chain = S3BFS_UNIVERSAL_BODY ? seq.substr(seq.find(t))
                            : t == 'T' ? std::string(S3BFS_TD_CHAIN, 'T')
                            : t == 'B' ? std::string(S3BFS_BU_CHAIN, 'B') : std::string(1, t);
    s3bfs_status r = add_chain(sp.conditional.phGraph_out[bi], chain, nullptr, nullptr);
    if (r != S3BFS_OK) return r;
  }

  CK(h, cudaGraphInstantiate(&h->exec, g, 0));
  return S3BFS_OK;
}

}  // namespace

extern "C" {

const char *s3bfs_status_string(s3bfs_status s) {
  switch (s) {
    case S3BFS_OK: return "ok";
    case S3BFS_ERR_INVALID_ARGUMENT: return "invalid argument";
    case S3BFS_ERR_UNSUPPORTED: return "unsupported";
    case S3BFS_ERR_OUT_OF_MEMORY: return "out of memory";
    case S3BFS_ERR_CUDA: return "CUDA error";
    case S3BFS_ERR_INVALID_GRAPH: return "invalid CSR graph";
  }
  return "unknown status";
}

s3bfs_status s3bfs_last_error(s3bfs_handle h, const char **msg) {
  if (!msg) return S3BFS_ERR_INVALID_ARGUMENT;
  *msg = h ? h->err.c_str() : g_err.c_str();
  return S3BFS_OK;
}

}  // extern "C"

namespace {
// create (share == NULL) or clone (share = the handle whose prepared graph is reused)
s3bfs_status create_impl(s3bfs_handle *out, int32_t n, int64_t nnz, const int32_t *row_offsets,
                         const int32_t *col_indices, const s3bfs_options *opts,
                         s3bfs_stream_t stream_, const s3bfs_ctx *share) {
  if (!out) return fail(nullptr, S3BFS_ERR_INVALID_ARGUMENT, "out is NULL");
  *out = nullptr;
  if (n <= 0) return fail(nullptr, S3BFS_ERR_INVALID_ARGUMENT, "n must be >= 1");
  if (n > INT32_MAX - 256)  // internal ids incl. the bitmap sentinel (Params::v_sent) fit int32
    return fail(nullptr, S3BFS_ERR_INVALID_ARGUMENT, "n out of [1, INT32_MAX - 256]");
  if (nnz < 0 || nnz > INT32_MAX) return fail(nullptr, S3BFS_ERR_INVALID_ARGUMENT, "nnz out of [0, INT32_MAX]");
  if (!row_offsets || (nnz > 0 && !col_indices))
    return fail(nullptr, S3BFS_ERR_INVALID_ARGUMENT, "null graph pointer");
  if (!is_device_ptr(row_offsets) || (nnz > 0 && !is_device_ptr(col_indices)))
    return fail(nullptr, S3BFS_ERR_INVALID_ARGUMENT, "graph arrays must be device memory");
  cudaStream_t stream = (cudaStream_t)stream_;

  s3bfs_ctx *h = new (std::nothrow) s3bfs_ctx;
  if (!h) return fail(nullptr, S3BFS_ERR_OUT_OF_MEMORY, "host allocation failed");
  auto bail = [&](s3bfs_status s) {
    g_err = h->err;
    s3bfs_destroy(h);
    return s;
  };
  h->n = n;
  h->nnz = nnz;
  h->ro = row_offsets;
  h->col = col_indices;
  if (opts) h->opt = *opts;
  if (share) {
    h->gs = share->gs;
    h->gs->refs++;
  } else {
    h->gs = new (std::nothrow) GraphStore;
    if (!h->gs) return bail(fail(h, S3BFS_ERR_OUT_OF_MEMORY, "host allocation failed"));
  }
  cudaError_t e;
  if ((e = cudaGetDevice(&h->dev)) != cudaSuccess) return bail(cuda_fail(h, e, "cudaGetDevice"));
  cudaDeviceProp prop;
  if ((e = cudaGetDeviceProperties(&prop, h->dev)) != cudaSuccess)
    return bail(cuda_fail(h, e, "cudaGetDeviceProperties"));
  if (prop.major != 10)
    return bail(fail(h, S3BFS_ERR_UNSUPPORTED,
                     "needs a compute capability 10.x device (sm_100a build), got " +
                         std::to_string(prop.major) + "." + std::to_string(prop.minor)));
  h->num_sms = prop.multiProcessorCount;

  // ---- (f) tunables ----
  int occ_x = 0, occ_c = 0;
  if ((e = cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ_x, k_explore<false>, KD_THREADS, 0)) != cudaSuccess)
    return bail(cuda_fail(h, e, "occupancy(k_explore)"));
  if ((e = cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ_c, k_compact, KD_THREADS, 0)) != cudaSuccess)
    return bail(cuda_fail(h, e, "occupancy(k_compact)"));
  int occ = occ_x < occ_c ? occ_x : occ_c;
  if (occ < 1) occ = 1;
  int p_max = h->num_sms * occ;  // every CTA resident: the look-back never waits on a CTA
  if (h->opt.max_ctas > 0 && h->opt.max_ctas < p_max) p_max = h->opt.max_ctas;
  if (p_max > KD_THREADS) p_max = KD_THREADS;  // k_compact's one-round-trip prefix: a thread per tile
  const int grain = h->opt.edges_per_cta > 0 ? h->opt.edges_per_cta : 1024;
  // cluster tier: T0 < e_l <= tc_max (one 8-CTA cluster); tier 0 keeps the small levels
  int tc_max = h->opt.cluster_max_edges == 0 ? KC_CL * KC_ECTA : h->opt.cluster_max_edges;
  if (tc_max > KC_CL * KC_ECTA) tc_max = KC_CL * KC_ECTA;
  if (h->opt.cluster_max_edges < 0 || h->opt.variant == 1) tc_max = -1;
  int t0 = h->opt.tier0_max_edges == 0 ? (tc_max > 0 ? S3BFS_T0_WITH_CLUSTER : KS_ECAP)
                                       : h->opt.tier0_max_edges;
  if (t0 > KS_ECAP) t0 = KS_ECAP;
  if (h->opt.variant == 1) t0 = -1;
  h->loop_graph = h->opt.loop_mode == 2 ? 0 : 1;
  const int dist_size = h->opt.dist_size > 1 ? h->opt.dist_size : 1;
  const int dist_rank = dist_size > 1 ? h->opt.dist_rank : 0;
  if (dist_size > 1) {  // NEXT-4: host-driven per-level protocol, every level on tier 1
    if (dist_size > DIST_MAX)
      return bail(fail(h, S3BFS_ERR_UNSUPPORTED, "dist_size > 8 (ranks of one node)"));
    if (share) return bail(fail(h, S3BFS_ERR_UNSUPPORTED, "clones of a dist_size > 1 handle"));
    if (dist_rank < 0 || dist_rank >= dist_size)
      return bail(fail(h, S3BFS_ERR_INVALID_ARGUMENT, "dist_rank not in [0, dist_size)"));
    if (h->opt.direction == 1)
      return bail(fail(h, S3BFS_ERR_UNSUPPORTED, "dist_size > 1 with direction = 1"));
    h->loop_graph = 0;
    t0 = -1;
    tc_max = -1;
  }
  const int collect = h->opt.collect_stats >= 0 ? 1 : 0;

  // ---- workspace (one allocation) ----
  h->cand_cap = nnz + (int64_t)p_max * (KD_WARPS + 1 + KD_SLACK) + 64;
  if (h->cand_cap >= INT32_MAX)
    return bail(fail(h, S3BFS_ERR_UNSUPPORTED, "nnz too large for int32 candidate slots"));
  const int stats_cap = n + 1 < (1 << 16) ? n + 1 : (1 << 16);
  // vertex-indexed arrays: n entries, or this rank's local slots with dist_size > 1
  const long long nblk = ((long long)n + 31) / 32;
  const long long nloc = dist_size > 1 ? (nblk + dist_size - 1) / dist_size * 32 : n;
  const long long nv = (nloc > n ? nloc : n) + 32;
  const size_t nb = (size_t)nv * 4, nb1 = (size_t)(nv + 1) * 4;
  size_t off = 0;
  auto take = [&](size_t bytes) { size_t o = off; off += align256(bytes); return o; };
  const size_t o_vinfo = take((size_t)nv * 32);  // 32-byte vertex records (Params::vinfo)
  const size_t o_vs16 = take((size_t)nv * 16);   // dense copy of their static halves
  size_t o_f[2], o_frs[2], o_fex[2];
  for (int i = 0; i < 2; ++i) { o_f[i] = take(nb); o_frs[i] = take(nb); o_fex[i] = take(nb1 + 16); }
  const size_t o_cand = take((size_t)h->cand_cap * 4);
  const size_t o_crd = take((size_t)h->cand_cap * 8);
  const size_t bm_bytes = ((size_t)n + 127) / 128 * 16;  // 16 B padded (vector clears)
  const size_t o_bm = take(bm_bytes + 16);  // + the sentinel block (Params::v_sent)
  // claim slots: a power of two >= max(n, a floor) (claim_slot's hash is mod 2^k); the floor
  // spreads a small graph's tags over more L2 lines (fewer same-line probes and stores)
  size_t claim_n = 16;
  while (claim_n < (size_t)n || claim_n < (size_t)S3BFS_CLAIM_MIN_BYTES) claim_n <<= 1;
  const size_t o_claim = take(claim_n);
  const size_t o_fb0 = take(bm_bytes), o_fb1 = take(bm_bytes);
  const bool bu_on = h->opt.direction == 1;  // NEXT-3: dense labels of bottom-up finds
  const size_t o_lpd = take(bu_on ? (size_t)nv * 8 : 0), o_bub = take(bu_on ? bm_bytes : 0);
  const size_t o_wcnt = take((size_t)p_max * KD_WARPS * 4);
  const size_t o_status = take((size_t)p_max * (dist_size > 1 ? dist_size : 1) * 8 + 8);
  // NEXT-3 bottom-up tiles: width = the power of two >= words / (tiles-per-CTA x P_max), at
  // least 64 words (one BU_W-word round for each of a CTA's 16 warps)
  const long long bu_words = (((long long)n + 127) >> 7) << 2;
  int bu_tile_w = 64;
  while ((long long)bu_tile_w * S3BFS_BU_TILES_PER_CTA * p_max < bu_words) bu_tile_w <<= 1;
  const int bu_tiles = h->opt.direction == 1 ? (int)((bu_words + bu_tile_w - 1) / bu_tile_w) : 0;
  const size_t o_bustatus = take((size_t)(bu_tiles + 1) * 8);
  const size_t o_ctl = take(sizeof(Ctl));
  const size_t o_stats = take((size_t)stats_cap * sizeof(s3bfs_level_stat));
  h->ws_bytes = off;
  if ((e = cudaMalloc(&h->ws, h->ws_bytes)) != cudaSuccess) return bail(cuda_fail(h, e, "cudaMalloc(workspace)"));
  char *base = (char *)h->ws;
  Params &P = h->P;
  P.col = col_indices;
  P.n = n;
  P.ctl = (Ctl *)(base + o_ctl);
  P.vinfo = (int4 *)(base + o_vinfo);
  P.vs16 = (const int4 *)(base + o_vs16);
  for (int i = 0; i < 2; ++i) {
    P.f[i] = (int32_t *)(base + o_f[i]);
    P.frs[i] = (int32_t *)(base + o_frs[i]);
    P.fex[i] = (int32_t *)(base + o_fex[i]);
  }
  P.cand = (int32_t *)(base + o_cand);
  P.cand_rd = (int2 *)(base + o_crd);
  P.bm = (uint32_t *)(base + o_bm);
  P.v_sent = (int32_t)(bm_bytes * 8);
  P.claim = (uint8_t *)(base + o_claim);
  P.claim_mask = (uint32_t)(claim_n - 1);
  // k_explore's visited test: ids < hub through the bitmap first (hot, L1-resident words once
  // the graph is degree-ordered), the rest by their discovery tag alone (R26)
  {
    const long long hv = h->opt.hub_vertices;
    long long hub = hv < 0 ? n : hv > 0 ? hv : (h->opt.reorder >= 0 ? (1LL << 19) : n);
    P.hub = (int32_t)(hub < n ? hub : n);
    const int tp = h->opt.tag_mode_pct;
    P.tag_pct = tp == 0 ? S3BFS_TAG_MODE_PCT : tp < 0 ? -1 : tp;
    // level passes (plan_pass): defaults from the R-MAT 24 sweep (profiles/r02_level_passes.log)
    const int sm = h->opt.split_min_edges, sp = h->opt.split_first_pct, sn = h->opt.split_passes;
    P.split_min = sm == 0 ? S3BFS_SPLIT_MIN_EDGES : sm;
    P.split_pct = sp <= 0 ? S3BFS_SPLIT_FIRST_PCT : sp > 99 ? 99 : sp;
    P.split_passes = sn == 0 ? S3BFS_SPLIT_PASSES : sn;
  }
  P.lpd = bu_on ? (int2 *)(base + o_lpd) : nullptr;
  P.bub = bu_on ? (uint32_t *)(base + o_bub) : nullptr;
  P.fb[0] = (uint32_t *)(base + o_fb0);
  P.fb[1] = (uint32_t *)(base + o_fb1);
  P.wcnt = (int32_t *)(base + o_wcnt);
  P.status = (unsigned long long *)(base + o_status);
  P.bu_status = (unsigned long long *)(base + o_bustatus);
  P.bu_tiles = bu_tiles;
  P.bu_tile_w = bu_tile_w;
  P.stats = (s3bfs_level_stat *)(base + o_stats);
  P.stats_cap = stats_cap;
  P.p_max = p_max;
  P.grain = grain;
  P.t0 = t0;
  P.tc_max = tc_max;
  P.variant = h->opt.variant == 1 ? 1 : 0;
  P.collect_stats = collect;
  P.use_graph = 0;
  P.n2o = nullptr;
  P.o2n = nullptr;
  P.direction = h->opt.direction == 1 ? 1 : 0;
  P.do_alpha = h->opt.do_alpha > 0 ? h->opt.do_alpha : 14;
  P.do_beta = h->opt.do_beta != 0 ? h->opt.do_beta : 24;
  P.n_scan = n;
  P.nnz = nnz;
  P.nnz_all = nnz;
  P.cand_cap = h->cand_cap;
  P.dist_size = dist_size;
  P.dist_rank = dist_rank;
  P.nloc = n;
  if (share) {  // a clone: the prepared graph is the source handle's; vertex records copied
    P.col = share->P.col;
    P.n2o = share->P.n2o;
    P.o2n = share->P.o2n;
    P.n_scan = share->P.n_scan;
    P.tro = share->P.tro;
    P.tcol = share->P.tcol;
    h->ro_int = share->ro_int;
    if ((e = cudaMemcpyAsync(P.vinfo, share->P.vinfo, (size_t)n * 32, cudaMemcpyDeviceToDevice,
                             stream)) != cudaSuccess ||
        (e = cudaMemcpyAsync(const_cast<int4 *>(P.vs16), share->P.vs16, (size_t)n * 16,
                             cudaMemcpyDeviceToDevice, stream)) != cudaSuccess)
      return bail(cuda_fail(h, e, "copy vertex records"));
  }
  if (!share && h->opt.validate_csr) {
    int h_err = 0;
    AsyncTmp err_b(stream);
    if ((e = err_b.alloc(4)) != cudaSuccess) return bail(cuda_fail(h, e, "cudaMallocAsync"));
    int *d_err = err_b.as<int>();
    cudaMemsetAsync(d_err, 0, 4, stream);
    k_validate<<<h->num_sms * 8, 256, 0, stream>>>(row_offsets, col_indices, n, nnz, d_err);
    cudaMemcpyAsync(&h_err, d_err, 4, cudaMemcpyDeviceToHost, stream);
    if ((e = cudaStreamSynchronize(stream)) != cudaSuccess) return bail(cuda_fail(h, e, "validate_csr"));
    if (h_err) {
      std::string m = "CSR invalid:";
      if (h_err & 1) m += " row_offsets[0] != 0;";
      if (h_err & 2) m += " row_offsets decreasing;";
      if (h_err & 4) m += " row_offsets[n] != nnz;";
      if (h_err & 8) m += " column index out of [0, n);";
      return bail(fail(h, S3BFS_ERR_INVALID_GRAPH, m));
    }
  }
  if (share) {
  } else if (h->opt.reorder >= 0) {
    s3bfs_status rs = build_reordered(h, stream);
    if (rs != S3BFS_OK) return bail(rs);
  } else {
    k_build_vinfo<<<h->num_sms * 8, 256, 0, stream>>>(row_offsets, nullptr, n, P.vinfo,
                                                      const_cast<int4 *>(P.vs16));
    if ((e = cudaGetLastError()) != cudaSuccess) return bail(cuda_fail(h, e, "k_build_vinfo"));
    h->ro_int = row_offsets;
  }
  if (dist_size > 1) {
    s3bfs_status ds = build_dist(h, stream, (int)nloc);
    if (ds != S3BFS_OK) return bail(ds);
  }
  P.col_vec = (((uintptr_t)P.col) & 15) == 0 ? 1 : 0;
  if (P.direction && !share) {
    s3bfs_status ts = build_in_adjacency(h, stream);
    if (ts != S3BFS_OK) return bail(ts);
  }
  {  // L2 policy descriptors (uniform kernel parameters of k_explore)
    unsigned long long h_pol[2] = {0, 0};
    AsyncTmp pol_b(stream);
    if ((e = pol_b.alloc(16)) != cudaSuccess) return bail(cuda_fail(h, e, "cudaMallocAsync"));
    unsigned long long *d_pol = pol_b.as<unsigned long long>();
    k_policies<<<1, 1, 0, stream>>>(d_pol);
    cudaMemcpyAsync(h_pol, d_pol, 16, cudaMemcpyDeviceToHost, stream);
    if ((e = cudaStreamSynchronize(stream)) != cudaSuccess) return bail(cuda_fail(h, e, "k_policies"));
    P.pol_first = h_pol[0];
    P.pol_last = h_pol[1];
  }
  if ((e = cudaMemsetAsync(P.ctl, 0, sizeof(Ctl), stream)) != cudaSuccess) return bail(cuda_fail(h, e, "memset(ctl)"));
  if ((e = cudaMemsetAsync(P.status, 0, (size_t)p_max * dist_size * 8 + 8, stream)) != cudaSuccess) return bail(cuda_fail(h, e, "memset(status)"));
  if (h->opt.debug_poison) {
    k_poison<<<h->num_sms * 4, 256, 0, stream>>>(P.vinfo, n, (int)h->cand_cap);
    if ((e = cudaGetLastError()) != cudaSuccess) return bail(cuda_fail(h, e, "k_poison"));
  }

  h->ks_smem = (size_t)(3 * KS_NCAP + 4 + (S3BFS_KS_ONCHIP ? KS_TAB : 2 * KS_ECAP)) * 4;
  if ((e = cudaFuncSetAttribute(k_small, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)h->ks_smem)) != cudaSuccess)
    return bail(cuda_fail(h, e, "cudaFuncSetAttribute(k_small)"));
  h->kc_smem = (size_t)(3 * KC_FCAP + 4 + 2 * KC_ECTA) * 4;
  if ((e = cudaFuncSetAttribute(k_cluster, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)h->kc_smem)) != cudaSuccess)
    return bail(cuda_fail(h, e, "cudaFuncSetAttribute(k_cluster)"));

  if (h->loop_graph) {
    s3bfs_status s = build_graph(h);
    if (s != S3BFS_OK) return bail(s);
  } else {
    if ((e = cudaMallocHost((void **)&h->h_ctl, sizeof(Ctl))) != cudaSuccess) return bail(cuda_fail(h, e, "cudaMallocHost"));
    if (h->opt.time_kernels) {
      h->time_kernels = true;
      for (auto &ev : h->ev)
        if ((e = cudaEventCreate(&ev)) != cudaSuccess) return bail(cuda_fail(h, e, "cudaEventCreate"));
    }
  }
  if ((e = cudaStreamSynchronize(stream)) != cudaSuccess) return bail(cuda_fail(h, e, "create sync"));
  *out = h;
  return S3BFS_OK;
}
}  // namespace

extern "C" {

s3bfs_status s3bfs_create(s3bfs_handle *out, int32_t n, int64_t nnz, const int32_t *row_offsets,
                          const int32_t *col_indices, const s3bfs_options *opts,
                          s3bfs_stream_t stream) {
  return create_impl(out, n, nnz, row_offsets, col_indices, opts, stream, nullptr);
}

s3bfs_status s3bfs_clone(s3bfs_handle src, s3bfs_handle *out, s3bfs_stream_t stream) {
  if (!src) return fail(nullptr, S3BFS_ERR_INVALID_ARGUMENT, "source handle is NULL");
  return create_impl(out, src->n, src->nnz, src->ro, src->col, &src->opt, stream, src);
}

s3bfs_status s3bfs_run(s3bfs_handle h, int32_t source, int32_t *level, int32_t *parent,
                       s3bfs_stream_t stream_) {
  if (!h) return fail(nullptr, S3BFS_ERR_INVALID_ARGUMENT, "handle is NULL");
  if (source < 0 || source >= h->n)
    return fail(h, S3BFS_ERR_INVALID_ARGUMENT, "source " + std::to_string(source) + " not in [0, n)");
  if (!level || !parent) return fail(h, S3BFS_ERR_INVALID_ARGUMENT, "level/parent is NULL");
  if (!is_device_ptr(level) || !is_device_ptr(parent))
    return fail(h, S3BFS_ERR_INVALID_ARGUMENT, "level/parent must be device memory");
  if (h->P.dist_size > 1)
    return fail(h, S3BFS_ERR_UNSUPPORTED, "a dist_size > 1 handle is driven by s3bfs_dist_*");
  cudaStream_t stream = (cudaStream_t)stream_;
  h->last_stream = stream;
  h->ran = true;
  if (h->loop_graph) {
    void *iargs[] = {&h->P, &source, &level, &parent};
    cudaKernelNodeParams ki = {};
    ki.func = (void *)k_init;
    ki.gridDim = dim3(init_grid(h));
    ki.blockDim = dim3(256);
    ki.kernelParams = iargs;
    CK(h, cudaGraphExecKernelNodeSetParams(h->exec, h->init_node, &ki));
    CK(h, cudaGraphLaunch(h->exec, stream));
    return S3BFS_OK;
  }
  k_init<<<init_grid(h), 256, 0, stream>>>(h->P, source, level, parent);
  CK(h, cudaGetLastError());
  // host-driven loop: one control-block read per level (debug / timing mode)
  h->kt = s3bfs_kernel_times{};
  int pending = -1;  // tier of the launch whose events are not yet read
  for (;;) {
    CK(h, cudaMemcpyAsync(h->h_ctl, h->P.ctl, sizeof(Ctl), cudaMemcpyDeviceToHost, stream));
    CK(h, cudaStreamSynchronize(stream));
    if (pending >= 0) {
      float a = 0.f, b = 0.f;
      if (pending == TIER_SMALL || pending == TIER_CLUSTER) {
        CK(h, cudaEventElapsedTime(&a, h->ev[0], h->ev[1]));
        h->kt.small_ms += a;
        h->kt.small_launches++;
      } else if (pending == TIER_BU) {
        CK(h, cudaEventElapsedTime(&a, h->ev[0], h->ev[1]));
        h->kt.bottom_up_ms += a;
        h->kt.bottom_up_launches++;
      } else {
        CK(h, cudaEventElapsedTime(&a, h->ev[0], h->ev[1]));
        CK(h, cudaEventElapsedTime(&b, h->ev[1], h->ev[2]));
        h->kt.explore_ms += a;
        h->kt.compact_ms += b;
        h->kt.explore_launches++;
        h->kt.compact_launches++;
      }
      pending = -1;
    }
    const Ctl c = *h->h_ctl;
    if (c.tier == TIER_DONE) {
      if (h->P.bub) k_finalize<true><<<finalize_grid(h), 256, 0, stream>>>(h->P);
      else k_finalize<false><<<finalize_grid(h), 256, 0, stream>>>(h->P);
      CK(h, cudaGetLastError());
      break;
    }
    if (h->time_kernels) CK(h, cudaEventRecord(h->ev[0], stream));
    if (c.tier == TIER_SMALL) {
      k_small<<<1, KS_THREADS, h->ks_smem, stream>>>(h->P);
      if (h->time_kernels) CK(h, cudaEventRecord(h->ev[1], stream));
    } else if (c.tier == TIER_CLUSTER) {
      k_cluster<<<KC_CL, KC_THREADS, h->kc_smem, stream>>>(h->P);
      if (h->time_kernels) CK(h, cudaEventRecord(h->ev[1], stream));
    } else if (c.tier == TIER_BU) {
      k_fb_clear<<<h->num_sms * 4, 256, 0, stream>>>(h->P);
      k_fb_set<<<h->num_sms * 4, 256, 0, stream>>>(h->P);
      k_bottom_up<<<h->P.p_max, KD_THREADS, 0, stream>>>(h->P);
      if (h->time_kernels) CK(h, cudaEventRecord(h->ev[1], stream));
    } else {
      k_explore<false><<<c.p_l, KD_THREADS, 0, stream>>>(h->P);
      if (h->time_kernels) CK(h, cudaEventRecord(h->ev[1], stream));
      k_compact<<<c.p_l, KD_THREADS, 0, stream>>>(h->P);
      if (h->time_kernels) CK(h, cudaEventRecord(h->ev[2], stream));
    }
    CK(h, cudaGetLastError());
    if (h->time_kernels) pending = c.tier;
  }
  return S3BFS_OK;
}

// ---- NEXT-4: one traversal over G ranks, 1-D vertex partition (include/s3bfs.h) ----------------
s3bfs_status s3bfs_dist_status(s3bfs_handle h, s3bfs_stream_t stream_, int32_t *done,
                               int64_t *n_next);
static s3bfs_status dist_check(s3bfs_handle h) {
  if (!h) return fail(nullptr, S3BFS_ERR_INVALID_ARGUMENT, "handle is NULL");
  if (h->P.dist_size <= 1) return fail(h, S3BFS_ERR_UNSUPPORTED, "handle has dist_size <= 1");
  return S3BFS_OK;
}

s3bfs_status s3bfs_dist_export(s3bfs_handle h, s3bfs_dist_peer *out) {
  s3bfs_status s = dist_check(h);
  if (s != S3BFS_OK) return s;
  if (!out) return fail(h, S3BFS_ERR_INVALID_ARGUMENT, "out is NULL");
  std::memset(out, 0, sizeof(*out));
  out->rank = h->P.dist_rank;
  out->size = h->P.dist_size;
  out->base = (uint64_t)(uintptr_t)h->xws;
  out->recv = (uint64_t)(uintptr_t)h->P.recv;
  out->rcnt = (uint64_t)(uintptr_t)h->P.rcnt;
  out->rmeta = (uint64_t)(uintptr_t)h->P.rmeta;
  out->rtot = (uint64_t)(uintptr_t)h->P.rtot;
  out->bm = (uint64_t)(uintptr_t)h->P.bm;
  out->vinfo = (uint64_t)(uintptr_t)h->P.vinfo;
  static_assert(sizeof(cudaIpcMemHandle_t) <= sizeof(out->ipc), "IPC handle size");
  cudaIpcMemHandle_t ih;
  cudaError_t e = cudaIpcGetMemHandle(&ih, h->xws);
  if (e == cudaSuccess) std::memcpy(out->ipc, &ih, sizeof(ih));
  else cudaGetLastError();  // no IPC (e.g. a sandbox): loopback connections still work
  out->ipc_valid = e == cudaSuccess ? 1 : 0;
  return S3BFS_OK;
}

s3bfs_status s3bfs_dist_connect(s3bfs_handle h, const s3bfs_dist_peer *peers, int32_t count,
                                int32_t use_ipc) {
  s3bfs_status s = dist_check(h);
  if (s != S3BFS_OK) return s;
  const int G = h->P.dist_size, me = h->P.dist_rank;
  if (!peers || count != G) return fail(h, S3BFS_ERR_INVALID_ARGUMENT, "need one peer record per rank");
  for (int d = 0; d < G; ++d)
    if (peers[d].rank != d || peers[d].size != G)
      return fail(h, S3BFS_ERR_INVALID_ARGUMENT, "peer records must be in rank order, same size");
  Params &P = h->P;
  for (int d = 0; d < G; ++d) {
    const s3bfs_dist_peer &q = peers[d];
    char *base = (char *)(uintptr_t)q.base;
    if (d == me) {
      base = (char *)h->xws;
    } else if (use_ipc) {
      if (!q.ipc_valid) return fail(h, S3BFS_ERR_UNSUPPORTED, "peer exported no IPC handle");
      if (h->ipc_open[d]) { cudaIpcCloseMemHandle(h->ipc_open[d]); h->ipc_open[d] = nullptr; }
      cudaIpcMemHandle_t ih;
      std::memcpy(&ih, q.ipc, sizeof(ih));
      void *p = nullptr;
      CK(h, cudaIpcOpenMemHandle(&p, ih, cudaIpcMemLazyEnablePeerAccess));
      h->ipc_open[d] = p;
      base = (char *)p;
    }
    auto map = [&](uint64_t a) { return base + (a - q.base); };  // same layout, rebased
    P.p_recv[d] = (int2 *)map(q.recv);
    P.p_rcnt[d] = (int32_t *)map(q.rcnt);
    P.p_rmeta[d] = (int2 *)map(q.rmeta);
    P.p_rtot[d] = (int2 *)map(q.rtot);
    P.p_bm[d] = (uint32_t *)map(q.bm);
    P.p_vinfo[d] = (int4 *)map(q.vinfo);
  }
  return S3BFS_OK;
}

s3bfs_status s3bfs_dist_begin(s3bfs_handle h, int32_t source, int32_t *level, int32_t *parent,
                              s3bfs_stream_t stream_) {
  s3bfs_status s = dist_check(h);
  if (s != S3BFS_OK) return s;
  if (source < 0 || source >= h->n)
    return fail(h, S3BFS_ERR_INVALID_ARGUMENT, "source " + std::to_string(source) + " not in [0, n)");
  if (!level || !parent || !is_device_ptr(level) || !is_device_ptr(parent))
    return fail(h, S3BFS_ERR_INVALID_ARGUMENT, "level/parent must be device memory");
  cudaStream_t stream = (cudaStream_t)stream_;
  h->last_stream = stream;
  h->ran = true;
  h->d_level = level;
  h->d_parent = parent;
  CK(h, cudaMemsetAsync(level, 0xff, (size_t)h->n * 4, stream));   // -1: not this rank's
  CK(h, cudaMemsetAsync(parent, 0xff, (size_t)h->n * 4, stream));  //     (or unreached)
  k_dist_init<<<init_grid(h), 256, 0, stream>>>(h->P, source);
  CK(h, cudaGetLastError());
  return S3BFS_OK;
}

s3bfs_status s3bfs_dist_explore(s3bfs_handle h, s3bfs_stream_t stream_) {
  s3bfs_status s = dist_check(h);
  if (s != S3BFS_OK) return s;
  // P_max CTAs: the level's P_l <= P_max is read on the device (surplus CTAs return at once)
  k_explore<true><<<h->P.p_max, KD_THREADS, 0, (cudaStream_t)stream_>>>(h->P);
  CK(h, cudaGetLastError());
  return S3BFS_OK;
}

s3bfs_status s3bfs_dist_dedup(s3bfs_handle h, s3bfs_stream_t stream_) {
  s3bfs_status s = dist_check(h);
  if (s != S3BFS_OK) return s;
  cudaStream_t stream = (cudaStream_t)stream_;
  k_dist_keep<<<h->P.p_max, KD_THREADS, 0, stream>>>(h->P);
  CK(h, cudaGetLastError());
  return S3BFS_OK;
}

s3bfs_status s3bfs_dist_advance(s3bfs_handle h, s3bfs_stream_t stream_, int32_t *done,
                                int64_t *n_next) {
  s3bfs_status s = dist_check(h);
  if (s != S3BFS_OK) return s;
  cudaStream_t stream = (cudaStream_t)stream_;
  k_dist_advance<<<1, 32, 0, stream>>>(h->P, nullptr);
  CK(h, cudaGetLastError());
  if (!done && !n_next) return S3BFS_OK;
  return s3bfs_dist_status(h, stream_, done, n_next);
}

s3bfs_status s3bfs_dist_advance_flag(s3bfs_handle h, s3bfs_stream_t stream_, int64_t *flag) {
  s3bfs_status s = dist_check(h);
  if (s != S3BFS_OK) return s;
  if (!flag) return fail(h, S3BFS_ERR_INVALID_ARGUMENT, "flag is NULL");
  k_dist_advance<<<1, 32, 0, (cudaStream_t)stream_>>>(h->P, (long long *)flag);
  CK(h, cudaGetLastError());
  return S3BFS_OK;
}

s3bfs_status s3bfs_dist_status(s3bfs_handle h, s3bfs_stream_t stream_, int32_t *done,
                               int64_t *n_next) {
  s3bfs_status s = dist_check(h);
  if (s != S3BFS_OK) return s;
  if (!done && !n_next) return fail(h, S3BFS_ERR_INVALID_ARGUMENT, "nothing to read");
  cudaStream_t stream = (cudaStream_t)stream_;
  if (!h->h_ctl) CK(h, cudaMallocHost((void **)&h->h_ctl, sizeof(Ctl)));
  CK(h, cudaMemcpyAsync(h->h_ctl, h->P.ctl, sizeof(Ctl), cudaMemcpyDeviceToHost, stream));
  CK(h, cudaStreamSynchronize(stream));
  if (done) *done = h->h_ctl->tier == TIER_DONE ? 1 : 0;
  if (n_next) *n_next = h->h_ctl->g_n_next;
  return S3BFS_OK;
}

s3bfs_status s3bfs_dist_end(s3bfs_handle h, s3bfs_stream_t stream_) {
  s3bfs_status s = dist_check(h);
  if (s != S3BFS_OK) return s;
  if (!h->d_level) return fail(h, S3BFS_ERR_INVALID_ARGUMENT, "no traversal begun");
  const long long want = ((long long)h->P.nloc + 255) / 256;
  const int grid = (int)(want < h->num_sms * 8 ? (want < 1 ? 1 : want) : h->num_sms * 8);
  k_dist_finalize<<<grid, 256, 0, (cudaStream_t)stream_>>>(h->P, h->d_level, h->d_parent);
  CK(h, cudaGetLastError());
  return S3BFS_OK;
}

s3bfs_status s3bfs_destroy(s3bfs_handle h) {
  if (!h) return S3BFS_OK;
  if (h->ran && h->last_stream) cudaStreamSynchronize(h->last_stream);
  else cudaDeviceSynchronize();
  if (h->exec) cudaGraphExecDestroy(h->exec);
  if (h->graph) cudaGraphDestroy(h->graph);
  if (h->ws) cudaFree(h->ws);
  for (auto &p : h->ipc_open)
    if (p) cudaIpcCloseMemHandle(p);
  if (h->xws) cudaFree(h->xws);
  if (h->dgraph) cudaFree(h->dgraph);
  if (h->gs && --h->gs->refs == 0) delete h->gs;
  if (h->h_ctl) cudaFreeHost(h->h_ctl);
  for (auto &ev : h->ev)
    if (ev) cudaEventDestroy(ev);
  delete h;
  return S3BFS_OK;
}

s3bfs_status s3bfs_get_level_stats(s3bfs_handle h, s3bfs_level_stat *out, int32_t cap,
                                   int32_t *num_levels) {
  if (!h || !num_levels || cap < 0 || (cap > 0 && !out)) return fail(h, S3BFS_ERR_INVALID_ARGUMENT, "bad arguments");
  *num_levels = 0;
  if (!h->ran) return S3BFS_OK;
  CK(h, cudaStreamSynchronize(h->last_stream));
  Ctl c;
  CK(h, cudaMemcpy(&c, h->P.ctl, sizeof(Ctl), cudaMemcpyDeviceToHost));
  *num_levels = c.num_levels;
  int k = c.num_levels < cap ? c.num_levels : cap;
  if (k > h->P.stats_cap) k = h->P.stats_cap;
  if (k > 0) CK(h, cudaMemcpy(out, h->P.stats, (size_t)k * sizeof(s3bfs_level_stat), cudaMemcpyDeviceToHost));
  return S3BFS_OK;
}

s3bfs_status s3bfs_get_kernel_times(s3bfs_handle h, s3bfs_kernel_times *out) {
  if (!h || !out) return fail(h, S3BFS_ERR_INVALID_ARGUMENT, "bad arguments");
  if (h->ran) CK(h, cudaStreamSynchronize(h->last_stream));
  *out = h->kt;
  return S3BFS_OK;
}

s3bfs_status s3bfs_debug_timeline(s3bfs_handle h, uint64_t out[4]) {
  if (!h || !out) return fail(h, S3BFS_ERR_INVALID_ARGUMENT, "bad arguments");
  if (h->ran) CK(h, cudaStreamSynchronize(h->last_stream));
  Ctl c;
  CK(h, cudaMemcpy(&c, h->P.ctl, sizeof(Ctl), cudaMemcpyDeviceToHost));
  for (int i = 0; i < 4; ++i) out[i] = c.t_dbg[i];
  return S3BFS_OK;
}

s3bfs_status s3bfs_get_info(s3bfs_handle h, s3bfs_info *out) {
  if (!h || !out) return fail(h, S3BFS_ERR_INVALID_ARGUMENT, "bad arguments");
  out->num_sms = h->num_sms;
  out->p_max = h->P.p_max;
  out->edges_per_cta = h->P.grain;
  out->tier0_max_edges = h->P.t0;
  out->kd_threads = KD_THREADS;
  out->kd_tile_edges = KX_GROUPS * 32;
  out->ksmall_threads = KS_THREADS;
  out->ksmall_max_frontier = KS_NCAP;
  out->td_chain = S3BFS_TD_CHAIN;
  out->bu_chain = S3BFS_BU_CHAIN;
  out->universal_body = S3BFS_UNIVERSAL_BODY;
  out->prologue = graph_prologue(h) ? 1 : 0;
  out->workspace_bytes = (int64_t)(h->ws_bytes + (h->gs ? h->gs->b2 + h->gs->b3 : 0));
  return S3BFS_OK;
}

s3bfs_status s3bfs_debug_exclusive_scan(const int32_t *in, int32_t *out, int32_t n,
                                        s3bfs_stream_t stream_) {
  if (n < 0 || !out || (n > 0 && !in)) return fail(nullptr, S3BFS_ERR_INVALID_ARGUMENT, "bad arguments");
  cudaStream_t stream = (cudaStream_t)stream_;
  if (n == 0) {
    cudaError_t e = cudaMemsetAsync(out, 0, 4, stream);
    return e == cudaSuccess ? S3BFS_OK : cuda_fail(nullptr, e, "memset");
  }
  const int tiles = (int)(((long long)n + SCAN_TILE - 1) / SCAN_TILE);
  AsyncTmp status_b(stream);
  cudaError_t e = status_b.alloc((size_t)(tiles + 1) * 8);  // + the tile counter
  if (e != cudaSuccess) return cuda_fail(nullptr, e, "cudaMallocAsync(status)");
  unsigned long long *status = status_b.as<unsigned long long>();
  cudaMemsetAsync(status, 0, (size_t)(tiles + 1) * 8, stream);
  k_scan_u32<<<tiles, SCAN_THREADS, 0, stream>>>(in, out, n, status);
  e = cudaGetLastError();
  return e == cudaSuccess ? S3BFS_OK : cuda_fail(nullptr, e, "k_scan_u32");
}

s3bfs_status s3bfs_debug_find_start_points(const int32_t *excl, int32_t n_l, int32_t chunk,
                                           int32_t p_l, int32_t *out_u, int32_t *out_off,
                                           s3bfs_stream_t stream_) {
  if (!excl || n_l < 1 || chunk < 1 || p_l < 0 || (p_l > 0 && (!out_u || !out_off)))
    return fail(nullptr, S3BFS_ERR_INVALID_ARGUMENT, "bad arguments");
  if (p_l == 0) return S3BFS_OK;
  const int threads = 256;
  const long long blocks = ((long long)p_l * 32 + threads - 1) / threads;
  k_find_start<<<(unsigned)blocks, threads, 0, (cudaStream_t)stream_>>>(excl, n_l, chunk, p_l, out_u, out_off);
  cudaError_t e = cudaGetLastError();
  return e == cudaSuccess ? S3BFS_OK : cuda_fail(nullptr, e, "k_find_start");
}

}  // extern "C"
