// lv_api.cu — C-ABI entry points (include/leann_b200.h) and the host search loop.
//
// lv_index_create mirrors Engine.open's loaders (index.py:235-274): the CSR
// levels, PQ codebooks/codes and the delete bitset are copied into HBM once.
// lv_search_batch mirrors run_search (search.py:434-443) over a batch of
// queries: matrix source = one persistent frontier launch; encoder source =
// a host loop alternating frontier launches with one packed encoder forward
// over every in-flight query's recompute request (dynamic batching).
#include <cstdlib>
#include <cstdio>
#include <algorithm>
#include <atomic>
#include <cmath>
#include <cstring>
#include <mutex>
#include <string>
#include <vector>

#include "lv_common.cuh"
#include "lv_encoder.cuh"
#include "lv_search.cuh"

namespace lv {

static thread_local std::string g_last_error;
void set_error(const std::string &msg) { g_last_error = msg; }
static std::atomic<long long> g_launches{0};
void note_launch(long long n) { g_launches.fetch_add(n, std::memory_order_relaxed); }

template <typename T>
static int dalloc(T **p, size_t count) {
  *p = nullptr;
  if (count == 0) count = 1;
  cudaError_t e = cudaMalloc((void **)p, count * sizeof(T));
  if (e != cudaSuccess) {
    set_error(std::string("cudaMalloc(") + std::to_string(count * sizeof(T)) +
              " bytes) failed: " + cudaGetErrorString(e));
    return LV_ERR_INTERNAL;
  }
  return LV_OK;
}
template <typename T>
static void dfree(T *&p) {
  if (p) cudaFree((void *)p);
  p = nullptr;
}

// Grow-only device buffer.
template <typename T>
struct DBuf {
  T *ptr = nullptr;
  size_t cap = 0;
  int ensure(size_t count) {
    if (count <= cap && ptr) return LV_OK;
    dfree(ptr);
    cap = 0;
    LV_TRY(dalloc(&ptr, count));
    cap = count;
    return LV_OK;
  }
  ~DBuf() { dfree(ptr); }
};

struct Workspace {
  DBuf<SlotState> st;
  DBuf<float> eq_d;
  DBuf<uint32_t> eq_id;
  DBuf<unsigned long long> aq;
  DBuf<uint32_t> abits, xbits;
  DBuf<uint32_t> aset, xset;  // bounded hash sets (hash visited mode)
  DBuf<int32_t> xlist, req, greq;
  DBuf<int32_t> counters;  // [0] greq_total, [1] queue_head, [2] done_count
  DBuf<unsigned long long> bytes;  // frontier algorithmic bytes
  DBuf<float> emb;
  DBuf<int32_t> hkeys, hvals, new_ids, emb_map, row_count;  // shared-recompute table
  DBuf<float> luts;
  DBuf<float> q, qn;
  DBuf<int64_t> out_ids, out_counters;
  DBuf<float> out_dist;
  DBuf<int32_t> out_count, out_status, visits, blog;
  int32_t *h_counters = nullptr;  // pinned
  // the per-slot bitmaps are all-zero between calls only when the last pass
  // finished every query (finish_query clears them); an early return leaves
  // this set and the next pass clears them in full
  bool bits_dirty = false;
  ~Workspace() {
    if (h_counters) cudaFreeHost(h_counters);
  }
};

}  // namespace lv

using namespace lv;

struct lv_index {
  int device = 0;
  int64_t n = 0;
  int32_t dim = 0, metric = 0, max_degree = 0, level_count = 0;
  int64_t entry = 0;
  std::vector<uint64_t *> offs;
  std::vector<uint32_t *> nbrs;
  std::vector<uint64_t> nnz;
  uint32_t *deleted_bits = nullptr;
  int32_t m = 0, padded = 0;
  float *codebooks = nullptr;
  uint8_t *codes = nullptr;
  float *matrix = nullptr;
  bool own_matrix = false;
  uint32_t *cached_bits = nullptr;
  int32_t *cache_slot = nullptr;
  float *cache_rows = nullptr;
  int64_t n_cached = 0;
  lv_encoder *enc = nullptr;
  void *tokens = nullptr;
  bool own_tokens = false;
  int32_t token_bytes = 0, seq_len = 0;
  lv_fetch_fn fetch = nullptr;  // LV_SOURCE_CALLBACK: host provider (ProviderSource.fetch)
  void *fetch_user = nullptr;
  Workspace ws;
  lv_search_stats stats{};
  ~lv_index() {
    for (auto p : offs) dfree(p);
    for (auto p : nbrs) dfree(p);
    dfree(deleted_bits);
    dfree(codebooks);
    dfree(codes);
    if (own_matrix) dfree(matrix);
    dfree(cached_bits);
    dfree(cache_slot);
    dfree(cache_rows);
    if (own_tokens && tokens) cudaFree(tokens);
  }
};

namespace {

int upload(void *dst, const void *src, size_t bytes, bool src_on_device, cudaStream_t s) {
  if (bytes == 0) return LV_OK;
  LV_CHECK_CUDA(cudaMemcpyAsync(dst, src, bytes,
                                src_on_device ? cudaMemcpyDeviceToDevice : cudaMemcpyHostToDevice,
                                s));
  return LV_OK;
}

// bool[n] -> packed u32 bit words on the device
int upload_bits(uint32_t **dst, const uint8_t *flags, int64_t n, bool on_device) {
  std::vector<uint8_t> host;
  const uint8_t *src = flags;
  if (on_device) {
    host.resize(n);
    LV_CHECK_CUDA(cudaMemcpy(host.data(), flags, n, cudaMemcpyDeviceToHost));
    src = host.data();
  }
  int64_t words = (n + 31) / 32;
  std::vector<uint32_t> packed(words, 0u);
  for (int64_t i = 0; i < n; ++i)
    if (src[i]) packed[i >> 5] |= 1u << (i & 31);
  if (!*dst) LV_TRY(dalloc(dst, words));
  LV_CHECK_CUDA(cudaMemcpy(*dst, packed.data(), words * 4, cudaMemcpyHostToDevice));
  return LV_OK;
}

}  // namespace

extern "C" {

const char *lv_last_error(void) { return g_last_error.c_str(); }
int lv_version(void) { return 1; }
long long lv_kernel_launches(void) { return g_launches.load(); }

int lv_index_create(const lv_index_desc *d, int device, lv_index **out) {
  LV_REQUIRE(d && out, LV_ERR_USAGE, "lv_index_create: null argument");
  *out = nullptr;
  LV_REQUIRE(d->n >= 1, LV_ERR_DATA, "graph.header: n must be >= 1");
  LV_REQUIRE(d->dim >= 1, LV_ERR_USAGE, "dim must be >= 1");
  LV_REQUIRE(d->metric >= 0 && d->metric <= 2, LV_ERR_DATA, "pq.metric: unknown metric tag");
  LV_REQUIRE(d->level_count >= 1 && d->level_count <= kMaxLevels, LV_ERR_DATA,
             "graph.header: level_count out of range");
  LV_REQUIRE(d->entry_point >= 0 && d->entry_point < d->n, LV_ERR_DATA,
             "graph.entry: entry point out of range");
  LV_REQUIRE(d->max_degree >= 1 && d->max_degree <= 1024, LV_ERR_DATA,
             "graph.header: max_degree out of range");
  LV_REQUIRE(d->n < (int64_t(1) << 31), LV_ERR_USAGE, "n must be < 2^31");
  if (d->pq_m > 0) {
    LV_REQUIRE(d->pq_m <= 256, LV_ERR_USAGE, "pq m > 256 is not supported");
    LV_REQUIRE(d->pq_padded_dim % d->pq_m == 0 && d->pq_padded_dim >= d->dim, LV_ERR_DATA,
               "pq.header: invalid geometry");
  }
  DeviceGuard guard(device);
  auto *ix = new lv_index();
  ix->device = device;
  ix->n = d->n;
  ix->dim = d->dim;
  ix->metric = d->metric;
  ix->max_degree = d->max_degree;
  ix->level_count = d->level_count;
  ix->entry = d->entry_point;
  int rc = LV_OK;
  for (int l = 0; l < d->level_count && rc == LV_OK; ++l) {
    uint64_t *o = nullptr;
    uint32_t *nb = nullptr;
    // CSR sanity (graph.py:100-135): the frontier's scratch is sized from
    // max_degree and the bitmaps are indexed by neighbour id, so every row
    // must fit max_degree and every id must be < n (O(nnz) host pass)
    const uint64_t *ho = d->level_offsets[l];
    const std::string sec = "graph.level" + std::to_string(l);
    if (ho[0] != 0 || ho[d->n] != d->level_nnz[l]) {
      set_error(sec + ".offsets: offsets[n] != neighbor count");
      rc = LV_ERR_DATA;
      break;
    }
    for (int64_t v = 0; v < d->n && rc == LV_OK; ++v) {
      if (ho[v + 1] < ho[v]) {
        set_error(sec + ".offsets: not monotone at node " + std::to_string(v));
        rc = LV_ERR_DATA;
      } else if (ho[v + 1] - ho[v] > (uint64_t)d->max_degree) {
        set_error(sec + ".degree: node " + std::to_string(v) + " exceeds M");
        rc = LV_ERR_DATA;
      }
    }
    if (rc != LV_OK) break;
    const uint32_t *hn = d->level_neighbors[l];
    for (uint64_t e = 0; e < d->level_nnz[l]; ++e) {
      if ((int64_t)hn[e] >= d->n) {
        set_error(sec + ".neighbors: id " + std::to_string(hn[e]) + " out of range");
        rc = LV_ERR_DATA;
        break;
      }
    }
    if (rc != LV_OK) break;
    rc = dalloc(&o, d->n + 1);
    if (rc == LV_OK) rc = dalloc(&nb, d->level_nnz[l]);
    ix->offs.push_back(o);
    ix->nbrs.push_back(nb);
    ix->nnz.push_back(d->level_nnz[l]);
    if (rc == LV_OK && cudaMemcpy(o, ho, (d->n + 1) * 8, cudaMemcpyHostToDevice) != cudaSuccess)
      rc = LV_ERR_INTERNAL;
    if (rc == LV_OK && d->level_nnz[l] &&
        cudaMemcpy(nb, d->level_neighbors[l], d->level_nnz[l] * 4, cudaMemcpyHostToDevice) !=
            cudaSuccess)
      rc = LV_ERR_INTERNAL;
  }
  if (rc == LV_OK && d->deleted) rc = upload_bits(&ix->deleted_bits, d->deleted, d->n, false);
  if (rc == LV_OK && d->pq_m > 0) {
    ix->m = d->pq_m;
    ix->padded = d->pq_padded_dim;
    size_t cb = (size_t)d->pq_m * kCentroids * (d->pq_padded_dim / d->pq_m);
    rc = dalloc(&ix->codebooks, cb);
    if (rc == LV_OK) rc = dalloc(&ix->codes, (size_t)d->n * d->pq_m);
    if (rc == LV_OK && cudaMemcpy(ix->codebooks, d->pq_codebooks, cb * 4,
                                  cudaMemcpyHostToDevice) != cudaSuccess)
      rc = LV_ERR_INTERNAL;
    if (rc == LV_OK && cudaMemcpy(ix->codes, d->pq_codes, (size_t)d->n * d->pq_m,
                                  cudaMemcpyHostToDevice) != cudaSuccess)
      rc = LV_ERR_INTERNAL;
  }
  if (rc != LV_OK) {
    if (g_last_error.empty()) set_error("lv_index_create: device copy failed");
    delete ix;
    return rc;
  }
  *out = ix;
  return LV_OK;
}

void lv_index_destroy(lv_index *ix) {
  if (!ix) return;
  DeviceGuard guard(ix->device);
  delete ix;
}

int lv_index_set_matrix(lv_index *ix, const float *matrix, int flags) {
  LV_REQUIRE(ix, LV_ERR_USAGE, "null index");
  DeviceGuard guard(ix->device);
  if (ix->own_matrix) dfree(ix->matrix);
  ix->matrix = nullptr;
  ix->own_matrix = false;
  if (!matrix) return LV_OK;
  if (flags & LV_IO_DEVICE) {  // borrowed device matrix (caller keeps it alive)
    ix->matrix = const_cast<float *>(matrix);
    return LV_OK;
  }
  LV_TRY(dalloc(&ix->matrix, (size_t)ix->n * ix->dim));
  ix->own_matrix = true;
  LV_CHECK_CUDA(cudaMemcpy(ix->matrix, matrix, (size_t)ix->n * ix->dim * 4, cudaMemcpyHostToDevice));
  return LV_OK;
}

int lv_index_set_deleted(lv_index *ix, const uint8_t *deleted, int flags) {
  LV_REQUIRE(ix, LV_ERR_USAGE, "null index");
  DeviceGuard guard(ix->device);
  if (!deleted) {
    dfree(ix->deleted_bits);
    return LV_OK;
  }
  return upload_bits(&ix->deleted_bits, deleted, ix->n, flags & LV_IO_DEVICE);
}

// EmbeddingCache (search.py:113-142): membership bitmap; for the encoder
// source the pinned vectors are computed once with the attached encoder.
int lv_index_set_cache(lv_index *ix, const int64_t *ids, int64_t count, int flags) {
  LV_REQUIRE(ix, LV_ERR_USAGE, "null index");
  DeviceGuard guard(ix->device);
  dfree(ix->cached_bits);
  dfree(ix->cache_slot);
  dfree(ix->cache_rows);
  ix->n_cached = 0;
  if (!ids || count <= 0) return LV_OK;
  std::vector<int64_t> h(count);
  if (flags & LV_IO_DEVICE)
    LV_CHECK_CUDA(cudaMemcpy(h.data(), ids, count * 8, cudaMemcpyDeviceToHost));
  else
    std::memcpy(h.data(), ids, count * 8);
  std::vector<uint8_t> mask(ix->n, 0);
  std::vector<int32_t> slot(ix->n, -1);
  std::vector<int32_t> order;
  for (int64_t i = 0; i < count; ++i) {
    LV_REQUIRE(h[i] >= 0 && h[i] < ix->n, LV_ERR_USAGE, "cache id out of range");
    if (!mask[h[i]]) {
      mask[h[i]] = 1;
      slot[h[i]] = (int32_t)order.size();
      order.push_back((int32_t)h[i]);
    }
  }
  LV_TRY(upload_bits(&ix->cached_bits, mask.data(), ix->n, false));
  LV_TRY(dalloc(&ix->cache_slot, ix->n));
  LV_CHECK_CUDA(cudaMemcpy(ix->cache_slot, slot.data(), ix->n * 4, cudaMemcpyHostToDevice));
  ix->n_cached = (int64_t)order.size();
  if (ix->enc && ix->tokens) {
    LV_TRY(dalloc(&ix->cache_rows, (size_t)ix->n_cached * ix->dim));
    int32_t *d_ids = nullptr;
    LV_TRY(dalloc(&d_ids, order.size()));
    LV_CHECK_CUDA(cudaMemcpy(d_ids, order.data(), order.size() * 4, cudaMemcpyHostToDevice));
    int rc = encode_node_rows(ix->enc, ix->tokens, ix->token_bytes, ix->seq_len, d_ids,
                              (int64_t)order.size(), ix->cache_rows, 0);
    cudaStreamSynchronize(0);
    cudaFree(d_ids);
    LV_TRY(rc);
  }
  return LV_OK;
}

int lv_index_attach_encoder(lv_index *ix, lv_encoder *enc, const void *tokens, int32_t token_bytes,
                            int32_t seq_len, int flags) {
  LV_REQUIRE(ix, LV_ERR_USAGE, "null index");
  LV_REQUIRE(token_bytes == 2 || token_bytes == 4, LV_ERR_USAGE, "token_bytes must be 2 or 4");
  LV_REQUIRE(seq_len >= 1, LV_ERR_USAGE, "seq_len must be >= 1");
  DeviceGuard guard(ix->device);
  if (ix->own_tokens && ix->tokens) cudaFree(ix->tokens);
  ix->tokens = nullptr;
  ix->own_tokens = false;
  ix->enc = enc;
  ix->token_bytes = token_bytes;
  ix->seq_len = seq_len;
  if (!enc) return LV_OK;
  LV_REQUIRE(encoder_hidden(enc) == ix->dim, LV_ERR_USAGE, "encoder hidden size != index dim");
  if (flags & LV_IO_DEVICE) {
    ix->tokens = const_cast<void *>(tokens);
  } else {
    size_t bytes = (size_t)ix->n * seq_len * token_bytes;
    LV_CHECK_CUDA(cudaMalloc(&ix->tokens, bytes));
    ix->own_tokens = true;
    LV_CHECK_CUDA(cudaMemcpy(ix->tokens, tokens, bytes, cudaMemcpyHostToDevice));
  }
  return LV_OK;
}

int lv_index_set_fetch(lv_index *ix, lv_fetch_fn fn, void *user) {
  LV_REQUIRE(ix, LV_ERR_USAGE, "null index");
  ix->fetch = fn;
  ix->fetch_user = user;
  return LV_OK;
}

// Pinned vectors of the lv_index_set_cache ids, in the order those ids were
// given (the reference EmbeddingCache.vectors, search.py:113-128).
int lv_index_set_cache_rows(lv_index *ix, const float *rows, int flags) {
  LV_REQUIRE(ix && rows, LV_ERR_USAGE, "lv_index_set_cache_rows: null argument");
  LV_REQUIRE(ix->n_cached > 0, LV_ERR_USAGE, "lv_index_set_cache_rows: no cache ids set");
  DeviceGuard guard(ix->device);
  dfree(ix->cache_rows);
  LV_TRY(dalloc(&ix->cache_rows, (size_t)ix->n_cached * ix->dim));
  LV_CHECK_CUDA(cudaMemcpy(ix->cache_rows, rows, (size_t)ix->n_cached * ix->dim * 4,
                           (flags & LV_IO_DEVICE) ? cudaMemcpyDeviceToDevice
                                                  : cudaMemcpyHostToDevice));
  return LV_OK;
}

int lv_last_search_stats(const lv_index *ix, lv_search_stats *stats) {
  LV_REQUIRE(ix && stats, LV_ERR_USAGE, "null argument");
  *stats = ix->stats;
  return LV_OK;
}

}  // extern "C"

namespace {

// LV_TRACE_ITERS=1: one stderr line per recompute iteration (profiling aid)
bool trace_iters() {
  static const bool on = [] {
    const char *v = std::getenv("LV_TRACE_ITERS");
    return v && v[0] == '1';
  }();
  return on;
}

__global__ void gather_rows_kernel(const float *src, const int32_t *idx, int64_t n, int dim,
                                   float *dst);

// One pass of the batched search over B device-resident queries.
int search_pass(lv_index *ix, const float *d_q, const float *d_qn, int B, const lv_search_params &p,
                int aq_cap_override, int64_t *d_ids, float *d_dist, int32_t *d_count,
                int64_t *d_counters, int32_t *d_status, int32_t *d_visits, int32_t visits_cap,
                int32_t *d_blog, int32_t blog_cap, cudaStream_t s) {
  Workspace &ws = ix->ws;
  const bool two_level = p.mode == LV_MODE_TWO_LEVEL;
  const bool enc_src = p.source == LV_SOURCE_ENCODER || p.source == LV_SOURCE_CALLBACK;
  const bool callback = p.source == LV_SOURCE_CALLBACK;
  // LV_SMEM_LUT (matrix source, two-level): each warp stages its query's LUT in
  // shared memory with one bulk copy. Measured 3x slower than the default
  // per-lookup global reads at config-2 shape (profiles/r02_frontier_lut_ab.txt):
  // a 64 KiB table per warp leaves 3 warps per SM, and this latency-bound
  // traversal needs the ~16 warps per SM the small-footprint kernel keeps.
  const bool lut_smem = !enc_src && two_level && (p.flags & LV_SMEM_LUT) && ix->m > 0;
  int sms = 148;
  {
    int dev = 0;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  }
  int auto_slots = enc_src ? 4096 : sms * 16;
  if (lut_smem) {  // the warps whose LUTs fit on the SMs at once
    const size_t per = frontier_smem_per_warp_lut(ix->max_degree, 2 * ix->max_degree + 2, ix->m);
    const int wpb = (int)std::max<size_t>(1, std::min<size_t>(kWarpsPerBlock, (227 * 1024) / per));
    const int bps = (int)std::max<size_t>(1, (228 * 1024) / (per * wpb + 1024));
    auto_slots = sms * wpb * bps;
  }
  int slots = p.max_inflight > 0 ? p.max_inflight : auto_slots;
  slots = std::max(1, std::min(slots, B));
  const int req_cap = 2 * ix->max_degree + 2;
  int64_t aq_cap = aq_cap_override > 0 ? aq_cap_override
                                        : std::max<int64_t>(4096, (int64_t)p.ef * ix->max_degree * 2);
  aq_cap = std::min<int64_t>(aq_cap, ix->n);
  aq_cap = std::max<int64_t>(aq_cap, 1);
  const int xl_cap = 4096;
  const int64_t words = (ix->n + 31) / 32;
  LV_TRY(ws.st.ensure(slots));
  LV_TRY(ws.eq_d.ensure((size_t)slots * p.ef));
  LV_TRY(ws.eq_id.ensure((size_t)slots * p.ef));
  LV_TRY(ws.aq.ensure((size_t)slots * (two_level ? aq_cap : 1)));
  // visited sets (approx_known / exact_known): dense bitmaps cost 2 x slots x n/8
  // bytes (1 GB at config-2 with 4096 slots, 41 GB at 10M nodes with 16k);
  // above a 4 GiB budget (or with LV_HASH_VISITED) two-level searches use
  // bounded per-slot hash sets of 2 x aq_cap entries instead (the AQ bounds
  // approx_known; overflow re-runs use bitmaps with <= 64 slots)
  const double bitmap_bytes = 2.0 * slots * (double)words * 4;
  const bool hashed = two_level && aq_cap_override == 0 &&
                      ((p.flags & LV_HASH_VISITED) || bitmap_bytes > 4.0 * (1ull << 30));
  uint32_t vmask = 0;
  if (hashed) {
    uint64_t cap = 1;
    while (cap < (uint64_t)(2 * aq_cap + 4096)) cap <<= 1;
    vmask = (uint32_t)(cap - 1);
    const size_t need = (size_t)slots * cap;
    const bool fresh = ws.aset.cap < need;
    LV_TRY(ws.aset.ensure(need));
    LV_TRY(ws.xset.ensure(need));
    if (fresh || ws.bits_dirty) {  // finish_query resets a finished slot's tables
      LV_CHECK_CUDA(cudaMemsetAsync(ws.aset.ptr, 0xff, ws.aset.cap * 4, s));
      LV_CHECK_CUDA(cudaMemsetAsync(ws.xset.ptr, 0xff, ws.xset.cap * 4, s));
    }
  } else {
    bool fresh_bits = ws.abits.cap < (size_t)slots * words;
    LV_TRY(ws.abits.ensure((size_t)slots * words));
    LV_TRY(ws.xbits.ensure((size_t)slots * words));
    if (fresh_bits || ws.bits_dirty) {  // kept all-zero between queries by finish_query
      LV_CHECK_CUDA(cudaMemsetAsync(ws.abits.ptr, 0, ws.abits.cap * 4, s));
      LV_CHECK_CUDA(cudaMemsetAsync(ws.xbits.ptr, 0, ws.xbits.cap * 4, s));
    }
  }
  ws.bits_dirty = true;  // cleared below once every query has finished
  LV_TRY(ws.xlist.ensure((size_t)slots * xl_cap));
  LV_TRY(ws.req.ensure((size_t)slots * req_cap));
  LV_TRY(ws.counters.ensure(4));
  LV_TRY(ws.bytes.ensure(1));
  LV_CHECK_CUDA(cudaMemsetAsync(ws.bytes.ptr, 0, 8, s));
  const int greq_cap = enc_src ? slots * req_cap : 0;
  const bool shared = enc_src && !(p.flags & LV_NO_SHARED_RECOMPUTE);
  int64_t tab_rows = greq_cap;
  uint32_t hmask = 0;
  if (enc_src) {
    LV_TRY(ws.greq.ensure(greq_cap));
    if (shared) {
      // step-wide table of recomputed rows (each distinct node is encoded once
      // per call while the table has room; a full table is reset). Sized to
      // hold every node when HBM allows — at 10M nodes and 16k queries in
      // flight an 8 GiB table reset every few iterations and lost most of the
      // sharing — keeping 12 GiB + 30% of the free memory for the encoder.
      const int64_t row_bytes = (int64_t)ix->dim * 4;
      size_t free_b = 0, total_b = 0;
      cudaMemGetInfo(&free_b, &total_b);
      const int64_t spare = std::max<int64_t>(0, ((int64_t)free_b - ((int64_t)12 << 30)) * 7 / 10);
      const int64_t budget = std::max<int64_t>(((int64_t)8 << 30), spare) / row_bytes;
      tab_rows = std::max<int64_t>(greq_cap, std::min<int64_t>(budget, ix->n));
      uint64_t hs = 1;
      while (hs < (uint64_t)(2 * tab_rows)) hs <<= 1;
      hmask = (uint32_t)(hs - 1);
      LV_TRY(ws.hkeys.ensure(hs));
      LV_TRY(ws.hvals.ensure(hs));
      LV_TRY(ws.new_ids.ensure(greq_cap));
      LV_TRY(ws.emb_map.ensure(greq_cap));
      LV_TRY(ws.row_count.ensure(1));
    }
    LV_TRY(ws.emb.ensure((size_t)tab_rows * ix->dim));
  }
  if (two_level) {
    LV_TRY(ws.luts.ensure((size_t)B * ix->m * kCentroids));
    LV_CHECK_CUDA(launch_lut(d_q, d_qn, B, ix->dim, ix->metric, ix->codebooks, ix->m, ix->padded,
                             ws.luts.ptr, s));
  }
  if (!ws.h_counters) LV_CHECK_CUDA(cudaMallocHost(&ws.h_counters, 32));
  LV_CHECK_CUDA(launch_slot_reset(ws.st.ptr, slots, s));
  LV_CHECK_CUDA(cudaMemsetAsync(ws.counters.ptr, 0, 16, s));

  SearchCtx c{};
  c.n = ix->n;
  c.dim = ix->dim;
  c.metric = ix->metric;
  c.max_degree = ix->max_degree;
  c.level_count = ix->level_count;
  c.entry = (int32_t)ix->entry;
  for (int l = 0; l < ix->level_count; ++l) {
    c.offs[l] = ix->offs[l];
    c.nbrs[l] = ix->nbrs[l];
  }
  c.deleted_bits = ix->deleted_bits;
  c.cached_bits = p.use_cache ? ix->cached_bits : nullptr;
  c.cache_slot = ix->cache_slot;
  c.cache_rows = ix->cache_rows;
  c.m = ix->m;
  c.codes = ix->codes;
  c.luts = ws.luts.ptr;
  c.source = enc_src ? LV_SOURCE_ENCODER : p.source;  // the kernels see callback = encoder
  c.matrix = ix->matrix;
  c.emb_buf = ws.emb.ptr;
  c.emb_map = shared ? ws.emb_map.ptr : nullptr;
  c.B = B;
  c.q = d_q;
  c.qn = d_qn;
  c.k = p.k;
  c.ef = p.ef;
  c.mode = p.mode;
  c.alpha = p.rerank_percent / 100.0;
  c.slots = slots;
  c.aq_cap = (int32_t)aq_cap;
  c.req_cap = req_cap;
  c.xl_cap = xl_cap;
  c.words = words;
  c.st = ws.st.ptr;
  c.eq_d = ws.eq_d.ptr;
  c.eq_id = ws.eq_id.ptr;
  c.aq = ws.aq.ptr;
  c.abits = hashed ? nullptr : ws.abits.ptr;
  c.xbits = hashed ? nullptr : ws.xbits.ptr;
  c.aset = hashed ? ws.aset.ptr : nullptr;
  c.xset = hashed ? ws.xset.ptr : nullptr;
  c.vmask = vmask;
  c.xlist = ws.xlist.ptr;
  c.req = ws.req.ptr;
  c.greq = ws.greq.ptr;
  c.greq_total = ws.counters.ptr + 0;
  c.greq_cap = greq_cap;
  c.queue_head = ws.counters.ptr + 1;
  c.done_count = ws.counters.ptr + 2;
  c.bytes_total = ws.bytes.ptr;
  c.out_ids = d_ids;
  c.out_dist = d_dist;
  c.out_count = d_count;
  c.out_counters = d_counters;
  c.out_status = d_status;
  c.visits = d_visits;
  c.visits_cap = visits_cap;
  c.blog = d_blog;
  c.blog_cap = blog_cap;
  c.lut_smem = lut_smem ? 1 : 0;
  c.warps_per_block = kWarpsPerBlock;

  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  float frontier_ms = 0.f, encoder_ms = 0.f;
  int64_t iterations = 0, physical = 0;
  if (!enc_src) {
    cudaEventRecord(e0, s);
    LV_CHECK_CUDA(launch_frontier(c, s));
    cudaEventRecord(e1, s);
    LV_CHECK_CUDA(cudaEventSynchronize(e1));
    cudaEventElapsedTime(&frontier_ms, e0, e1);
    iterations = 1;
  } else {
    const bool dry = (p.flags & LV_DRY_RECOMPUTE) != 0;
    LV_REQUIRE(dry ? ix->matrix != nullptr
                   : (callback ? ix->fetch != nullptr : (ix->enc && ix->tokens)), LV_ERR_USAGE,
               dry ? "LV_DRY_RECOMPUTE requires lv_index_set_matrix"
                   : (callback ? "callback source requires lv_index_set_fetch"
                               : "encoder source requires lv_index_attach_encoder"));
    std::vector<int32_t> h_ids;
    std::vector<int64_t> h_ids64;
    std::vector<float> h_rows;
    int32_t row_base = 0;
    auto reset_table = [&]() -> int {
      LV_CHECK_CUDA(cudaMemsetAsync(ws.hkeys.ptr, 0xff, ((size_t)hmask + 1) * 4, s));
      LV_CHECK_CUDA(cudaMemsetAsync(ws.hvals.ptr, 0xff, ((size_t)hmask + 1) * 4, s));
      LV_CHECK_CUDA(cudaMemsetAsync(ws.row_count.ptr, 0, 4, s));
      row_base = 0;
      return LV_OK;
    };
    if (shared) LV_TRY(reset_table());
    while (true) {
      LV_CHECK_CUDA(cudaMemsetAsync(ws.counters.ptr, 0, 4, s));  // greq_total
      cudaEventRecord(e0, s);
      LV_CHECK_CUDA(launch_frontier(c, s));
      cudaEventRecord(e1, s);
      LV_CHECK_CUDA(cudaMemcpyAsync(ws.h_counters, ws.counters.ptr, 12, cudaMemcpyDeviceToHost, s));
      LV_CHECK_CUDA(cudaStreamSynchronize(s));
      float ms = 0.f;
      cudaEventElapsedTime(&ms, e0, e1);
      frontier_ms += ms;
      ++iterations;
      const int total = ws.h_counters[0];
      if (total > 0) {
        const int32_t *enc_ids = ws.greq.ptr;
        int32_t n_new = total;
        float *enc_out = ws.emb.ptr;
        if (shared) {
          // one encode per distinct node of the step; repeats reuse its row
          if ((int64_t)row_base + total > tab_rows) LV_TRY(reset_table());
          LV_CHECK_CUDA(launch_dedup(ws.greq.ptr, total, ws.hkeys.ptr, ws.hvals.ptr, hmask,
                                     ws.row_count.ptr, row_base, ws.new_ids.ptr, ws.emb_map.ptr,
                                     s));
          LV_CHECK_CUDA(cudaMemcpyAsync(ws.h_counters + 3, ws.row_count.ptr, 4,
                                        cudaMemcpyDeviceToHost, s));
          LV_CHECK_CUDA(cudaStreamSynchronize(s));
          n_new = ws.h_counters[3] - row_base;
          enc_ids = ws.new_ids.ptr;
          enc_out = ws.emb.ptr + (size_t)row_base * ix->dim;
          row_base = ws.h_counters[3];
        }
        cudaEventRecord(e0, s);
        if (n_new > 0 && dry) {
          gather_rows_kernel<<<(unsigned)(((int64_t)n_new * ix->dim + 255) / 256), 256, 0, s>>>(
              ix->matrix, enc_ids, n_new, ix->dim, enc_out);
          note_launch();
          LV_CHECK_CUDA(cudaGetLastError());
        } else if (n_new > 0 && callback) {
          // host provider: ProviderSource.fetch(ids) (search.py:103-110) on the
          // new ids, rows back into the step table
          h_ids.resize(n_new);
          h_ids64.resize(n_new);
          h_rows.resize((size_t)n_new * ix->dim);
          LV_CHECK_CUDA(cudaMemcpyAsync(h_ids.data(), enc_ids, (size_t)n_new * 4,
                                        cudaMemcpyDeviceToHost, s));
          LV_CHECK_CUDA(cudaStreamSynchronize(s));
          for (int32_t i = 0; i < n_new; ++i) h_ids64[i] = h_ids[i];
          const int frc = ix->fetch(ix->fetch_user, h_ids64.data(), n_new, h_rows.data());
          LV_REQUIRE(frc == 0, LV_ERR_PROVIDER, "provider fetch failed");
          LV_CHECK_CUDA(cudaMemcpyAsync(enc_out, h_rows.data(), h_rows.size() * 4,
                                        cudaMemcpyHostToDevice, s));
        } else if (n_new > 0) {
          LV_TRY(encode_node_rows(ix->enc, ix->tokens, ix->token_bytes, ix->seq_len, enc_ids,
                                  n_new, enc_out, s));
        }
        cudaEventRecord(e1, s);
        LV_CHECK_CUDA(cudaEventSynchronize(e1));
        cudaEventElapsedTime(&ms, e0, e1);
        encoder_ms += ms;
        physical += n_new;
        if (trace_iters())
          std::fprintf(stderr, "[lv] iter %lld requests %d encoded %d encoder_ms %.3f\n",
                       (long long)iterations, total, n_new, ms);
      } else if (ws.h_counters[2] >= B) {
        break;
      }
      LV_REQUIRE(iterations < (int64_t)1 << 40, LV_ERR_INTERNAL, "search loop did not terminate");
    }
  }
  cudaEventDestroy(e0);
  cudaEventDestroy(e1);
  ws.bits_dirty = false;  // every query finished: finish_query cleared its bits
  unsigned long long bytes = 0;
  LV_CHECK_CUDA(cudaMemcpyAsync(&bytes, ws.bytes.ptr, 8, cudaMemcpyDeviceToHost, s));
  LV_CHECK_CUDA(cudaStreamSynchronize(s));
  ix->stats.adc_bytes += (int64_t)bytes;
  ix->stats.iterations += iterations;
  ix->stats.physical_encodes += physical;
  ix->stats.frontier_ms += frontier_ms;
  ix->stats.encoder_ms += encoder_ms;
  return LV_OK;
}

__global__ void gather_rows_kernel(const float *src, const int32_t *idx, int64_t n, int dim,
                                   float *dst) {
  int64_t t = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (t >= n * dim) return;
  int64_t r = t / dim;
  dst[t] = src[(int64_t)idx[r] * dim + (t % dim)];
}

}  // namespace

extern "C" int lv_search_batch(lv_index *ix, const float *q, const float *qnorm, int32_t B,
                               const lv_search_params *p, const lv_search_outputs *out,
                               void *stream) {
  LV_REQUIRE(ix && p && out, LV_ERR_USAGE, "lv_search_batch: null argument");
  // SearchParams.__post_init__ (search.py:45-54)
  LV_REQUIRE(p->k >= 1 && p->ef >= p->k, LV_ERR_USAGE, "need ef >= k >= 1");
  LV_REQUIRE(p->rerank_percent > 0 && p->rerank_percent <= 100, LV_ERR_USAGE,
             "rerank_percent must be in (0, 100]");
  LV_REQUIRE(p->batch_size >= 1, LV_ERR_USAGE, "batch_size must be >= 1");
  LV_REQUIRE(p->mode == LV_MODE_TWO_LEVEL || p->mode == LV_MODE_EXACT_BESTFIRST, LV_ERR_USAGE,
             "unknown mode");
  LV_REQUIRE(p->mode != LV_MODE_TWO_LEVEL || ix->m > 0, LV_ERR_USAGE,
             "two_level mode requires PQ artifacts");
  LV_REQUIRE(p->source == LV_SOURCE_MATRIX || p->source == LV_SOURCE_ENCODER ||
                 p->source == LV_SOURCE_CALLBACK,
             LV_ERR_USAGE, "unknown source");
  LV_REQUIRE(p->source != LV_SOURCE_MATRIX || ix->matrix, LV_ERR_USAGE,
             "matrix source requires lv_index_set_matrix");
  LV_REQUIRE(!p->use_cache || ix->cached_bits, LV_ERR_USAGE, "cache requested but not built");
  LV_REQUIRE(p->source == LV_SOURCE_MATRIX || !p->use_cache || ix->cache_rows, LV_ERR_USAGE,
             "recompute-source cache needs cached vectors (attach the encoder before the cache, "
             "or lv_index_set_cache_rows)");
  LV_REQUIRE(p->ef <= (1 << 24), LV_ERR_USAGE, "ef too large");
  LV_REQUIRE(B >= 0, LV_ERR_USAGE, "B must be >= 0");
  LV_REQUIRE(out->ids && out->dist && out->count && out->counters, LV_ERR_USAGE,
             "lv_search_batch: missing output buffer");
  if (B == 0) return LV_OK;
  LV_REQUIRE(q, LV_ERR_USAGE, "null queries");
  DeviceGuard guard(ix->device);
  cudaStream_t s = (cudaStream_t)stream;
  Workspace &ws = ix->ws;
  const bool dev_io = p->flags & LV_IO_DEVICE;
  const int k = p->k;
  ix->stats = lv_search_stats{};
  cudaEvent_t t0, t1;
  cudaEventCreate(&t0);
  cudaEventCreate(&t1);
  cudaEventRecord(t0, s);

  const float *d_q = q, *d_qn = qnorm;
  if (!dev_io) {
    LV_TRY(ws.q.ensure((size_t)B * ix->dim));
    LV_TRY(upload(ws.q.ptr, q, (size_t)B * ix->dim * 4, false, s));
    d_q = ws.q.ptr;
  }
  if (!qnorm) {
    // qn on the device (sequential fp32 sum of squares). Bit parity with the
    // reference needs the host value np.float32(np.sqrt(np.dot(q, q)))
    // (vectors.py:138, BLAS sdot order), so parity callers pass qnorm.
    LV_TRY(ws.qn.ensure(B));
    LV_CHECK_CUDA(launch_qnorm(d_q, B, ix->dim, ws.qn.ptr, s));
    d_qn = ws.qn.ptr;
  } else if (!dev_io) {
    LV_TRY(ws.qn.ensure(B));
    LV_TRY(upload(ws.qn.ptr, qnorm, (size_t)B * 4, false, s));
    d_qn = ws.qn.ptr;
  }
  if (ix->metric == LV_METRIC_COSINE && p->mode == LV_MODE_TWO_LEVEL) {
    // adc_build raises for a zero query under cosine (pq.py:163-166)
    LV_TRY(ws.counters.ensure(4));
    LV_CHECK_CUDA(cudaMemsetAsync(ws.counters.ptr + 3, 0, 4, s));
    LV_CHECK_CUDA(launch_count_zero(d_qn, B, ws.counters.ptr + 3, s));
    int32_t zeros = 0;
    LV_CHECK_CUDA(cudaMemcpyAsync(&zeros, ws.counters.ptr + 3, 4, cudaMemcpyDeviceToHost, s));
    LV_CHECK_CUDA(cudaStreamSynchronize(s));
    LV_REQUIRE(zeros == 0, LV_ERR_USAGE, "cosine ADC undefined for zero query");
  }
  int64_t *d_ids = out->ids;
  float *d_dist = out->dist;
  int32_t *d_count = out->count;
  int64_t *d_counters = out->counters;
  int32_t *d_status = out->status;
  int32_t *d_visits = out->visits;
  int32_t *d_blog = out->batch_log;
  if (!dev_io) {
    LV_TRY(ws.out_ids.ensure((size_t)B * k));
    LV_TRY(ws.out_dist.ensure((size_t)B * k));
    LV_TRY(ws.out_count.ensure(B));
    LV_TRY(ws.out_counters.ensure((size_t)B * 4));
    LV_TRY(ws.out_status.ensure(B));
    d_ids = ws.out_ids.ptr;
    d_dist = ws.out_dist.ptr;
    d_count = ws.out_count.ptr;
    d_counters = ws.out_counters.ptr;
    d_status = ws.out_status.ptr;
    d_visits = nullptr;
    d_blog = nullptr;
    if (out->visits && out->visits_cap > 0) {
      LV_TRY(ws.visits.ensure((size_t)B * out->visits_cap));
      d_visits = ws.visits.ptr;
    }
    if (out->batch_log && out->batch_log_cap > 0) {
      LV_TRY(ws.blog.ensure((size_t)B * out->batch_log_cap));
      d_blog = ws.blog.ptr;
    }
  } else if (!d_status) {
    LV_TRY(ws.out_status.ensure(B));
    d_status = ws.out_status.ptr;
  }
  if (d_visits) LV_CHECK_CUDA(cudaMemsetAsync(d_visits, 0xff, (size_t)B * out->visits_cap * 4, s));
  if (d_blog) LV_CHECK_CUDA(cudaMemsetAsync(d_blog, 0xff, (size_t)B * out->batch_log_cap * 4, s));

  LV_TRY(search_pass(ix, d_q, d_qn, B, *p, 0, d_ids, d_dist, d_count, d_counters, d_status,
                     d_visits, out->visits_cap, d_blog, out->batch_log_cap, s));

  // queries whose approximate queue overflowed are re-run with capacity n
  std::vector<int32_t> status(B);
  LV_CHECK_CUDA(cudaMemcpyAsync(status.data(), d_status, (size_t)B * 4, cudaMemcpyDeviceToHost, s));
  LV_CHECK_CUDA(cudaStreamSynchronize(s));
  std::vector<int32_t> redo;
  for (int b = 0; b < B; ++b) {
    if (status[b] == LV_Q_AQ_OVERFLOW) redo.push_back(b);
    else if (status[b] != LV_Q_OK) {
      set_error("query " + std::to_string(b) + " failed inside the search kernel");
      return LV_ERR_INTERNAL;
    }
  }
  if (!redo.empty()) {
    const int R = (int)redo.size();
    DBuf<float> rq, rqn, rdist;
    DBuf<int64_t> rids, rcnt;
    DBuf<int32_t> rcount, rstatus, ridx, rvis, rblog;
    LV_TRY(rq.ensure((size_t)R * ix->dim));
    LV_TRY(rqn.ensure(R));
    LV_TRY(rids.ensure((size_t)R * k));
    LV_TRY(rdist.ensure((size_t)R * k));
    LV_TRY(rcount.ensure(R));
    LV_TRY(rcnt.ensure((size_t)R * 4));
    LV_TRY(rstatus.ensure(R));
    LV_TRY(ridx.ensure(R));
    LV_CHECK_CUDA(cudaMemcpyAsync(ridx.ptr, redo.data(), R * 4, cudaMemcpyHostToDevice, s));
    gather_rows_kernel<<<(unsigned)(((int64_t)R * ix->dim + 255) / 256), 256, 0, s>>>(
        d_q, ridx.ptr, R, ix->dim, rq.ptr);
        note_launch();
    gather_rows_kernel<<<(R + 255) / 256, 256, 0, s>>>(d_qn, ridx.ptr, R, 1, rqn.ptr);
    note_launch();
    int32_t *pv = nullptr, *pb = nullptr;
    if (d_visits) {
      LV_TRY(rvis.ensure((size_t)R * out->visits_cap));
      LV_CHECK_CUDA(cudaMemsetAsync(rvis.ptr, 0xff, (size_t)R * out->visits_cap * 4, s));
      pv = rvis.ptr;
    }
    if (d_blog) {
      LV_TRY(rblog.ensure((size_t)R * out->batch_log_cap));
      LV_CHECK_CUDA(cudaMemsetAsync(rblog.ptr, 0xff, (size_t)R * out->batch_log_cap * 4, s));
      pb = rblog.ptr;
    }
    lv_search_params rp = *p;
    rp.max_inflight = std::min(R, 64);
    LV_TRY(search_pass(ix, rq.ptr, rqn.ptr, R, rp, (int)std::min<int64_t>(ix->n, INT32_MAX),
                       rids.ptr, rdist.ptr, rcount.ptr, rcnt.ptr, rstatus.ptr, pv, out->visits_cap,
                       pb, out->batch_log_cap, s));
    for (int i = 0; i < R; ++i) {
      int b = redo[i];
      LV_CHECK_CUDA(cudaMemcpyAsync(d_ids + (size_t)b * k, rids.ptr + (size_t)i * k, k * 8,
                                    cudaMemcpyDeviceToDevice, s));
      LV_CHECK_CUDA(cudaMemcpyAsync(d_dist + (size_t)b * k, rdist.ptr + (size_t)i * k, k * 4,
                                    cudaMemcpyDeviceToDevice, s));
      LV_CHECK_CUDA(cudaMemcpyAsync(d_count + b, rcount.ptr + i, 4, cudaMemcpyDeviceToDevice, s));
      LV_CHECK_CUDA(cudaMemcpyAsync(d_counters + (size_t)b * 4, rcnt.ptr + (size_t)i * 4, 32,
                                    cudaMemcpyDeviceToDevice, s));
      LV_CHECK_CUDA(cudaMemcpyAsync(d_status + b, rstatus.ptr + i, 4, cudaMemcpyDeviceToDevice, s));
      if (pv)
        LV_CHECK_CUDA(cudaMemcpyAsync(d_visits + (size_t)b * out->visits_cap,
                                      pv + (size_t)i * out->visits_cap, out->visits_cap * 4,
                                      cudaMemcpyDeviceToDevice, s));
      if (pb)
        LV_CHECK_CUDA(cudaMemcpyAsync(d_blog + (size_t)b * out->batch_log_cap,
                                      pb + (size_t)i * out->batch_log_cap, out->batch_log_cap * 4,
                                      cudaMemcpyDeviceToDevice, s));
    }
    LV_CHECK_CUDA(cudaStreamSynchronize(s));
  }

  if (!dev_io) {
    LV_CHECK_CUDA(cudaMemcpyAsync(out->ids, d_ids, (size_t)B * k * 8, cudaMemcpyDeviceToHost, s));
    LV_CHECK_CUDA(cudaMemcpyAsync(out->dist, d_dist, (size_t)B * k * 4, cudaMemcpyDeviceToHost, s));
    LV_CHECK_CUDA(cudaMemcpyAsync(out->count, d_count, (size_t)B * 4, cudaMemcpyDeviceToHost, s));
    LV_CHECK_CUDA(cudaMemcpyAsync(out->counters, d_counters, (size_t)B * 32, cudaMemcpyDeviceToHost, s));
    if (out->status)
      LV_CHECK_CUDA(cudaMemcpyAsync(out->status, d_status, (size_t)B * 4, cudaMemcpyDeviceToHost, s));
    if (d_visits)
      LV_CHECK_CUDA(cudaMemcpyAsync(out->visits, d_visits, (size_t)B * out->visits_cap * 4,
                                    cudaMemcpyDeviceToHost, s));
    if (d_blog)
      LV_CHECK_CUDA(cudaMemcpyAsync(out->batch_log, d_blog, (size_t)B * out->batch_log_cap * 4,
                                    cudaMemcpyDeviceToHost, s));
  }
  cudaEventRecord(t1, s);
  LV_CHECK_CUDA(cudaStreamSynchronize(s));
  float total_ms = 0.f;
  cudaEventElapsedTime(&total_ms, t0, t1);
  cudaEventDestroy(t0);
  cudaEventDestroy(t1);
  ix->stats.total_ms = total_ms;
  return LV_OK;
}

extern "C" int lv_adc_tables(lv_index *ix, const float *q, const float *qnorm, int32_t B,
                             float *tables, int flags, void *stream) {
  LV_REQUIRE(ix && q && qnorm && tables, LV_ERR_USAGE, "lv_adc_tables: null argument");
  LV_REQUIRE(ix->m > 0, LV_ERR_USAGE, "index has no PQ artifacts");
  if (B <= 0) return LV_OK;
  DeviceGuard guard(ix->device);
  cudaStream_t s = (cudaStream_t)stream;
  const size_t tsz = (size_t)B * ix->m * kCentroids;
  if (flags & LV_IO_DEVICE) {
    LV_CHECK_CUDA(launch_lut(q, qnorm, B, ix->dim, ix->metric, ix->codebooks, ix->m, ix->padded,
                             tables, s));
    return LV_OK;
  }
  DBuf<float> dq, dqn, dt;
  LV_TRY(dq.ensure((size_t)B * ix->dim));
  LV_TRY(dqn.ensure(B));
  LV_TRY(dt.ensure(tsz));
  LV_TRY(upload(dq.ptr, q, (size_t)B * ix->dim * 4, false, s));
  LV_TRY(upload(dqn.ptr, qnorm, (size_t)B * 4, false, s));
  LV_CHECK_CUDA(launch_lut(dq.ptr, dqn.ptr, B, ix->dim, ix->metric, ix->codebooks, ix->m,
                           ix->padded, dt.ptr, s));
  LV_CHECK_CUDA(cudaMemcpyAsync(tables, dt.ptr, tsz * 4, cudaMemcpyDeviceToHost, s));
  LV_CHECK_CUDA(cudaStreamSynchronize(s));
  return LV_OK;
}

extern "C" int lv_adc_score(lv_index *ix, const float *table, const int64_t *ids, int64_t count,
                            float *out, int flags, void *stream) {
  LV_REQUIRE(ix && table && ids && out, LV_ERR_USAGE, "lv_adc_score: null argument");
  LV_REQUIRE(ix->m > 0, LV_ERR_USAGE, "index has no PQ artifacts");
  if (count <= 0) return LV_OK;
  DeviceGuard guard(ix->device);
  cudaStream_t s = (cudaStream_t)stream;
  if (flags & LV_IO_DEVICE) {
    LV_CHECK_CUDA(launch_adc_score(table, ix->m, ix->codes, ids, count, out, s));
    return LV_OK;
  }
  for (int64_t i = 0; i < count; ++i)
    LV_REQUIRE(ids[i] >= 0 && ids[i] < ix->n, LV_ERR_USAGE, "node id out of range");
  DBuf<float> dt, dout;
  DBuf<int64_t> dids;
  LV_TRY(dt.ensure((size_t)ix->m * kCentroids));
  LV_TRY(dids.ensure(count));
  LV_TRY(dout.ensure(count));
  LV_TRY(upload(dt.ptr, table, (size_t)ix->m * kCentroids * 4, false, s));
  LV_TRY(upload(dids.ptr, ids, count * 8, false, s));
  LV_CHECK_CUDA(launch_adc_score(dt.ptr, ix->m, ix->codes, dids.ptr, count, dout.ptr, s));
  LV_CHECK_CUDA(cudaMemcpyAsync(out, dout.ptr, count * 4, cudaMemcpyDeviceToHost, s));
  LV_CHECK_CUDA(cudaStreamSynchronize(s));
  return LV_OK;
}

extern "C" int lv_distance_many(int32_t metric, const float *rows, int64_t nrows, int32_t dim,
                                const float *q, float qnorm, float *out, int flags, void *stream) {
  LV_REQUIRE(rows && q && out, LV_ERR_USAGE, "lv_distance_many: null argument");
  LV_REQUIRE(metric >= 0 && metric <= 2, LV_ERR_USAGE, "unknown metric");
  LV_REQUIRE(dim >= 1, LV_ERR_USAGE, "dim must be >= 1");
  if (nrows <= 0) return LV_OK;
  cudaStream_t s = (cudaStream_t)stream;
  if (flags & LV_IO_DEVICE) {
    LV_CHECK_CUDA(launch_distance_many(metric, rows, nrows, dim, q, qnorm, out, s));
    return LV_OK;
  }
  DBuf<float> dr, dq, dout;
  LV_TRY(dr.ensure((size_t)nrows * dim));
  LV_TRY(dq.ensure(dim));
  LV_TRY(dout.ensure(nrows));
  LV_TRY(upload(dr.ptr, rows, (size_t)nrows * dim * 4, false, s));
  LV_TRY(upload(dq.ptr, q, (size_t)dim * 4, false, s));
  LV_CHECK_CUDA(launch_distance_many(metric, dr.ptr, nrows, dim, dq.ptr, qnorm, dout.ptr, s));
  LV_CHECK_CUDA(cudaMemcpyAsync(out, dout.ptr, nrows * 4, cudaMemcpyDeviceToHost, s));
  LV_CHECK_CUDA(cudaStreamSynchronize(s));
  return LV_OK;
}

// Engine.search's pending-buffer merge (index.py:320-327 over buffer_scan,
// update.py:483-488): see include/leann_b200.h.
extern "C" int lv_merge_pending(int32_t metric, const float *pending, const int64_t *pending_ids,
                                int64_t n_pending, int32_t dim, const float *q,
                                const float *qnorm, int32_t B, int32_t k, int64_t *ids,
                                float *dist, int32_t *count, int flags, void *stream) {
  LV_REQUIRE(ids && dist && count, LV_ERR_USAGE, "lv_merge_pending: null output");
  LV_REQUIRE(metric >= 0 && metric <= 2, LV_ERR_USAGE, "unknown metric");
  LV_REQUIRE(dim >= 1 && k >= 1 && B >= 0 && n_pending >= 0, LV_ERR_USAGE,
             "lv_merge_pending: bad sizes");
  if (B == 0 || n_pending == 0) return LV_OK;
  LV_REQUIRE(pending && pending_ids && q, LV_ERR_USAGE, "lv_merge_pending: null input");
  cudaStream_t s = (cudaStream_t)stream;
  const bool dev = flags & LV_IO_DEVICE;
  DBuf<float> dp, dq, dqn, dd, scratch;
  DBuf<int64_t> dpi, di;
  DBuf<int32_t> dc, bad;
  const float *p_pend = pending, *p_q = q, *p_qn = qnorm;
  const int64_t *p_pid = pending_ids;
  int64_t *p_ids = ids;
  float *p_dist = dist;
  int32_t *p_count = count;
  if (!dev) {
    LV_TRY(dp.ensure((size_t)n_pending * dim));
    LV_TRY(dpi.ensure(n_pending));
    LV_TRY(dq.ensure((size_t)B * dim));
    LV_TRY(di.ensure((size_t)B * k));
    LV_TRY(dd.ensure((size_t)B * k));
    LV_TRY(dc.ensure(B));
    LV_TRY(upload(dp.ptr, pending, (size_t)n_pending * dim * 4, false, s));
    LV_TRY(upload(dpi.ptr, pending_ids, (size_t)n_pending * 8, false, s));
    LV_TRY(upload(dq.ptr, q, (size_t)B * dim * 4, false, s));
    LV_TRY(upload(di.ptr, ids, (size_t)B * k * 8, false, s));
    LV_TRY(upload(dd.ptr, dist, (size_t)B * k * 4, false, s));
    LV_TRY(upload(dc.ptr, count, (size_t)B * 4, false, s));
    p_pend = dp.ptr;
    p_pid = dpi.ptr;
    p_q = dq.ptr;
    p_ids = di.ptr;
    p_dist = dd.ptr;
    p_count = dc.ptr;
    if (qnorm) {
      LV_TRY(dqn.ensure(B));
      LV_TRY(upload(dqn.ptr, qnorm, (size_t)B * 4, false, s));
      p_qn = dqn.ptr;
    }
  }
  if (!p_qn) {
    LV_TRY(dqn.ensure(B));
    LV_CHECK_CUDA(launch_qnorm(p_q, B, dim, dqn.ptr, s));
    p_qn = dqn.ptr;
  }
  LV_TRY(scratch.ensure((size_t)B * n_pending));
  LV_TRY(bad.ensure(1));
  LV_CHECK_CUDA(cudaMemsetAsync(bad.ptr, 0, 4, s));
  LV_CHECK_CUDA(launch_pending_merge(metric, p_pend, p_pid, n_pending, dim, p_q, p_qn, B, k, p_ids,
                                     p_dist, p_count, scratch.ptr, bad.ptr, s));
  int32_t h_bad = 0;
  LV_CHECK_CUDA(cudaMemcpyAsync(&h_bad, bad.ptr, 4, cudaMemcpyDeviceToHost, s));
  if (!dev) {
    LV_CHECK_CUDA(cudaMemcpyAsync(ids, p_ids, (size_t)B * k * 8, cudaMemcpyDeviceToHost, s));
    LV_CHECK_CUDA(cudaMemcpyAsync(dist, p_dist, (size_t)B * k * 4, cudaMemcpyDeviceToHost, s));
    LV_CHECK_CUDA(cudaMemcpyAsync(count, p_count, (size_t)B * 4, cudaMemcpyDeviceToHost, s));
  }
  LV_CHECK_CUDA(cudaStreamSynchronize(s));
  LV_REQUIRE(!h_bad, LV_ERR_USAGE, "cosine distance undefined for zero vector");
  return LV_OK;
}

// qn = np.float32(np.sqrt(np.dot(q, q))) per row in the OpenBLAS sdot order
// (vectors.py:138, pq.py:163) — what lv_search_batch uses when qnorm is NULL.
extern "C" int lv_query_norms(const float *q, int32_t B, int32_t dim, float *out, int flags,
                              void *stream) {
  LV_REQUIRE(q && out, LV_ERR_USAGE, "lv_query_norms: null argument");
  LV_REQUIRE(dim >= 1 && B >= 0, LV_ERR_USAGE, "lv_query_norms: bad sizes");
  if (B == 0) return LV_OK;
  cudaStream_t s = (cudaStream_t)stream;
  if (flags & LV_IO_DEVICE) {
    LV_CHECK_CUDA(launch_qnorm(q, B, dim, out, s));
    return LV_OK;
  }
  DBuf<float> dq, dn;
  LV_TRY(dq.ensure((size_t)B * dim));
  LV_TRY(dn.ensure(B));
  LV_TRY(upload(dq.ptr, q, (size_t)B * dim * 4, false, s));
  LV_CHECK_CUDA(launch_qnorm(dq.ptr, B, dim, dn.ptr, s));
  LV_CHECK_CUDA(cudaMemcpyAsync(out, dn.ptr, (size_t)B * 4, cudaMemcpyDeviceToHost, s));
  LV_CHECK_CUDA(cudaStreamSynchronize(s));
  return LV_OK;
}

// distance_many (vectors.py:120-140) of each query against a gathered list of
// rows: out[b][c] = d(q_b, matrix[ids[b][c]]) in the reference's einsum order
// (ids < 0 -> +inf). Device pointers only; qnorm NULL -> lv_query_norms order.
extern "C" int lv_distance_gather(int32_t metric, const float *matrix, int32_t dim,
                                  const int64_t *ids, int32_t B, int32_t C, const float *q,
                                  const float *qnorm, float *out, void *stream) {
  LV_REQUIRE(matrix && ids && q && out, LV_ERR_USAGE, "lv_distance_gather: null argument");
  LV_REQUIRE(metric >= 0 && metric <= 2 && dim >= 1 && B >= 0 && C >= 0, LV_ERR_USAGE,
             "lv_distance_gather: bad arguments");
  if (B == 0 || C == 0) return LV_OK;
  cudaStream_t s = (cudaStream_t)stream;
  DBuf<float> dqn;
  const float *p_qn = qnorm;
  if (!p_qn) {
    LV_TRY(dqn.ensure(B));
    LV_CHECK_CUDA(launch_qnorm(q, B, dim, dqn.ptr, s));
    p_qn = dqn.ptr;
  }
  LV_CHECK_CUDA(launch_distance_gather(metric, matrix, dim, ids, B, C, q, p_qn, out, s));
  if (dqn.ptr) LV_CHECK_CUDA(cudaStreamSynchronize(s));  // dqn is freed on return
  return LV_OK;
}
