// lv_search.cuh — host/device contract of the batched search kernels.
#pragma once
#include "lv_common.cuh"

namespace lv {

enum Phase : int32_t { PH_IDLE = 0, PH_ENTRY = 1, PH_DESCENT = 2, PH_BASE = 3, PH_FINISHED = 4 };

constexpr uint32_t kVisited = 0x80000000u;
constexpr int kWarpsPerBlock = 4;

// Scalar state of one query slot (kept in registers by its warp while running).
struct SlotState {
  int32_t qi;        // query index being served, -1 when idle
  int32_t phase;     // Phase
  int32_t level;     // current upper level during descent
  int32_t cur;       // descent position
  float cur_d;
  int32_t eq_size;
  int32_t eq_hint;   // every EQ entry before this index is visited
  int32_t aq_len;
  int32_t xl_len;
  int32_t req_n;     // ids in the pending request
  int32_t req_off;   // offset of this slot's misses in the global request buffer
  int32_t n_elig;    // eligible (not yet promoted) AQ entries
  int32_t status;
  int32_t visits_n;
  int32_t blog_n;
  int32_t pad_;
  long long recomps;
  long long approx;
  long long hits;
  long long expansions;
  long long bytes;   // algorithmic HBM bytes of this query's traversal
};

struct SearchCtx {
  // graph (graph.py:30-73)
  int64_t n;
  int32_t dim, metric, max_degree, level_count;
  int32_t entry;
  const uint64_t *offs[kMaxLevels];
  const uint32_t *nbrs[kMaxLevels];
  const uint32_t *deleted_bits;  // may be null
  const uint32_t *cached_bits;   // may be null (cache off)
  const int32_t *cache_slot;     // node -> row of cache_rows (encoder source)
  const float *cache_rows;
  // PQ (pq.py:40-76)
  int32_t m;
  const uint8_t *codes;
  const float *luts;  // [B][m][256]
  // exact-vector source
  int32_t source;
  const float *matrix;   // [n][dim]  (LV_SOURCE_MATRIX)
  const float *emb_buf;  // recomputed rows (LV_SOURCE_ENCODER)
  const int32_t *emb_map;  // request index -> row of emb_buf (shared-recompute table), or null
  // queries
  int32_t B;
  const float *q;   // [B][dim]
  const float *qn;  // [B]
  // params (search.py:37-56)
  int32_t k, ef, mode;
  double alpha;     // rerank_percent / 100.0, computed on the host in float64
  // slots
  int32_t slots, aq_cap, req_cap, xl_cap;
  int64_t words;    // bitmap words per slot
  SlotState *st;
  float *eq_d;
  uint32_t *eq_id;
  unsigned long long *aq;
  uint32_t *abits, *xbits;   // dense per-slot bitmaps [slots][words] (vmask == 0)
  // bounded per-slot open-addressing sets [slots][vmask + 1] of node ids
  // (0xffffffff = empty), used instead of the bitmaps when vmask != 0: memory
  // O(slots x aq_cap) instead of O(slots x n) (config-3/5: 16k slots x 10M nodes)
  uint32_t *aset, *xset;
  uint32_t vmask;
  int32_t *xlist;
  int32_t *req;
  // global request buffer (encoder source)
  int32_t *greq;
  int32_t *greq_total;
  int32_t greq_cap;
  int32_t *queue_head;
  int32_t *done_count;
  unsigned long long *bytes_total;  // summed SlotState::bytes of finished queries
  // outputs
  int64_t *out_ids;
  float *out_dist;
  int32_t *out_count;
  int64_t *out_counters;
  int32_t *out_status;
  int32_t *visits;
  int32_t visits_cap;
  int32_t *blog;
  int32_t blog_cap;
  // LUT staging: 1 = each warp copies its query's LUT into shared memory with
  // one bulk (TMA-engine) copy when it claims the query (matrix source: a
  // warp runs its queries to completion, so each LUT crosses HBM once)
  int32_t lut_smem;
  int32_t warps_per_block;
};

__host__ __device__ inline size_t frontier_smem_per_warp(int max_degree, int req_cap) {
  size_t per = (size_t)max_degree * 16 + (size_t)req_cap * 8 + (size_t)max_degree * 4;
  return (per + 15) & ~size_t(15);
}
// with the LUT in shared memory: LUT (m x 256 fp32) + its mbarrier + the scratch
__host__ __device__ inline size_t frontier_smem_per_warp_lut(int max_degree, int req_cap, int m) {
  return (size_t)m * 256 * 4 + 16 + frontier_smem_per_warp(max_degree, req_cap);
}

// launchers (lv_search.cu)
cudaError_t launch_lut(const float *q, const float *qn, int B, int dim, int metric,
                       const float *codebooks, int m, int padded, float *luts, cudaStream_t s);
cudaError_t launch_adc_score(const float *lut, int m, const uint8_t *codes, const int64_t *ids,
                             int64_t count, float *out, cudaStream_t s);
cudaError_t launch_distance_many(int metric, const float *rows, int64_t nrows, int dim,
                                 const float *q, float qn, float *out, cudaStream_t s);
// Shared recomputation (cross-query dedup): map each of the `total` requested
// node ids to a row of the step's embedding table, claiming new rows for ids
// not seen before in this step (their ids are appended to new_ids at
// row - *base). keys/vals: open-addressing table of `mask + 1` slots.
cudaError_t launch_dedup(const int32_t *greq, int total, int32_t *keys, int32_t *vals,
                         uint32_t mask, int32_t *row_count, int32_t base, int32_t *new_ids,
                         int32_t *map, cudaStream_t s);
cudaError_t launch_qnorm(const float *q, int B, int dim, float *qn, cudaStream_t s);
cudaError_t launch_distance_gather(int metric, const float *rows, int dim, const int64_t *ids,
                                   int B, int C, const float *q, const float *qn, float *out,
                                   cudaStream_t s);
// buffer_scan + Engine.search merge (update.py:483-488, index.py:320-327);
// scratch holds B * np_ floats, *bad is set on a zero cosine denominator.
cudaError_t launch_pending_merge(int metric, const float *pend, const int64_t *pids, int64_t np_,
                                 int dim, const float *q, const float *qn, int B, int k,
                                 int64_t *ids, float *dist, int32_t *count, float *scratch,
                                 int *bad, cudaStream_t s);
cudaError_t launch_slot_reset(SlotState *st, int slots, cudaStream_t s);
cudaError_t launch_count_zero(const float *v, int n, int32_t *count, cudaStream_t s);
cudaError_t launch_frontier(SearchCtx &ctx, cudaStream_t s);
size_t frontier_smem_bytes(const SearchCtx &ctx);

}  // namespace lv
