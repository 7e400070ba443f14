/*
 * leann_b200.h — C-ABI of the B200-native LEANN search hot path.
 *
 * This is the drop-in boundary for the reference's query path. The reference
 * (slimvec 0.1.0, pure Python) has no FFI; its boundaries are Python duck
 * types, and each entry point below replaces one of them:
 *
 *   lv_index_create      <- Engine.open loaders: load_graph (graph.py:151-193),
 *                           load_pq (pq.py:213-244), load_deleted (graph.py:204-216)
 *   lv_index_set_matrix  <- MatrixSource(matrix) oracle source (search.py:78-93)
 *   lv_index_set_fetch   <- ProviderSource.fetch (search.py:103-110) of a HOST provider
 *                           (any reference provider object): the device traversal calls it
 *                           once per iteration with the step's new ids (LV_SOURCE_CALLBACK)
 *   lv_index_set_cache_rows
 *                        <- EmbeddingCache.vectors (search.py:113-128): the pinned rows
 *   lv_query_norms       <- the host np.float32(np.sqrt(np.dot(q, q))) of vectors.py:138 /
 *                           pq.py:163, on the device in the same BLAS order
 *   lv_merge_pending     <- Engine.search's merge of the pending (buffered-add) items
 *                           (index.py:320-327) over MutableIndex.buffer_scan
 *                           (update.py:483-488) with distance() (vectors.py:94-116)
 *   lv_index_set_cache   <- build_embedding_cache / EmbeddingCache (search.py:113-142)
 *   lv_index_attach_encoder
 *                        <- ProviderSource(provider, store.get) (search.py:96-110)
 *                           + provider.embed_batch (vectors.py:201-211)
 *   lv_search_batch      <- run_search(graph, q, params, source, metric, pq_model,
 *                           pq_codes, cache) (search.py:434-443), batched over B queries:
 *                           two_level_search (search.py:331-431) and
 *                           best_first_search (search.py:288-328)
 *   lv_adc_tables        <- adc_build (pq.py:153-178)
 *   lv_adc_score         <- approx_distance_many (pq.py:186-189)
 *   lv_distance_many     <- distance_many (vectors.py:120-140)
 *   lv_distance_gather   <- distance_many over gathered rows, for brute_force_topk /
 *                           ground_truth (evaluation.py:82-105)
 *   lv_encoder_create / lv_encode
 *                        <- provider.embed_batch for token payloads (vectors.py:201-211);
 *                           lv_encoder_profile / lv_encoder_stats replace the reference's
 *                           SearchReport.stage_times["embed"] instrumentation (search.py:66,
 *                           :159-187) with device-timed GEMM counters
 *   lv_gemm_bf16         <- the dense contraction inside embed_batch (no reference
 *                           counterpart: the reference's provider is a hash, vectors.py:168-189);
 *                           exported for unit tests of the tcgen05 GEMM
 *   lv_attention_bf16 / lv_attention_gqa_bf16
 *                        <- the encoder's attention (BERT-style MHA; config-4 causal GQA),
 *                           exported for unit tests of the tcgen05 attention kernels
 *   lv_encoder_set_fused_ln, lv_encoder_set_split_residual, lv_set_gemm_mode,
 *   lv_set_attention_mode, lv_set_fused_qkv_attention
 *                        <- kernel-variant switches for parity tests and A/B measurements
 *
 * Conventions: plain pointers and sizes only. Unless LV_IO_DEVICE is set in a
 * call's flags, array arguments are HOST pointers and the call copies them
 * through pinned staging on `stream` and synchronises before returning.
 * With LV_IO_DEVICE they are device pointers and the call is stream-ordered.
 * Return codes map onto the reference's SlimvecError.code (errors.py:11-93):
 * usage -> LV_ERR_USAGE, data -> LV_ERR_DATA, provider -> LV_ERR_PROVIDER,
 * internal -> LV_ERR_INTERNAL (same numbers as the CLI exit codes, cli.py:16).
 * A handle is used by one host thread at a time; one handle per GPU/rank.
 */
#ifndef LEANN_B200_H
#define LEANN_B200_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define LV_OK 0
#define LV_ERR_USAGE 2
#define LV_ERR_DATA 3
#define LV_ERR_PROVIDER 4
#define LV_ERR_INTERNAL 5

/* metric tags: the LPQ1 header byte order (pq.py:193-195, vectors.py:19) */
#define LV_METRIC_L2 0
#define LV_METRIC_IP 1
#define LV_METRIC_COSINE 2

/* search modes (search.py:32) */
#define LV_MODE_EXACT_BESTFIRST 0
#define LV_MODE_TWO_LEVEL 1

/* exact-vector sources */
#define LV_SOURCE_MATRIX 0   /* resident matrix (MatrixSource) */
#define LV_SOURCE_ENCODER 1  /* recompute with the attached encoder (ProviderSource) */
#define LV_SOURCE_CALLBACK 2 /* recompute through a host provider (lv_index_set_fetch) */

#define LV_IO_DEVICE 1       /* pointer arguments are device pointers */
#define LV_NO_SHARED_RECOMPUTE 2  /* lv_search_params.flags: encode every request, even
                                     when another in-flight query recomputed the node
                                     earlier in the same call (results are identical) */
#define LV_DRY_RECOMPUTE 4   /* lv_search_params.flags, encoder source: fill recomputed rows
                                from the resident matrix (lv_index_set_matrix) instead of
                                running the encoder. Same results and counters (the encoder
                                is batch-invariant); measures a configuration's physical
                                recompute count cheaply (tuning) */

#define LV_SMEM_LUT 8         /* lv_search_params.flags, matrix source: stage each query's ADC
                                lookup table in shared memory with one bulk copy instead of
                                reading it from global memory per lookup (A/B; slower at
                                config-2 shape: 64 KiB per warp caps residency at 3 warps/SM) */

#define LV_HASH_VISITED 16    /* lv_search_params.flags, two-level: per-query visited sets as
                                bounded hash sets (2 x AQ capacity) instead of dense n-bit
                                bitmaps; automatic when the bitmaps would exceed 4 GiB */

/* per-query status codes written to lv_search_outputs.status */
#define LV_Q_OK 0
#define LV_Q_AQ_OVERFLOW 1   /* retried internally with a larger queue; never returned */
#define LV_Q_FAILED 2

typedef struct lv_index lv_index;
/* Host provider: write the exact float32 vectors of ids[0..n) into rows[n][dim];
 * return 0, or non-zero for a provider failure (-> LV_ERR_PROVIDER). */
typedef int (*lv_fetch_fn)(void *user, const int64_t *ids, int32_t n, float *rows);
typedef struct lv_encoder lv_encoder;

/* One loaded index (LGR1 graph + LPQ1 PQ + LDL1 deletes), host arrays. */
typedef struct {
  int64_t n;                                /* nodes */
  int32_t dim;                              /* embedding dim */
  int32_t metric;                           /* LV_METRIC_* */
  int32_t max_degree;                       /* LGR1 M (caps every CSR row) */
  int32_t level_count;                      /* >= 1 */
  int64_t entry_point;
  const uint64_t *const *level_offsets;     /* [level_count] x u64[n+1] */
  const uint32_t *const *level_neighbors;   /* [level_count] x u32[nnz_l] */
  const uint64_t *level_nnz;                /* [level_count] */
  const uint8_t *deleted;                   /* u8[n] 0/1, or NULL */
  int32_t pq_m;                             /* 0 = no PQ (best-first only) */
  int32_t pq_padded_dim;
  const float *pq_codebooks;                /* f32[m][256][padded/m] */
  const uint8_t *pq_codes;                  /* u8[n][m] */
} lv_index_desc;

typedef struct {
  int32_t k;
  int32_t ef;
  double rerank_percent;   /* (0, 100] */
  int32_t batch_size;      /* only shapes the host-side batch log */
  int32_t mode;            /* LV_MODE_* */
  int32_t source;          /* LV_SOURCE_* */
  int32_t use_cache;       /* consult the lv_index_set_cache set */
  int32_t max_inflight;    /* concurrent query slots; 0 = automatic */
  int32_t flags;           /* LV_IO_DEVICE */
} lv_search_params;

typedef struct {
  int64_t *ids;            /* [B*k], -1 padded */
  float *dist;             /* [B*k] */
  int32_t *count;          /* [B] results returned (<= k) */
  int64_t *counters;       /* [B*4]: recomputations, approx_lookups, cache_hits, expansions */
  int32_t *status;         /* [B] LV_Q_*; may be NULL */
  int32_t *visits;         /* optional [B*visits_cap]: base-layer expansion order */
  int32_t visits_cap;
  int32_t *batch_log;      /* optional [B*batch_log_cap]: per-call recompute sizes */
  int32_t batch_log_cap;
} lv_search_outputs;

/* Aggregate statistics of the last lv_search_batch on a handle. */
typedef struct {
  int64_t iterations;        /* frontier launches (encoder mode) */
  int64_t logical_recomputes;
  int64_t physical_encodes;  /* passages run through the encoder */
  double frontier_ms;        /* device time in frontier kernels */
  double encoder_ms;         /* device time in the encoder */
  double total_ms;
  int64_t adc_bytes;         /* algorithmic bytes of the frontier kernels */
} lv_search_stats;

typedef struct {
  int64_t passages;       /* sequences encoded since the last reset */
  int64_t gemm_launches;  /* timed GEMM launches (profile mode) */
  double gemm_ms;         /* summed CUDA-event time of those launches */
  double gemm_flops;      /* 2*M*N*K summed over those launches */
  double gemm_bytes;      /* algorithmic bytes: A + W + out (+ residual) */
  int64_t attn_launches;  /* timed attention launches (profile mode) */
  double attn_ms;
  double attn_flops;      /* 4*S^2*dh*H per sequence */
  double attn_bytes;      /* qkv read + context written */
  int64_t fused_launches; /* timed fused QKV-projection + attention launches (S = 256, dh = 64) */
  double fused_ms;
  double fused_flops;     /* 2*M*3d*d (projection) + 4*S^2*dh*H per sequence (attention) */
  double fused_bytes;     /* x read + W_qkv + context written */
} lv_encoder_stats_t;

typedef struct {
  int32_t arch;         /* 0 = BERT-style post-LN GELU, mean pool (C1-C3);
                           1 = decoder-style (Qwen3-shaped, C4): pre-RMSNorm, GQA with
                           per-head q/k RMSNorm + RoPE, causal, SwiGLU, last-token pool */
  int32_t layers;
  int32_t hidden;
  int32_t heads;
  int32_t ffn;
  int32_t vocab;
  int32_t max_seq;
  int32_t precision;    /* 0 = fp32 (parity mode), 1 = bf16 tcgen05 (arch 1: bf16 only) */
  int32_t kv_heads;     /* arch 1: key/value heads (0 = heads) */
  int32_t head_dim;     /* arch 1: per-head dimension (0 = hidden / heads) */
  float rope_theta;     /* arch 1 */
  float norm_eps;       /* arch 1: RMSNorm epsilon */
} lv_encoder_config;

const char *lv_last_error(void);
int lv_version(void);
/* number of kernels this library has launched in the process (evidence counter) */
long long lv_kernel_launches(void);

int lv_index_create(const lv_index_desc *desc, int device, lv_index **out);
void lv_index_destroy(lv_index *index);
int lv_index_set_matrix(lv_index *index, const float *matrix, int flags);
int lv_index_set_deleted(lv_index *index, const uint8_t *deleted, int flags);
int lv_index_set_cache(lv_index *index, const int64_t *ids, int64_t count, int flags);
int lv_index_attach_encoder(lv_index *index, lv_encoder *enc, const void *tokens,
                            int32_t token_bytes, int32_t seq_len, int flags);
/* Host provider for LV_SOURCE_CALLBACK (fn = NULL detaches). Called on the
 * thread that runs lv_search_batch, once per traversal iteration. */
int lv_index_set_fetch(lv_index *index, lv_fetch_fn fn, void *user);
/* rows[count][dim]: the exact vectors of the ids last passed to lv_index_set_cache,
 * in that order (replaces vectors the attached encoder computed). */
int lv_index_set_cache_rows(lv_index *index, const float *rows, int flags);

/* qnorm may be NULL: norms are then computed on the device in the reference's
 * np.dot order (OpenBLAS SkylakeX sdot, bit-exact for dim % 32 == 0; vectors.py:138,
 * pq.py:163). A zero query norm under cosine two_level -> LV_ERR_USAGE (pq.py:163-166). */
int lv_search_batch(lv_index *index, const float *q, const float *qnorm, int32_t B,
                    const lv_search_params *params, const lv_search_outputs *out,
                    void *stream);
int lv_last_search_stats(const lv_index *index, lv_search_stats *stats);

int lv_adc_tables(lv_index *index, const float *q, const float *qnorm, int32_t B,
                  float *tables, int flags, void *stream);
int lv_adc_score(lv_index *index, const float *table, const int64_t *ids, int64_t count,
                 float *out, int flags, void *stream);
int lv_distance_many(int32_t metric, const float *rows, int64_t nrows, int32_t dim,
                     const float *q, float qnorm, float *out, int flags, void *stream);
/* distance_many (vectors.py:120-140) of query q[b] against matrix rows ids[b][0..C)
 * in the reference's einsum order, out [B][C] (ids < 0 -> +inf); DEVICE pointers,
 * stream-ordered. qnorm NULL -> computed as lv_query_norms. Used to re-rank
 * brute-force candidates into the reference's ground truth (evaluation.py:82-95). */
int lv_distance_gather(int32_t metric, const float *matrix, int32_t dim, const int64_t *ids,
                       int32_t B, int32_t C, const float *q, const float *qnorm, float *out,
                       void *stream);
/* qn = np.float32(np.sqrt(np.dot(q, q))) of each row q[b] (B x dim) in the
 * OpenBLAS sdot order (bit-exact with numpy on a SkylakeX-kernel host for
 * dim % 32 == 0; vectors.py:138, pq.py:163). */
int lv_query_norms(const float *q, int32_t B, int32_t dim, float *out, int flags, void *stream);
/* Pending-buffer merge: distance(q_b, pending_p) for every query b and pending
 * item p (vectors.py:94-116; np.dot in the OpenBLAS sdot order), merged with
 * the graph's results ids/dist/count (in-out, [B*k] / [B]) by (distance, id)
 * keeping the first k (index.py:320-327). qnorm may be NULL (computed on the
 * device in the same sdot order). A zero cosine denominator -> LV_ERR_USAGE. */
int lv_merge_pending(int32_t metric, const float *pending, const int64_t *pending_ids,
                     int64_t n_pending, int32_t dim, const float *q, const float *qnorm,
                     int32_t B, int32_t k, int64_t *ids, float *dist, int32_t *count,
                     int flags, void *stream);

int lv_encoder_create(const lv_encoder_config *cfg, const float *const *weights,
                      int32_t n_weights, int device, lv_encoder **out);
void lv_encoder_destroy(lv_encoder *enc);
int lv_encode(lv_encoder *enc, const void *tokens, int32_t token_bytes, int64_t n_seqs,
              int32_t seq_len, float *out, int flags, void *stream);
int lv_encoder_profile(lv_encoder *enc, int enable);
int lv_encoder_stats(lv_encoder *enc, lv_encoder_stats_t *stats);
int lv_encoder_reset_stats(lv_encoder *enc);
/* bf16 encoder: 1 = LayerNorms folded into the GEMM epilogues (default when
 * hidden, ffn % 256 == 0), 0 = standalone LayerNorm kernels. */
int lv_encoder_set_fused_ln(lv_encoder *enc, int enable);
/* bf16 encoder with fused LayerNorms: 1 (default) = the residual stream is carried
 * as bf16 plus an int8 correction (~15-bit mantissa) through the residual GEMM
 * epilogues and the pooling, 0 = bf16 residual stream. */
int lv_encoder_set_split_residual(lv_encoder *enc, int enable);

/* out[M][N] = epi(A[M][K] . W[N][K]^T (+ bias) ...), bf16 device pointers, fp32 bias;
 * epi: 0 bias, 1 bias + erf-GELU, 2 bias + residual. N % 128 == 0, K % 64 == 0. */
int lv_gemm_bf16(const void *A, const void *W, const float *bias, const void *residual,
                 void *out, int32_t M, int32_t N, int32_t K, int32_t epi, void *stream);
/* Multi-head bidirectional attention of the encoder, bf16 device pointers:
 * qkv [n_seqs*S][3*H*dh] (q | k | v), out [n_seqs*S][H*dh]. S % 64 == 0, dh in {64, 128}. */
int lv_attention_bf16(const void *qkv, void *out, int32_t n_seqs, int32_t S, int32_t H,
                      int32_t dh, void *stream);
/* Grouped-query attention (decoder-style encoder, config-4), bf16 device
 * pointers: qkv [n_seqs*S][(Hq + 2*Hkv)*dh] (q heads | k heads | v heads),
 * out [n_seqs*S][Hq*dh]; causal != 0 masks keys after the query. S % 64 == 0,
 * dh in {64, 128}, Hq % Hkv == 0. */
int lv_attention_gqa_bf16(const void *qkv, void *out, int32_t n_seqs, int32_t S, int32_t Hq,
                          int32_t Hkv, int32_t dh, int32_t causal, void *stream);
/* GEMM kernel selection: 0 = auto (2-CTA cta_group::2 kernel when N % 256 == 0),
 * 1 = 1-CTA kernel only; + 4 = the
 * 2-buffer/4-stage kernel also for long-K (K > 1024) residual GEMMs instead of the
 * default 1-buffer/5-stage one; + 8 = the 1-buffer/5-stage split-residual kernel also
 * for short-K split-residual GEMMs (default: 2-buffer/3-stage).
 * Returns the previous mode. */
int lv_set_gemm_mode(int mode);
/* Attention kernel selection: 0 = auto (tcgen05/TMEM kernel for dh == 64 and
 * S in {128, 256}, else the mma.sync kernel), 1 = mma.sync kernel only, any other value =
 * tcgen05 kernel where it applies. Returns the previous mode. */
int lv_set_attention_mode(int mode);
/* 1 (default): the bf16 BERT encoder at S = 256, dh = 64 runs the QKV projection
 * and the attention of a layer as one SM-pair kernel (qkv never written to HBM);
 * 0: the unfused pair GEMM + attn_tc_kernel (bit-identical results). Returns the
 * previous setting. */
int lv_set_fused_qkv_attention(int enable);

#ifdef __cplusplus
}
#endif
#endif /* LEANN_B200_H */
