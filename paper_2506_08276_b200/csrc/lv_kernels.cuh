// lv_kernels.cuh — launchers of the passage-encoder kernels (lv_encoder.cu,
// lv_gemm_tc.cu, lv_attn.cu). Activations are token-major [T][width] with
// T = n_seqs * seq_len; every kernel is batch-invariant (a row's result never
// depends on which other rows share the launch): fixed K order, no split-K.
#pragma once
#include <cuda.h>
#include <cuda_bf16.h>

#include "lv_common.cuh"

namespace lv {

enum Epi : int {
  EPI_BIAS = 0,           // out = acc + bias
  EPI_BIAS_GELU = 1,      // out = gelu_erf(acc + bias)
  EPI_BIAS_RESIDUAL = 2,  // out = acc + bias + residual
};

// ---- bf16 tcgen05 GEMM (lv_gemm_tc.cu): out[M][N] = epi(A[M][K] . W[N][K]^T)
// A, W, residual, out bf16 row-major; bias fp32. Requires N % 128 == 0,
// K % 64 == 0, 16-byte aligned rows. Persistent, warp-specialised:
// TMA producer / single-thread tcgen05.mma issuer / 4 epilogue warps.
struct TcGemmPlan;  // cached tensor maps for one (A, W, M, N, K)

// Generalised epilogue of the 2-CTA kernel (flags combine):
//   v = acc + bias                                   (default)
//   v = rstd_r * (acc - mean_r * colc) + bias        (EPF_LN_IN: A rows are raw
//        pre-LayerNorm activations y and W was pre-scaled by the LN gamma, so
//        W.LN(y) + b = rstd (W'.y - mean W'.1) + (W.beta + b) — the LayerNorm
//        never materialises)
//   v = gelu(v)                                      (EPF_GELU)
//   v += res                                         (EPF_RES)
//   v += (res - mean_r) * rstd_r * res_g + res_b     (EPF_RES | EPF_RES_LN)
//   stats[row][col / 64] = (mean, M2) of the bf16-rounded outputs of each
//        64-column box (EPF_STATS; combined by ln_stats_finalize)
//   EPF_SPLIT (with EPF_RES): the residual stream is carried to ~2^-14
//        absolute precision as hi = bf16(v) plus an int8 correction lo
//        (lo8_encode: the rounding error in units of 2^-13): the
//        residual is res + lo8_decode(res_lo), the output is written as out
//        (hi) and out_lo, and the statistics are taken from the unrounded v.
//        The consuming GEMMs read hi as their A operand; only the residual
//        adds and the LayerNorm statistics see the pair. (Rounding the
//        post-LN residual stream to bf16 at every sublayer was the dominant
//        error of the bf16 encoder against the fp32 one; the int8 half costs
//        1 byte per element per read / write.)
//   out[:, j] = silu(acc[:, g(j)]) * acc[:, u(j)]   (EPF_SWIGLU, alone: weight
//        rows interleaved per 64 as [gate 64 | up 64]; output width N / 2)
enum EpiFlag : int {
  EPF_GELU = 1, EPF_RES = 2, EPF_RES_LN = 4, EPF_LN_IN = 8, EPF_STATS = 16, EPF_SWIGLU = 32,
  EPF_SPLIT = 64
};
struct EpiParams {
  const float *bias = nullptr;    // [N]
  const float *colc = nullptr;    // [N]  EPF_LN_IN
  const float2 *ln_in = nullptr;  // [M]  (mean, rstd) of the A rows, EPF_LN_IN
  const float2 *res_ln = nullptr; // [M]  (mean, rstd) of the residual rows, EPF_RES_LN
  const float *res_g = nullptr;   // [N]  EPF_RES_LN
  const float *res_b = nullptr;   // [N]  EPF_RES_LN
  float2 *stats = nullptr;        // [M][N / 64]  EPF_STATS
  const int8_t *res_lo = nullptr;  // [M][N]  EPF_SPLIT: int8 correction of the residual
  int8_t *out_lo = nullptr;        // [M][N]  EPF_SPLIT: int8 correction of the output
  int flags = 0;
};
// 2-CTA kernel with the generalised epilogue; needs N % 256 == 0, K % 64 == 0.
int tc_gemm_ex(const __nv_bfloat16 *A, const __nv_bfloat16 *W, const __nv_bfloat16 *residual,
               __nv_bfloat16 *out, int M, int N, int K, const EpiParams &ep, cudaStream_t s);
int tc_gemm(const __nv_bfloat16 *A, const __nv_bfloat16 *W, const float *bias,
            const __nv_bfloat16 *residual, __nv_bfloat16 *out, int M, int N, int K, int epi,
            cudaStream_t s);
int tc_gemm_num_sms();
// Row-major bf16 [rows][cols] tensor map (row stride in bytes), box
// (box_cols x box_rows), 128-byte swizzle (box_cols * 2 must be 128).
// Split residual stream (EPF_SPLIT): v ~= hi + lo * 2^-13 with hi = bf16(v) and
// lo = the bf16 rounding error in units of 2^-13, saturated to an int8 and
// stored offset-binary (byte = lo + 128). |lo| <= 127 covers bf16's half-ulp
// for |v| < 8, the range of the post-LayerNorm stream; larger values
// saturate, so a correction is never worse than bf16 alone. Absolute error
// <= 2^-14. Four corrections per 32-bit word (byte k = column k).
constexpr float kLo8Scale = 8192.f;
__device__ __forceinline__ uint32_t lo8_s8(float scaled) {   // round-to-nearest, saturate
  uint32_t q;
  asm("cvt.rni.sat.s8.f32 %0, %1;" : "=r"(q) : "f"(scaled));
  return q;
}
// v[0..3], hi[0..3] -> one word of offset-binary corrections
__device__ __forceinline__ uint32_t lo8_pack4(const float *v, const float *hi) {
  const uint32_t q0 = lo8_s8((v[0] - hi[0]) * kLo8Scale), q1 = lo8_s8((v[1] - hi[1]) * kLo8Scale);
  const uint32_t q2 = lo8_s8((v[2] - hi[2]) * kLo8Scale), q3 = lo8_s8((v[3] - hi[3]) * kLo8Scale);
  return __byte_perm(__byte_perm(q0, q1, 0x0040), __byte_perm(q2, q3, 0x0040), 0x5410) ^
         0x80808080u;
}
// correction of column k (0..3) of a word, as a float (exact), times 2^-13 by the caller
__device__ __forceinline__ float lo8_get(uint32_t w, int k) {
  return __int_as_float(__byte_perm(w, 0x4B00u, 0x5440u | (uint32_t)k)) - 8388736.f;
}
constexpr float kLo8Inv = 1.f / kLo8Scale;
// Row-major int8 [rows][cols] tensor map, box (box_cols x box_rows), 64-byte
// swizzle (box_cols must be 64): 16-byte chunk j of box row r lands at chunk
// j ^ ((r >> 1) & 3).
bool make_tma_2d_u8(CUtensorMap *m, const void *ptr, uint64_t cols, uint64_t rows,
                    uint64_t row_stride_bytes, int box_cols, int box_rows);
bool make_tma_2d_bf16(CUtensorMap *m, const void *ptr, uint64_t cols, uint64_t rows,
                      uint64_t row_stride_bytes, int box_cols, int box_rows);
extern int g_gemm_mode;  // 0 auto (2-CTA pair kernel when N % 256 == 0), 1 force 1-CTA
extern int g_long_k_single;  // residual pair GEMMs with K > 1024: 1-buffer / 5-stage kernel
extern int g_split_single;   // split-residual pair GEMMs with K <= 1024: kMode 5 (1 buffer)

// ---- fp32 SIMT GEMM (parity mode, lv_encoder.cu): same contract in fp32.
cudaError_t f32_gemm(const float *A, const float *W, const float *bias, const float *residual,
                     float *out, int M, int N, int K, int epi, cudaStream_t s);

// ---- attention (lv_attn.cu). qkv [T][3*H*dh] (q | k | v, head-major inside
// each), out [T][H*dh]; bidirectional softmax(q k^T / sqrt(dh)) v per sequence.
cudaError_t attention_bf16(const __nv_bfloat16 *qkv, __nv_bfloat16 *out, int n_seqs, int S,
                           int H, int dh, cudaStream_t s);
// grouped-query attention, optional causal mask (decoder-style encoder, config-4):
// qkv [T][(Hq + 2 Hkv) * dh] = q heads | k heads | v heads, out [T][Hq * dh];
// dh in {64, 128}, S % 64 == 0.
cudaError_t attention_gqa_bf16(const __nv_bfloat16 *qkv, __nv_bfloat16 *out, int n_seqs, int S,
                               int Hq, int Hkv, int dh, bool causal, cudaStream_t s);
extern int g_attn_mode;  // see lv_set_attention_mode (leann_b200.h)
// Fused QKV projection + attention of a post-LN BERT layer on an SM pair
// (lv_qkv_attn.cu): ctx = attention(epi(x . W_qkv^T)) with the QKV epilogue of
// tc_gemm_ex (bias; LN-in when ln_in != null: rstd (acc - mean colc) + bias);
// S = 256, dh = 64, K % 64 == 0. Bit-identical to tc_gemm_ex + attention_bf16.
int qkv_attention_fused(const __nv_bfloat16 *x, const __nv_bfloat16 *w_qkv, const float *bias,
                        const float *colc, const float2 *ln_in, __nv_bfloat16 *ctx, int n_seqs,
                        int S, int H, int dh, int K, cudaStream_t s);
extern int g_fuse_qkv_attn;  // see lv_set_fused_qkv_attention (leann_b200.h)
cudaError_t attention_f32(const float *qkv, float *out, int n_seqs, int S, int H, int dh,
                          cudaStream_t s);

}  // namespace lv
