// lv_encoder.cu — the passage encoder behind the recompute source.
//
// The reference's provider boundary (provider.embed_batch, vectors.py:201-211,
// called from ProviderSource.fetch, search.py:103-110) maps item payloads to
// unit vectors. Here the payload of node v is its row of the token store
// (items.dat with packed u16/u32 token ids) and the provider is
// a random-init BERT-style encoder (post-LN, erf-GELU, mean-pool + L2 norm):
//
//   x = LN(tok[id] + pos[p])
//   per layer: x = LN1(x + Wo.attn(Wqkv.x + b) + bo); x = LN2(x + W2.gelu(W1.x + b1) + b2)
//   out = normalize(mean_p x)
//
// precision 1 (bf16): weights/activations bf16, fp32 accumulate/statistics;
//   GEMMs on tcgen05 (lv_gemm_tc.cu), attention on tensor cores (lv_attn.cu).
// precision 0 (fp32): SIMT fp32 GEMM and attention — the parity mode checked
//   against the torch fp32 oracle (oracle/encoder_ref.py).
// Both are batch-invariant: a passage's embedding never depends on the batch
// it rides in (the test_vectors.py:145-152 contract).
#include <algorithm>
#include <cstdlib>
#include <cmath>
#include <cstring>
#include <type_traits>
#include <vector>

#include "lv_encoder.cuh"
#include "lv_kernels.cuh"

namespace lv {
namespace {

constexpr unsigned kFull = 0xffffffffu;
constexpr float kLnEps = 1e-12f;

template <typename T>
__device__ __forceinline__ float to_f(T v);
template <>
__device__ __forceinline__ float to_f<float>(float v) { return v; }
template <>
__device__ __forceinline__ float to_f<__nv_bfloat16>(__nv_bfloat16 v) { return __bfloat162float(v); }
template <typename T>
__device__ __forceinline__ T from_f(float v);
template <>
__device__ __forceinline__ float from_f<float>(float v) { return v; }
template <>
__device__ __forceinline__ __nv_bfloat16 from_f<__nv_bfloat16>(float v) { return __float2bfloat16_rn(v); }

__device__ __forceinline__ float warp_sum(float v) {
  for (int o = 16; o; o >>= 1) v += __shfl_xor_sync(kFull, v, o);
  return v;
}

// One warp per token row: gather token + position embedding, LayerNorm.
// Row r of sequence n reads token store row ids[n] (or n when ids is null).
template <typename T>
__global__ void embed_ln_kernel(const void *__restrict__ tokens, int token_bytes, int S,
                                const int32_t *__restrict__ ids, int64_t seq0, int64_t n_seqs,
                                const float *__restrict__ tok_emb, const float *__restrict__ pos_emb,
                                int vocab, const float *__restrict__ g,
                                const float *__restrict__ b, int d, T *__restrict__ out,
                                int8_t *__restrict__ out_lo = nullptr) {
  const int64_t row = (int64_t)blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5);
  const int lane = threadIdx.x & 31;
  if (row >= n_seqs * S) return;
  const int64_t n = seq0 + row / S;
  const int p = (int)(row % S);
  const int64_t src = ids ? (int64_t)__ldg(ids + n) : n;
  uint32_t tok = token_bytes == 2
                     ? (uint32_t)__ldg(reinterpret_cast<const uint16_t *>(tokens) + src * S + p)
                     : __ldg(reinterpret_cast<const uint32_t *>(tokens) + src * S + p);
  if (tok >= (uint32_t)vocab) tok = vocab - 1;  // ids are validated on the host path
  const float *te = tok_emb + (size_t)tok * d;
  const float *pe = pos_emb + (size_t)p * d;
  float v[32];
  const int per = d / 32;
  float s = 0.f;
#pragma unroll
  for (int i = 0; i < 32; ++i) {
    if (i < per) {
      const int c = i * 32 + lane;
      v[i] = __ldg(te + c) + __ldg(pe + c);
      s += v[i];
    }
  }
  const float mean = warp_sum(s) / d;
  float q = 0.f;
#pragma unroll
  for (int i = 0; i < 32; ++i)
    if (i < per) {
      const float t = v[i] - mean;
      q += t * t;
    }
  const float rstd = rsqrtf(warp_sum(q) / d + kLnEps);
  T *o = out + row * d;
#pragma unroll
  for (int i = 0; i < 32; ++i)
    if (i < per) {
      const int c = i * 32 + lane;
      const float val = (v[i] - mean) * rstd * __ldg(g + c) + __ldg(b + c);
      const T hi = from_f<T>(val);
      o[c] = hi;
      if (out_lo)  // split stream: offset-binary correction byte (lv_kernels.cuh)
        out_lo[row * d + c] = (int8_t)((lo8_s8((val - to_f<T>(hi)) * kLo8Scale) & 0xff) ^ 0x80);
    }
}

// out = LN(in), one warp per row.
template <typename T>
__global__ void ln_kernel(const T *__restrict__ in, T *__restrict__ out, const float *__restrict__ g,
                          const float *__restrict__ b, int64_t rows, int d) {
  const int64_t row = (int64_t)blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5);
  const int lane = threadIdx.x & 31;
  if (row >= rows) return;
  const T *x = in + row * d;
  float v[32];
  const int per = d / 32;
  float s = 0.f;
#pragma unroll
  for (int i = 0; i < 32; ++i)
    if (i < per) {
      v[i] = to_f<T>(x[i * 32 + lane]);
      s += v[i];
    }
  const float mean = warp_sum(s) / d;
  float q = 0.f;
#pragma unroll
  for (int i = 0; i < 32; ++i)
    if (i < per) {
      const float t = v[i] - mean;
      q += t * t;
    }
  const float rstd = rsqrtf(warp_sum(q) / d + kLnEps);
  T *o = out + row * d;
#pragma unroll
  for (int i = 0; i < 32; ++i)
    if (i < per) {
      const int c = i * 32 + lane;
      o[c] = from_f<T>((v[i] - mean) * rstd * __ldg(g + c) + __ldg(b + c));
    }
}

// bf16 LayerNorm with 16-byte accesses (d % 256 == 0): lane owns chunks
// i*32 + lane of 8 elements; HBM-bound, one warp per row.
template <int NV>
__global__ void ln_bf16_vec_kernel(const __nv_bfloat16 *__restrict__ in,
                                   __nv_bfloat16 *__restrict__ out, const float *__restrict__ g,
                                   const float *__restrict__ b, int64_t rows) {
  constexpr int d = NV * 256;
  const int64_t row = (int64_t)blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5);
  const int lane = threadIdx.x & 31;
  if (row >= rows) return;
  const uint4 *x = reinterpret_cast<const uint4 *>(in + row * d);
  float v[NV][8];
  float s = 0.f;
#pragma unroll
  for (int i = 0; i < NV; ++i) {
    uint4 u = __ldg(x + i * 32 + lane);
    const __nv_bfloat162 *h = reinterpret_cast<const __nv_bfloat162 *>(&u);
#pragma unroll
    for (int e = 0; e < 4; ++e) {
      float2 f = __bfloat1622float2(h[e]);
      v[i][2 * e] = f.x;
      v[i][2 * e + 1] = f.y;
      s += f.x + f.y;
    }
  }
  const float mean = warp_sum(s) / d;
  float q = 0.f;
#pragma unroll
  for (int i = 0; i < NV; ++i)
#pragma unroll
    for (int e = 0; e < 8; ++e) {
      const float t = v[i][e] - mean;
      q += t * t;
    }
  const float rstd = rsqrtf(warp_sum(q) / d + kLnEps);
  uint4 *o = reinterpret_cast<uint4 *>(out + row * d);
#pragma unroll
  for (int i = 0; i < NV; ++i) {
    const int c0 = (i * 32 + lane) * 8;
    const float4 g0 = __ldg(reinterpret_cast<const float4 *>(g + c0));
    const float4 g1 = __ldg(reinterpret_cast<const float4 *>(g + c0 + 4));
    const float4 b0 = __ldg(reinterpret_cast<const float4 *>(b + c0));
    const float4 b1 = __ldg(reinterpret_cast<const float4 *>(b + c0 + 4));
    const float gg[8] = {g0.x, g0.y, g0.z, g0.w, g1.x, g1.y, g1.z, g1.w};
    const float bb[8] = {b0.x, b0.y, b0.z, b0.w, b1.x, b1.y, b1.z, b1.w};
    uint4 u;
    uint32_t *w = reinterpret_cast<uint32_t *>(&u);
#pragma unroll
    for (int e = 0; e < 4; ++e) {
      __nv_bfloat162 h = __floats2bfloat162_rn((v[i][2 * e] - mean) * rstd * gg[2 * e] + bb[2 * e],
                                               (v[i][2 * e + 1] - mean) * rstd * gg[2 * e + 1] +
                                                   bb[2 * e + 1]);
      w[e] = *reinterpret_cast<uint32_t *>(&h);
    }
    o[i * 32 + lane] = u;
  }
}

template <typename T>
void launch_ln(const T *in, T *out, const float *g, const float *b, int64_t rows, int d,
               cudaStream_t s) {
  const unsigned blocks = (unsigned)((rows + 7) / 8);
  if constexpr (sizeof(T) == 2) {
    if (d == 256) {
      ln_bf16_vec_kernel<1><<<blocks, 256, 0, s>>>(in, out, g, b, rows);
      note_launch();
      return;
    }
    if (d == 768) {
      ln_bf16_vec_kernel<3><<<blocks, 256, 0, s>>>(in, out, g, b, rows);
      note_launch();
      return;
    }
    if (d == 1024) {
      ln_bf16_vec_kernel<4><<<blocks, 256, 0, s>>>(in, out, g, b, rows);
      note_launch();
      return;
    }
  }
  ln_kernel<T><<<blocks, 256, 0, s>>>(in, out, g, b, rows, d);
  note_launch();
}

// Mean over the S token rows of each sequence, then L2 normalisation
// (x / max(||x||, 1e-12)). One block per sequence, fixed summation order.
template <typename T>
__global__ void pool_kernel(const T *__restrict__ x, float *__restrict__ out, int S, int d) {
  __shared__ float red[32];
  const int64_t seq = blockIdx.x;
  const T *base = x + seq * S * d;
  float local = 0.f;
  float mv[4];
  int nv = 0;
  for (int c = threadIdx.x; c < d; c += blockDim.x) {
    float s = 0.f;
    for (int p = 0; p < S; ++p) s += to_f<T>(base[(size_t)p * d + c]);
    s /= (float)S;
    mv[nv++] = s;
    local += s * s;
  }
  local = warp_sum(local);
  if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = local;
  __syncthreads();
  if (threadIdx.x < 32) {
    float t = threadIdx.x < (blockDim.x >> 5) ? red[threadIdx.x] : 0.f;
    t = warp_sum(t);
    if (threadIdx.x == 0) red[0] = t;
  }
  __syncthreads();
  const float inv = 1.0f / fmaxf(sqrtf(red[0]), 1e-12f);
  nv = 0;
  for (int c = threadIdx.x; c < d; c += blockDim.x) out[seq * d + c] = mv[nv++] * inv;
}

// Row LayerNorm statistics from the per-64-column-box (mean, M2) partials the
// GEMM epilogue wrote (EPF_STATS): Chan's parallel combination in a fixed
// order, population variance like the LayerNorm kernels, one thread per row.
__global__ void ln_stats_finalize_kernel(const float2 *__restrict__ parts, int nbox,
                                         float2 *__restrict__ out, int64_t rows) {
  const int64_t r = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (r >= rows) return;
  const float2 *p = parts + r * nbox;
  float m[32];
  float mean = 0.f, m2 = 0.f;
  for (int b = 0; b < nbox; ++b) {
    const float2 t = __ldg(p + b);
    m[b] = t.x;
    mean += t.x;
    m2 += t.y;
  }
  mean /= (float)nbox;
  for (int b = 0; b < nbox; ++b) {
    const float dm = m[b] - mean;
    m2 = fmaf(64.f * dm, dm, m2);
  }
  out[r] = make_float2(mean, rsqrtf(m2 / (64.f * nbox) + kLnEps));
}

// pool_kernel over LN(y): mean_p LN(y_p) = g * mean_p((y_p - mu_p) * rstd_p) + b,
// then L2 normalisation. One block per sequence; thread t owns columns
// [8t, 8t + 8) (16-byte loads, d % 8 == 0, d <= 1024), fixed summation order.
__global__ void __launch_bounds__(128) pool_ln_kernel(const __nv_bfloat16 *__restrict__ y,
                                                      const int8_t *__restrict__ y_lo,
                                                      const float2 *__restrict__ st,
                                                      const float *__restrict__ g,
                                                      const float *__restrict__ b,
                                                      float *__restrict__ out, int S, int d) {
  __shared__ float red[4];
  __shared__ float2 sst[512];
  const int64_t seq = blockIdx.x;
  for (int p = threadIdx.x; p < S; p += blockDim.x) sst[p] = st[seq * S + p];
  __syncthreads();
  const int c0 = 8 * threadIdx.x;
  const bool live = c0 < d;
  float acc[8] = {0.f, 0.f, 0.f, 0.f, 0.f, 0.f, 0.f, 0.f};
  if (live) {
    const uint4 *base = reinterpret_cast<const uint4 *>(y + seq * S * d + c0);
    const int stride = d / 8;
    const uint2 *base_lo =
        y_lo ? reinterpret_cast<const uint2 *>(y_lo + seq * S * d + c0) : nullptr;
    for (int p = 0; p < S; ++p) {
      const uint4 u = __ldg(base + (size_t)p * stride);
      const __nv_bfloat162 *h = reinterpret_cast<const __nv_bfloat162 *>(&u);
      uint2 ul = make_uint2(0x80808080u, 0x80808080u);   // offset-binary zero corrections
      if (base_lo) ul = __ldg(base_lo + (size_t)p * stride);  // split residual: y = hi + lo
      const float mu = sst[p].x, rs = sst[p].y;
#pragma unroll
      for (int e = 0; e < 4; ++e) {
        const float2 f = __bfloat1622float2(h[e]);
        const uint32_t w = e < 2 ? ul.x : ul.y;
        const float y0 = fmaf(lo8_get(w, (2 * e) & 3), kLo8Inv, f.x);
        const float y1 = fmaf(lo8_get(w, (2 * e + 1) & 3), kLo8Inv, f.y);
        acc[2 * e] = fmaf(y0 - mu, rs, acc[2 * e]);
        acc[2 * e + 1] = fmaf(y1 - mu, rs, acc[2 * e + 1]);
      }
    }
  }
  float v[8], local = 0.f;
#pragma unroll
  for (int e = 0; e < 8; ++e) {
    v[e] = live ? fmaf(g[c0 + e], acc[e] / (float)S, b[c0 + e]) : 0.f;
    local += v[e] * v[e];
  }
  local = warp_sum(local);
  if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = local;
  __syncthreads();
  const float tot = (red[0] + red[1]) + (red[2] + red[3]);
  const float inv = 1.0f / fmaxf(sqrtf(tot), 1e-12f);
  if (live) {
    float4 *o = reinterpret_cast<float4 *>(out + seq * d + c0);
    o[0] = make_float4(v[0] * inv, v[1] * inv, v[2] * inv, v[3] * inv);
    o[1] = make_float4(v[4] * inv, v[5] * inv, v[6] * inv, v[7] * inv);
  }
}

// ---- decoder-style encoder (arch 1, Qwen3-shaped, config-4) kernels --------

// x[row] = tok_emb[token of row] (fp32 table -> bf16), one warp per row.
__global__ void embed_gather_kernel(const void *__restrict__ tokens, int token_bytes, int S,
                                    const int32_t *__restrict__ ids, int64_t seq0, int64_t n_seqs,
                                    const float *__restrict__ tok_emb, int vocab, int d,
                                    __nv_bfloat16 *__restrict__ out,
                                    float2 *__restrict__ st = nullptr, float eps = 0.f) {
  const int64_t row = (int64_t)blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5);
  const int lane = threadIdx.x & 31;
  if (row >= n_seqs * S) return;
  const int64_t n = seq0 + row / S;
  const int p = (int)(row % S);
  const int64_t src = ids ? (int64_t)__ldg(ids + n) : n;
  uint32_t tok = token_bytes == 2
                     ? (uint32_t)__ldg(reinterpret_cast<const uint16_t *>(tokens) + src * S + p)
                     : __ldg(reinterpret_cast<const uint32_t *>(tokens) + src * S + p);
  if (tok >= (uint32_t)vocab) tok = vocab - 1;
  const float4 *te = reinterpret_cast<const float4 *>(tok_emb + (size_t)tok * d);
  uint2 *o = reinterpret_cast<uint2 *>(out + row * d);
  float ss = 0.f;  // sum of squares of the stored (bf16) values
  for (int c = lane; c < d / 4; c += 32) {
    const float4 v = __ldg(te + c);
    uint2 u;
    __nv_bfloat162 a = __floats2bfloat162_rn(v.x, v.y), b = __floats2bfloat162_rn(v.z, v.w);
    const float2 fa = __bfloat1622float2(a), fb = __bfloat1622float2(b);
    ss = fmaf(fa.x, fa.x, fmaf(fa.y, fa.y, fmaf(fb.x, fb.x, fmaf(fb.y, fb.y, ss))));
    u.x = *reinterpret_cast<uint32_t *>(&a);
    u.y = *reinterpret_cast<uint32_t *>(&b);
    o[c] = u;
  }
  if (st) {  // RMSNorm statistics (mean 0, rstd) of the row for the folded consumer GEMM
    ss = warp_sum(ss);
    if (lane == 0) st[row] = make_float2(0.f, rsqrtf(ss / d + eps));
  }
}

// RMSNorm statistics from the per-64-column-box (mean, M2) partials of an
// EPF_STATS epilogue: (0, rsqrt(mean(x^2) + eps)), one thread per row.
__global__ void rms_stats_finalize_kernel(const float2 *__restrict__ parts, int nbox, float eps,
                                          float2 *__restrict__ out, int64_t rows) {
  const int64_t r = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (r >= rows) return;
  const float2 *p = parts + r * nbox;
  float ss = 0.f;
  for (int b = 0; b < nbox; ++b) {
    const float2 t = __ldg(p + b);
    ss += fmaf(64.f * t.x, t.x, t.y);
  }
  out[r] = make_float2(0.f, rsqrtf(ss / (64.f * nbox) + eps));
}

// out = x * rsqrt(mean(x^2) + eps) * g (RMSNorm), bf16 rows, one warp per row,
// d % 256 == 0 (16-byte accesses).
__global__ void rmsnorm_bf16_kernel(const __nv_bfloat16 *__restrict__ in,
                                    __nv_bfloat16 *__restrict__ out, const float *__restrict__ g,
                                    int64_t rows, int d, float eps) {
  const int64_t row = (int64_t)blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5);
  const int lane = threadIdx.x & 31;
  if (row >= rows) return;
  const uint4 *x = reinterpret_cast<const uint4 *>(in + row * d);
  const int nv = d / 256;
  float v[4][8];
  float ss = 0.f;
#pragma unroll
  for (int i = 0; i < 4; ++i) {
    if (i >= nv) break;
    const uint4 u = __ldg(x + i * 32 + lane);
    const __nv_bfloat162 *h = reinterpret_cast<const __nv_bfloat162 *>(&u);
#pragma unroll
    for (int e = 0; e < 4; ++e) {
      const float2 f = __bfloat1622float2(h[e]);
      v[i][2 * e] = f.x;
      v[i][2 * e + 1] = f.y;
      ss = fmaf(f.x, f.x, fmaf(f.y, f.y, ss));
    }
  }
  const float r = rsqrtf(warp_sum(ss) / d + eps);
  uint4 *o = reinterpret_cast<uint4 *>(out + row * d);
#pragma unroll
  for (int i = 0; i < 4; ++i) {
    if (i >= nv) break;
    const int c0 = (i * 32 + lane) * 8;
    uint4 u;
    uint32_t *w = reinterpret_cast<uint32_t *>(&u);
    const float4 g0 = __ldg(reinterpret_cast<const float4 *>(g + c0));
    const float4 g1 = __ldg(reinterpret_cast<const float4 *>(g + c0 + 4));
    const float gg[8] = {g0.x, g0.y, g0.z, g0.w, g1.x, g1.y, g1.z, g1.w};
#pragma unroll
    for (int e = 0; e < 4; ++e) {
      __nv_bfloat162 hh = __floats2bfloat162_rn(v[i][2 * e] * r * gg[2 * e],
                                                v[i][2 * e + 1] * r * gg[2 * e + 1]);
      w[e] = *reinterpret_cast<uint32_t *>(&hh);
    }
    o[i * 32 + lane] = u;
  }
}

// In place on the q and k heads of qkv rows: per-head RMSNorm (q_norm /
// k_norm gammas) then rotary embedding (rotate-half convention) with the
// precomputed table rope[p][i] = (cos, sin)(p * theta^(-2i/dh)), position
// p = row % S. One warp per token row, looping over its q and k heads (one
// warp per (row, head) measured 143 us vs 93 us per config-4 layer); dh/32
// elements per lane, element j pairs with j + dh/2 inside the same lane.
template <int DH>
__global__ void qk_norm_rope_kernel(__nv_bfloat16 *__restrict__ qkv, int64_t rows, int S, int Hq,
                                    int Hkv, const float *__restrict__ qg,
                                    const float *__restrict__ kg, float eps,
                                    const float2 *__restrict__ rope) {
  constexpr int E = DH / 32;
  const int64_t row = (int64_t)blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5);
  const int lane = threadIdx.x & 31;
  if (row >= rows) return;  // one warp per token row, all q and k heads
  const int p = (int)(row % S);
  const float2 *rp = rope + (size_t)p * (DH / 2);
  float2 cs[E];
  float gq[E], gk[E];
#pragma unroll
  for (int e = 0; e < E; ++e) {
    const int j = e * 32 + lane;
    cs[e] = __ldg(rp + j % (DH / 2));
    gq[e] = __ldg(qg + j);
    gk[e] = __ldg(kg + j);
  }
  __nv_bfloat16 *base = qkv + row * (int64_t)(Hq + 2 * Hkv) * DH;
#pragma unroll 2
  for (int hd = 0; hd < Hq + Hkv; ++hd) {
    __nv_bfloat16 *x = base + hd * DH;
    const bool isq = hd < Hq;
    float v[E];
    float ss = 0.f;
#pragma unroll
    for (int e = 0; e < E; ++e) {
      v[e] = __bfloat162float(x[e * 32 + lane]);
      ss = fmaf(v[e], v[e], ss);
    }
    const float r = rsqrtf(warp_sum(ss) / DH + eps);
#pragma unroll
    for (int e = 0; e < E; ++e) v[e] *= r * (isq ? gq[e] : gk[e]);
#pragma unroll
    for (int e = 0; e < E; ++e) {
      const int pe = e < E / 2 ? e + E / 2 : e - E / 2;  // partner j +- dh/2
      const float rot = e < E / 2 ? -v[pe] : v[pe];
      x[e * 32 + lane] = __float2bfloat16_rn(fmaf(v[e], cs[e].x, rot * cs[e].y));
    }
  }
}

// Last-token pooling: final RMSNorm of row S-1 of each sequence, then L2
// normalisation. One warp per sequence.
__global__ void pool_last_kernel(const __nv_bfloat16 *__restrict__ x, const float *__restrict__ g,
                                 float *__restrict__ out, int64_t n_seqs, int S, int d, float eps) {
  const int64_t seq = (int64_t)blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5);
  const int lane = threadIdx.x & 31;
  if (seq >= n_seqs) return;
  const __nv_bfloat16 *r = x + (seq * S + S - 1) * d;
  float ss = 0.f;
  for (int c = lane; c < d; c += 32) {
    const float v = __bfloat162float(r[c]);
    ss = fmaf(v, v, ss);
  }
  const float rn = rsqrtf(warp_sum(ss) / d + eps);
  float nn = 0.f;
  for (int c = lane; c < d; c += 32) {
    const float v = __bfloat162float(r[c]) * rn * g[c];
    nn = fmaf(v, v, nn);
  }
  const float inv = 1.0f / fmaxf(sqrtf(warp_sum(nn)), 1e-12f);
  for (int c = lane; c < d; c += 32) out[seq * d + c] = __bfloat162float(r[c]) * rn * g[c] * inv;
}

// fp32 SIMT GEMM, 64x64 tile, 4x4 per thread; sequential fmaf over K.
__global__ void __launch_bounds__(256)
    f32_gemm_kernel(const float *__restrict__ A, const float *__restrict__ W,
                    const float *__restrict__ bias, const float *__restrict__ res,
                    float *__restrict__ out, int M, int N, int K, int epi) {
  __shared__ float As[16][68], Ws[16][68];
  const int tx = threadIdx.x & 15, ty = threadIdx.x >> 4;
  const int m0 = blockIdx.y * 64, n0 = blockIdx.x * 64;
  float acc[4][4] = {};
  for (int k0 = 0; k0 < K; k0 += 16) {
    for (int i = threadIdx.x; i < 1024; i += 256) {
      const int r = i >> 4, c = i & 15;
      const int gm = m0 + r, gn = n0 + r, gk = k0 + c;
      As[c][r] = (gm < M && gk < K) ? __ldg(A + (size_t)gm * K + gk) : 0.f;
      Ws[c][r] = (gn < N && gk < K) ? __ldg(W + (size_t)gn * K + gk) : 0.f;
    }
    __syncthreads();
#pragma unroll
    for (int kk = 0; kk < 16; ++kk) {
      float a[4], w[4];
#pragma unroll
      for (int i = 0; i < 4; ++i) {
        a[i] = As[kk][ty * 4 + i];
        w[i] = Ws[kk][tx * 4 + i];
      }
#pragma unroll
      for (int i = 0; i < 4; ++i)
#pragma unroll
        for (int j = 0; j < 4; ++j) acc[i][j] = fmaf(a[i], w[j], acc[i][j]);
    }
    __syncthreads();
  }
#pragma unroll
  for (int i = 0; i < 4; ++i) {
    const int gm = m0 + ty * 4 + i;
    if (gm >= M) continue;
#pragma unroll
    for (int j = 0; j < 4; ++j) {
      const int gn = n0 + tx * 4 + j;
      if (gn >= N) continue;
      float v = acc[i][j] + bias[gn];
      if (epi == EPI_BIAS_GELU) v = 0.5f * v * (1.0f + erff(v * 0.70710678118654752f));
      else if (epi == EPI_BIAS_RESIDUAL) v += res[(size_t)gm * N + gn];
      out[(size_t)gm * N + gn] = v;
    }
  }
}

__global__ void f32_to_bf16_kernel(const float *__restrict__ in, __nv_bfloat16 *__restrict__ out,
                                   int64_t n) {
  int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i < n) out[i] = __float2bfloat16_rn(in[i]);
}

}  // namespace

cudaError_t f32_gemm(const float *A, const float *W, const float *bias, const float *residual,
                     float *out, int M, int N, int K, int epi, cudaStream_t s) {
  dim3 grid((N + 63) / 64, (M + 63) / 64);
  f32_gemm_kernel<<<grid, 256, 0, s>>>(A, W, bias, residual, out, M, N, K, epi);
  note_launch();
  return cudaGetLastError();
}

}  // namespace lv

using namespace lv;

struct EncLayer {
  void *w_qkv = nullptr, *w_o = nullptr, *w_1 = nullptr, *w_2 = nullptr;
  float *b_qkv = nullptr, *b_o = nullptr, *b_1 = nullptr, *b_2 = nullptr;
  float *ln1_g = nullptr, *ln1_b = nullptr, *ln2_g = nullptr, *ln2_b = nullptr;
  // LayerNorm folded into the consuming GEMM (bf16 fused mode): W' = W diag(gamma)
  // (bf16), colc = W'.1, bias' = W.beta + b, for W_qkv (previous layer's LN2;
  // layer >= 1) and W_1 (this layer's LN1)
  void *w_qkv_f = nullptr, *w_1_f = nullptr;
  float *c_qkv = nullptr, *e_qkv = nullptr, *c_1 = nullptr, *e_1 = nullptr;
};

// decoder-style (arch 1) layer: pre-RMSNorm, GQA, SwiGLU
struct DecLayer {
  float *ln1_g = nullptr, *qn_g = nullptr, *kn_g = nullptr, *ln2_g = nullptr;
  void *w_qkv = nullptr, *w_o = nullptr, *w_gu = nullptr /* [gate; up] */, *w_down = nullptr;
  // RMSNorm gammas folded into the consuming weights (fused mode): W diag(g)
  void *w_qkv_f = nullptr, *w_gu_f = nullptr;
};

struct lv_encoder {
  lv_encoder_config cfg{};
  std::vector<DecLayer> dec;           // arch 1
  float *final_g = nullptr;            // arch 1 final RMSNorm
  float *zeros = nullptr;              // arch 1: zero bias for bias-free projections
  float2 *rope = nullptr;              // arch 1: (cos, sin) table [max_seq][head_dim / 2]
  int device = 0;
  float *tok_emb = nullptr, *pos_emb = nullptr, *emb_g = nullptr, *emb_b = nullptr;
  std::vector<EncLayer> layers;
  std::vector<void *> allocs;
  // activation workspace (element size 2 or 4), grown on demand
  int64_t cap_tokens = 0;
  void *x = nullptr, *qkv = nullptr, *ctx = nullptr, *y = nullptr, *h = nullptr;
  void *x_lo = nullptr, *y_lo = nullptr;  // split residual stream: int8 corrections (lo8)
  float2 *st_part = nullptr, *st1 = nullptr, *st2 = nullptr;  // LN statistics (fused mode)
  bool fuse_ln = false;  // bf16: LayerNorms folded into the GEMM epilogues
  bool split_res = true;  // fused bf16: residual stream as (hi, lo) bf16 pairs (EPF_SPLIT)
  // profiling of the dense GEMMs (lv_encoder_profile)
  bool profile = false;
  std::vector<cudaEvent_t> ev_pool;
  std::vector<std::pair<cudaEvent_t, cudaEvent_t>> ev_used;
  std::vector<double> ev_flops, ev_bytes;  // algorithmic work of each timed launch
  std::vector<int> ev_kind;                // 0 GEMM, 1 attention, 2 fused QKV + attention
  double gemm_bytes = 0.0;
  int64_t attn_launches = 0;
  double attn_ms = 0.0, attn_flops = 0.0, attn_bytes = 0.0;
  double gemm_ms = 0.0, gemm_flops = 0.0;
  int64_t fused_launches = 0;
  double fused_ms = 0.0, fused_flops = 0.0, fused_bytes = 0.0;
  int64_t gemm_launches = 0;
  int64_t passages = 0;
  ~lv_encoder() {
    for (void *p : allocs) cudaFree(p);
    cudaFree(x);
    cudaFree(qkv);
    cudaFree(ctx);
    cudaFree(y);
    cudaFree(h);
    cudaFree(x_lo);
    cudaFree(y_lo);
    cudaFree(st_part);
    cudaFree(st1);
    cudaFree(st2);
    for (auto e : ev_pool) cudaEventDestroy(e);
    for (auto &pr : ev_used) {
      cudaEventDestroy(pr.first);
      cudaEventDestroy(pr.second);
    }
  }
  size_t esize() const { return cfg.precision == 1 ? 2 : 4; }
};

namespace lv {
namespace {

// round-to-nearest-even to bf16, kept in a float (host)
float bf16_round_host(float f) {
  uint32_t u;
  std::memcpy(&u, &f, 4);
  if ((u & 0x7f800000u) == 0x7f800000u) return f;
  u = (u + 0x7fffu + ((u >> 16) & 1u)) & 0xffff0000u;
  std::memcpy(&f, &u, 4);
  return f;
}

int dev_alloc(lv_encoder *e, void **p, size_t bytes) {
  LV_CHECK_CUDA(cudaMalloc(p, bytes));
  e->allocs.push_back(*p);
  return LV_OK;
}

int upload_f32(lv_encoder *e, float **dst, const float *src, size_t n) {
  LV_TRY(dev_alloc(e, (void **)dst, n * 4));
  LV_CHECK_CUDA(cudaMemcpy(*dst, src, n * 4, cudaMemcpyHostToDevice));
  return LV_OK;
}

// matrices: bf16 copies for the tensor-core path, fp32 for parity mode
int upload_mat(lv_encoder *e, void **dst, const float *src, size_t n) {
  if (e->cfg.precision == 0) return upload_f32(e, (float **)dst, src, n);
  float *tmp = nullptr;
  LV_CHECK_CUDA(cudaMalloc(&tmp, n * 4));
  LV_CHECK_CUDA(cudaMemcpy(tmp, src, n * 4, cudaMemcpyHostToDevice));
  int rc = dev_alloc(e, dst, n * 2);
  if (rc == LV_OK) {
    f32_to_bf16_kernel<<<(unsigned)((n + 255) / 256), 256>>>(tmp, (__nv_bfloat16 *)*dst,
                                                            (int64_t)n);
    if (cudaDeviceSynchronize() != cudaSuccess) rc = LV_ERR_INTERNAL;
  }
  cudaFree(tmp);
  return rc;
}

int ensure_ws(lv_encoder *e, int64_t tokens) {
  if (tokens <= e->cap_tokens) return LV_OK;
  cudaFree(e->x);
  cudaFree(e->qkv);
  cudaFree(e->ctx);
  cudaFree(e->y);
  cudaFree(e->h);
  cudaFree(e->x_lo);
  cudaFree(e->y_lo);
  cudaFree(e->st_part);
  cudaFree(e->st1);
  cudaFree(e->st2);
  e->x = e->qkv = e->ctx = e->y = e->h = e->x_lo = e->y_lo = nullptr;
  e->st_part = e->st1 = e->st2 = nullptr;
  e->cap_tokens = 0;
  const size_t es = e->esize();
  const size_t d = e->cfg.hidden, ff = e->cfg.ffn;
  size_t w_qkv = 3 * d, w_ctx = d, w_h = ff;
  if (e->cfg.arch == 1) {
    const size_t dh = e->cfg.head_dim, hq = e->cfg.heads, hk = e->cfg.kv_heads;
    w_qkv = (hq + 2 * hk) * dh;
    w_ctx = hq * dh;
    w_h = ff;  // SwiGLU activation (the GEMM epilogue writes it directly)
  }
  LV_CHECK_CUDA(cudaMalloc(&e->x, tokens * d * es));
  LV_CHECK_CUDA(cudaMalloc(&e->qkv, tokens * w_qkv * es));
  LV_CHECK_CUDA(cudaMalloc(&e->ctx, tokens * w_ctx * es));
  LV_CHECK_CUDA(cudaMalloc(&e->y, tokens * d * es));
  LV_CHECK_CUDA(cudaMalloc(&e->h, tokens * w_h * es));
  if (e->cfg.precision == 1 && e->cfg.arch == 0) {  // int8 corrections of the split stream
    LV_CHECK_CUDA(cudaMalloc(&e->x_lo, tokens * d));
    LV_CHECK_CUDA(cudaMalloc(&e->y_lo, tokens * d));
  }
  if (e->cfg.precision == 1) {
    LV_CHECK_CUDA(cudaMalloc(&e->st_part, tokens * (d / 64) * sizeof(float2)));
    LV_CHECK_CUDA(cudaMalloc(&e->st1, tokens * sizeof(float2)));
    LV_CHECK_CUDA(cudaMalloc(&e->st2, tokens * sizeof(float2)));
  }
  e->cap_tokens = tokens;
  return LV_OK;
}

cudaEvent_t take_event(lv_encoder *e) {
  if (!e->ev_pool.empty()) {
    cudaEvent_t ev = e->ev_pool.back();
    e->ev_pool.pop_back();
    return ev;
  }
  cudaEvent_t ev;
  cudaEventCreate(&ev);
  return ev;
}

template <typename T>
int gemm(lv_encoder *e, const void *A, const void *W, const float *bias, const void *res, void *out,
         int M, int N, int K, int epi, cudaStream_t s) {
  cudaEvent_t e0 = nullptr, e1 = nullptr;
  if (e->profile) {
    e0 = take_event(e);
    e1 = take_event(e);
    cudaEventRecord(e0, s);
  }
  if constexpr (sizeof(T) == 2) {
    LV_TRY(tc_gemm((const __nv_bfloat16 *)A, (const __nv_bfloat16 *)W, bias,
                   (const __nv_bfloat16 *)res, (__nv_bfloat16 *)out, M, N, K, epi, s));
  } else {
    LV_CHECK_CUDA(f32_gemm((const float *)A, (const float *)W, bias, (const float *)res,
                           (float *)out, M, N, K, epi, s));
  }
  if (e->profile) {
    cudaEventRecord(e1, s);
    e->ev_used.emplace_back(e0, e1);
    e->ev_flops.push_back(2.0 * M * (double)N * K);
    e->ev_bytes.push_back((double)sizeof(T) *
                          ((double)M * K + (double)N * K + (double)M * N * (res ? 2 : 1)));
    e->ev_kind.push_back(0);
  }
  return LV_OK;
}

// bf16 forward with the LayerNorms folded into the GEMM epilogues (x0 = the
// embedding LN output is already in e->x). Per layer l (y2 of layer l-1 in x):
//   qkv = LN2(y2).Wqkv + b        (l = 0: x0.Wqkv + b)            EPF_LN_IN
//   y1  = ctx.Wo + bo + LN2(y2)   (l = 0: + x0), + row stats       EPF_RES[_LN] | EPF_STATS
//   h   = gelu(LN1(y1).W1 + b1)                                    EPF_LN_IN | EPF_GELU
//   y2  = h.W2 + b2 + LN1(y1), + row stats                         EPF_RES_LN | EPF_STATS
// and the pooled output reads LN2(y2) through the statistics. No LayerNorm
// output ever round-trips through HBM.
int fused_gemm(lv_encoder *e, const void *A, const void *W, const void *res, void *out, int M,
               int N, int K, const EpiParams &ep, cudaStream_t s) {
  cudaEvent_t e0 = nullptr, e1 = nullptr;
  if (e->profile) {
    e0 = take_event(e);
    e1 = take_event(e);
    cudaEventRecord(e0, s);
  }
  LV_TRY(tc_gemm_ex((const __nv_bfloat16 *)A, (const __nv_bfloat16 *)W,
                    (const __nv_bfloat16 *)res, (__nv_bfloat16 *)out, M, N, K, ep, s));
  if (e->profile) {
    cudaEventRecord(e1, s);
    e->ev_used.emplace_back(e0, e1);
    e->ev_flops.push_back(2.0 * M * (double)N * K);
    const double n_out = (ep.flags & EPF_SWIGLU) ? N / 2 : N;
    e->ev_bytes.push_back(2.0 * ((double)M * K + (double)N * K +
                                 (double)M * n_out * ((ep.flags & EPF_RES) ? 2 : 1)));
    e->ev_kind.push_back(0);
  }
  return LV_OK;
}

// bf16 attention with optional CUDA-event timing (profile mode): algorithmic
// work 4*S^2*dh*H FLOPs and qkv + context bytes per sequence
// Hkv > 0: grouped-query causal attention (decoder-style encoder, causal
// FLOPs counted at half); bytes = q, k, v read + context written.
int timed_attention(lv_encoder *e, const __nv_bfloat16 *qkv, __nv_bfloat16 *ctx, int ns, int S,
                    int H, int dh, cudaStream_t s, int Hkv = 0) {
  cudaEvent_t e0 = nullptr, e1 = nullptr;
  if (e->profile) {
    e0 = take_event(e);
    e1 = take_event(e);
    cudaEventRecord(e0, s);
  }
  if (Hkv > 0)
    LV_CHECK_CUDA(attention_gqa_bf16(qkv, ctx, ns, S, H, Hkv, dh, true, s));
  else
    LV_CHECK_CUDA(attention_bf16(qkv, ctx, ns, S, H, dh, s));
  if (e->profile) {
    cudaEventRecord(e1, s);
    e->ev_used.emplace_back(e0, e1);
    const double heads_io = Hkv > 0 ? 2.0 * H + 2.0 * Hkv : 4.0 * H;
    e->ev_flops.push_back((Hkv > 0 ? 2.0 : 4.0) * ns * (double)S * S * dh * H);
    e->ev_bytes.push_back(2.0 * ns * (double)S * heads_io * dh);
    e->ev_kind.push_back(1);
  }
  return LV_OK;
}

// fused QKV projection + attention (S = 256, dh = 64) with optional CUDA-event
// timing: algorithmic work = the projection's 2*M*3d*d plus attention's
// 4*S^2*dh*H FLOPs per sequence; bytes = x + W_qkv read, context written
int fused_qkv_attention(lv_encoder *e, const __nv_bfloat16 *x, const void *w_qkv,
                        const EpiParams &q, __nv_bfloat16 *ctx, int ns, int S, int H, int dh,
                        cudaStream_t s) {
  cudaEvent_t e0 = nullptr, e1 = nullptr;
  if (e->profile) {
    e0 = take_event(e);
    e1 = take_event(e);
    cudaEventRecord(e0, s);
  }
  const int d = H * dh;
  LV_TRY(qkv_attention_fused(x, (const __nv_bfloat16 *)w_qkv, q.bias, q.colc,
                             (q.flags & EPF_LN_IN) ? q.ln_in : nullptr, ctx, ns, S, H, dh, d, s));
  if (e->profile) {
    cudaEventRecord(e1, s);
    e->ev_used.emplace_back(e0, e1);
    const double M = (double)ns * S;
    e->ev_flops.push_back(2.0 * M * 3.0 * d * d + 4.0 * ns * (double)S * S * dh * H);
    e->ev_bytes.push_back(2.0 * (M * d + 3.0 * d * (double)d + M * d));
    e->ev_kind.push_back(2);
  }
  return LV_OK;
}

int finalize_stats(lv_encoder *e, float2 *dst, int M, cudaStream_t s) {
  ln_stats_finalize_kernel<<<(unsigned)((M + 255) / 256), 256, 0, s>>>(
      e->st_part, e->cfg.hidden / 64, dst, M);
  note_launch();
  LV_CHECK_CUDA(cudaGetLastError());
  return LV_OK;
}

int forward_fused(lv_encoder *e, int64_t ns, int S, int M, float *out, cudaStream_t s) {
  const auto &c = e->cfg;
  const int d = c.hidden, ff = c.ffn, H = c.heads, dh = c.hidden / c.heads;
  using bf = __nv_bfloat16;
  bf *x = (bf *)e->x, *qkv = (bf *)e->qkv, *ctx = (bf *)e->ctx, *y = (bf *)e->y, *h = (bf *)e->h;
  const bool split = e->split_res;
  int8_t *x_lo = split ? (int8_t *)e->x_lo : nullptr, *y_lo = split ? (int8_t *)e->y_lo : nullptr;
  for (size_t l = 0; l < e->layers.size(); ++l) {
    const EncLayer &L = e->layers[l];
    const EncLayer *P = l ? &e->layers[l - 1] : nullptr;
    EpiParams q;
    if (P) {
      q.bias = L.e_qkv;
      q.colc = L.c_qkv;
      q.ln_in = e->st2;
      q.flags = EPF_LN_IN;
    } else {
      q.bias = L.b_qkv;
    }
    const void *w_qkv = P ? L.w_qkv_f : L.w_qkv;
    if (g_fuse_qkv_attn && S == 256 && dh == 64) {  // qkv stays on chip (lv_qkv_attn.cu)
      LV_TRY(fused_qkv_attention(e, x, w_qkv, q, ctx, (int)ns, S, H, dh, s));
    } else {
      LV_TRY(fused_gemm(e, x, w_qkv, nullptr, qkv, M, 3 * d, d, q, s));
      LV_TRY(timed_attention(e, qkv, ctx, (int)ns, S, H, dh, s));
    }
    EpiParams o;
    o.bias = L.b_o;
    o.flags = EPF_RES | EPF_STATS | (split ? EPF_SPLIT : 0);
    o.stats = e->st_part;
    o.res_lo = x_lo;
    o.out_lo = y_lo;
    if (P) {
      o.flags |= EPF_RES_LN;
      o.res_ln = e->st2;
      o.res_g = P->ln2_g;
      o.res_b = P->ln2_b;
    }
    LV_TRY(fused_gemm(e, ctx, L.w_o, x, y, M, d, d, o, s));
    LV_TRY(finalize_stats(e, e->st1, M, s));
    EpiParams f1;
    f1.bias = L.e_1;
    f1.colc = L.c_1;
    f1.ln_in = e->st1;
    f1.flags = EPF_LN_IN | EPF_GELU;
    LV_TRY(fused_gemm(e, y, L.w_1_f, nullptr, h, M, ff, d, f1, s));
    EpiParams f2;
    f2.bias = L.b_2;
    f2.flags = EPF_RES | EPF_RES_LN | EPF_STATS | (split ? EPF_SPLIT : 0);
    f2.res_lo = y_lo;
    f2.out_lo = x_lo;
    f2.res_ln = e->st1;
    f2.res_g = L.ln1_g;
    f2.res_b = L.ln1_b;
    f2.stats = e->st_part;
    LV_TRY(fused_gemm(e, h, L.w_2, y, x, M, d, ff, f2, s));
    LV_TRY(finalize_stats(e, e->st2, M, s));
  }
  const EncLayer &Z = e->layers.back();
  pool_ln_kernel<<<(unsigned)ns, 128, 0, s>>>(x, x_lo, e->st2, Z.ln2_g, Z.ln2_b, out, S, d);
  note_launch();
  LV_CHECK_CUDA(cudaGetLastError());
  return LV_OK;
}

// tokens per encoder chunk (activations of one chunk live at once); LV_CHUNK_TOKENS
// overrides the default 2^19 for measurements
int64_t chunk_tokens(const lv_encoder *) {
  static const int64_t v = [] {
    const char *s = std::getenv("LV_CHUNK_TOKENS");
    const long long x = s ? std::atoll(s) : 0;
    return x > 0 ? (int64_t)x : ((int64_t)1 << 19);
  }();
  return v;
}

template <typename T>
int forward(lv_encoder *e, const void *tokens, int token_bytes, int S, const int32_t *d_ids,
            int64_t n_seqs, float *out, cudaStream_t s) {
  const auto &c = e->cfg;
  const int d = c.hidden, ff = c.ffn, H = c.heads, dh = c.hidden / c.heads;
  const int64_t max_tokens = std::max<int64_t>(S, chunk_tokens(e));
  const int64_t chunk = std::max<int64_t>(1, max_tokens / S);
  LV_TRY(ensure_ws(e, std::min<int64_t>(n_seqs, chunk) * S));
  T *x = (T *)e->x, *qkv = (T *)e->qkv, *ctx = (T *)e->ctx, *y = (T *)e->y, *h = (T *)e->h;
  for (int64_t s0 = 0; s0 < n_seqs; s0 += chunk) {
    const int64_t ns = std::min(chunk, n_seqs - s0);
    const int M = (int)(ns * S);
    int8_t *x_lo = nullptr;
    if constexpr (sizeof(T) == 2)
      if (e->fuse_ln && e->split_res) x_lo = (int8_t *)e->x_lo;
    embed_ln_kernel<T><<<(unsigned)((M + 7) / 8), 256, 0, s>>>(
        tokens, token_bytes, S, d_ids, s0, ns, e->tok_emb, e->pos_emb, c.vocab, e->emb_g,
        e->emb_b, d, x, x_lo);
        note_launch();
    LV_CHECK_CUDA(cudaGetLastError());
    if constexpr (sizeof(T) == 2) {
      if (e->fuse_ln) {
        LV_TRY(forward_fused(e, ns, S, M, out + s0 * d, s));
        continue;
      }
    }
    for (const EncLayer &L : e->layers) {
      LV_TRY(gemm<T>(e, x, L.w_qkv, L.b_qkv, nullptr, qkv, M, 3 * d, d, EPI_BIAS, s));
      if constexpr (sizeof(T) == 2) {
        LV_TRY(timed_attention(e, (const __nv_bfloat16 *)qkv, (__nv_bfloat16 *)ctx, (int)ns, S,
                               H, dh, s));
      } else {
        LV_CHECK_CUDA(attention_f32((const float *)qkv, (float *)ctx, (int)ns, S, H, dh, s));
      }
      LV_TRY(gemm<T>(e, ctx, L.w_o, L.b_o, x, y, M, d, d, EPI_BIAS_RESIDUAL, s));
      launch_ln<T>(y, x, L.ln1_g, L.ln1_b, M, d, s);
      LV_TRY(gemm<T>(e, x, L.w_1, L.b_1, nullptr, h, M, ff, d, EPI_BIAS_GELU, s));
      LV_TRY(gemm<T>(e, h, L.w_2, L.b_2, x, y, M, d, ff, EPI_BIAS_RESIDUAL, s));
      launch_ln<T>(y, x, L.ln2_g, L.ln2_b, M, d, s);
    }
    pool_kernel<T><<<(unsigned)ns, 256, 0, s>>>(x, out + s0 * d, S, d);
    note_launch();
    LV_CHECK_CUDA(cudaGetLastError());
  }
  e->passages += n_seqs;
  return LV_OK;
}

// Decoder-style encoder (arch 1), bf16 only. Per layer (residual stream x):
//   h = RMSNorm(x) ; qkv = h.Wqkv ; q, k <- RoPE(RMSNorm_head(q | k))
//   x = x + GQA_causal(q, k, v).Wo ; h = RMSNorm(x)
//   x = x + (silu(h.Wg) * (h.Wu)).Wd
// out = normalize(RMSNorm_final(x[last token])).
int forward_decoder(lv_encoder *e, const void *tokens, int token_bytes, int S,
                    const int32_t *d_ids, int64_t n_seqs, float *out, cudaStream_t s) {
  using bf = __nv_bfloat16;
  const auto &c = e->cfg;
  const int d = c.hidden, ff = c.ffn, Hq = c.heads, Hk = c.kv_heads, dh = c.head_dim;
  const int nqkv = (Hq + 2 * Hk) * dh;
  const int64_t max_tokens = std::max<int64_t>(S, (int64_t)1 << 18);
  const int64_t chunk = std::max<int64_t>(1, max_tokens / S);
  LV_TRY(ensure_ws(e, std::min<int64_t>(n_seqs, chunk) * S));
  bf *cur = (bf *)e->x, *tmp = (bf *)e->y, *qkv = (bf *)e->qkv, *ctx = (bf *)e->ctx,
     *gu = (bf *)e->h;
  for (int64_t s0 = 0; s0 < n_seqs; s0 += chunk) {
    const int64_t ns = std::min(chunk, n_seqs - s0);
    const int M = (int)(ns * S);
    cur = (bf *)e->x;
    tmp = (bf *)e->y;
    const bool fuse = e->fuse_ln;
    embed_gather_kernel<<<(unsigned)((M + 7) / 8), 256, 0, s>>>(
        tokens, token_bytes, S, d_ids, s0, ns, e->tok_emb, c.vocab, d, cur,
        fuse ? e->st2 : nullptr, c.norm_eps);
    note_launch();
    const unsigned rn_blocks = (unsigned)((M + 7) / 8);
    if (fuse) {
      // RMSNorms folded: producers emit row statistics, consumers use gamma-
      // scaled weights and scale their accumulators by rstd (EPF_LN_IN, mean 0)
      auto rms_final = [&](float2 *dst) -> int {
        rms_stats_finalize_kernel<<<(unsigned)((M + 255) / 256), 256, 0, s>>>(
            e->st_part, d / 64, c.norm_eps, dst, M);
        note_launch();
        LV_CHECK_CUDA(cudaGetLastError());
        return LV_OK;
      };
      for (const DecLayer &L : e->dec) {
        EpiParams q;
        q.bias = e->zeros;
        q.colc = e->zeros;
        q.ln_in = e->st2;
        q.flags = EPF_LN_IN;
        LV_TRY(fused_gemm(e, cur, L.w_qkv_f, nullptr, qkv, M, nqkv, d, q, s));
        if (dh == 128)
          qk_norm_rope_kernel<128><<<rn_blocks, 256, 0, s>>>(qkv, M, S, Hq, Hk, L.qn_g, L.kn_g,
                                                              c.norm_eps, e->rope);
        else
          qk_norm_rope_kernel<64><<<rn_blocks, 256, 0, s>>>(qkv, M, S, Hq, Hk, L.qn_g, L.kn_g,
                                                             c.norm_eps, e->rope);
        note_launch();
        LV_TRY(timed_attention(e, qkv, ctx, (int)ns, S, Hq, dh, s, Hk));
        EpiParams o;
        o.bias = e->zeros;
        o.flags = EPF_RES | EPF_STATS;
        o.stats = e->st_part;
        LV_TRY(fused_gemm(e, ctx, L.w_o, cur, tmp, M, d, Hq * dh, o, s));
        std::swap(cur, tmp);
        LV_TRY(rms_final(e->st1));
        EpiParams sg;
        sg.flags = EPF_SWIGLU | EPF_LN_IN;
        sg.ln_in = e->st1;
        LV_TRY(fused_gemm(e, cur, L.w_gu_f, nullptr, gu, M, 2 * ff, d, sg, s));
        EpiParams dn;
        dn.bias = e->zeros;
        dn.flags = EPF_RES | EPF_STATS;
        dn.stats = e->st_part;
        LV_TRY(fused_gemm(e, gu, L.w_down, cur, tmp, M, d, ff, dn, s));
        std::swap(cur, tmp);
        LV_TRY(rms_final(e->st2));
      }
    }
    for (const DecLayer &L : e->dec) {
      if (fuse) break;
      rmsnorm_bf16_kernel<<<rn_blocks, 256, 0, s>>>(cur, tmp, L.ln1_g, M, d, c.norm_eps);
      note_launch();
      LV_TRY(gemm<bf>(e, tmp, L.w_qkv, e->zeros, nullptr, qkv, M, nqkv, d, EPI_BIAS, s));
      const int64_t items = M;  // one warp per token row
      if (dh == 128)
        qk_norm_rope_kernel<128><<<(unsigned)((items + 7) / 8), 256, 0, s>>>(
            qkv, M, S, Hq, Hk, L.qn_g, L.kn_g, c.norm_eps, e->rope);
      else
        qk_norm_rope_kernel<64><<<(unsigned)((items + 7) / 8), 256, 0, s>>>(
            qkv, M, S, Hq, Hk, L.qn_g, L.kn_g, c.norm_eps, e->rope);
      note_launch();
      LV_TRY(timed_attention(e, qkv, ctx, (int)ns, S, Hq, dh, s, Hk));
      LV_TRY(gemm<bf>(e, ctx, L.w_o, e->zeros, cur, tmp, M, d, Hq * dh, EPI_BIAS_RESIDUAL, s));
      std::swap(cur, tmp);
      rmsnorm_bf16_kernel<<<rn_blocks, 256, 0, s>>>(cur, tmp, L.ln2_g, M, d, c.norm_eps);
      note_launch();
      EpiParams sg;
      sg.flags = EPF_SWIGLU;  // act = silu(h.Wg) * (h.Wu), straight from the accumulators
      LV_TRY(fused_gemm(e, tmp, L.w_gu, nullptr, gu, M, 2 * ff, d, sg, s));
      LV_TRY(gemm<bf>(e, gu, L.w_down, e->zeros, cur, tmp, M, d, ff, EPI_BIAS_RESIDUAL, s));
      std::swap(cur, tmp);
    }
    pool_last_kernel<<<(unsigned)((ns + 7) / 8), 256, 0, s>>>(cur, e->final_g, out + s0 * d, ns, S,
                                                              d, c.norm_eps);
    note_launch();
    LV_CHECK_CUDA(cudaGetLastError());
  }
  e->passages += n_seqs;
  return LV_OK;
}

}  // namespace

int encoder_hidden(const lv_encoder *enc) { return enc ? enc->cfg.hidden : 0; }

int encode_node_rows(lv_encoder *enc, const void *tokens, int token_bytes, int seq_len,
                     const int32_t *d_ids, int64_t count, float *out, cudaStream_t s) {
  LV_REQUIRE(enc, LV_ERR_USAGE, "null encoder");
  LV_REQUIRE(seq_len <= enc->cfg.max_seq, LV_ERR_USAGE, "seq_len exceeds the encoder's max_seq");
  if (count <= 0) return LV_OK;
  if (enc->cfg.arch == 1)
    return forward_decoder(enc, tokens, token_bytes, seq_len, d_ids, count, out, s);
  if (enc->cfg.precision == 1)
    return forward<__nv_bfloat16>(enc, tokens, token_bytes, seq_len, d_ids, count, out, s);
  return forward<float>(enc, tokens, token_bytes, seq_len, d_ids, count, out, s);
}

// Resolve the recorded GEMM events (after the stream has been synchronised).
void encoder_collect_profile(lv_encoder *enc) {
  if (!enc) return;
  for (size_t i = 0; i < enc->ev_used.size(); ++i) {
    float ms = 0.f;
    if (cudaEventElapsedTime(&ms, enc->ev_used[i].first, enc->ev_used[i].second) == cudaSuccess) {
      if (enc->ev_kind[i] == 0) {
        enc->gemm_ms += ms;
        enc->gemm_flops += enc->ev_flops[i];
        enc->gemm_bytes += enc->ev_bytes[i];
        enc->gemm_launches += 1;
      } else if (enc->ev_kind[i] == 2) {
        enc->fused_ms += ms;
        enc->fused_flops += enc->ev_flops[i];
        enc->fused_bytes += enc->ev_bytes[i];
        enc->fused_launches += 1;
      } else {
        enc->attn_ms += ms;
        enc->attn_flops += enc->ev_flops[i];
        enc->attn_bytes += enc->ev_bytes[i];
        enc->attn_launches += 1;
      }
    }
    enc->ev_pool.push_back(enc->ev_used[i].first);
    enc->ev_pool.push_back(enc->ev_used[i].second);
  }
  enc->ev_used.clear();
  enc->ev_flops.clear();
  enc->ev_bytes.clear();
  enc->ev_kind.clear();
}

}  // namespace lv

namespace {
int create_decoder(const lv_encoder_config *cfg_in, const float *const *weights, int32_t n_weights,
                   int device, lv_encoder **out) {
  lv_encoder_config cfg = *cfg_in;
  if (cfg.kv_heads <= 0) cfg.kv_heads = cfg.heads;
  if (cfg.head_dim <= 0) cfg.head_dim = cfg.heads ? cfg.hidden / cfg.heads : 0;
  if (cfg.norm_eps <= 0.f) cfg.norm_eps = 1e-6f;
  if (cfg.rope_theta <= 0.f) cfg.rope_theta = 1e6f;
  LV_REQUIRE(cfg.precision == 1, LV_ERR_USAGE, "the decoder-style encoder (arch 1) is bf16 only");
  LV_REQUIRE(cfg.layers >= 1 && cfg.heads >= 1 && cfg.kv_heads >= 1 &&
                 cfg.heads % cfg.kv_heads == 0 && (cfg.head_dim == 64 || cfg.head_dim == 128),
             LV_ERR_USAGE, "arch 1: need heads % kv_heads == 0 and head_dim in {64, 128}");
  const int nqkv = (cfg.heads + 2 * cfg.kv_heads) * cfg.head_dim;
  LV_REQUIRE(cfg.hidden % 256 == 0 && cfg.hidden <= 1024 && cfg.ffn % 256 == 0 && nqkv % 256 == 0 &&
                 (cfg.heads * cfg.head_dim) % 64 == 0,
             LV_ERR_USAGE, "arch 1: hidden, ffn, (heads + 2 kv_heads) * head_dim % 256 == 0");
  LV_REQUIRE(cfg.vocab >= 1 && cfg.max_seq >= 1 && cfg.max_seq <= 4096, LV_ERR_USAGE,
             "bad encoder geometry");
  LV_REQUIRE(n_weights == 2 + 9 * cfg.layers, LV_ERR_USAGE,
             "arch 1 weights: expected 2 + 9 * layers arrays");
  DeviceGuard guard(device);
  auto *e = new lv_encoder();
  e->cfg = cfg;
  e->device = device;
  const size_t d = cfg.hidden, ff = cfg.ffn, dh = cfg.head_dim, hq = cfg.heads;
  int rc = LV_OK;
  auto up = [&](float **dst, int idx, size_t n) {
    if (rc == LV_OK) rc = upload_f32(e, dst, weights[idx], n);
  };
  auto upm = [&](void **dst, int idx, size_t n) {
    if (rc == LV_OK) rc = upload_mat(e, dst, weights[idx], n);
  };
  up(&e->tok_emb, 0, (size_t)cfg.vocab * d);
  e->dec.resize(cfg.layers);
  std::vector<float> gu;
  for (int l = 0; l < cfg.layers && rc == LV_OK; ++l) {
    DecLayer &L = e->dec[l];
    const int b = 1 + 9 * l;
    up(&L.ln1_g, b + 0, d);
    upm(&L.w_qkv, b + 1, (size_t)nqkv * d);
    up(&L.qn_g, b + 2, dh);
    up(&L.kn_g, b + 3, dh);
    upm(&L.w_o, b + 4, d * hq * dh);
    up(&L.ln2_g, b + 5, d);
    // [gate | up] interleaved per 64 rows: one GEMM with the SwiGLU epilogue
    gu.resize(2 * ff * d);
    for (size_t blk = 0; blk < ff / 64; ++blk) {
      std::memcpy(gu.data() + (2 * blk) * 64 * d, weights[b + 6] + blk * 64 * d, 64 * d * 4);
      std::memcpy(gu.data() + (2 * blk + 1) * 64 * d, weights[b + 7] + blk * 64 * d, 64 * d * 4);
    }
    if (rc == LV_OK) rc = upload_mat(e, &L.w_gu, gu.data(), 2 * ff * d);
    upm(&L.w_down, b + 8, d * ff);
    // folded copies: columns scaled by the RMSNorm gamma of their input
    const float *g1 = weights[b + 0], *g2 = weights[b + 5];
    std::vector<float> wq((size_t)nqkv * d);
    for (size_t n = 0; n < (size_t)nqkv; ++n)
      for (size_t k = 0; k < d; ++k) wq[n * d + k] = weights[b + 1][n * d + k] * g1[k];
    if (rc == LV_OK) rc = upload_mat(e, &L.w_qkv_f, wq.data(), wq.size());
    for (size_t n = 0; n < 2 * ff; ++n)
      for (size_t k = 0; k < d; ++k) gu[n * d + k] *= g2[k];
    if (rc == LV_OK) rc = upload_mat(e, &L.w_gu_f, gu.data(), 2 * ff * d);
  }
  e->fuse_ln = rc == LV_OK;
  up(&e->final_g, 1 + 9 * cfg.layers, d);
  if (rc == LV_OK) {
    const size_t nz = std::max<size_t>(std::max<size_t>(nqkv, 2 * ff), d);
    std::vector<float> z(nz, 0.f);
    rc = upload_f32(e, &e->zeros, z.data(), nz);
  }
  if (rc == LV_OK) {  // RoPE table, fp32 like the reference formulation
    std::vector<float> t((size_t)cfg.max_seq * dh);
    for (int p = 0; p < cfg.max_seq; ++p)
      for (size_t i = 0; i < dh / 2; ++i) {
        const float inv = 1.0f / std::pow(cfg.rope_theta, (float)(2 * i) / (float)dh);
        const float a = (float)p * inv;
        t[((size_t)p * (dh / 2) + i) * 2] = std::cos(a);
        t[((size_t)p * (dh / 2) + i) * 2 + 1] = std::sin(a);
      }
    rc = upload_f32(e, reinterpret_cast<float **>(&e->rope), t.data(), t.size());
  }
  if (rc != LV_OK) {
    delete e;
    return rc;
  }
  *out = e;
  return LV_OK;
}
}  // namespace

extern "C" {

int lv_encoder_create(const lv_encoder_config *cfg, const float *const *weights, int32_t n_weights,
                      int device, lv_encoder **out) {
  LV_REQUIRE(cfg && weights && out, LV_ERR_USAGE, "lv_encoder_create: null argument");
  *out = nullptr;
  LV_REQUIRE(cfg->arch == 0 || cfg->arch == 1, LV_ERR_USAGE, "arch must be 0 or 1");
  if (cfg->arch == 1) return create_decoder(cfg, weights, n_weights, device, out);
  LV_REQUIRE(cfg->precision == 0 || cfg->precision == 1, LV_ERR_USAGE, "precision must be 0 or 1");
  LV_REQUIRE(cfg->layers >= 1 && cfg->heads >= 1 && cfg->hidden % cfg->heads == 0, LV_ERR_USAGE,
             "bad encoder geometry");
  LV_REQUIRE(cfg->hidden % 32 == 0 && cfg->hidden <= 1024, LV_ERR_USAGE,
             "hidden must be a multiple of 32 and <= 1024");
  LV_REQUIRE(cfg->vocab >= 1 && cfg->max_seq >= 1 && cfg->ffn >= 1, LV_ERR_USAGE,
             "bad encoder geometry");
  if (cfg->precision == 1) {
    const int dh = cfg->hidden / cfg->heads;
    LV_REQUIRE(cfg->hidden % 128 == 0 && cfg->ffn % 128 == 0 && (dh == 64 || dh == 128),
               LV_ERR_USAGE, "bf16 encoder needs hidden, ffn % 128 == 0 and head dim 64/128");
  }
  LV_REQUIRE(n_weights == 4 + 12 * cfg->layers, LV_ERR_USAGE,
             "weights: expected 4 + 12 * layers arrays");
  DeviceGuard guard(device);
  auto *e = new lv_encoder();
  e->cfg = *cfg;
  e->device = device;
  const size_t d = cfg->hidden, ff = cfg->ffn;
  int rc = LV_OK;
  auto up = [&](float **dst, int idx, size_t n) {
    if (rc == LV_OK) rc = upload_f32(e, dst, weights[idx], n);
  };
  auto upm = [&](void **dst, int idx, size_t n) {
    if (rc == LV_OK) rc = upload_mat(e, dst, weights[idx], n);
  };
  up(&e->tok_emb, 0, (size_t)cfg->vocab * d);
  up(&e->pos_emb, 1, (size_t)cfg->max_seq * d);
  up(&e->emb_g, 2, d);
  up(&e->emb_b, 3, d);
  e->layers.resize(cfg->layers);
  for (int l = 0; l < cfg->layers; ++l) {
    EncLayer &L = e->layers[l];
    const int b = 4 + 12 * l;
    upm(&L.w_qkv, b + 0, 3 * d * d);
    up(&L.b_qkv, b + 1, 3 * d);
    upm(&L.w_o, b + 2, d * d);
    up(&L.b_o, b + 3, d);
    up(&L.ln1_g, b + 4, d);
    up(&L.ln1_b, b + 5, d);
    upm(&L.w_1, b + 6, ff * d);
    up(&L.b_1, b + 7, ff);
    upm(&L.w_2, b + 8, d * ff);
    up(&L.b_2, b + 9, d);
    up(&L.ln2_g, b + 10, d);
    up(&L.ln2_b, b + 11, d);
  }
  // bf16: fold each LayerNorm into the GEMM that consumes it (see forward_fused)
  if (rc == LV_OK && cfg->precision == 1 && d % 256 == 0 && ff % 256 == 0) {
    std::vector<float> wf, cv, ev;
    auto fold = [&](int wi, int bi, int gi, int be, size_t N, size_t K, void **wd, float **cd,
                    float **ed) {
      if (rc != LV_OK) return;
      const float *W = weights[wi], *bias = weights[bi], *g = weights[gi], *beta = weights[be];
      wf.resize(N * K);
      cv.resize(N);
      ev.resize(N);
      for (size_t n = 0; n < N; ++n) {
        double cs = 0.0, es = bias[n];
        for (size_t k = 0; k < K; ++k) {
          const float wr = bf16_round_host(W[n * K + k] * g[k]);
          wf[n * K + k] = wr;
          cs += wr;
          es += (double)W[n * K + k] * beta[k];
        }
        cv[n] = (float)cs;
        ev[n] = (float)es;
      }
      rc = upload_mat(e, wd, wf.data(), N * K);
      if (rc == LV_OK) rc = upload_f32(e, cd, cv.data(), N);
      if (rc == LV_OK) rc = upload_f32(e, ed, ev.data(), N);
    };
    for (int l = 0; l < cfg->layers; ++l) {
      EncLayer &L = e->layers[l];
      const int b = 4 + 12 * l;
      if (l > 0) fold(b + 0, b + 1, b - 2, b - 1, 3 * d, d, &L.w_qkv_f, &L.c_qkv, &L.e_qkv);
      fold(b + 6, b + 7, b + 4, b + 5, ff, d, &L.w_1_f, &L.c_1, &L.e_1);
    }
    e->fuse_ln = rc == LV_OK;
  }
  if (rc != LV_OK) {
    delete e;
    return rc;
  }
  *out = e;
  return LV_OK;
}

void lv_encoder_destroy(lv_encoder *enc) {
  if (!enc) return;
  DeviceGuard guard(enc->device);
  delete enc;
}

int lv_encode(lv_encoder *enc, const void *tokens, int32_t token_bytes, int64_t n_seqs,
              int32_t seq_len, float *out, int flags, void *stream) {
  LV_REQUIRE(enc && tokens && out, LV_ERR_USAGE, "lv_encode: null argument");
  LV_REQUIRE(token_bytes == 2 || token_bytes == 4, LV_ERR_USAGE, "token_bytes must be 2 or 4");
  LV_REQUIRE(seq_len >= 1 && seq_len <= enc->cfg.max_seq, LV_ERR_USAGE,
             "seq_len must be in [1, max_seq]");
  if (enc->cfg.precision == 1)
    LV_REQUIRE(seq_len % 64 == 0, LV_ERR_USAGE, "bf16 encoder needs seq_len % 64 == 0");
  if (n_seqs <= 0) return LV_OK;
  DeviceGuard guard(enc->device);
  cudaStream_t s = (cudaStream_t)stream;
  const size_t tok_n = (size_t)n_seqs * seq_len;
  if (flags & LV_IO_DEVICE)
    return encode_node_rows(enc, tokens, token_bytes, seq_len, nullptr, n_seqs, out, s);
  // host tokens: validate ids (the reference raises on bad payloads), stage, encode, copy back
  for (size_t i = 0; i < tok_n; ++i) {
    uint32_t t = token_bytes == 2 ? ((const uint16_t *)tokens)[i] : ((const uint32_t *)tokens)[i];
    LV_REQUIRE(t < (uint32_t)enc->cfg.vocab, LV_ERR_DATA, "token id out of vocabulary");
  }
  void *dt = nullptr;
  float *dout = nullptr;
  LV_CHECK_CUDA(cudaMalloc(&dt, tok_n * token_bytes));
  if (cudaMalloc(&dout, (size_t)n_seqs * enc->cfg.hidden * 4) != cudaSuccess) {
    cudaFree(dt);
    set_error("cudaMalloc failed");
    return LV_ERR_INTERNAL;
  }
  int rc = LV_OK;
  if (cudaMemcpyAsync(dt, tokens, tok_n * token_bytes, cudaMemcpyHostToDevice, s) != cudaSuccess)
    rc = LV_ERR_INTERNAL;
  if (rc == LV_OK) rc = encode_node_rows(enc, dt, token_bytes, seq_len, nullptr, n_seqs, dout, s);
  if (rc == LV_OK &&
      cudaMemcpyAsync(out, dout, (size_t)n_seqs * enc->cfg.hidden * 4, cudaMemcpyDeviceToHost,
                      s) != cudaSuccess)
    rc = LV_ERR_INTERNAL;
  if (cudaStreamSynchronize(s) != cudaSuccess && rc == LV_OK) {
    set_error(std::string("encoder failed: ") + cudaGetErrorString(cudaGetLastError()));
    rc = LV_ERR_INTERNAL;
  }
  cudaFree(dt);
  cudaFree(dout);
  return rc;
}

int lv_gemm_bf16(const void *A, const void *W, const float *bias, const void *residual, void *out,
                 int32_t M, int32_t N, int32_t K, int32_t epi, void *stream) {
  LV_REQUIRE(A && W && bias && out, LV_ERR_USAGE, "lv_gemm_bf16: null argument");
  LV_REQUIRE(epi >= 0 && epi <= 2, LV_ERR_USAGE, "lv_gemm_bf16: unknown epilogue");
  return tc_gemm((const __nv_bfloat16 *)A, (const __nv_bfloat16 *)W, bias,
                 (const __nv_bfloat16 *)residual, (__nv_bfloat16 *)out, M, N, K, epi,
                 (cudaStream_t)stream);
}

int lv_attention_bf16(const void *qkv, void *out, int32_t n_seqs, int32_t S, int32_t H,
                      int32_t dh, void *stream) {
  LV_REQUIRE(qkv && out, LV_ERR_USAGE, "lv_attention_bf16: null argument");
  LV_REQUIRE(S % 64 == 0 && (dh == 64 || dh == 128), LV_ERR_USAGE,
             "lv_attention_bf16: need S % 64 == 0 and dh in {64, 128}");
  LV_CHECK_CUDA(attention_bf16((const __nv_bfloat16 *)qkv, (__nv_bfloat16 *)out, n_seqs, S, H, dh,
                               (cudaStream_t)stream));
  return LV_OK;
}

int lv_attention_gqa_bf16(const void *qkv, void *out, int32_t n_seqs, int32_t S, int32_t Hq,
                          int32_t Hkv, int32_t dh, int32_t causal, void *stream) {
  LV_REQUIRE(qkv && out, LV_ERR_USAGE, "lv_attention_gqa_bf16: null argument");
  LV_REQUIRE(S % 64 == 0 && (dh == 64 || dh == 128) && Hkv >= 1 && Hq % Hkv == 0, LV_ERR_USAGE,
             "lv_attention_gqa_bf16: need S % 64 == 0, dh in {64, 128}, Hq % Hkv == 0");
  LV_CHECK_CUDA(attention_gqa_bf16((const __nv_bfloat16 *)qkv, (__nv_bfloat16 *)out, n_seqs, S, Hq,
                                   Hkv, dh, causal != 0, (cudaStream_t)stream));
  return LV_OK;
}

int lv_set_gemm_mode(int mode) {
  const int prev = g_gemm_mode | (g_long_k_single ? 0 : 4) | (g_split_single ? 8 : 0);
  g_gemm_mode = mode & 1;
  g_long_k_single = (mode & 4) ? 0 : 1;
  g_split_single = (mode & 8) ? 1 : 0;
  return prev;
}

int lv_encoder_set_split_residual(lv_encoder *enc, int enable) {
  LV_REQUIRE(enc, LV_ERR_USAGE, "null encoder");
  enc->split_res = enable != 0;
  return LV_OK;
}

int lv_encoder_set_fused_ln(lv_encoder *enc, int enable) {
  LV_REQUIRE(enc, LV_ERR_USAGE, "null encoder");
  const bool can = enc->cfg.precision == 1 &&
                   ((!enc->layers.empty() && enc->layers[0].w_1_f) ||
                    (!enc->dec.empty() && enc->dec[0].w_qkv_f));
  LV_REQUIRE(!enable || can, LV_ERR_USAGE,
             "fused LayerNorm needs the bf16 encoder with hidden, ffn % 256 == 0");
  enc->fuse_ln = enable != 0;
  return LV_OK;
}

int lv_set_fused_qkv_attention(int enable) {
  const int prev = g_fuse_qkv_attn;
  g_fuse_qkv_attn = enable != 0;
  return prev;
}

int lv_set_attention_mode(int mode) {
  const int prev = g_attn_mode;
  g_attn_mode = mode;
  return prev;
}

int lv_encoder_profile(lv_encoder *enc, int enable) {
  LV_REQUIRE(enc, LV_ERR_USAGE, "null encoder");
  enc->profile = enable != 0;
  return LV_OK;
}

int lv_encoder_stats(lv_encoder *enc, lv_encoder_stats_t *st) {
  LV_REQUIRE(enc && st, LV_ERR_USAGE, "null argument");
  DeviceGuard guard(enc->device);
  cudaDeviceSynchronize();
  encoder_collect_profile(enc);
  st->passages = enc->passages;
  st->gemm_launches = enc->gemm_launches;
  st->gemm_ms = enc->gemm_ms;
  st->gemm_flops = enc->gemm_flops;
  st->gemm_bytes = enc->gemm_bytes;
  st->attn_launches = enc->attn_launches;
  st->attn_ms = enc->attn_ms;
  st->attn_flops = enc->attn_flops;
  st->attn_bytes = enc->attn_bytes;
  st->fused_launches = enc->fused_launches;
  st->fused_ms = enc->fused_ms;
  st->fused_flops = enc->fused_flops;
  st->fused_bytes = enc->fused_bytes;
  return LV_OK;
}

int lv_encoder_reset_stats(lv_encoder *enc) {
  LV_REQUIRE(enc, LV_ERR_USAGE, "null encoder");
  DeviceGuard guard(enc->device);
  cudaDeviceSynchronize();
  encoder_collect_profile(enc);
  enc->passages = 0;
  enc->gemm_launches = 0;
  enc->gemm_ms = 0.0;
  enc->gemm_flops = 0.0;
  enc->gemm_bytes = 0.0;
  enc->attn_launches = 0;
  enc->attn_ms = enc->attn_flops = enc->attn_bytes = 0.0;
  enc->fused_launches = 0;
  enc->fused_ms = enc->fused_flops = enc->fused_bytes = 0.0;
  return LV_OK;
}

}  // extern "C"
