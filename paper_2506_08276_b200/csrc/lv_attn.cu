// lv_attn.cu — bidirectional multi-head attention of the passage encoder.
//
// Each passage is an independent sequence (no padding: every chunk of the
// token store holds exactly seq_len ids), so one CTA owns one (sequence,
// head) pair and the whole K/V of that head fits in shared memory.
//
//   attention_bf16: flash-style, scores and P.V on tensor cores (mma.sync
//     m16n8k16 bf16 -> fp32, fragments via ldmatrix / ldmatrix.trans), online
//     softmax in fp32 registers; Q/K/V staged with cp.async. Attention is ~5% of the encoder FLOPs at S <= 512 (the GEMMs in
//     lv_gemm_tc.cu carry the rest).
//   attention_f32: parity-mode reference path (one warp per query row, fixed
//     summation order), used by the fp32 encoder.
#include <cfloat>

#include "lv_kernels.cuh"

namespace lv {
namespace {

constexpr unsigned kFull = 0xffffffffu;

__device__ __forceinline__ void mma_bf16_16816(float (&c)[4], const uint32_t (&a)[4], uint32_t b0,
                                               uint32_t b1) {
  asm volatile(
      "mma.sync.aligned.m16n8k16.row.col.f32.bf16.bf16.f32 {%0,%1,%2,%3}, {%4,%5,%6,%7}, "
      "{%8,%9}, {%0,%1,%2,%3};"
      : "+f"(c[0]), "+f"(c[1]), "+f"(c[2]), "+f"(c[3])
      : "r"(a[0]), "r"(a[1]), "r"(a[2]), "r"(a[3]), "r"(b0), "r"(b1));
}

__device__ __forceinline__ uint32_t pack2(float a, float b) {
  __nv_bfloat162 h = __floats2bfloat162_rn(a, b);
  return *reinterpret_cast<uint32_t *>(&h);
}

__device__ __forceinline__ void cp_async16(void *smem, const void *gmem) {
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"(
                   (uint32_t)__cvta_generic_to_shared(smem)),
               "l"(gmem)
               : "memory");
}
__device__ __forceinline__ void ldsm_x4(uint32_t (&r)[4], const void *p) {
  asm volatile("ldmatrix.sync.aligned.m8n8.x4.shared.b16 {%0,%1,%2,%3}, [%4];"
               : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3])
               : "r"((uint32_t)__cvta_generic_to_shared(p)));
}
__device__ __forceinline__ void ldsm_x4_t(uint32_t (&r)[4], const void *p) {
  asm volatile("ldmatrix.sync.aligned.m8n8.x4.trans.shared.b16 {%0,%1,%2,%3}, [%4];"
               : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3])
               : "r"((uint32_t)__cvta_generic_to_shared(p)));
}

// One CTA per (sequence, head). Q, K, V of the head are staged with 16-byte
// cp.async into row-major shared memory padded to DH + 8 elements (row stride
// = 16 * odd bytes, so the 8 rows of every ldmatrix 8x8 tile hit distinct bank
// groups). Fragments come from ldmatrix.x4 (Q as A, K as B) and
// ldmatrix.x4.trans (V as B of P.V), so no transposing stores are needed.
template <int DH>
__global__ void __launch_bounds__(256, DH == 64 ? 2 : 1) attn_bf16_kernel(const __nv_bfloat16 *__restrict__ qkv,
                                                            __nv_bfloat16 *__restrict__ out,
                                                            int S, int H, float scale_log2) {
  extern __shared__ __align__(16) uint8_t smem[];
  constexpr int LD = DH + 8;
  __nv_bfloat16 *Qs = reinterpret_cast<__nv_bfloat16 *>(smem);
  __nv_bfloat16 *Ks = Qs + S * LD;
  __nv_bfloat16 *Vs = Ks + S * LD;
  const int seq = blockIdx.x / H, h = blockIdx.x % H;
  const int D = H * DH;
  const size_t row0 = (size_t)seq * S;
  const __nv_bfloat16 *base = qkv + row0 * 3 * D + h * DH;
  constexpr int kVec = DH / 8;
  for (int i = threadIdx.x; i < S * kVec; i += blockDim.x) {
    const int j = i / kVec, c = (i % kVec) * 8;
    const __nv_bfloat16 *rp = base + (size_t)j * 3 * D + c;
    cp_async16(Qs + j * LD + c, rp);
    cp_async16(Ks + j * LD + c, rp + D);
    cp_async16(Vs + j * LD + c, rp + 2 * D);
  }
  asm volatile("cp.async.commit_group;\ncp.async.wait_group 0;" ::: "memory");
  __syncthreads();

  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int g = lane >> 2, t = lane & 3;
  const int nwarps = blockDim.x >> 5;
  const int lr = lane & 7, lm = lane >> 3;  // ldmatrix: row within tile, tile index
  for (int rb = warp; rb < S / 16; rb += nwarps) {
    const int r0 = rb * 16;
    uint32_t qa[DH / 16][4];
#pragma unroll
    for (int ks = 0; ks < DH / 16; ++ks)
      ldsm_x4(qa[ks], Qs + (r0 + (lane & 15)) * LD + ks * 16 + (lane >> 4) * 8);
    float o[DH / 8][4];
#pragma unroll
    for (int i = 0; i < DH / 8; ++i) o[i][0] = o[i][1] = o[i][2] = o[i][3] = 0.f;
    float m0 = -FLT_MAX, m1 = -FLT_MAX, l0 = 0.f, l1 = 0.f;
    for (int kv0 = 0; kv0 < S; kv0 += 64) {
      float s[8][4];
#pragma unroll
      for (int nt = 0; nt < 8; ++nt) s[nt][0] = s[nt][1] = s[nt][2] = s[nt][3] = 0.f;
#pragma unroll
      for (int np = 0; np < 4; ++np) {      // pairs of 8-key n-tiles
#pragma unroll
        for (int ks = 0; ks < DH / 16; ++ks) {
          uint32_t b[4];  // tiles: (keys +0..7, dims +0..7), (+0..7, +8..15), (+8..15, +0..7), (+8..15, +8..15)
          ldsm_x4(b, Ks + (kv0 + np * 16 + (lm >> 1) * 8 + lr) * LD + ks * 16 + (lm & 1) * 8);
          mma_bf16_16816(s[2 * np], qa[ks], b[0], b[1]);
          mma_bf16_16816(s[2 * np + 1], qa[ks], b[2], b[3]);
        }
      }
      float mx0 = m0, mx1 = m1;
#pragma unroll
      for (int nt = 0; nt < 8; ++nt) {
        mx0 = fmaxf(mx0, fmaxf(s[nt][0], s[nt][1]));
        mx1 = fmaxf(mx1, fmaxf(s[nt][2], s[nt][3]));
      }
      mx0 = fmaxf(mx0, __shfl_xor_sync(kFull, mx0, 1));
      mx0 = fmaxf(mx0, __shfl_xor_sync(kFull, mx0, 2));
      mx1 = fmaxf(mx1, __shfl_xor_sync(kFull, mx1, 1));
      mx1 = fmaxf(mx1, __shfl_xor_sync(kFull, mx1, 2));
      const float c0 = exp2f((m0 - mx0) * scale_log2), c1 = exp2f((m1 - mx1) * scale_log2);
      m0 = mx0;
      m1 = mx1;
      const float sm0 = mx0 * scale_log2, sm1 = mx1 * scale_log2;
      l0 *= c0;
      l1 *= c1;
#pragma unroll
      for (int i = 0; i < DH / 8; ++i) {
        o[i][0] *= c0;
        o[i][1] *= c0;
        o[i][2] *= c1;
        o[i][3] *= c1;
      }
      uint32_t pa[4][4];
#pragma unroll
      for (int nt = 0; nt < 8; ++nt) {
        float p0 = exp2f(fmaf(s[nt][0], scale_log2, -sm0));
        float p1 = exp2f(fmaf(s[nt][1], scale_log2, -sm0));
        float p2 = exp2f(fmaf(s[nt][2], scale_log2, -sm1));
        float p3 = exp2f(fmaf(s[nt][3], scale_log2, -sm1));
        l0 += p0 + p1;
        l1 += p2 + p3;
        const int j = nt >> 1, hi = nt & 1;
        pa[j][hi ? 2 : 0] = pack2(p0, p1);
        pa[j][hi ? 3 : 1] = pack2(p2, p3);
      }
#pragma unroll
      for (int j = 0; j < 4; ++j) {          // 16-key k-steps
#pragma unroll
        for (int dp = 0; dp < DH / 16; ++dp) {  // pairs of 8-dim n-tiles
          uint32_t b[4];  // tiles (keys +0..7, dims +0..7), (+8..15, +0..7), (+0..7, +8..15), (+8..15, +8..15)
          ldsm_x4_t(b, Vs + (kv0 + j * 16 + (lm & 1) * 8 + lr) * LD + dp * 16 + (lm >> 1) * 8);
          mma_bf16_16816(o[2 * dp], pa[j], b[0], b[1]);
          mma_bf16_16816(o[2 * dp + 1], pa[j], b[2], b[3]);
        }
      }
    }
    l0 += __shfl_xor_sync(kFull, l0, 1);
    l0 += __shfl_xor_sync(kFull, l0, 2);
    l1 += __shfl_xor_sync(kFull, l1, 1);
    l1 += __shfl_xor_sync(kFull, l1, 2);
    const float i0 = 1.f / l0, i1 = 1.f / l1;
    __nv_bfloat16 *o0 = out + (row0 + r0 + g) * D + h * DH;
    __nv_bfloat16 *o1 = o0 + (size_t)8 * D;
#pragma unroll
    for (int nt = 0; nt < DH / 8; ++nt) {
      *reinterpret_cast<uint32_t *>(o0 + nt * 8 + 2 * t) = pack2(o[nt][0] * i0, o[nt][1] * i0);
      *reinterpret_cast<uint32_t *>(o1 + nt * 8 + 2 * t) = pack2(o[nt][2] * i1, o[nt][3] * i1);
    }
  }
}


// fp32 reference-order attention: one warp per (sequence, head, query row).
__global__ void attn_f32_kernel(const float *__restrict__ qkv, float *__restrict__ out, int n_seqs,
                                int S, int H, int dh, float scale) {
  extern __shared__ float sm[];
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int nw = blockDim.x >> 5;
  float *qv = sm + warp * (dh + S);
  float *sc = qv + dh;
  const long long item = (long long)blockIdx.x * nw + warp;
  const long long total = (long long)n_seqs * H * S;
  if (item >= total) return;
  const int r = (int)(item % S);
  const int h = (int)((item / S) % H);
  const long long seq = item / ((long long)S * H);
  const int D = H * dh;
  const float *base = qkv + (size_t)seq * S * 3 * D;
  for (int d = lane; d < dh; d += 32) qv[d] = base[(size_t)r * 3 * D + h * dh + d];
  __syncwarp();
  float mx = -FLT_MAX;
  for (int j = lane; j < S; j += 32) {
    const float *kr = base + (size_t)j * 3 * D + D + h * dh;
    float acc = 0.f;
    for (int d = 0; d < dh; ++d) acc = fmaf(qv[d], __ldg(kr + d), acc);
    acc *= scale;
    sc[j] = acc;
    mx = fmaxf(mx, acc);
  }
  for (int o = 16; o; o >>= 1) mx = fmaxf(mx, __shfl_xor_sync(kFull, mx, o));
  float sum = 0.f;
  for (int j = lane; j < S; j += 32) {
    float p = expf(sc[j] - mx);
    sc[j] = p;
    sum += p;
  }
  for (int o = 16; o; o >>= 1) sum += __shfl_xor_sync(kFull, sum, o);
  __syncwarp();
  const float inv = 1.f / sum;
  for (int d = lane; d < dh; d += 32) {
    float acc = 0.f;
    const float *vc = base + 2 * D + h * dh + d;
    for (int j = 0; j < S; ++j) acc = fmaf(sc[j], __ldg(vc + (size_t)j * 3 * D), acc);
    out[((size_t)seq * S + r) * D + h * dh + d] = acc * inv;
  }
}

}  // namespace

cudaError_t attention_bf16(const __nv_bfloat16 *qkv, __nv_bfloat16 *out, int n_seqs, int S, int H,
                           int dh, cudaStream_t s) {
  if (n_seqs <= 0) return cudaSuccess;
  if (S % 64 != 0 || dh % 16 != 0) return cudaErrorInvalidValue;
  const size_t smem = (size_t)3 * S * (dh + 8) * 2;
  const int threads = std::min(256, std::max(32, (S / 16) * 32));
  const float scale_log2 = 1.4426950408889634f / sqrtf((float)dh);
  cudaError_t e;
  if (dh == 64) {
    e = cudaFuncSetAttribute(attn_bf16_kernel<64>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                             (int)smem);
    if (e != cudaSuccess) return e;
    attn_bf16_kernel<64><<<n_seqs * H, threads, smem, s>>>(qkv, out, S, H, scale_log2);
    note_launch();
  } else if (dh == 128) {
    e = cudaFuncSetAttribute(attn_bf16_kernel<128>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                             (int)smem);
    if (e != cudaSuccess) return e;
    attn_bf16_kernel<128><<<n_seqs * H, threads, smem, s>>>(qkv, out, S, H, scale_log2);
    note_launch();
  } else {
    return cudaErrorInvalidValue;
  }
  return cudaGetLastError();
}

cudaError_t attention_f32(const float *qkv, float *out, int n_seqs, int S, int H, int dh,
                          cudaStream_t s) {
  if (n_seqs <= 0) return cudaSuccess;
  const int warps = 8;
  const size_t smem = (size_t)warps * (dh + S) * 4;
  const long long items = (long long)n_seqs * H * S;
  cudaError_t e = cudaFuncSetAttribute(attn_f32_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                       (int)smem);
  if (e != cudaSuccess) return e;
  attn_f32_kernel<<<(unsigned)((items + warps - 1) / warps), warps * 32, smem, s>>>(
      qkv, out, n_seqs, S, H, dh, 1.0f / sqrtf((float)dh));
      note_launch();
  return cudaGetLastError();
}

}  // namespace lv
