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
#include "lv_tc.cuh"

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


// ---------------------------------------------------------------------------
// attn_tc_kernel: the same attention on the 5th-gen tensor cores.
//
// Work item = one (sequence, head); S in {128, 256}, dh = 64. Persistent, one
// CTA per SM, warp-specialised:
//   warp 0      TMA: Q, K, V of an item ([S][64] bf16 boxes of the qkv rows,
//               128-byte swizzle) into a 2-stage shared-memory ring;
//   warp 1      one lane issues tcgen05.mma: per 128-row Q tile t,
//                 S_t = Q_t . K^T   (SS, M=128, N=S, K=64)   -> TMEM region r
//                 O_t = P_t . V     (TS, M=128, N=64, K=S)   -> same region
//               with P_t read from TMEM (A operand) and V as an MN-major
//               shared-memory operand (no transpose anywhere);
//   warps 2-9   two softmax groups of 4 warps (group r owns TMEM region r =
//               256 columns; tiles alternate between the groups so the MMA of
//               one tile overlaps the softmax of the other). A thread owns one
//               query row: pass 1 row max over S columns, pass 2
//               p = 2^(s*c - max*c) (MUFU ex2), row sum in fp32, P packed to
//               bf16 and written back over the consumed score columns
//               (tcgen05.st); after the P.V MMA it reads O, scales by 1/sum and
//               stores its 128-byte head slice of the context row.
// No mask (every passage is exactly S tokens) and no online rescaling (a row
// of scores fits in TMEM). Batch-invariant: each item is a fixed-order
// computation independent of the launch.
namespace atc {
constexpr int kThreads = 64 + 8 * 32;
template <int S>
struct Cfg {
  static constexpr int kTileBytes = S * 128;  // [S][64] bf16
  static constexpr int kStageBytes = 3 * kTileBytes;
  static constexpr int kStages = 2;
  static constexpr int kQTiles = S / 128;
  static constexpr int kSmem = kStages * kStageBytes + 1024 + 256;
};
}  // namespace atc

__device__ __forceinline__ float ex2_approx(float x) {
  float y;
  asm("ex2.approx.ftz.f32 %0, %1;" : "=f"(y) : "f"(x));
  return y;
}

template <int S>
__global__ void __launch_bounds__(atc::kThreads, 1)
    attn_tc_kernel(const __grid_constant__ CUtensorMap tm, __nv_bfloat16 *__restrict__ out,
                   int n_items, int H, float scale_log2) {
  using namespace tc;
  using C = atc::Cfg<S>;
  extern __shared__ uint8_t smem_raw[];
  uint8_t *smem = smem_raw + ((1024u - (tc::smem_u32(smem_raw) & 1023u)) & 1023u);  // 1 KB aligned, still shared space
  // Q|K and V of a stage have separate full/empty barriers: Q and K are free
  // once the item's last Q.K^T MMA completes, so the next item's Q|K load
  // starts a softmax earlier than a per-stage release would allow
  uint64_t *full = reinterpret_cast<uint64_t *>(smem + C::kStages * C::kStageBytes);  // Q|K
  uint64_t *empty = full + 2;
  uint64_t *full_v = empty + 2;
  uint64_t *empty_v = full_v + 2;
  uint64_t *s_full = empty_v + 2;
  uint64_t *p_full = s_full + 2;
  uint64_t *o_full = p_full + 2;
  uint64_t *r_free = o_full + 2;
  uint32_t *tslot = reinterpret_cast<uint32_t *>(r_free + 2);

  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  if (threadIdx.x == 0) {
    for (int i = 0; i < 2; ++i) {
      mbar_init(&full[i], 1);
      mbar_init(&empty[i], 1);
      mbar_init(&full_v[i], 1);
      mbar_init(&empty_v[i], 1);
      mbar_init(&s_full[i], 1);
      mbar_init(&p_full[i], 4);
      mbar_init(&o_full[i], 1);
      mbar_init(&r_free[i], 4);
    }
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  if (warp == 1) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(
                     smem_u32(tslot)),
                 "r"(512));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
  }
  fence_before();
  __syncthreads();
  fence_after();
  const uint32_t tmem = *tslot;
  const int D = H * 64;
  const int n_local = n_items > (int)blockIdx.x
                          ? (n_items - (int)blockIdx.x + (int)gridDim.x - 1) / (int)gridDim.x
                          : 0;
  const int total = n_local * C::kQTiles;  // Q tiles this CTA processes

  if (warp == 0) {
    if (lane == 0) {
      asm volatile("prefetch.tensormap [%0];" ::"l"(&tm) : "memory");
      uint64_t pol;
      asm volatile("createpolicy.fractional.L2::evict_first.b64 %0, 1.0;" : "=l"(pol));
      for (int i = 0; i < n_local; ++i) {
        const int st = i & 1;
        mbar_wait(&empty[st], ((i >> 1) & 1) ^ 1);
        const int item = (int)blockIdx.x + i * (int)gridDim.x;
        const int seq = item / H, h = item - seq * H;
        uint8_t *base = smem + st * C::kStageBytes;
        mbar_expect_tx(&full[st], 2 * C::kTileBytes);
        tma_load_2d(base, &tm, &full[st], h * 64, seq * S, pol);
        tma_load_2d(base + C::kTileBytes, &tm, &full[st], D + h * 64, seq * S, pol);
        mbar_wait(&empty_v[st], ((i >> 1) & 1) ^ 1);
        mbar_expect_tx(&full_v[st], C::kTileBytes);
        tma_load_2d(base + 2 * C::kTileBytes, &tm, &full_v[st], 2 * D + h * 64, seq * S, pol);
      }
    }
  } else if (warp == 1) {
    if (lane == 0) {
      constexpr uint32_t idesc_s = idesc_bf16(128, S);
      constexpr uint32_t idesc_o = idesc_bf16(128, 64, true);
      auto issue_s = [&](int j) {
        const int i = j / C::kQTiles, t = j % C::kQTiles, r = j & 1;
        if (t == 0) mbar_wait(&full[i & 1], (i >> 1) & 1);
        mbar_wait(&r_free[r], ((j >> 1) & 1) ^ 1);
        fence_after();
        const uint8_t *base = smem + (i & 1) * C::kStageBytes;
        const uint64_t a = sw128_desc(smem_u32(base + t * 128 * 128));
        const uint64_t b = sw128_desc(smem_u32(base + C::kTileBytes));
#pragma unroll
        for (int k = 0; k < 4; ++k) umma_ss(tmem + r * 256, a + 2 * k, b + 2 * k, idesc_s, k);
        umma_commit(&s_full[r]);
        if (t == C::kQTiles - 1) umma_commit(&empty[i & 1]);  // Q|K of the stage consumed
      };
      auto issue_pv = [&](int j) {
        const int i = j / C::kQTiles, t = j % C::kQTiles, r = j & 1;
        if (t == 0) mbar_wait(&full_v[i & 1], (i >> 1) & 1);
        mbar_wait(&p_full[r], (j >> 1) & 1);
        fence_after();
        const uint8_t *base = smem + (i & 1) * C::kStageBytes;
        const uint64_t v = sw128_desc(smem_u32(base + 2 * C::kTileBytes), 1024, 16);
#pragma unroll
        for (int k = 0; k < S / 16; ++k)  // 16 keys = 2 swizzle atoms (2048 B) of V per step
          umma_ts(tmem + r * 256 + S / 2, tmem + r * 256 + 8 * k, v + (uint64_t)(128 * k), idesc_o,
                  k);
        umma_commit(&o_full[r]);
        if (t == C::kQTiles - 1) umma_commit(&empty_v[i & 1]);
      };
      if (total > 0) issue_s(0);
      if (total > 1) issue_s(1);
      for (int j = 0; j < total; ++j) {
        issue_pv(j);
        if (j + 2 < total) issue_s(j + 2);
      }
    }
  } else {
    const int g = (warp - 2) >> 2;  // softmax group = TMEM region
    const int q = warp & 3;         // TMEM lane quarter
    const uint32_t tb = tmem + ((uint32_t)(q * 32) << 16) + (uint32_t)(g * 256);
    for (int j = g; j < total; j += 2) {
      const uint32_t ph = (uint32_t)(j >> 1) & 1;
      mbar_wait(&s_full[g], ph);
      fence_after();
      // pass 1: row max
      float mx = -FLT_MAX;
#pragma unroll 1
      for (int c = 0; c < S / 32; c += 2) {
        uint32_t r0[32], r1[32];
        tmem_ld32_nowait(tb + 32 * c, r0);
        tmem_ld32_nowait(tb + 32 * c + 32, r1);
        tmem_ld_wait();
#pragma unroll
        for (int e = 0; e < 32; ++e)
          mx = fmaxf(mx, fmaxf(__uint_as_float(r0[e]), __uint_as_float(r1[e])));
      }
      const float mc = mx * scale_log2;
      // pass 2: p = 2^(s*c - max*c), row sum, P (bf16) over the consumed columns
      // the row sum is kept as two halves (columns [0, S/2) and [S/2, S)) added at
      // the end: the order the fused QKV + attention kernel (lv_qkv_attn.cu), whose
      // two warps per row each own one half, reproduces bit for bit
      float sum_a = 0.f, sum = 0.f;
#pragma unroll 1
      for (int c = 0; c < S / 32; ++c) {
        if (c == S / 64) {
          sum_a = sum;
          sum = 0.f;
        }
        uint32_t r0[32];
        tmem_ld32(tb + 32 * c, r0);
        uint32_t w[16];
#pragma unroll
        for (int e = 0; e < 16; ++e) {
          const float x0 = fmaf(__uint_as_float(r0[2 * e]), scale_log2, -mc);
          const float x1 = fmaf(__uint_as_float(r0[2 * e + 1]), scale_log2, -mc);
          const float p0 = ex2_approx(x0);
          const float p1 = ex2_approx(x1);
          sum += p0 + p1;
          w[e] = pack_bf16(p0, p1);
        }
        tmem_st16(tb + 16 * c, w);
      }
      sum = sum_a + sum;
      tmem_st_wait();
      fence_before();
      __syncwarp();
      if (lane == 0) mbar_arrive(&p_full[g]);
      // epilogue: O / sum -> context row slice
      const int i = j / C::kQTiles, t = j % C::kQTiles;
      const int item = (int)blockIdx.x + i * (int)gridDim.x;
      const int seq = item / H, h = item - seq * H;
      const size_t row = (size_t)seq * S + t * 128 + q * 32 + lane;
      mbar_wait(&o_full[g], ph);
      fence_after();
      uint32_t o0[32], o1[32];
      tmem_ld32_nowait(tb + S / 2, o0);
      tmem_ld32_nowait(tb + S / 2 + 32, o1);
      tmem_ld_wait();
      fence_before();
      __syncwarp();
      if (lane == 0) mbar_arrive(&r_free[g]);
      const float inv = 1.f / sum;
      uint4 *op = reinterpret_cast<uint4 *>(out + row * D + h * 64);
#pragma unroll
      for (int v = 0; v < 4; ++v) {
        uint4 u;
        u.x = pack_bf16(__uint_as_float(o0[8 * v + 0]) * inv, __uint_as_float(o0[8 * v + 1]) * inv);
        u.y = pack_bf16(__uint_as_float(o0[8 * v + 2]) * inv, __uint_as_float(o0[8 * v + 3]) * inv);
        u.z = pack_bf16(__uint_as_float(o0[8 * v + 4]) * inv, __uint_as_float(o0[8 * v + 5]) * inv);
        u.w = pack_bf16(__uint_as_float(o0[8 * v + 6]) * inv, __uint_as_float(o0[8 * v + 7]) * inv);
        op[v] = u;
      }
#pragma unroll
      for (int v = 0; v < 4; ++v) {
        uint4 u;
        u.x = pack_bf16(__uint_as_float(o1[8 * v + 0]) * inv, __uint_as_float(o1[8 * v + 1]) * inv);
        u.y = pack_bf16(__uint_as_float(o1[8 * v + 2]) * inv, __uint_as_float(o1[8 * v + 3]) * inv);
        u.z = pack_bf16(__uint_as_float(o1[8 * v + 4]) * inv, __uint_as_float(o1[8 * v + 5]) * inv);
        u.w = pack_bf16(__uint_as_float(o1[8 * v + 6]) * inv, __uint_as_float(o1[8 * v + 7]) * inv);
        op[4 + v] = u;
      }
    }
  }
  fence_before();
  __syncthreads();
  if (warp == 1) {
    fence_after();
    asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem), "r"(512));
  }
}

template <int S>
cudaError_t launch_attn_tc(const __nv_bfloat16 *qkv, __nv_bfloat16 *out, int n_seqs, int H,
                           cudaStream_t s) {
  using C = atc::Cfg<S>;
  CUtensorMap tm;
  const uint64_t D3 = (uint64_t)3 * H * 64;
  if (!make_tma_2d_bf16(&tm, qkv, D3, (uint64_t)n_seqs * S, D3 * 2, 64, S))
    return cudaErrorInvalidValue;
  static unsigned long long attr = 0;  // per device (first_on_device)
  if (first_on_device(attr)) {
    cudaError_t e = cudaFuncSetAttribute(attn_tc_kernel<S>,
                                         cudaFuncAttributeMaxDynamicSharedMemorySize, C::kSmem);
    if (e != cudaSuccess) return e;
  }
  const int items = n_seqs * H;
  const int grid = std::min(items, tc_gemm_num_sms());
  attn_tc_kernel<S><<<grid, atc::kThreads, C::kSmem, s>>>(tm, out, items, H,
                                                                 1.4426950408889634f / 8.0f);
  note_launch();
  return cudaGetLastError();
}


// ---------------------------------------------------------------------------
// attn_flash_kernel: grouped-query attention with an optional causal mask for
// the decoder-style (Qwen3-shaped, config-4) encoder: q heads Hq, k/v heads
// Hkv (q head h reads k/v head h / (Hq / Hkv)), head dim DH in {64, 128}, any
// S % 64 == 0 (S = 512 at config-4 does not fit shared memory whole, so K/V
// stream through a 2-stage cp.async ring of 64-key blocks with an online
// softmax). Row layout of qkv: [q heads | k heads | v heads] x DH.
// One CTA = 64 query rows of one (sequence, q head), 4 warps x 16 rows;
// tensor-core math as attn_bf16_kernel (mma.sync m16n8k16, ldmatrix).
template <int DH, bool CAUSAL>
__global__ void __launch_bounds__(128) attn_flash_kernel(const __nv_bfloat16 *__restrict__ qkv,
                                                         __nv_bfloat16 *__restrict__ out, int S,
                                                         int Hq, int Hkv, float scale_log2) {
  extern __shared__ __align__(16) uint8_t smem[];
  constexpr int LD = DH + 8;
  constexpr int kVec = DH / 8;
  __nv_bfloat16 *Qs = reinterpret_cast<__nv_bfloat16 *>(smem);
  __nv_bfloat16 *Ks = Qs + 64 * LD;       // [2][64][LD]
  __nv_bfloat16 *Vs = Ks + 2 * 64 * LD;   // [2][64][LD]
  // causal: the longest rows (last q blocks) are scheduled first for a short tail
  const int qb = CAUSAL ? (int)gridDim.x - 1 - (int)blockIdx.x : (int)blockIdx.x;
  const int seq = blockIdx.y / Hq, h = blockIdx.y % Hq, g = h / (Hq / Hkv);
  const int RS = (Hq + 2 * Hkv) * DH;
  const size_t row0 = (size_t)seq * S;
  const __nv_bfloat16 *qbase = qkv + row0 * RS + h * DH;
  const __nv_bfloat16 *kbase = qkv + row0 * RS + (Hq + g) * DH;
  const __nv_bfloat16 *vbase = qkv + row0 * RS + (Hq + Hkv + g) * DH;
  for (int i = threadIdx.x; i < 64 * kVec; i += blockDim.x) {
    const int j = i / kVec, c = (i % kVec) * 8;
    cp_async16(Qs + j * LD + c, qbase + (size_t)(qb * 64 + j) * RS + c);
  }
  auto load_kv = [&](int kb, int st) {
    for (int i = threadIdx.x; i < 64 * kVec; i += blockDim.x) {
      const int j = i / kVec, c = (i % kVec) * 8;
      const size_t r = (size_t)(kb * 64 + j) * RS + c;
      cp_async16(Ks + (st * 64 + j) * LD + c, kbase + r);
      cp_async16(Vs + (st * 64 + j) * LD + c, vbase + r);
    }
  };
  const int nkv = CAUSAL ? qb + 1 : S / 64;
  load_kv(0, 0);
  asm volatile("cp.async.commit_group;" ::: "memory");

  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int gq = lane >> 2, t = lane & 3;
  const int lr = lane & 7, lm = lane >> 3;
  const int r0 = warp * 16;                 // this warp's rows within the block
  const int qrow0 = qb * 64 + r0 + gq;      // query index of accumulator rows c[0..1]
  uint32_t qa[DH / 16][4];
  float o[DH / 8][4];
#pragma unroll
  for (int i = 0; i < DH / 8; ++i) o[i][0] = o[i][1] = o[i][2] = o[i][3] = 0.f;
  float m0 = -FLT_MAX, m1 = -FLT_MAX, l0 = 0.f, l1 = 0.f;
  for (int kb = 0; kb < nkv; ++kb) {
    const int st = kb & 1;
    if (kb + 1 < nkv) load_kv(kb + 1, st ^ 1);
    asm volatile("cp.async.commit_group;" ::: "memory");
    asm volatile("cp.async.wait_group 1;" ::: "memory");
    __syncthreads();
    if (kb == 0) {
#pragma unroll
      for (int ks = 0; ks < DH / 16; ++ks)
        ldsm_x4(qa[ks], Qs + (r0 + (lane & 15)) * LD + ks * 16 + (lane >> 4) * 8);
    }
    const __nv_bfloat16 *Kb = Ks + st * 64 * LD, *Vb = Vs + st * 64 * LD;
    float sc[8][4];
#pragma unroll
    for (int nt = 0; nt < 8; ++nt) sc[nt][0] = sc[nt][1] = sc[nt][2] = sc[nt][3] = 0.f;
#pragma unroll
    for (int np = 0; np < 4; ++np) {
#pragma unroll
      for (int ks = 0; ks < DH / 16; ++ks) {
        uint32_t b[4];
        ldsm_x4(b, Kb + (np * 16 + (lm >> 1) * 8 + lr) * LD + ks * 16 + (lm & 1) * 8);
        mma_bf16_16816(sc[2 * np], qa[ks], b[0], b[1]);
        mma_bf16_16816(sc[2 * np + 1], qa[ks], b[2], b[3]);
      }
    }
    if (CAUSAL && kb == qb) {  // diagonal block: key > query is masked
#pragma unroll
      for (int nt = 0; nt < 8; ++nt) {
        const int key = kb * 64 + nt * 8 + 2 * t;
        if (key > qrow0) sc[nt][0] = -INFINITY;
        if (key + 1 > qrow0) sc[nt][1] = -INFINITY;
        if (key > qrow0 + 8) sc[nt][2] = -INFINITY;
        if (key + 1 > qrow0 + 8) sc[nt][3] = -INFINITY;
      }
    }
    float mx0 = m0, mx1 = m1;
#pragma unroll
    for (int nt = 0; nt < 8; ++nt) {
      mx0 = fmaxf(mx0, fmaxf(sc[nt][0], sc[nt][1]));
      mx1 = fmaxf(mx1, fmaxf(sc[nt][2], sc[nt][3]));
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
      const float p0 = exp2f(fmaf(sc[nt][0], scale_log2, -sm0));
      const float p1 = exp2f(fmaf(sc[nt][1], scale_log2, -sm0));
      const float p2 = exp2f(fmaf(sc[nt][2], scale_log2, -sm1));
      const float p3 = exp2f(fmaf(sc[nt][3], scale_log2, -sm1));
      l0 += p0 + p1;
      l1 += p2 + p3;
      const int j = nt >> 1, hi = nt & 1;
      pa[j][hi ? 2 : 0] = pack2(p0, p1);
      pa[j][hi ? 3 : 1] = pack2(p2, p3);
    }
#pragma unroll
    for (int j = 0; j < 4; ++j) {
#pragma unroll
      for (int dp = 0; dp < DH / 16; ++dp) {
        uint32_t b[4];
        ldsm_x4_t(b, Vb + (j * 16 + (lm & 1) * 8 + lr) * LD + dp * 16 + (lm >> 1) * 8);
        mma_bf16_16816(o[2 * dp], pa[j], b[0], b[1]);
        mma_bf16_16816(o[2 * dp + 1], pa[j], b[2], b[3]);
      }
    }
    __syncthreads();  // the next iteration's prefetch overwrites this stage
  }
  l0 += __shfl_xor_sync(kFull, l0, 1);
  l0 += __shfl_xor_sync(kFull, l0, 2);
  l1 += __shfl_xor_sync(kFull, l1, 1);
  l1 += __shfl_xor_sync(kFull, l1, 2);
  const float i0 = 1.f / l0, i1 = 1.f / l1;
  const int D = Hq * DH;
  __nv_bfloat16 *o0 = out + (row0 + qrow0) * D + h * DH;
  __nv_bfloat16 *o1 = o0 + (size_t)8 * D;
#pragma unroll
  for (int nt = 0; nt < DH / 8; ++nt) {
    *reinterpret_cast<uint32_t *>(o0 + nt * 8 + 2 * t) = pack2(o[nt][0] * i0, o[nt][1] * i0);
    *reinterpret_cast<uint32_t *>(o1 + nt * 8 + 2 * t) = pack2(o[nt][2] * i1, o[nt][3] * i1);
  }
}

template <int DH, bool CAUSAL>
cudaError_t launch_flash(const __nv_bfloat16 *qkv, __nv_bfloat16 *out, int n_seqs, int S, int Hq,
                         int Hkv, cudaStream_t s) {
  const size_t smem = (size_t)5 * 64 * (DH + 8) * 2;
  cudaError_t e = cudaFuncSetAttribute(attn_flash_kernel<DH, CAUSAL>,
                                       cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  if (e != cudaSuccess) return e;
  dim3 grid(S / 64, n_seqs * Hq);
  attn_flash_kernel<DH, CAUSAL><<<grid, 128, smem, s>>>(qkv, out, S, Hq, Hkv,
                                                        1.4426950408889634f / sqrtf((float)DH));
  note_launch();
  return cudaGetLastError();
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

int g_attn_mode = 0;

cudaError_t attention_bf16(const __nv_bfloat16 *qkv, __nv_bfloat16 *out, int n_seqs, int S, int H,
                           int dh, cudaStream_t s) {
  if (n_seqs <= 0) return cudaSuccess;
  if (S % 64 != 0 || dh % 16 != 0) return cudaErrorInvalidValue;
  if (g_attn_mode != 1 && dh == 64 && (S == 128 || S == 256)) {
    if (((uintptr_t)qkv & 15) != 0 || ((uintptr_t)out & 15) != 0) return cudaErrorInvalidValue;
    return S == 256 ? launch_attn_tc<256>(qkv, out, n_seqs, H, s)
                    : launch_attn_tc<128>(qkv, out, n_seqs, H, s);
  }
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

// ---------------------------------------------------------------------------
// attn_tc_causal_kernel: causal grouped-query attention on the 5th-gen tensor
// cores for the decoder-style encoder (config-4: dh = 128, S % 128 == 0).
//
// Work item = one 128-row query tile t of one (sequence, q head); its keys are
// the (t + 1) 128-key blocks up to the diagonal. Two passes over the key
// blocks replace the online rescaling of O (which would need O read-modify-
// written in TMEM between P.V MMAs): pass A computes S = Q.K_b^T per block for
// the exact row max; pass B recomputes S, writes P = 2^(s*c - max*c) (bf16,
// masked above the diagonal) over the scores in TMEM and accumulates
// O += P.V_b (TS-MMA, V as an MN-major operand spanning two 64-column swizzle
// atoms). Q.K^T runs twice (1.5x the attention MMA work), cheap next to the
// softmax exponentials.
//   warp 0 / 10  TMA producers of softmax group 0 / 1 (Q, then the K blocks of
//                pass A, then K, V of pass B through a 2-slot ring per group)
//   warp 1       single MMA issuer; polls both groups' barriers and issues
//                whichever operation is ready
//   warps 2-9    two softmax groups of 4 warps (one TMEM lane quarter each);
//                group r owns TMEM columns [256 r, 256 r + 256): S/P in the
//                first 128, O in the second, and every second work item
namespace atq {
constexpr int kThreads = 11 * 32;
constexpr int kTile = 128 * 128 * 2;        // [128][128] bf16 = two 64-column atoms
constexpr int kGroupBytes = 3 * kTile;      // Q + 2 ring slots
constexpr int kSmem = 2 * kGroupBytes + 1024 + 512;
}  // namespace atq

__global__ void __launch_bounds__(atq::kThreads, 1)
    attn_tc_causal_kernel(const __grid_constant__ CUtensorMap tm, __nv_bfloat16 *__restrict__ out,
                          int n_seqs, int S, int Hq, int Hkv) {
  using namespace tc;
  extern __shared__ uint8_t smem_raw[];
  uint8_t *smem = smem_raw + ((1024u - (tc::smem_u32(smem_raw) & 1023u)) & 1023u);  // 1 KB aligned, still shared space
  uint64_t *bars = reinterpret_cast<uint64_t *>(smem + 2 * atq::kGroupBytes);
  // per group r: [0] q_full [1] q_free [2,3] ring_full [4,5] ring_free [6] s_full
  // [7] s_free [8] p_full [9] pv_done [10] o_full [11] o_free
  auto B = [&](int r, int i) { return bars + r * 12 + i; };
  uint32_t *tslot = reinterpret_cast<uint32_t *>(bars + 24);
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  if (threadIdx.x == 0) {
    for (int r = 0; r < 2; ++r) {
      mbar_init(B(r, 0), 1);
      mbar_init(B(r, 1), 1);
      for (int k = 2; k < 6; ++k) mbar_init(B(r, k), 1);
      mbar_init(B(r, 6), 1);
      mbar_init(B(r, 7), 4);
      mbar_init(B(r, 8), 4);
      mbar_init(B(r, 9), 1);
      mbar_init(B(r, 10), 1);
      mbar_init(B(r, 11), 4);
    }
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  if (warp == 1) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(
                     smem_u32(tslot)),
                 "r"(512));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
  }
  fence_before();
  __syncthreads();
  fence_after();
  const uint32_t tmem = *tslot;
  const int nT = S / 128;
  const int n_items = n_seqs * Hq * nT;
  const int RS = (Hq + 2 * Hkv) * 128;  // qkv row width
  // local items of this CTA: j = 0, 1, ...; item = blockIdx.x + j * gridDim.x,
  // t-major decode (longest tiles first), group r = j & 1
  const int n_local =
      n_items > (int)blockIdx.x ? (n_items - (int)blockIdx.x + (int)gridDim.x - 1) / (int)gridDim.x
                                : 0;
  auto decode = [&](int j, int &seq, int &h, int &t) {
    const int item = (int)blockIdx.x + j * (int)gridDim.x;
    const int per_t = n_seqs * Hq;
    t = nT - 1 - item / per_t;
    const int rem = item % per_t;
    seq = rem / Hq;
    h = rem % Hq;
  };

  if (warp == 0 || warp == 10) {
    const int r = warp == 0 ? 0 : 1;
    if (lane == 0) {
      asm volatile("prefetch.tensormap [%0];" ::"l"(&tm) : "memory");
      uint64_t pol;
      asm volatile("createpolicy.fractional.L2::evict_last.b64 %0, 1.0;" : "=l"(pol));
      uint8_t *qs = smem + r * atq::kGroupBytes;
      uint8_t *ring = qs + atq::kTile;
      uint32_t nq = 0, nr = 0;  // Q loads / ring loads so far
      auto load_tile = [&](uint8_t *dst, uint64_t *bar, int col, int row) {
        mbar_expect_tx(bar, atq::kTile);
        tma_load_2d(dst, &tm, bar, col, row, pol);
        tma_load_2d(dst + atq::kTile / 2, &tm, bar, col + 64, row, pol);
      };
      auto ring_load = [&](int col, int row) {
        const int sl = nr & 1;
        mbar_wait(B(r, 4 + sl), ((nr >> 1) & 1) ^ 1);
        load_tile(ring + sl * atq::kTile, B(r, 2 + sl), col, row);
        ++nr;
      };
      for (int j = r; j < n_local; j += 2) {
        int seq, h, t;
        decode(j, seq, h, t);
        const int g = h / (Hq / Hkv);
        const int row0 = seq * S;
        mbar_wait(B(r, 1), (nq & 1) ^ 1);
        load_tile(qs, B(r, 0), h * 128, row0 + t * 128);
        ++nq;
        for (int kb = 0; kb <= t; ++kb) ring_load((Hq + g) * 128, row0 + kb * 128);
        for (int kb = 0; kb <= t; ++kb) {
          ring_load((Hq + g) * 128, row0 + kb * 128);
          ring_load((Hq + Hkv + g) * 128, row0 + kb * 128);
        }
      }
    }
  } else if (warp == 1) {
    if (lane == 0) {
      constexpr uint32_t idesc_s = idesc_bf16(128, 128);
      constexpr uint32_t idesc_o = idesc_bf16(128, 128, true);
      struct GS {
        int j, t, op;          // local item, its tile, next op index within the item
        uint32_t nq, nr;       // Q loads consumed / ring slots consumed
        uint32_t ns, npv;      // S ops issued / P.V ops issued (this group)
        uint32_t nsa;          // pass-A S ops whose s_free is awaited
        bool prev_pv;          // the previous S op was followed by a P.V reading P
        uint32_t nitems;       // items started (o_free parity)
      } gs[2];
      for (int r = 0; r < 2; ++r) {
        gs[r] = GS{r, 0, 0, 0, 0, 0, 0, 0, false, 0};
        if (r < n_local) {
          int a, b2;
          decode(r, a, b2, gs[r].t);
        }
      }
      int done = 0;
      const int want = (n_local > 0) + (n_local > 1);
      while (done < want) {
        for (int r = 0; r < 2; ++r) {
          GS &G = gs[r];
          if (G.j >= n_local) continue;
          const int t = G.t;
          const int nA = t + 1;
          const int nops = nA + 2 * (t + 1);
          const int op = G.op;
          const uint32_t rb = tmem + r * 256;
          const uint8_t *qs = smem + r * atq::kGroupBytes;
          const uint8_t *ring = qs + atq::kTile;
          const bool is_s = op < nA || ((op - nA) & 1) == 0;
          const int sl = G.nr & 1;
          if (!mbar_test(B(r, 2 + sl), (G.nr >> 1) & 1)) continue;  // operand tile landed
          if (is_s) {
            if (op == 0 && !mbar_test(B(r, 0), G.nq & 1)) continue;  // Q landed
            // the S/P region is free: the softmax consumed the previous pass-A
            // S, or the P.V that read the previous P completed
            if (G.ns > 0) {
              if (G.prev_pv) {
                if (!mbar_test(B(r, 9), (G.npv - 1) & 1)) continue;
              } else if (!mbar_test(B(r, 7), (G.nsa - 1) & 1)) {
                continue;
              }
            }
            fence_after();
            const uint64_t a = sw128_desc(smem_u32(qs));
            const uint64_t b = sw128_desc(smem_u32(ring + sl * atq::kTile));
#pragma unroll
            for (int k = 0; k < 8; ++k) {  // K = 128: two 64-column atoms, 4 steps each
              const uint64_t off = (uint64_t)((k >> 2) * (atq::kTile / 2 / 16) + 2 * (k & 3));
              umma_ss(rb, a + off, b + off, idesc_s, k);
            }
            umma_commit(B(r, 6));
            umma_commit(B(r, 4 + sl));
            ++G.ns;
            if (op < nA) {
              ++G.nsa;
              G.prev_pv = false;
            } else {
              G.prev_pv = true;
            }
            if (op == nops - 2) umma_commit(B(r, 1));  // last Q.K^T: Q slot free
          } else {
            const int kb = (op - nA) >> 1;
            if (!mbar_test(B(r, 8), G.npv & 1)) continue;                       // P written
            if (kb == 0 && !mbar_test(B(r, 11), (G.nitems & 1) ^ 1)) continue;  // O drained
            fence_after();
            const uint64_t v = sw128_desc(smem_u32(ring + sl * atq::kTile), 1024, atq::kTile / 2);
#pragma unroll
            for (int k = 0; k < 8; ++k)  // 16 keys per step = 2048 B of each V atom
              umma_ts(rb + 128, rb + 8 * k, v + (uint64_t)(128 * k), idesc_o, kb > 0 || k > 0);
            umma_commit(B(r, 9));
            umma_commit(B(r, 4 + sl));
            ++G.npv;
            if (kb == t) umma_commit(B(r, 10));
          }
          ++G.nr;
          if (op == 0) ++G.nq;
          G.op = op + 1;
          if (G.op == nops) {  // next item of this group
            G.op = 0;
            ++G.nitems;
            G.j += 2;
            if (G.j < n_local) {
              int a, b2;
              decode(G.j, a, b2, G.t);
            } else {
              ++done;
            }
          }
        }
      }
    }
  } else {
    const int g = (warp - 2) >> 2;
    const int q = warp & 3;
    const int rrow = q * 32 + lane;
    const uint32_t tb = tmem + ((uint32_t)(q * 32) << 16) + (uint32_t)(g * 256);
    constexpr float kC = 0.12751743082459868f;  // log2(e) / sqrt(128)
    uint32_t ns = 0, nitems = 0;
    for (int j = g; j < n_local; j += 2, ++nitems) {
      int seq, h, t;
      decode(j, seq, h, t);
      const int qi = t * 128 + rrow;  // query position
      float m = -FLT_MAX;
      for (int kb = 0; kb <= t; ++kb, ++ns) {  // pass A: row max
        mbar_wait(B(g, 6), ns & 1);
        fence_after();
        uint32_t r0[32], r1[32];
#pragma unroll
        for (int c = 0; c < 128; c += 64) {
          tmem_ld32_nowait(tb + c, r0);
          tmem_ld32_nowait(tb + c + 32, r1);
          tmem_ld_wait();
#pragma unroll
          for (int e = 0; e < 32; ++e) {
            const int k0 = kb * 128 + c + e;
            const float a0 = k0 <= qi ? __uint_as_float(r0[e]) : -FLT_MAX;
            const float a1 = k0 + 32 <= qi ? __uint_as_float(r1[e]) : -FLT_MAX;
            m = fmaxf(m, fmaxf(a0, a1));
          }
        }
        fence_before();
        __syncwarp();
        if (lane == 0) mbar_arrive(B(g, 7));
      }
      const float mc = m * kC;
      float s4[4] = {0.f, 0.f, 0.f, 0.f};
      for (int kb = 0; kb <= t; ++kb, ++ns) {  // pass B: P over the scores
        mbar_wait(B(g, 6), ns & 1);
        fence_after();
#pragma unroll 1
        for (int c = 0; c < 128; c += 32) {
          uint32_t r0[32];
          tmem_ld32(tb + c, r0);
          uint32_t w[16];
#pragma unroll
          for (int e = 0; e < 16; ++e) {
            const int k0 = kb * 128 + c + 2 * e;
            const float p0 = k0 <= qi ? ex2_approx(fmaf(__uint_as_float(r0[2 * e]), kC, -mc)) : 0.f;
            const float p1 =
                k0 + 1 <= qi ? ex2_approx(fmaf(__uint_as_float(r0[2 * e + 1]), kC, -mc)) : 0.f;
            s4[(2 * e) & 3] += p0;
            s4[(2 * e + 1) & 3] += p1;
            w[e] = pack_bf16(p0, p1);
          }
          tmem_st16(tb + c / 2, w);
        }
        tmem_st_wait();
        fence_before();
        __syncwarp();
        if (lane == 0) mbar_arrive(B(g, 8));
      }
      // epilogue: O / rowsum -> context row slice [h*128, +128)
      mbar_wait(B(g, 10), nitems & 1);
      fence_after();
      uint32_t o[4][32];
#pragma unroll
      for (int c = 0; c < 4; ++c) tmem_ld32_nowait(tb + 128 + 32 * c, o[c]);
      tmem_ld_wait();
      fence_before();
      __syncwarp();
      if (lane == 0) mbar_arrive(B(g, 11));
      const float inv = 1.f / ((s4[0] + s4[1]) + (s4[2] + s4[3]));
      uint4 *op = reinterpret_cast<uint4 *>(out + ((size_t)seq * S + qi) * (size_t)(Hq * 128) +
                                            h * 128);
#pragma unroll
      for (int c = 0; c < 4; ++c)
#pragma unroll
        for (int v = 0; v < 4; ++v) {
          uint4 u;
          u.x = pack_bf16(__uint_as_float(o[c][8 * v + 0]) * inv, __uint_as_float(o[c][8 * v + 1]) * inv);
          u.y = pack_bf16(__uint_as_float(o[c][8 * v + 2]) * inv, __uint_as_float(o[c][8 * v + 3]) * inv);
          u.z = pack_bf16(__uint_as_float(o[c][8 * v + 4]) * inv, __uint_as_float(o[c][8 * v + 5]) * inv);
          u.w = pack_bf16(__uint_as_float(o[c][8 * v + 6]) * inv, __uint_as_float(o[c][8 * v + 7]) * inv);
          op[4 * c + v] = u;
        }
    }
  }
  fence_before();
  __syncthreads();
  if (warp == 1) {
    fence_after();
    asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem), "r"(512));
  }
}

cudaError_t launch_attn_tc_causal(const __nv_bfloat16 *qkv, __nv_bfloat16 *out, int n_seqs, int S,
                                  int Hq, int Hkv, cudaStream_t s) {
  CUtensorMap tm;
  const uint64_t W = (uint64_t)(Hq + 2 * Hkv) * 128;
  if (!make_tma_2d_bf16(&tm, qkv, W, (uint64_t)n_seqs * S, W * 2, 64, 128))
    return cudaErrorInvalidValue;
  static unsigned long long attr = 0;  // per device (first_on_device)
  if (first_on_device(attr)) {
    cudaError_t e = cudaFuncSetAttribute(attn_tc_causal_kernel,
                                         cudaFuncAttributeMaxDynamicSharedMemorySize, atq::kSmem);
    if (e != cudaSuccess) return e;
  }
  const int items = n_seqs * Hq * (S / 128);
  const int grid = std::min(items, tc_gemm_num_sms());
  attn_tc_causal_kernel<<<grid, atq::kThreads, atq::kSmem, s>>>(tm, out, n_seqs, S, Hq, Hkv);
  note_launch();
  return cudaGetLastError();
}


cudaError_t attention_gqa_bf16(const __nv_bfloat16 *qkv, __nv_bfloat16 *out, int n_seqs, int S,
                               int Hq, int Hkv, int dh, bool causal, cudaStream_t s) {
  if (n_seqs <= 0) return cudaSuccess;
  if (S % 64 != 0 || Hkv <= 0 || Hq % Hkv != 0) return cudaErrorInvalidValue;
  if (dh == 64)
    return causal ? launch_flash<64, true>(qkv, out, n_seqs, S, Hq, Hkv, s)
                  : launch_flash<64, false>(qkv, out, n_seqs, S, Hq, Hkv, s);
  if (dh == 128 && causal && S % 128 == 0 && g_attn_mode != 1 &&
      ((uintptr_t)qkv & 15) == 0 && ((uintptr_t)out & 15) == 0)
    return launch_attn_tc_causal(qkv, out, n_seqs, S, Hq, Hkv, s);
  if (dh == 128)
    return causal ? launch_flash<128, true>(qkv, out, n_seqs, S, Hq, Hkv, s)
                  : launch_flash<128, false>(qkv, out, n_seqs, S, Hq, Hkv, s);
  return cudaErrorInvalidValue;
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
