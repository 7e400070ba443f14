// lv_qkv_attn.cu — the QKV projection and the attention of one encoder layer in
// ONE kernel on an SM pair (tcgen05 cta_group::2), sm_100a: qkv never leaves
// the chip.
//
//   ctx[s, :, h] = softmax(Q_h K_h^T / 8) V_h,   [Q_h | K_h | V_h] = epi(x[s] . W_h^T)
//
// This is the recompute half of LEANN's two-level search (provider.embed_batch,
// vectors.py:201-211, batched over every in-flight query's candidates). The
// unfused encoder wrote qkv ([T][3d] bf16, 4.6 KB per token) from the QKV GEMM
// and read it back in attn_tc_kernel: 10.7% of the config-2 step, bound by that
// HBM round trip (profiles/r02_summary.md).
//
// Work item = (sequence s, head h), S = 256 tokens, dh = 64. CTA r of the pair
// owns token rows [128 r, 128 r + 128) of the sequence:
//  1. GEMM (M = 256, N = 192, K = d): A = x rows of the sequence (TMA, 128-byte
//     swizzle), B = the 192 weight rows of head h (q_h | k_h | v_h, three 32-row
//     TMA boxes per CTA out of the unpermuted nn.Linear weight) -> TMEM columns
//     [0, 192) of each CTA: its 128 rows x (q | k | v).
//  2. Drain (8 epilogue warps): bias / LN-in rank-1 correction (the epilogue of
//     tc_gemm_pair_kernel, EPF_LN_IN, same expression), bf16 round, then
//        Q -> own smem [128][64] (K-major, 128B swizzle)   A of S = Q.K^T
//        K -> own smem [128][64] (K-major, 128B swizzle)   B half of S (keys of CTA r)
//        V -> [256 keys][32 dims] MN-major 64B-swizzled halves: dims [0, 32) to
//             CTA 0, [32, 64) to CTA 1 (st.shared::cluster into the peer)  B of P.V
//  3. S = Q.K^T (pair MMA, M = 256, N = 256 keys, K = 64) -> TMEM [256, 512):
//     the B operand's N split across the pair IS the key split, so no K exchange.
//  4. Softmax: the two warps sharing a TMEM lane quarter own columns [0, 128) and
//     [128, 256) of a row (max / sum exchanged through shared memory); P (bf16)
//     written over the consumed scores (tcgen05.st).
//  5. O = P.V (pair TS-MMA: P from each CTA's TMEM, V MN-major, M = 256, N = 64)
//     -> TMEM [192, 256); ctx = O / rowsum, 64 bytes per thread and row.
// Pipelining (one MMA thread, cycle k): G(k), PV(k-2), S(k-1); epilogue cycle k:
// drain(k), O-epilogue(k-2), softmax(k-1) — the GEMM of item k runs on the tensor
// pipe while the epilogue warps do the softmax of item k-1. Q/K are double
// buffered, V triple buffered (P.V of item k-2 is issued after G(k)).
//
// Numerics: every value equals the unfused path bit for bit — the same fp32
// accumulators (fixed K order), the same epilogue expression, the same
// exponentials, the row sum in the two-half order attn_tc_kernel uses.
// Batch-invariant: an item never depends on other items.
#include <cuda.h>

#include <cfloat>

#include "lv_kernels.cuh"
#include "lv_tc.cuh"

namespace lv {
namespace {
using namespace tc;

namespace qa {
constexpr int kThreads = 64 + 8 * 32;
constexpr int kS = 256, kDh = 64;
constexpr int kStages = 3;
constexpr int kABytes = 128 * 64 * 2;   // A half per stage (128 rows x 64 K)
constexpr int kBBytes = 96 * 64 * 2;    // B half per stage (96 weight rows x 64 K)
constexpr int kQKBytes = 128 * 128;     // [128][64] bf16
constexpr int kVBytes = kS * 64;        // [256 keys][32 dims] bf16
constexpr int kOffB = kStages * kABytes;
constexpr int kOffQ = kOffB + kStages * kBBytes;
constexpr int kOffK = kOffQ + 2 * kQKBytes;
constexpr int kOffV = kOffK + 2 * kQKBytes;
constexpr int kOffRed = kOffV + 3 * kVBytes;    // float [2][2][128]: row max / sum halves
constexpr int kOffBar = kOffRed + 2 * 2 * 128 * 4;
constexpr int kSmem = kOffBar + 256 + 1024;
constexpr uint32_t kColAcc = 0, kColO = 192, kColS = 256;
static_assert(kOffQ % 1024 == 0 && kOffV % 1024 == 0, "swizzled regions need 1 KB alignment");
static_assert(kSmem <= 232448, "shared memory");
}  // namespace qa

__device__ __forceinline__ float ex2_fast(float x) {
  float y;
  asm("ex2.approx.ftz.f32 %0, %1;" : "=f"(y) : "f"(x));
  return y;
}

__global__ void __cluster_dims__(2, 1, 1) __launch_bounds__(qa::kThreads, 1)
    qkv_attn_pair_kernel(const __grid_constant__ CUtensorMap tmA,
                         const __grid_constant__ CUtensorMap tmB, const float *__restrict__ bias,
                         const float *__restrict__ colc, const float2 *__restrict__ ln_in,
                         __nv_bfloat16 *__restrict__ ctx, int n_items, int H, int K,
                         float scale_log2) {
  using namespace qa;
  extern __shared__ uint8_t smem_raw[];
  uint8_t *smem = reinterpret_cast<uint8_t *>(
      (reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  uint8_t *sA = smem, *sB = smem + kOffB, *sQ = smem + kOffQ, *sK = smem + kOffK,
          *sV = smem + kOffV;
  float *red = reinterpret_cast<float *>(smem + kOffRed);
  uint64_t *full = reinterpret_cast<uint64_t *>(smem + kOffBar);
  uint64_t *empty = full + kStages;
  uint64_t *acc_full = empty + kStages;
  uint64_t *acc_empty = acc_full + 1;
  uint64_t *qkv_ready = acc_empty + 1;  // [2]
  uint64_t *s_full = qkv_ready + 2;
  uint64_t *p_full = s_full + 1;        // [2]
  uint64_t *o_full = p_full + 2;
  uint64_t *o_empty = o_full + 1;
  uint32_t *tslot = reinterpret_cast<uint32_t *>(o_empty + 1);

  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const uint32_t rank = cluster_rank();
  const bool leader = rank == 0;
  if (threadIdx.x == 0) {
    for (int s = 0; s < kStages; ++s) {
      mbar_init(&full[s], 1);
      mbar_init(&empty[s], 1);
    }
    mbar_init(acc_full, 1);
    mbar_init(acc_empty, 16);
    mbar_init(&qkv_ready[0], 16);
    mbar_init(&qkv_ready[1], 16);
    mbar_init(s_full, 1);
    mbar_init(&p_full[0], 16);
    mbar_init(&p_full[1], 16);
    mbar_init(o_full, 1);
    mbar_init(o_empty, 16);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  if (warp == 1) {
    asm volatile("tcgen05.alloc.cta_group::2.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(
                     smem_u32(tslot)),
                 "r"(512));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::2.sync.aligned;");
  }
  fence_before();
  cluster_sync_all();
  fence_after();
  const uint32_t tmem = *tslot;

  const int pair = blockIdx.x >> 1, n_pairs = gridDim.x >> 1;
  const int n = n_items > pair ? (n_items - pair + n_pairs - 1) / n_pairs : 0;
  const int D = H * kDh;
  const int kblocks = K / 64;

  if (warp == 0) {
    if (lane == 0) {
      asm volatile("prefetch.tensormap [%0];" ::"l"(&tmA) : "memory");
      asm volatile("prefetch.tensormap [%0];" ::"l"(&tmB) : "memory");
      uint64_t pol_a, pol_b;  // x rows are read by the 12 heads of a sequence; weights stay
      asm volatile("createpolicy.fractional.L2::evict_normal.b64 %0, 1.0;" : "=l"(pol_a));
      asm volatile("createpolicy.fractional.L2::evict_last.b64 %0, 1.0;" : "=l"(pol_b));
      int stage = 0;
      uint32_t phase = 0;
      for (int i = 0; i < n; ++i) {
        const int item = pair + i * n_pairs;
        const int seq = item / H, h = item - seq * H;
        for (int kb = 0; kb < kblocks; ++kb) {
          mbar_wait(&empty[stage], phase ^ 1);
          const uint32_t fb = map_to_rank(&full[stage], 0);
          if (leader) mbar_expect_tx(&full[stage], 2 * (kABytes + kBBytes));
          tma_load_2d_pair(sA + stage * kABytes, &tmA, fb, kb * 64, seq * kS + (int)rank * 128,
                           pol_a);
          // weight rows of head h in accumulator-column order q | k | v, 32 rows per
          // box: CTA 0 loads q[0,64) k[0,32), CTA 1 loads k[32,64) v[0,64)
#pragma unroll
          for (int j = 0; j < 3; ++j) {
            const int seg = (int)rank * 3 + j;
            const int wrow = (seg >> 1) * D + h * kDh + (seg & 1) * 32;
            tma_load_2d_pair(sB + stage * kBBytes + j * 4096, &tmB, fb, kb * 64, wrow, pol_b);
          }
          if (++stage == kStages) {
            stage = 0;
            phase ^= 1;
          }
        }
      }
    }
  } else if (warp == 1) {
    if (leader && lane == 0) {
      constexpr uint32_t idesc_g = idesc_bf16(256, 192);
      constexpr uint32_t idesc_s = idesc_bf16(256, kS);
      constexpr uint32_t idesc_o = idesc_bf16(256, kDh, true);
      int stage = 0;
      uint32_t phase = 0;
      for (int k = 0; k < n + 2; ++k) {
        if (k < n) {  // G(k): the QKV projection of item k
          if (k > 0) mbar_wait(acc_empty, (uint32_t)(k - 1) & 1);
          fence_after();
          for (int kb = 0; kb < kblocks; ++kb) {
            mbar_wait(&full[stage], phase);
            fence_after();
            const uint64_t a0 = sw128_desc(smem_u32(sA + stage * kABytes));
            const uint64_t b0 = sw128_desc(smem_u32(sB + stage * kBBytes));
#pragma unroll
            for (int j = 0; j < 4; ++j)
              umma_bf16_pair(tmem + kColAcc, a0 + 2 * j, b0 + 2 * j, idesc_g, (kb | j) != 0);
            umma_commit_pair(&empty[stage]);
            if (++stage == kStages) {
              stage = 0;
              phase ^= 1;
            }
          }
          umma_commit_pair(acc_full);
        }
        if (k >= 2) {  // PV(k-2): P from TMEM, V from the pair's shared memory
          const int j = k - 2;
          mbar_wait(&p_full[j & 1], (uint32_t)(j >> 1) & 1);
          if (j >= 1) mbar_wait(o_empty, (uint32_t)(j - 1) & 1);
          fence_after();
          const uint32_t vb = smem_u32(sV + (j % 3) * kVBytes);
#pragma unroll
          for (int t = 0; t < kS / 16; ++t)  // 16 keys = 1024 bytes of V per K step
            umma_ts_pair(tmem + kColO, tmem + kColS + 8 * t, sw64_desc(vb + 1024 * t), idesc_o,
                         t != 0);
          umma_commit_pair(o_full);
        }
        if (k >= 1 && k - 1 < n) {  // S(k-1) = Q.K^T over the sequence's 256 keys
          const int j = k - 1;
          mbar_wait_acq_cluster(&qkv_ready[j & 1], (uint32_t)(j >> 1) & 1);
          fence_after();
          const uint64_t a0 = sw128_desc(smem_u32(sQ + (j & 1) * kQKBytes));
          const uint64_t b0 = sw128_desc(smem_u32(sK + (j & 1) * kQKBytes));
#pragma unroll
          for (int t = 0; t < kDh / 16; ++t)
            umma_bf16_pair(tmem + kColS, a0 + 2 * t, b0 + 2 * t, idesc_s, t != 0);
          umma_commit_pair(s_full);
        }
      }
    }
  } else {
    const int ew = warp - 2;
    const int q = warp & 3;     // TMEM lane quarter
    const int half = ew >> 2;   // column half of the row this warp owns
    const int row = q * 32 + lane;  // row of the CTA's 128
    const uint32_t lane_off = (uint32_t)(q * 32) << 16;
    const uint32_t acc_empty_l = map_to_rank(acc_empty, 0);
    const uint32_t o_empty_l = map_to_rank(o_empty, 0);
    const uint32_t qkv_ready_l0 = map_to_rank(&qkv_ready[0], 0);
    const uint32_t qkv_ready_l1 = map_to_rank(&qkv_ready[1], 0);
    const uint32_t p_full_l0 = map_to_rank(&p_full[0], 0), p_full_l1 = map_to_rank(&p_full[1], 0);
    const int bar_id = 1 + q;  // the two warps of this lane quarter
    float sum_prev = 1.f;      // row sum of the item whose softmax ran last
    for (int k = 0; k < n + 2; ++k) {
      if (k < n) {  // drain(k): accumulators -> Q, K, V tiles in shared memory
        const int item = pair + k * n_pairs;
        const int seq = item / H, h = item - seq * H;
        mbar_wait(acc_full, (uint32_t)k & 1);
        fence_after();
        uint32_t r[96];
        {
          uint32_t(&r0)[32] = *reinterpret_cast<uint32_t(*)[32]>(&r[0]);
          uint32_t(&r1)[32] = *reinterpret_cast<uint32_t(*)[32]>(&r[32]);
          uint32_t(&r2)[32] = *reinterpret_cast<uint32_t(*)[32]>(&r[64]);
          const uint32_t ta = tmem + lane_off + kColAcc + (uint32_t)(half * 96);
          tmem_ld32_nowait(ta, r0);
          tmem_ld32_nowait(ta + 32, r1);
          tmem_ld32_nowait(ta + 64, r2);
          tmem_ld_wait();
        }
        fence_before();
        __syncwarp();
        if (lane == 0) mbar_arrive_remote(acc_empty_l);
        const int grow = seq * kS + (int)rank * 128 + row;
        float mu = 0.f, rs = 1.f;
        if (ln_in) {
          const float2 st = __ldg(ln_in + grow);
          mu = st.x;
          rs = st.y;
        }
        const uint32_t sw = (uint32_t)(row & 7);
#pragma unroll
        for (int c = 0; c < 3; ++c) {
          const int n0 = half * 96 + 32 * c;  // accumulator column: q [0,64) k [64,128) v [128,192)
          const int part = n0 >> 6, dim0 = n0 & 63;
          const int gcol = part * D + h * kDh + dim0;  // column of the unfused qkv row
          const float4 *b4 = reinterpret_cast<const float4 *>(bias + gcol);
          const float4 *c4 = reinterpret_cast<const float4 *>(colc + gcol);
          uint32_t w[16];
#pragma unroll
          for (int j = 0; j < 8; ++j) {
            const float4 bb = __ldg(b4 + j);
            const float bv[4] = {bb.x, bb.y, bb.z, bb.w};
            float v[4];
            if (ln_in) {
              const float4 cc = __ldg(c4 + j);
              const float cv[4] = {cc.x, cc.y, cc.z, cc.w};
#pragma unroll
              for (int e = 0; e < 4; ++e)
                v[e] = fmaf(rs, fmaf(-mu, cv[e], __uint_as_float(r[32 * c + 4 * j + e])), bv[e]);
            } else {
#pragma unroll
              for (int e = 0; e < 4; ++e) v[e] = __uint_as_float(r[32 * c + 4 * j + e]) + bv[e];
            }
            w[2 * j] = pack_bf16(v[0], v[1]);
            w[2 * j + 1] = pack_bf16(v[2], v[3]);
          }
          if (part < 2) {  // Q or K: K-major [128][64], 128-byte swizzle
            uint8_t *dst = (part == 0 ? sQ : sK) + (k & 1) * kQKBytes + row * 128;
#pragma unroll
            for (int j = 0; j < 4; ++j) {
              const uint32_t chunk = (uint32_t)(dim0 >> 3) + j;
              *reinterpret_cast<uint4 *>(dst + ((chunk ^ sw) << 4)) =
                  make_uint4(w[4 * j], w[4 * j + 1], w[4 * j + 2], w[4 * j + 3]);
            }
          } else {  // V dims [dim0, dim0 + 32) -> CTA dim0 / 32, key row of the sequence
            const int key = (int)rank * 128 + row;
            const uint32_t kw = (uint32_t)((key >> 1) & 3);
            uint8_t *dst = sV + (k % 3) * kVBytes + key * 64;
            const uint32_t target = (uint32_t)(dim0 >> 5);
            if (target == rank) {
#pragma unroll
              for (int j = 0; j < 4; ++j)
                *reinterpret_cast<uint4 *>(dst + (((uint32_t)j ^ kw) << 4)) =
                    make_uint4(w[4 * j], w[4 * j + 1], w[4 * j + 2], w[4 * j + 3]);
            } else {
              const uint32_t rdst = map_to_rank(dst, target);
#pragma unroll
              for (int j = 0; j < 4; ++j)
                st_cluster_v4(rdst + (((uint32_t)j ^ kw) << 4),
                              make_uint4(w[4 * j], w[4 * j + 1], w[4 * j + 2], w[4 * j + 3]));
            }
          }
        }
        // generic-proxy writes (own and peer shared memory) before the MMA reads them
        asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
        asm volatile("fence.proxy.async.shared::cluster;" ::: "memory");
        __syncwarp();
        if (lane == 0) {
          asm volatile("fence.acq_rel.cluster;" ::: "memory");
          mbar_arrive_release_cluster((k & 1) ? qkv_ready_l1 : qkv_ready_l0);
        }
      }
      if (k >= 2) {  // O-epilogue(k-2): ctx row slice = O / rowsum
        const int j = k - 2;
        const int item = pair + j * n_pairs;
        const int seq = item / H, h = item - seq * H;
        mbar_wait(o_full, (uint32_t)j & 1);
        fence_after();
        uint32_t o[32];
        tmem_ld32(tmem + lane_off + kColO + (uint32_t)(half * 32), o);
        fence_before();
        __syncwarp();
        if (lane == 0) mbar_arrive_remote(o_empty_l);
        const float inv = 1.f / sum_prev;
        const size_t grow = (size_t)seq * kS + rank * 128 + row;
        uint4 *op = reinterpret_cast<uint4 *>(ctx + grow * D + h * kDh + half * 32);
#pragma unroll
        for (int v = 0; v < 4; ++v) {
          uint4 u;
          u.x = pack_bf16(__uint_as_float(o[8 * v + 0]) * inv, __uint_as_float(o[8 * v + 1]) * inv);
          u.y = pack_bf16(__uint_as_float(o[8 * v + 2]) * inv, __uint_as_float(o[8 * v + 3]) * inv);
          u.z = pack_bf16(__uint_as_float(o[8 * v + 4]) * inv, __uint_as_float(o[8 * v + 5]) * inv);
          u.w = pack_bf16(__uint_as_float(o[8 * v + 6]) * inv, __uint_as_float(o[8 * v + 7]) * inv);
          op[v] = u;
        }
      }
      if (k >= 1 && k - 1 < n) {  // softmax(k-1) over this warp's 128 score columns
        const int j = k - 1;
        mbar_wait(s_full, (uint32_t)j & 1);
        fence_after();
        uint32_t s[128];
        {
          const uint32_t tb = tmem + lane_off + kColS + (uint32_t)(half * 128);
          uint32_t(&s0)[32] = *reinterpret_cast<uint32_t(*)[32]>(&s[0]);
          uint32_t(&s1)[32] = *reinterpret_cast<uint32_t(*)[32]>(&s[32]);
          uint32_t(&s2)[32] = *reinterpret_cast<uint32_t(*)[32]>(&s[64]);
          uint32_t(&s3)[32] = *reinterpret_cast<uint32_t(*)[32]>(&s[96]);
          tmem_ld32_nowait(tb, s0);
          tmem_ld32_nowait(tb + 32, s1);
          tmem_ld32_nowait(tb + 64, s2);
          tmem_ld32_nowait(tb + 96, s3);
          tmem_ld_wait();
        }
        float mx = -FLT_MAX;
#pragma unroll
        for (int e = 0; e < 128; ++e) mx = fmaxf(mx, __uint_as_float(s[e]));
        red[half * 128 + row] = mx;
        named_sync(bar_id, 64);  // both halves' scores are in registers from here on
        mx = fmaxf(mx, red[(half ^ 1) * 128 + row]);
        const float mc = mx * scale_log2;
        float part = 0.f;
#pragma unroll
        for (int c = 0; c < 4; ++c) {
          uint32_t w[16];
#pragma unroll
          for (int e = 0; e < 16; ++e) {
            const float p0 = ex2_fast(fmaf(__uint_as_float(s[32 * c + 2 * e]), scale_log2, -mc));
            const float p1 =
                ex2_fast(fmaf(__uint_as_float(s[32 * c + 2 * e + 1]), scale_log2, -mc));
            part += p0 + p1;
            w[e] = pack_bf16(p0, p1);
          }
          tmem_st16(tmem + lane_off + kColS + (uint32_t)(half * 64 + 16 * c), w);
        }
        tmem_st_wait();
        red[256 + half * 128 + row] = part;
        fence_before();
        named_sync(bar_id, 64);
        sum_prev = half == 0 ? part + red[256 + 128 + row] : red[256 + row] + part;
        __syncwarp();
        if (lane == 0) mbar_arrive_remote((j & 1) ? p_full_l1 : p_full_l0);
      }
    }
  }
  fence_before();
  cluster_sync_all();
  if (warp == 1) {
    fence_after();
    asm volatile("tcgen05.dealloc.cta_group::2.sync.aligned.b32 %0, %1;" ::"r"(tmem), "r"(512));
  }
}

}  // namespace

int g_fuse_qkv_attn = 1;

int qkv_attention_fused(const __nv_bfloat16 *x, const __nv_bfloat16 *w_qkv, const float *bias,
                        const float *colc, const float2 *ln_in, __nv_bfloat16 *ctx, int n_seqs,
                        int S, int H, int dh, int K, cudaStream_t s) {
  LV_REQUIRE(S == qa::kS && dh == qa::kDh && K % 64 == 0 && K > 0 && bias &&
                 (!ln_in || colc),
             LV_ERR_USAGE, "qkv_attention_fused: needs S = 256, dh = 64, K % 64 == 0");
  if (n_seqs <= 0) return LV_OK;
  const int D = H * dh;
  CUtensorMap ta, tb;
  LV_REQUIRE(make_tma_2d_bf16(&ta, x, (uint64_t)K, (uint64_t)n_seqs * S, (uint64_t)K * 2, 64, 128),
             LV_ERR_INTERNAL, "cuTensorMapEncodeTiled(x) failed");
  LV_REQUIRE(make_tma_2d_bf16(&tb, w_qkv, (uint64_t)K, (uint64_t)3 * D, (uint64_t)K * 2, 64, 32),
             LV_ERR_INTERNAL, "cuTensorMapEncodeTiled(W_qkv) failed");
  static bool attr = false;
  if (!attr) {
    LV_CHECK_CUDA(cudaFuncSetAttribute(qkv_attn_pair_kernel,
                                       cudaFuncAttributeMaxDynamicSharedMemorySize, qa::kSmem));
    attr = true;
  }
  const int items = n_seqs * H;
  const int pairs = std::min(items, tc_gemm_num_sms() / 2);
  qkv_attn_pair_kernel<<<2 * pairs, qa::kThreads, qa::kSmem, s>>>(
      ta, tb, bias, colc, ln_in, ctx, items, H, K, 1.4426950408889634f / 8.0f);
  note_launch();
  LV_CHECK_CUDA(cudaGetLastError());
  return LV_OK;
}

}  // namespace lv
