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
//        V -> [256 keys][32 dims] MN-major 64B-swizzled halves: dims [0, 32) live in
//             CTA 0, [32, 64) in CTA 1 (the peer's half: one bulk copy)   B of P.V
//  3. S = Q.K^T (pair MMA, M = 256, N = 256 keys, K = 64) -> TMEM [256, 512):
//     the B operand's N split across the pair IS the key split, so no K exchange.
//  4. Softmax: the two warps sharing a TMEM lane quarter own columns [0, 128) and
//     [128, 256) of a row (max / sum exchanged through shared memory); each writes
//     its P (bf16) over its own consumed scores (tcgen05.st).
//  5. O = P.V (pair TS-MMA: P from each CTA's TMEM, V MN-major, M = 256, N = 64)
//     -> TMEM [192, 256); ctx = O / rowsum through a swizzled shared-memory tile and
//     one TMA store per 32 rows (full 128-byte lines).
// Pipelining (one MMA thread, cycle k): G(k), PV(k-2), S(k-1); epilogue cycle k:
// drain(k), O-epilogue(k-2), softmax(k-1) — the GEMM of item k+1 runs on the
// tensor pipe while the epilogue warps do the softmax of item k-1. Q and K are
// single-buffered (drain(k) writes them once S(k-1) completed), V double-buffered
// (once P.V(k-2) completed), which leaves 4 operand stages in shared memory.
// Cross-CTA traffic is asynchronous only: the peer's V half goes as one 8 KB
// shared::cluster bulk copy completing on the receiver's mbarrier (no generic
// remote stores, so no cluster-scope memory fences on the critical path).
//
// Numerics: every value equals the unfused path bit for bit — the same fp32
// accumulators (fixed K order), the same epilogue expression, the same
// exponentials, the row sum in the two-half order attn_tc_kernel uses.
// Batch-invariant: an item never depends on other items.
#include <cuda.h>

#include <cfloat>
#include <cstdio>

#include "lv_kernels.cuh"
#include "lv_tc.cuh"

namespace lv {
namespace {
using namespace tc;

namespace qa {
constexpr int kThreads = 64 + 8 * 32;
constexpr int kS = 256, kDh = 64;
constexpr int kStages = 4;
constexpr int kABytes = 128 * 64 * 2;   // A half per stage (128 rows x 64 K)
constexpr int kBBytes = 96 * 64 * 2;    // B half per stage (96 weight rows x 64 K)
constexpr int kQKBytes = 128 * 128;     // [128][64] bf16
constexpr int kVBytes = kS * 64;        // [256 keys][32 dims] bf16
constexpr int kStgBytes = 128 * 64;     // this CTA's keys x the peer's 32 dims
constexpr int kOffB = kStages * kABytes;
constexpr int kOffQ = kOffB + kStages * kBBytes;
constexpr int kOffK = kOffQ + kQKBytes;
constexpr int kOffV = kOffK + kQKBytes;
constexpr int kOffStg = kOffV + 2 * kVBytes;
constexpr int kOffCtx = kOffStg + kStgBytes;     // [128 rows][64] bf16 context tile, 128B swizzle
constexpr int kOffCol = kOffCtx + kQKBytes;      // float [2 items][bias 192 | colc 192]
constexpr int kOffRed = kOffCol + 2 * 384 * 4;   // float [128 rows][max h0, max h1, sum h0, sum h1]
constexpr int kOffBar = kOffRed + 128 * 16;
constexpr int kSmem = kOffBar + 256 + 1024;
constexpr uint32_t kColAcc = 0, kColO = 192, kColS = 256;
constexpr int kBarDrain = 5;  // named barrier of the 8 epilogue warps (ids 1-4: row pairs)
static_assert(kOffQ % 1024 == 0 && kOffK % 1024 == 0 && kOffV % 1024 == 0 &&
                  kOffStg % 1024 == 0 && kOffCtx % 1024 == 0,
              "swizzled regions need 1 KB alignment");
static_assert(kSmem <= 232448, "shared memory");
}  // namespace qa

__device__ __forceinline__ float ex2_fast(float x) {
  float y;
  asm("ex2.approx.ftz.f32 %0, %1;" : "=f"(y) : "f"(x));
  return y;
}

// shared::cta -> shared::cluster bulk copy (async proxy), completion (complete_tx)
// on an mbarrier of the destination CTA
__device__ __forceinline__ void bulk_copy_to_peer(uint32_t dst, const void *src, uint32_t bytes,
                                                  uint32_t mbar) {
  asm volatile(
      "cp.async.bulk.shared::cluster.shared::cta.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::
          "r"(dst),
      "r"(smem_u32(src)), "r"(bytes), "r"(mbar)
      : "memory");
}

__global__ void __cluster_dims__(2, 1, 1) __launch_bounds__(qa::kThreads, 1)
    qkv_attn_pair_kernel(const __grid_constant__ CUtensorMap tmA,
                         const __grid_constant__ CUtensorMap tmB,
                         const __grid_constant__ CUtensorMap tmC, const float *__restrict__ bias,
                         const float *__restrict__ colc, const float2 *__restrict__ ln_in,
                         __nv_bfloat16 *__restrict__ ctx, int n_seqs, int H, int K,
                         int seq_major, float scale_log2) {
  using namespace qa;
  extern __shared__ uint8_t smem_raw[];
  uint8_t *smem = smem_raw + ((1024u - (tc::smem_u32(smem_raw) & 1023u)) & 1023u);  // 1 KB aligned, still shared space
  uint8_t *sA = smem, *sB = smem + kOffB, *sQ = smem + kOffQ, *sK = smem + kOffK,
          *sV = smem + kOffV, *sStg = smem + kOffStg, *sCtx = smem + kOffCtx;
  float *sCol = reinterpret_cast<float *>(smem + kOffCol);
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
  uint64_t *v_in = o_empty + 1;         // [2] the peer's V half landed here (complete_tx)
  uint64_t *v_fwd = v_in + 2;           // [2] leader: the peer's v_in completed
  uint32_t *tslot = reinterpret_cast<uint32_t *>(v_fwd + 2);

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
    mbar_init(s_full, 1);
    mbar_init(o_full, 1);
    mbar_init(o_empty, 16);
    for (int i = 0; i < 2; ++i) {
      mbar_init(&qkv_ready[i], 16);
      mbar_init(&p_full[i], 16);
      mbar_init(&v_in[i], 1);
      mbar_init(&v_fwd[i], 1);
    }
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
  // Work assignment. seq_major (large launches): pair p owns sequences p, p + P, ... and
  // runs their H heads back to back, so a sequence's x rows come from DRAM once (head 0)
  // and from L2 for the other heads, and the producer prefetches the next sequence's
  // rows into L2 one K block per head. Otherwise items (sequence, head) are dealt out
  // round-robin (small launches: every pair busy).
  const int n_items = n_seqs * H;
  const int n = seq_major ? (n_seqs > pair ? (n_seqs - pair + n_pairs - 1) / n_pairs : 0) * H
                          : (n_items > pair ? (n_items - pair + n_pairs - 1) / n_pairs : 0);
  auto item_of = [&](int i, int &seq, int &h) {
    if (seq_major) {
      const int t = i / H;
      seq = pair + t * n_pairs;
      h = i - t * H;
    } else {
      const int item = pair + i * n_pairs;
      seq = item / H;
      h = item - seq * H;
    }
  };
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
        int seq, h;
        item_of(i, seq, h);
        if (seq_major && h < kblocks && seq + n_pairs < n_seqs)  // next sequence's K block h -> L2
          asm volatile("cp.async.bulk.prefetch.tensor.2d.L2.global.tile [%0, {%1, %2}];" ::"l"(&tmA),
                       "r"(h * 64), "r"((seq + n_pairs) * kS + (int)rank * 128)
                       : "memory");
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
          const uint32_t vb = smem_u32(sV + (j & 1) * kVBytes);
#pragma unroll
          for (int t = 0; t < kS / 16; ++t)  // 16 keys = 1024 bytes of V per K step; P of
            // keys [128, 256) sits at S-region columns [128, 192) (softmax, below)
            umma_ts_pair(tmem + kColO, tmem + kColS + 8 * t + (t >= 8 ? 64 : 0),
                         sw64_desc(vb + 1024 * t), idesc_o, t != 0);
          umma_commit_pair(o_full);
        }
        if (k >= 1 && k - 1 < n) {  // S(k-1) = Q.K^T over the sequence's 256 keys
          const int j = k - 1;
          const uint32_t ph = (uint32_t)(j >> 1) & 1;
          mbar_wait(&qkv_ready[j & 1], ph);  // Q, K, own V halves written (both CTAs)
          mbar_wait(&v_in[j & 1], ph);       // the peer's V half landed in the leader
          mbar_wait(&v_fwd[j & 1], ph);      // ... and the leader's half in the peer
          fence_after();
          const uint64_t a0 = sw128_desc(smem_u32(sQ));
          const uint64_t b0 = sw128_desc(smem_u32(sK));
#pragma unroll
          for (int t = 0; t < kDh / 16; ++t)
            umma_bf16_pair(tmem + kColS, a0 + 2 * t, b0 + 2 * t, idesc_s, t != 0);
          umma_commit_pair(s_full);
        }
      }
    } else if (!leader && lane == 0) {  // forward the completion of this CTA's V copies
      const uint32_t fwd0 = map_to_rank(&v_fwd[0], 0), fwd1 = map_to_rank(&v_fwd[1], 0);
      for (int j = 0; j < n; ++j) {
        mbar_wait(&v_in[j & 1], (uint32_t)(j >> 1) & 1);
        mbar_arrive_remote((j & 1) ? fwd1 : fwd0);
      }
    }
  } else {
    const int ew = warp - 2;
    const int q = warp & 3;     // TMEM lane quarter
    const int half = ew >> 2;   // column half of the row this warp owns
    const int row = q * 32 + lane;  // row of the CTA's 128
    const int et = ew * 32 + lane;  // epilogue thread 0..255
    const bool elected = et == 0;
    const uint32_t lane_off = (uint32_t)(q * 32) << 16;
    const uint32_t acc_empty_l = map_to_rank(acc_empty, 0);
    const uint32_t o_empty_l = map_to_rank(o_empty, 0);
    const uint32_t qkv_ready_l0 = map_to_rank(&qkv_ready[0], 0);
    const uint32_t qkv_ready_l1 = map_to_rank(&qkv_ready[1], 0);
    const uint32_t p_full_l0 = map_to_rank(&p_full[0], 0), p_full_l1 = map_to_rank(&p_full[1], 0);
    const uint32_t peer = rank ^ 1u;
    const uint32_t peer_vin0 = map_to_rank(&v_in[0], peer), peer_vin1 = map_to_rank(&v_in[1], peer);
    const uint32_t peer_v0 = map_to_rank(sV + rank * kStgBytes, peer);  // my keys in the peer's V
    const int bar_id = 1 + q;  // the two warps of this lane quarter
    // column vectors (bias, LN-in colc) of item i -> sCol[i & 1] by cp.async, one item ahead
    auto load_cols = [&](int i) {
      if (et < 96) {
        int seq, h;
        item_of(i, seq, h);
        const int v = et / 48, c = et % 48;  // vector, 16-byte chunk of its 192 columns
        const int col = c * 4;               // 0..188: q [0,64) k [64,128) v [128,192)
        const int gcol = (col >> 6) * D + h * kDh + (col & 63);
        const float *src = v ? colc : bias;
        if (src)
          asm volatile("cp.async.ca.shared.global [%0], [%1], 16;" ::"r"(
                           smem_u32(sCol + (i & 1) * 384 + v * 192 + col)),
                       "l"(src + gcol)
                       : "memory");
      }
      asm volatile("cp.async.commit_group;" ::: "memory");
    };
    if (n > 0) load_cols(0);
    float sum_prev = 1.f;      // row sum of the item whose softmax ran last
    for (int k = 0; k < n + 2; ++k) {
      if (k < n) {  // drain(k): accumulators -> Q, K, V tiles in shared memory
        int seq, h_unused;
        item_of(k, seq, h_unused);
        const int grow = seq * kS + (int)rank * 128 + row;
        float mu = 0.f, rs = 1.f;
        if (ln_in) {
          const float2 st = __ldg(ln_in + grow);
          mu = st.x;
          rs = st.y;
        }
        asm volatile("cp.async.wait_group 0;" ::: "memory");
        named_sync(kBarDrain, 256);  // item k's column vectors visible; buffer (k+1)&1 free
        if (k + 1 < n) load_cols(k + 1);
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
        // epilogue of tc_gemm_pair_kernel (EPF_LN_IN or bias only), bf16 packed in place
        const float *cb = sCol + (k & 1) * 384 + half * 96;
#pragma unroll
        for (int c = 0; c < 3; ++c) {
#pragma unroll
          for (int j = 0; j < 8; ++j) {
            const float4 bb = *reinterpret_cast<const float4 *>(cb + 32 * c + 4 * j);
            const float bv[4] = {bb.x, bb.y, bb.z, bb.w};
            float v[4];
            if (ln_in) {
              const float4 cc = *reinterpret_cast<const float4 *>(cb + 192 + 32 * c + 4 * j);
              const float cv[4] = {cc.x, cc.y, cc.z, cc.w};
#pragma unroll
              for (int e = 0; e < 4; ++e)
                v[e] = fmaf(rs, fmaf(-mu, cv[e], __uint_as_float(r[32 * c + 4 * j + e])), bv[e]);
            } else {
#pragma unroll
              for (int e = 0; e < 4; ++e) v[e] = __uint_as_float(r[32 * c + 4 * j + e]) + bv[e];
            }
            r[16 * c + 2 * j] = pack_bf16(v[0], v[1]);
            r[16 * c + 2 * j + 1] = pack_bf16(v[2], v[3]);
          }
        }
        // Q / K of item k-1 consumed and its V copies complete (S(k-1) waited for them);
        // V slot k&1 (item k-2) consumed by P.V(k-2) in both CTAs
        if (k >= 1) mbar_wait(s_full, (uint32_t)(k - 1) & 1);
        if (k >= 2) mbar_wait(o_full, (uint32_t)(k - 2) & 1);
        const uint32_t sw = (uint32_t)(row & 7), kw = (uint32_t)((row >> 1) & 3);
#pragma unroll
        for (int c = 0; c < 3; ++c) {
          const int n0 = half * 96 + 32 * c;  // accumulator column: q [0,64) k [64,128) v [128,192)
          const int part = n0 >> 6, dim0 = n0 & 63;
          const uint32_t *w = &r[16 * c];
          if (part < 2) {  // Q or K: K-major [128][64], 128-byte swizzle
            uint8_t *dst = (part == 0 ? sQ : sK) + row * 128;
#pragma unroll
            for (int j = 0; j < 4; ++j) {
              const uint32_t chunk = (uint32_t)(dim0 >> 3) + j;
              *reinterpret_cast<uint4 *>(dst + ((chunk ^ sw) << 4)) =
                  make_uint4(w[4 * j], w[4 * j + 1], w[4 * j + 2], w[4 * j + 3]);
            }
          } else {  // V dims [dim0, dim0 + 32) belong to CTA dim0 / 32; key = 128 rank + row
            uint8_t *dst = (uint32_t)(dim0 >> 5) == rank
                               ? sV + (k & 1) * kVBytes + ((int)rank * 128 + row) * 64
                               : sStg + row * 64;  // byte image of the peer's rows
#pragma unroll
            for (int j = 0; j < 4; ++j)
              *reinterpret_cast<uint4 *>(dst + (((uint32_t)j ^ kw) << 4)) =
                  make_uint4(w[4 * j], w[4 * j + 1], w[4 * j + 2], w[4 * j + 3]);
          }
        }
        fence_async_smem();            // generic writes -> visible to the async proxy
        named_sync(kBarDrain, 256);    // the CTA's Q, K, V and staging rows are written
        if (elected) {
          mbar_expect_tx(&v_in[k & 1], kStgBytes);  // the peer's 8 KB for item k
          bulk_copy_to_peer(peer_v0 + (uint32_t)((k & 1) * kVBytes), sStg, kStgBytes,
                            (k & 1) ? peer_vin1 : peer_vin0);
        }
        __syncwarp();
        if (lane == 0) mbar_arrive_remote((k & 1) ? qkv_ready_l1 : qkv_ready_l0);
      }
      if (k >= 2) {  // O-epilogue(k-2): ctx = O / rowsum, staged per lane quarter, TMA store
        const int j = k - 2;
        int seq, h;
        item_of(j, seq, h);
        mbar_wait(o_full, (uint32_t)j & 1);
        fence_after();
        uint32_t o[32];
        tmem_ld32(tmem + lane_off + kColO + (uint32_t)(half * 32), o);
        fence_before();
        __syncwarp();
        if (lane == 0) mbar_arrive_remote(o_empty_l);
        const float inv = 1.f / sum_prev;
        uint32_t w[16];
#pragma unroll
        for (int e = 0; e < 16; ++e)
          w[e] = pack_bf16(__uint_as_float(o[2 * e]) * inv, __uint_as_float(o[2 * e + 1]) * inv);
        uint8_t *tile = sCtx + q * 32 * 128;  // this lane quarter's [32 rows][64] box
        if (half == 0 && lane == 0) bulk_wait_read<0>();  // the previous store has read it
        named_sync(bar_id, 64);
#pragma unroll
        for (int v = 0; v < 4; ++v)
          *reinterpret_cast<uint4 *>(tile + lane * 128 + ((uint32_t)((4 * half + v) ^ (lane & 7)) << 4)) =
              make_uint4(w[4 * v], w[4 * v + 1], w[4 * v + 2], w[4 * v + 3]);
        fence_async_smem();
        named_sync(bar_id, 64);
        if (half == 0 && lane == 0) {
          tma_store_2d(&tmC, tile, h * kDh, seq * kS + (int)rank * 128 + q * 32);
          bulk_commit();
        }
      }
      if (k >= 1 && k - 1 < n) {  // softmax(k-1) over this warp's 128 score columns
        const int j = k - 1;
        mbar_wait(s_full, (uint32_t)j & 1);
        fence_after();
        // scores in two passes over TMEM (pass 1: row max, pass 2: exponentials); each
        // half writes its P over its own consumed score columns: keys [0, 128) at TMEM
        // columns [0, 64) of the S region, keys [128, 256) at [128, 192)
        const uint32_t tb = tmem + lane_off + kColS + (uint32_t)(half * 128);
        float *rr = red + row * 4;  // this row's max / sum halves, shared by the row's two warps
        float mx = -FLT_MAX;
#pragma unroll 1
        for (int c = 0; c < 4; c += 2) {
          uint32_t s0[32], s1[32];
          tmem_ld32_nowait(tb + 32 * c, s0);
          tmem_ld32_nowait(tb + 32 * c + 32, s1);
          tmem_ld_wait();
#pragma unroll
          for (int e = 0; e < 32; ++e)
            mx = fmaxf(mx, fmaxf(__uint_as_float(s0[e]), __uint_as_float(s1[e])));
        }
        rr[half] = mx;
        named_sync(bar_id, 64);
        mx = fmaxf(mx, rr[half ^ 1]);
        const float mc = mx * scale_log2;
        float part = 0.f;
#pragma unroll 1
        for (int c = 0; c < 4; ++c) {
          uint32_t s0[32];
          tmem_ld32(tb + 32 * c, s0);
          uint32_t w[16];
#pragma unroll
          for (int e = 0; e < 16; ++e) {
            const float p0 = ex2_fast(fmaf(__uint_as_float(s0[2 * e]), scale_log2, -mc));
            const float p1 = ex2_fast(fmaf(__uint_as_float(s0[2 * e + 1]), scale_log2, -mc));
            part += p0 + p1;
            w[e] = pack_bf16(p0, p1);
          }
          tmem_st16(tb + 16 * c, w);
        }
        tmem_st_wait();
        rr[2 + half] = part;
        fence_before();
        named_sync(bar_id, 64);
        sum_prev = half == 0 ? part + rr[3] : rr[2] + part;
        __syncwarp();
        if (lane == 0) mbar_arrive_remote((j & 1) ? p_full_l1 : p_full_l0);
      }
    }
  }
  if (warp >= 2 && lane == 0) bulk_wait<0>();  // context stores complete before exit
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
  CUtensorMap tc_;
  LV_REQUIRE(make_tma_2d_bf16(&tc_, ctx, (uint64_t)D, (uint64_t)n_seqs * S, (uint64_t)D * 2, 64, 32),
             LV_ERR_INTERNAL, "cuTensorMapEncodeTiled(ctx) failed");
  static unsigned long long attr = 0;  // per device (first_on_device)
  if (first_on_device(attr)) {
    LV_CHECK_CUDA(cudaFuncSetAttribute(qkv_attn_pair_kernel,
                                       cudaFuncAttributeMaxDynamicSharedMemorySize, qa::kSmem));
  }
  const int items = n_seqs * H;
  const int pairs = std::min(items, tc_gemm_num_sms() / 2);
  const int seq_major = n_seqs >= 8 * pairs;
  qkv_attn_pair_kernel<<<2 * pairs, qa::kThreads, qa::kSmem, s>>>(
      ta, tb, tc_, bias, colc, ln_in, ctx, n_seqs, H, K, seq_major, 1.4426950408889634f / 8.0f);
  note_launch();
  const cudaError_t err = cudaGetLastError();
  if (err != cudaSuccess) {
    cudaFuncAttributes fa{};
    cudaFuncGetAttributes(&fa, qkv_attn_pair_kernel);
    std::fprintf(stderr, "qkv_attn_pair_kernel launch: %s (regs %d, static smem %zu, max dyn %d, "
                 "max threads %d, requested smem %d)\n", cudaGetErrorString(err), fa.numRegs,
                 fa.sharedSizeBytes, fa.maxDynamicSharedSizeBytes, fa.maxThreadsPerBlock,
                 qa::kSmem);
  }
  LV_CHECK_CUDA(err);
  return LV_OK;
}

}  // namespace lv
