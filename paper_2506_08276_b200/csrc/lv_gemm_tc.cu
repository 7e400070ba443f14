// lv_gemm_tc.cu — bf16 GEMM on the 5th-gen tensor cores (tcgen05 + TMEM + TMA), sm_100a.
//
//   out[M][N] = epi(A[M][K] . W[N][K]^T)      A = activations, W = nn.Linear weight
//
// This is the encoder's dense contraction (the "recompute" half of LEANN's
// two-level search: provider.embed_batch, vectors.py:201-211, becomes a packed
// encoder forward over every in-flight query's candidates).
//
// Structure (persistent, one CTA per SM, warp-specialised):
//   warp 0      one elected lane issues TMA loads of A/W K-slices (128B swizzle)
//               into a STAGES-deep shared-memory ring (mbarrier full/empty);
//   warp 1      allocates 512 TMEM columns; one lane issues tcgen05.mma
//               (M=128, N=BN, K=16, bf16 -> fp32) into one of two TMEM
//               accumulators and tcgen05.commit's the ring slot / accumulator;
//   warps 2..9  epilogue: tcgen05.ld the accumulator (each warp owns its TMEM
//               lane quarter and half of the columns), fused bias / erf-GELU /
//               residual, bf16 pack, 16-byte global stores; then release the
//               accumulator so the MMA of tile i+1 overlaps the epilogue of i.
// Batch-invariance: each output element is one fixed-order K reduction, no
// split-K, so a row's result does not depend on M or on its tile neighbours.
#include <cuda.h>
#include <cudaTypedefs.h>

#include <mutex>

#include "lv_kernels.cuh"
#include "lv_tc.cuh"

namespace lv {
int g_long_k_single = 1;  // residual GEMMs with K > 1024: single box buffer, 5 stages (kMode 4)
int g_split_single = 0;   // split-residual GEMMs with K <= 1024: kMode 5 instead of 6
namespace {

constexpr int kBM = 128;
constexpr int kBK = 64;  // one 128-byte swizzle atom of bf16
constexpr int kEpiWarps = 8;
constexpr int kThreads = 64 + kEpiWarps * 32;

template <int BN>
struct Cfg {
  static constexpr int kStages = BN == 256 ? 4 : 6;
  static constexpr int kABytes = kBM * kBK * 2;
  static constexpr int kBBytes = BN * kBK * 2;
  static constexpr int kStageBytes = kABytes + kBBytes;
  static constexpr int kTmemCols = 2 * BN;  // two accumulators
  static constexpr int kSmem = kStages * kStageBytes + 1024 /*align*/ + 256 /*barriers*/;
};

using namespace tc;

// GELU in the bf16 epilogue: tanh form on the MUFU pipe (7 instructions vs ~25
// for erff). |gelu_tanh - gelu_erf| < 5e-4 over the real line, below the
// 2^-8 relative resolution of the bf16 output; the fp32 parity encoder keeps
// the exact erf form (lv_encoder.cu).
__device__ __forceinline__ float gelu_erf(float x) {
  const float u = x * fmaf(0.0356774081f, x * x, 0.7978845608f);
  float t;
  asm("tanh.approx.f32 %0, %1;" : "=f"(t) : "f"(u));
  const float hx = 0.5f * x;
  return fmaf(hx, t, hx);
}

template <int BN>
__global__ void __launch_bounds__(kThreads, 1)
    tc_gemm_kernel(const __grid_constant__ CUtensorMap tmA, const __grid_constant__ CUtensorMap tmB,
                   int M, int N, int K, const float *__restrict__ bias,
                   const __nv_bfloat16 *__restrict__ residual, __nv_bfloat16 *__restrict__ out,
                   int epi) {
  using C = Cfg<BN>;
  extern __shared__ uint8_t smem_raw[];
  uint8_t *smem = smem_raw + ((1024u - (tc::smem_u32(smem_raw) & 1023u)) & 1023u);  // 1 KB aligned, still shared space
  uint8_t *sA = smem;
  uint8_t *sB = smem + C::kStages * C::kABytes;
  uint64_t *full = reinterpret_cast<uint64_t *>(sB + C::kStages * C::kBBytes);
  uint64_t *empty = full + C::kStages;
  uint64_t *tfull = empty + C::kStages;
  uint64_t *tempty = tfull + 2;
  uint32_t *tslot = reinterpret_cast<uint32_t *>(tempty + 2);

  const int warp = threadIdx.x >> 5;
  const int lane = threadIdx.x & 31;
  if (threadIdx.x == 0) {
    for (int s = 0; s < C::kStages; ++s) {
      mbar_init(&full[s], 1);
      mbar_init(&empty[s], 1);
    }
    for (int a = 0; a < 2; ++a) {
      mbar_init(&tfull[a], 1);
      mbar_init(&tempty[a], kEpiWarps);
    }
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  if (warp == 1) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(
                     smem_u32(tslot)),
                 "r"(C::kTmemCols));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
  }
  fence_before();
  __syncthreads();
  fence_after();
  const uint32_t tmem_base = *tslot;

  const int m_tiles = (M + kBM - 1) / kBM;
  const int n_tiles = N / BN;
  const int num_tiles = m_tiles * n_tiles;
  const int kblocks = K / kBK;

  if (warp == 0) {
    if (lane == 0) {
      asm volatile("prefetch.tensormap [%0];" ::"l"(&tmA) : "memory");
      asm volatile("prefetch.tensormap [%0];" ::"l"(&tmB) : "memory");
      uint64_t pol_a, pol_b;  // A blocks are reused by every N tile; weights stay in L2
      asm volatile("createpolicy.fractional.L2::evict_normal.b64 %0, 1.0;" : "=l"(pol_a));
      asm volatile("createpolicy.fractional.L2::evict_last.b64 %0, 1.0;" : "=l"(pol_b));
      int stage = 0;
      uint32_t phase = 0;
      for (int tile = blockIdx.x; tile < num_tiles; tile += gridDim.x) {
        const int m0 = (tile / n_tiles) * kBM;
        const int n0 = (tile % n_tiles) * BN;
        for (int kb = 0; kb < kblocks; ++kb) {
          mbar_wait(&empty[stage], phase ^ 1);
          mbar_expect_tx(&full[stage], C::kStageBytes);
          tma_load_2d(sA + stage * C::kABytes, &tmA, &full[stage], kb * kBK, m0, pol_a);
          tma_load_2d(sB + stage * C::kBBytes, &tmB, &full[stage], kb * kBK, n0, pol_b);
          if (++stage == C::kStages) {
            stage = 0;
            phase ^= 1;
          }
        }
      }
    }
  } else if (warp == 1) {
    if (lane == 0) {
      constexpr uint32_t idesc = idesc_bf16(kBM, BN);
      int stage = 0;
      uint32_t phase = 0;
      int acc = 0;
      uint32_t acc_phase = 0;
      for (int tile = blockIdx.x; tile < num_tiles; tile += gridDim.x) {
        mbar_wait(&tempty[acc], acc_phase ^ 1);
        fence_after();
        const uint32_t d = tmem_base + (uint32_t)(acc * BN);
        for (int kb = 0; kb < kblocks; ++kb) {
          mbar_wait(&full[stage], phase);
          fence_after();
          const uint64_t a0 = sw128_desc(smem_u32(sA + stage * C::kABytes));
          const uint64_t b0 = sw128_desc(smem_u32(sB + stage * C::kBBytes));
#pragma unroll
          for (int k = 0; k < kBK / 16; ++k)  // +32 bytes per K=16 step inside the atom
            umma_ss(d, a0 + 2 * k, b0 + 2 * k, idesc, (kb | k) != 0);
          umma_commit(&empty[stage]);
          if (++stage == C::kStages) {
            stage = 0;
            phase ^= 1;
          }
        }
        umma_commit(&tfull[acc]);
        acc ^= 1;
        if (acc == 0) acc_phase ^= 1;
      }
    }
  } else {
    const int ew = warp - 2;
    const int q = warp & 3;            // TMEM lane quarter this warp may access
    const int half = ew >> 2;          // which half of the tile's columns
    constexpr int kCols = BN / 2;
    int acc = 0;
    uint32_t acc_phase = 0;
    for (int tile = blockIdx.x; tile < num_tiles; tile += gridDim.x) {
      const int m0 = (tile / n_tiles) * kBM;
      const int n0 = (tile % n_tiles) * BN;
      mbar_wait(&tfull[acc], acc_phase);
      fence_after();
      const int row = m0 + q * 32 + lane;
      const bool live = row < M;
#pragma unroll 1
      for (int c = 0; c < kCols; c += 32) {
        const int col = half * kCols + c;
        uint32_t r[32];
        tmem_ld32(tmem_base + ((uint32_t)(q * 32) << 16) + (uint32_t)(acc * BN + col), r);
        if (live) {
          const int gn = n0 + col;
          const float4 *b4 = reinterpret_cast<const float4 *>(bias + gn);
          float v[32];
#pragma unroll
          for (int j = 0; j < 8; ++j) {
            float4 bb = __ldg(b4 + j);
            v[4 * j + 0] = __uint_as_float(r[4 * j + 0]) + bb.x;
            v[4 * j + 1] = __uint_as_float(r[4 * j + 1]) + bb.y;
            v[4 * j + 2] = __uint_as_float(r[4 * j + 2]) + bb.z;
            v[4 * j + 3] = __uint_as_float(r[4 * j + 3]) + bb.w;
          }
          if (epi == EPI_BIAS_GELU) {
#pragma unroll
            for (int j = 0; j < 32; ++j) v[j] = gelu_erf(v[j]);
          } else if (epi == EPI_BIAS_RESIDUAL) {
            const uint4 *rp = reinterpret_cast<const uint4 *>(residual + (size_t)row * N + gn);
#pragma unroll
            for (int j = 0; j < 4; ++j) {
              uint4 u = __ldg(rp + j);
              const __nv_bfloat162 *h = reinterpret_cast<const __nv_bfloat162 *>(&u);
#pragma unroll
              for (int e = 0; e < 4; ++e) {
                float2 f = __bfloat1622float2(h[e]);
                v[8 * j + 2 * e] += f.x;
                v[8 * j + 2 * e + 1] += f.y;
              }
            }
          }
          uint4 *op = reinterpret_cast<uint4 *>(out + (size_t)row * N + gn);
#pragma unroll
          for (int j = 0; j < 4; ++j) {
            uint4 u;
            u.x = pack_bf16(v[8 * j + 0], v[8 * j + 1]);
            u.y = pack_bf16(v[8 * j + 2], v[8 * j + 3]);
            u.z = pack_bf16(v[8 * j + 4], v[8 * j + 5]);
            u.w = pack_bf16(v[8 * j + 6], v[8 * j + 7]);
            op[j] = u;
          }
        }
      }
      fence_before();
      __syncwarp();
      if (lane == 0) mbar_arrive(&tempty[acc]);
      acc ^= 1;
      if (acc == 0) acc_phase ^= 1;
    }
  }
  fence_before();
  __syncthreads();
  if (warp == 1) {
    fence_after();
    asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem_base),
                 "r"(C::kTmemCols));
  }
}

// ----------------------------------------------------------------------------
// 2-CTA variant (cta_group::2): an SM pair computes a 256 x 256 tile. CTA r of
// the pair TMA-loads A rows [m0 + 128 r, +128) and B rows [n0 + 128 r, +128)
// (its half of N) into its own ring; both loads complete on the LEADER's full
// barrier. The leader's single elected thread issues tcgen05.mma.cta_group::2
// (M=256, N=256, K=16), which reads A and B halves from both CTAs' shared
// memory and writes rows 0-127 of D to the leader's TMEM and rows 128-255 to
// the peer's. Commits are multicast to both CTAs (ring slot free / accumulator
// full); the peer's epilogue warps release the accumulator with a remote
// arrive on the leader's barrier. Per SM this loads (128 + 128) x 64 x 2 bytes
// per 128 x 256 x 64 MACs: 1.5x the MACs per L2 byte of the 1-CTA kernel,
// whose 50%-busy tensor pipe was bound by TMA/L2 throughput.
// Shared-memory budget per CTA (<= 227 KB): residual GEMMs double-buffer the
// epilogue boxes (residual prefetch one box ahead) and keep 4 operand stages;
// the others single-buffer the output box and keep 5.
template <int kMode>
struct PairCfg;
constexpr int kHalfBytes = 128 * kBK * 2;          // 16 KB: A or B half per stage
constexpr int kStageBytes2 = 2 * kHalfBytes;        // per CTA
// epilogue staging: per epilogue warp two [32 rows][64 cols] bf16 boxes (4 KB
// each, 128-byte swizzle) — residual tile in (TMA load), output tile out (TMA store)
constexpr int kBoxBytes = 32 * 64 * 2;
constexpr int kLoBoxBytes = 32 * 64;  // EPF_SPLIT: int8 [32 rows][64 cols], 64-byte swizzle
// per epilogue warp, two boxes' column vectors (bias, colc, gamma, beta: 64 fp32 each)
constexpr int kColVecBytes = 4 * 64 * 4;
constexpr int kColVecTotal = kEpiWarps * 2 * kColVecBytes;
// kMode 0: no residual (1 box buffer, 5 stages); 1: residual, 2 box buffers
// (the next box's residual prefetched), 4 stages. (A 3-buffer / 3-stage short-K
// variant measured slower and was removed.)
template <int kMode>
struct PairCfg {
  // kMode 3: SwiGLU epilogue (no residual; gate/up interleaved per 64 columns)
  // kMode 4: residual with a single box buffer and 5 stages (long-K GEMMs: the
  // epilogue has slack, the residual box is loaded when the box starts)
  // kMode 5: split residual (EPF_SPLIT), long K: one (hi bf16, lo int8) box
  //          pair per warp, 5 stages
  // kMode 6: split residual, short K: two box pairs (next box's residual
  //          prefetched), 3 stages
  static constexpr bool kRes = kMode == 1 || kMode == 4 || kMode >= 5;
  static constexpr bool kSplit = kMode >= 5;
  static constexpr int kStages = (kMode == 0 || kMode == 3 || kMode == 4 || kMode == 5) ? 5
                                 : kMode == 1 ? 4 : 3;
  static constexpr int kBufs = (kMode == 0 || kMode == 3 || kMode == 4 || kMode == 5) ? 1 : 2;
  static constexpr int kPairBytes = kBoxBytes + (kSplit ? kLoBoxBytes : 0);
  static constexpr int kStagingBytes = kEpiWarps * kBufs * kPairBytes;
  static constexpr int kSmem = kStages * kStageBytes2 + kStagingBytes + kColVecTotal + 1024 + 512;
};

template <int kMode>
__global__ void __cluster_dims__(2, 1, 1) __launch_bounds__(kThreads, 1)
    tc_gemm_pair_kernel(const __grid_constant__ CUtensorMap tmA,
                        const __grid_constant__ CUtensorMap tmB,
                        const __grid_constant__ CUtensorMap tmO,
                        const __grid_constant__ CUtensorMap tmR,
                        const __grid_constant__ CUtensorMap tmRL,
                        const __grid_constant__ CUtensorMap tmOL, int M, int N, int K,
                        const EpiParams ep) {
  constexpr int BN = 256;
  extern __shared__ uint8_t smem_raw[];
  uint8_t *smem = smem_raw + ((1024u - (tc::smem_u32(smem_raw) & 1023u)) & 1023u);  // 1 KB aligned, still shared space
  uint8_t *sA = smem;
  constexpr bool kRes = PairCfg<kMode>::kRes;
  constexpr bool kSplit = PairCfg<kMode>::kSplit;
  constexpr int kBufs = PairCfg<kMode>::kBufs;
  constexpr int kStages2 = PairCfg<kMode>::kStages;
  constexpr int kStagingBytes = PairCfg<kMode>::kStagingBytes;
  uint8_t *sB = smem + kStages2 * kHalfBytes;
  uint8_t *sStage = sB + kStages2 * kHalfBytes;
  float *sColVec = reinterpret_cast<float *>(sStage + kStagingBytes);
  uint64_t *full = reinterpret_cast<uint64_t *>(sStage + kStagingBytes + kColVecTotal);
  uint64_t *empty = full + kStages2;
  uint64_t *tfull = empty + kStages2;
  uint64_t *tempty = tfull + 2;
  uint64_t *rbar = tempty + 2;  // [kEpiWarps][3] residual-box arrivals
  uint32_t *tslot = reinterpret_cast<uint32_t *>(rbar + 3 * kEpiWarps);

  const int warp = threadIdx.x >> 5;
  const int lane = threadIdx.x & 31;
  const uint32_t rank = cluster_rank();
  const bool leader = rank == 0;
  if (threadIdx.x == 0) {
    for (int s = 0; s < kStages2; ++s) {
      mbar_init(&full[s], 1);
      mbar_init(&empty[s], 1);
    }
    for (int a = 0; a < 2; ++a) {
      mbar_init(&tfull[a], 1);
      mbar_init(&tempty[a], 2 * kEpiWarps);
    }
    for (int a = 0; a < 3 * kEpiWarps; ++a) mbar_init(&rbar[a], 1);
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
  const uint32_t tmem_base = *tslot;

  const int pair = blockIdx.x >> 1;
  const int n_pairs = gridDim.x >> 1;
  const int m_tiles = (M + 255) / 256;
  const int n_tiles = N / BN;
  const int num_tiles = m_tiles * n_tiles;
  const int kblocks = K / kBK;

  if (warp == 0) {
    if (lane == 0) {
      asm volatile("prefetch.tensormap [%0];" ::"l"(&tmA) : "memory");
      asm volatile("prefetch.tensormap [%0];" ::"l"(&tmB) : "memory");
      uint64_t pol_a, pol_b;
      asm volatile("createpolicy.fractional.L2::evict_normal.b64 %0, 1.0;" : "=l"(pol_a));
      asm volatile("createpolicy.fractional.L2::evict_last.b64 %0, 1.0;" : "=l"(pol_b));
      int stage = 0;
      uint32_t phase = 0;
      for (int tile = pair; tile < num_tiles; tile += n_pairs) {
        const int m0 = (tile / n_tiles) * 256 + (int)rank * 128;
        const int n0 = (tile % n_tiles) * BN + (int)rank * 128;
        for (int kb = 0; kb < kblocks; ++kb) {
          mbar_wait(&empty[stage], phase ^ 1);
          const uint32_t fb = map_to_rank(&full[stage], 0);
          if (leader) mbar_expect_tx(&full[stage], 2 * kStageBytes2);
          tma_load_2d_pair(sA + stage * kHalfBytes, &tmA, fb, kb * kBK, m0, pol_a);
          tma_load_2d_pair(sB + stage * kHalfBytes, &tmB, fb, kb * kBK, n0, pol_b);
          if (++stage == kStages2) {
            stage = 0;
            phase ^= 1;
          }
        }
      }
    }
  } else if (warp == 1) {
    if (leader && lane == 0) {
      constexpr uint32_t idesc = idesc_bf16(256, BN);
      int stage = 0;
      uint32_t phase = 0;
      int acc = 0;
      uint32_t acc_phase = 0;
      for (int tile = pair; tile < num_tiles; tile += n_pairs) {
        mbar_wait(&tempty[acc], acc_phase ^ 1);
        fence_after();
        const uint32_t d = tmem_base + (uint32_t)(acc * BN);
        for (int kb = 0; kb < kblocks; ++kb) {
          mbar_wait(&full[stage], phase);
          fence_after();
          const uint64_t a0 = sw128_desc(smem_u32(sA + stage * kHalfBytes));
          const uint64_t b0 = sw128_desc(smem_u32(sB + stage * kHalfBytes));
#pragma unroll
          for (int k = 0; k < kBK / 16; ++k)
            umma_bf16_pair(d, a0 + 2 * k, b0 + 2 * k, idesc, (kb | k) != 0);
          umma_commit_pair(&empty[stage]);
          if (++stage == kStages2) {
            stage = 0;
            phase ^= 1;
          }
        }
        umma_commit_pair(&tfull[acc]);
        acc ^= 1;
        if (acc == 0) acc_phase ^= 1;
      }
    }
  } else if constexpr (kMode == 3) {
    // SwiGLU epilogue: the weight rows are interleaved per 64 (gate block g,
    // then up block g), so a warp's 128 accumulator columns hold gate and up
    // of the same 64 output columns: out = silu(gate) * up, one [32 x 64]
    // output box per tile and warp (output width N / 2). Bias-free.
    const int ew = warp - 2;
    const int q = warp & 3;
    const int half = ew >> 2;
    uint8_t *box = sStage + ew * kBoxBytes;
    const uint32_t tempty_leader0 = map_to_rank(&tempty[0], 0);
    const uint32_t tempty_leader1 = map_to_rank(&tempty[1], 0);
    const uint32_t row_off = (uint32_t)lane * 128;
    const uint32_t sw = (uint32_t)(lane & 7);
    int acc = 0;
    uint32_t acc_phase = 0;
    for (int tile = pair; tile < num_tiles; tile += n_pairs) {
      const int y = (tile / n_tiles) * 256 + (int)rank * 128 + q * 32;
      const int xo = (tile % n_tiles) * (BN / 2) + half * 64;
      float rs = 1.f;  // RMSNorm folded in (EPF_LN_IN, mean 0): silu(rs g) * (rs u)
      if ((ep.flags & EPF_LN_IN) && y + lane < M) rs = __ldg(ep.ln_in + y + lane).y;
      mbar_wait(&tfull[acc], acc_phase);
      fence_after();
      if (lane == 0) bulk_wait_read<0>();  // the previous tile's store has read the box
      __syncwarp();
#pragma unroll 1
      for (int c = 0; c < 2; ++c) {
        uint32_t g[32], u[32];
        const uint32_t ta = tmem_base + ((uint32_t)(q * 32) << 16) +
                            (uint32_t)(acc * BN + half * 128 + c * 32);
        tmem_ld32_nowait(ta, g);
        tmem_ld32_nowait(ta + 64, u);
        tmem_ld_wait();
        if (c == 1) {  // accumulator fully read
          fence_before();
          __syncwarp();
          if (lane == 0) mbar_arrive_remote(acc ? tempty_leader1 : tempty_leader0);
        }
#pragma unroll
        for (int k = 0; k < 4; ++k) {
          uint32_t w[4];
#pragma unroll
          for (int e = 0; e < 4; ++e) {
            const float g0 = rs * __uint_as_float(g[8 * k + 2 * e]);
            const float g1 = rs * __uint_as_float(g[8 * k + 2 * e + 1]);
            const float s0 = __fdividef(g0, 1.f + __expf(-g0)), s1 = __fdividef(g1, 1.f + __expf(-g1));
            w[e] = pack_bf16(s0 * rs * __uint_as_float(u[8 * k + 2 * e]),
                             s1 * rs * __uint_as_float(u[8 * k + 2 * e + 1]));
          }
          *reinterpret_cast<uint4 *>(box + row_off + (((uint32_t)(c * 4 + k) ^ sw) << 4)) =
              make_uint4(w[0], w[1], w[2], w[3]);
        }
      }
      fence_async_smem();
      __syncwarp();
      if (lane == 0) {
        tma_store_2d(&tmO, box, xo, y);
        bulk_commit();
      }
      acc ^= 1;
      if (acc == 0) acc_phase ^= 1;
    }
    if (lane == 0) bulk_wait<0>();
  } else {
    // Epilogue: each warp owns 32 accumulator rows (its TMEM lane quarter) x
    // 128 columns (its half), processed as two 64-column boxes. A box goes
    // TMEM -> registers (+bias, GELU / +residual) -> swizzled shared-memory
    // staging -> one TMA store; the residual box arrives by TMA one box ahead.
    // Every global access is a coalesced bulk transfer (a thread-per-row
    // st.global would touch 32 cache lines per instruction).
    const int ew = warp - 2;
    const int q = warp & 3;
    const int half = ew >> 2;
    const int fl = ep.flags;
    constexpr bool has_res = kRes;
    // per buffer: the bf16 box, then (kSplit) its int8 correction box
    constexpr int kPair = PairCfg<kMode>::kPairBytes;
    uint8_t *stg = sStage + ew * kBufs * kPair;
    constexpr uint32_t kResBytes = kPair;
    uint64_t *rb = rbar + 3 * ew;
    uint32_t rph = 0;  // parity bit per buffer
    const uint32_t tempty_leader0 = map_to_rank(&tempty[0], 0);
    const uint32_t tempty_leader1 = map_to_rank(&tempty[1], 0);
    uint64_t pol_r = 0;
    if (has_res) asm volatile("createpolicy.fractional.L2::evict_first.b64 %0, 1.0;" : "=l"(pol_r));
    auto box_coords = [&](int tile, int b, int &x, int &y) {
      y = (tile / n_tiles) * 256 + (int)rank * 128 + q * 32;
      x = (tile % n_tiles) * BN + half * 128 + b * 64;
    };
    if (has_res && lane == 0 && pair < num_tiles) {
      int x, y;
      box_coords(pair, 0, x, y);
      mbar_expect_tx(&rb[0], kResBytes);
      tma_load_2d(stg, &tmR, &rb[0], x, y, pol_r);
      if constexpr (kSplit) tma_load_2d(stg + kBoxBytes, &tmRL, &rb[0], x, y, pol_r);
    }
    // column vectors of a box -> this warp's shared buffer, by cp.async (one
    // box ahead; reading them with per-chunk global loads exposed an L2 round
    // trip per 8 columns)
    float *cvw = sColVec + ew * 2 * (kColVecBytes / 4);
    auto load_colvecs = [&](int cbuf, int x) {
      float *dst = cvw + cbuf * (kColVecBytes / 4);
      const int l16 = lane & 15, hi = lane >> 4;
      const float *v0 = hi ? ep.colc : ep.bias;
      if (!hi || (fl & EPF_LN_IN))
        asm volatile("cp.async.ca.shared.global [%0], [%1], 16;" ::"r"(
                         smem_u32(dst + hi * 64 + 4 * l16)),
                     "l"(v0 + x + 4 * l16)
                     : "memory");
      if (fl & EPF_RES_LN) {
        const float *v1 = hi ? ep.res_b : ep.res_g;
        asm volatile("cp.async.ca.shared.global [%0], [%1], 16;" ::"r"(
                         smem_u32(dst + (2 + hi) * 64 + 4 * l16)),
                     "l"(v1 + x + 4 * l16)
                     : "memory");
      }
      asm volatile("cp.async.commit_group;" ::: "memory");
    };
    if (pair < num_tiles) {
      int x, y;
      box_coords(pair, 0, x, y);
      load_colvecs(0, x);
    }
    // 16-byte chunk c of row r of a 128-byte-swizzled box
    const uint32_t row_off = (uint32_t)lane * 128;
    const uint32_t sw = (uint32_t)(lane & 7);
    int acc = 0;
    uint32_t acc_phase = 0;
    int blk = 0;
    // per-row LayerNorm statistics (EPF_LN_IN / EPF_RES_LN) of a tile, loaded one
    // tile ahead so their global-load latency hides behind the current tile
    // (both boxes of a tile share rows)
    auto row_stats = [&](int t, float4 &st) {
      st = make_float4(0.f, 1.f, 0.f, 1.f);
      if (t >= num_tiles) return;
      const int row = (t / n_tiles) * 256 + (int)rank * 128 + q * 32 + lane;
      if (row >= M) return;
      if (fl & EPF_LN_IN) {
        const float2 v = __ldg(ep.ln_in + row);
        st.x = v.x;
        st.y = v.y;
      }
      if (fl & EPF_RES_LN) {
        const float2 v = __ldg(ep.res_ln + row);
        st.z = v.x;
        st.w = v.y;
      }
    };
    float4 st_cur, st_next;
    row_stats(pair, st_cur);
    for (int tile = pair; tile < num_tiles; tile += n_pairs) {
      row_stats(tile + n_pairs, st_next);
      mbar_wait(&tfull[acc], acc_phase);
      fence_after();
#pragma unroll 1
      for (int b = 0; b < 2; ++b, ++blk) {
        const int buf = blk & 1;            // column-vector buffer
        const int bb = blk % kBufs;         // epilogue box buffer
        const int nb = (blk + 1) % kBufs;   // the next box's buffer
        uint8_t *box = stg + bb * kPair;
        uint8_t *lobox = box + kBoxBytes + (uint32_t)lane * 64;  // kSplit: this row's int8s
        const uint32_t sw64 = (uint32_t)((lane >> 1) & 3);          // 64-byte swizzle of the row
        uint4 lo_in = make_uint4(0u, 0u, 0u, 0u);
        uint32_t lo_out[4] = {0u, 0u, 0u, 0u};
        int x, y;
        box_coords(tile, b, x, y);
        const int grow = y + lane;  // this thread's output row
        const bool live = grow < M;
        const float mu_i = st_cur.x, rs_i = st_cur.y, mu_r = st_cur.z, rs_r = st_cur.w;
        {  // next box's column vectors into the other buffer
          const int nt = b == 0 ? tile : tile + n_pairs;
          if (nt < num_tiles) {
            int nx, ny;
            box_coords(nt, b ^ 1, nx, ny);
            load_colvecs(buf ^ 1, nx);
          } else {
            asm volatile("cp.async.commit_group;" ::: "memory");
          }
        }
        uint32_t r[64];
        {
          uint32_t(&r0)[32] = *reinterpret_cast<uint32_t(*)[32]>(&r[0]);
          uint32_t(&r1)[32] = *reinterpret_cast<uint32_t(*)[32]>(&r[32]);
          const uint32_t ta = tmem_base + ((uint32_t)(q * 32) << 16) +
                              (uint32_t)(acc * BN + half * 128 + b * 64);
          tmem_ld32_nowait(ta, r0);
          tmem_ld32_nowait(ta + 32, r1);
          tmem_ld_wait();
        }
        if (b == 1) {  // accumulator fully read: the MMA of the next tile may reuse it
          fence_before();
          __syncwarp();
          if (lane == 0) mbar_arrive_remote(acc ? tempty_leader1 : tempty_leader0);
        }
        // next box's residual into the other buffer (its previous TMA store
        // must have finished reading it)
        if (lane == 0) {
          if constexpr (kRes && kBufs > 1) {
            const int nt = b == 0 ? tile : tile + n_pairs;
            if (nt < num_tiles) {
              bulk_wait_read<kBufs - 2>();  // the store that last used buffer nb has read it
              int nx, ny;
              box_coords(nt, b ^ 1, nx, ny);
              mbar_expect_tx(&rb[nb], kResBytes);
              tma_load_2d(stg + nb * kPair, &tmR, &rb[nb], nx, ny, pol_r);
              if constexpr (kSplit)
                tma_load_2d(stg + nb * kPair + kBoxBytes, &tmRL, &rb[nb], nx, ny, pol_r);
            }
          } else if constexpr (kRes) {  // single buffer: this box's residual (box 0: prologue)
            if (blk > 0) {
              bulk_wait_read<0>();
              mbar_expect_tx(&rb[0], kResBytes);
              tma_load_2d(stg, &tmR, &rb[0], x, y, pol_r);
              if constexpr (kSplit) tma_load_2d(stg + kBoxBytes, &tmRL, &rb[0], x, y, pol_r);
            }
          } else {
            bulk_wait_read<0>();  // the previous box's store has read the (single) buffer
          }
        }
        __syncwarp();
        if (has_res) {
          mbar_wait(&rb[bb], (rph >> bb) & 1);
          rph ^= 1u << bb;
        }
        asm volatile("cp.async.wait_group 1;" ::: "memory");  // this box's column vectors
        __syncwarp();
        const float *cv = cvw + buf * (kColVecBytes / 4);
        float sk = 0.f, s1 = 0.f, s2 = 0.f;  // shifted sums of the rounded outputs (EPF_STATS)
        const float4 *b4 = reinterpret_cast<const float4 *>(cv);
#pragma unroll
        for (int c = 0; c < 8; ++c) {  // 8 columns per 16-byte chunk
          const float4 bl = b4[2 * c], bh = b4[2 * c + 1];
          const float bb[8] = {bl.x, bl.y, bl.z, bl.w, bh.x, bh.y, bh.z, bh.w};
          float v[8];
          if (fl & EPF_LN_IN) {
            const float4 *c4 = reinterpret_cast<const float4 *>(cv + 64 + 8 * c);
            const float4 cl = c4[0], ch = c4[1];
            const float cc[8] = {cl.x, cl.y, cl.z, cl.w, ch.x, ch.y, ch.z, ch.w};
#pragma unroll
            for (int e = 0; e < 8; ++e)
              v[e] = fmaf(rs_i, fmaf(-mu_i, cc[e], __uint_as_float(r[8 * c + e])), bb[e]);
          } else {
#pragma unroll
            for (int e = 0; e < 8; ++e) v[e] = __uint_as_float(r[8 * c + e]) + bb[e];
          }
          uint4 *cp = reinterpret_cast<uint4 *>(box + row_off + (((uint32_t)c ^ sw) << 4));
          if (fl & EPF_GELU) {
#pragma unroll
            for (int e = 0; e < 8; ++e) v[e] = gelu_erf(v[e]);
          }
          // kSplit: the row's int8 corrections, 16 per 16-byte chunk (two column chunks)
          uint4 *cpl = reinterpret_cast<uint4 *>(lobox + (((uint32_t)(c >> 1) ^ sw64) << 4));
          if constexpr (kSplit)
            if ((c & 1) == 0) lo_in = *cpl;
          if (has_res) {
            const uint4 u = *cp;
            const __nv_bfloat162 *h = reinterpret_cast<const __nv_bfloat162 *>(&u);
            float rv[8];
#pragma unroll
            for (int e = 0; e < 4; ++e) {
              const float2 f = __bfloat1622float2(h[e]);
              rv[2 * e] = f.x;
              rv[2 * e + 1] = f.y;
            }
            if constexpr (kSplit) {  // residual = hi + lo * 2^-13
              const uint32_t w0 = (c & 1) ? lo_in.z : lo_in.x, w1 = (c & 1) ? lo_in.w : lo_in.y;
#pragma unroll
              for (int e = 0; e < 4; ++e) {
                rv[e] = fmaf(lo8_get(w0, e), kLo8Inv, rv[e]);
                rv[4 + e] = fmaf(lo8_get(w1, e), kLo8Inv, rv[4 + e]);
              }
            }
            if (fl & EPF_RES_LN) {
              const float4 *g4 = reinterpret_cast<const float4 *>(cv + 128 + 8 * c);
              const float4 *e4 = reinterpret_cast<const float4 *>(cv + 192 + 8 * c);
              const float4 gl = g4[0], gh = g4[1], el = e4[0], eh = e4[1];
              const float gg[8] = {gl.x, gl.y, gl.z, gl.w, gh.x, gh.y, gh.z, gh.w};
              const float be[8] = {el.x, el.y, el.z, el.w, eh.x, eh.y, eh.z, eh.w};
#pragma unroll
              for (int e = 0; e < 8; ++e) rv[e] = fmaf((rv[e] - mu_r) * rs_r, gg[e], be[e]);
            }
#pragma unroll
            for (int e = 0; e < 8; ++e) v[e] += rv[e];
          }
          uint4 o;
          o.x = pack_bf16(v[0], v[1]);
          o.y = pack_bf16(v[2], v[3]);
          o.z = pack_bf16(v[4], v[5]);
          o.w = pack_bf16(v[6], v[7]);
          *cp = o;
          if constexpr (kSplit) {  // int8 correction of hi; statistics of the unrounded v
            const uint32_t ow[4] = {o.x, o.y, o.z, o.w};
            float hf[8];
#pragma unroll
            for (int e = 0; e < 4; ++e) {   // the bf16 values just packed, back as floats
              hf[2 * e] = __uint_as_float(ow[e] << 16);
              hf[2 * e + 1] = __uint_as_float(ow[e] & 0xffff0000u);
            }
            lo_out[2 * (c & 1)] = lo8_pack4(v, hf);
            lo_out[2 * (c & 1) + 1] = lo8_pack4(v + 4, hf + 4);
            if (c & 1) *cpl = make_uint4(lo_out[0], lo_out[1], lo_out[2], lo_out[3]);
            if (fl & EPF_STATS) {
#pragma unroll
              for (int e = 0; e < 8; e += 2) {
                if (c == 0 && e == 0) sk = v[0];
                const float a0 = v[e] - sk, a1 = v[e + 1] - sk;
                s1 += a0 + a1;
                s2 = fmaf(a0, a0, fmaf(a1, a1, s2));
              }
            }
          } else if (fl & EPF_STATS) {
            const __nv_bfloat162 *h = reinterpret_cast<const __nv_bfloat162 *>(&o);
#pragma unroll
            for (int e = 0; e < 4; ++e) {
              const float2 f = __bfloat1622float2(h[e]);
              if (c == 0 && e == 0) sk = f.x;
              const float a0 = f.x - sk, a1 = f.y - sk;
              s1 += a0 + a1;
              s2 = fmaf(a0, a0, fmaf(a1, a1, s2));
            }
          }
        }
        if ((fl & EPF_STATS) && live)  // box (mean, M2) from sums shifted by its first value
          ep.stats[(size_t)grow * (N / 64) + (x >> 6)] =
              make_float2(sk + s1 * (1.f / 64.f), fmaxf(s2 - s1 * s1 * (1.f / 64.f), 0.f));
        fence_async_smem();
        __syncwarp();
        if (lane == 0) {
          tma_store_2d(&tmO, box, x, y);
          if constexpr (kSplit) tma_store_2d(&tmOL, box + kBoxBytes, x, y);
          bulk_commit();
        }
      }
      acc ^= 1;
      if (acc == 0) acc_phase ^= 1;
      st_cur = st_next;
    }
    if (lane == 0) bulk_wait<0>();
  }
  fence_before();
  cluster_sync_all();
  if (warp == 1) {
    fence_after();
    asm volatile("tcgen05.dealloc.cta_group::2.sync.aligned.b32 %0, %1;" ::"r"(tmem_base),
                 "r"(512));
  }
}

PFN_cuTensorMapEncodeTiled_v12000 encode_fn() {
  static PFN_cuTensorMapEncodeTiled_v12000 fn = nullptr;
  static std::once_flag once;
  std::call_once(once, [] {
    cudaDriverEntryPointQueryResult q;
    void *p = nullptr;
    if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q) ==
            cudaSuccess &&
        q == cudaDriverEntryPointSuccess)
      fn = reinterpret_cast<PFN_cuTensorMapEncodeTiled_v12000>(p);
  });
  return fn;
}

// 2-D bf16 row-major [rows][K] map with a (64 x box_rows) box, 128-byte swizzle.
bool make_map(CUtensorMap *m, const void *ptr, int rows, int K, int box_rows) {
  return make_tma_2d_bf16(m, ptr, (uint64_t)K, (uint64_t)rows, (uint64_t)K * 2, kBK, box_rows);
}

template <int BN>
int launch(const __nv_bfloat16 *A, const __nv_bfloat16 *W, const float *bias,
           const __nv_bfloat16 *residual, __nv_bfloat16 *out, int M, int N, int K, int epi,
           cudaStream_t s) {
  using C = Cfg<BN>;
  CUtensorMap ta, tb;
  LV_REQUIRE(make_map(&ta, A, M, K, kBM), LV_ERR_INTERNAL, "cuTensorMapEncodeTiled(A) failed");
  LV_REQUIRE(make_map(&tb, W, N, K, BN), LV_ERR_INTERNAL, "cuTensorMapEncodeTiled(W) failed");
  static unsigned long long attr_set = 0;  // per device (first_on_device)
  if (first_on_device(attr_set)) {
    LV_CHECK_CUDA(cudaFuncSetAttribute(tc_gemm_kernel<BN>,
                                       cudaFuncAttributeMaxDynamicSharedMemorySize, C::kSmem));
  }
  const int tiles = ((M + kBM - 1) / kBM) * (N / BN);
  const int grid = std::min(tiles, tc_gemm_num_sms());
  tc_gemm_kernel<BN><<<grid, kThreads, C::kSmem, s>>>(ta, tb, M, N, K, bias, residual, out, epi);
  note_launch();
  LV_CHECK_CUDA(cudaGetLastError());
  return LV_OK;
}

int launch_pair(const __nv_bfloat16 *A, const __nv_bfloat16 *W, const __nv_bfloat16 *residual,
                __nv_bfloat16 *out, int M, int N, int K, const EpiParams &ep, cudaStream_t s) {
  CUtensorMap ta, tb, to, tr;
  LV_REQUIRE(make_map(&ta, A, M, K, 128), LV_ERR_INTERNAL, "cuTensorMapEncodeTiled(A) failed");
  LV_REQUIRE(make_map(&tb, W, N, K, 128), LV_ERR_INTERNAL, "cuTensorMapEncodeTiled(W) failed");
  const int n_out = (ep.flags & EPF_SWIGLU) ? N / 2 : N;
  LV_REQUIRE(make_tma_2d_bf16(&to, out, n_out, M, (uint64_t)n_out * 2, 64, 32), LV_ERR_INTERNAL,
             "cuTensorMapEncodeTiled(out) failed");
  LV_REQUIRE(make_tma_2d_bf16(&tr, residual ? residual : out, N, M, (uint64_t)N * 2, 64, 32),
             LV_ERR_INTERNAL, "cuTensorMapEncodeTiled(residual) failed");
  CUtensorMap trl = tr, tol = to;
  const bool split = (ep.flags & EPF_SPLIT) != 0;
  if (split) {
    LV_REQUIRE(make_tma_2d_u8(&trl, ep.res_lo, N, M, (uint64_t)N, 64, 32), LV_ERR_INTERNAL,
               "cuTensorMapEncodeTiled(residual lo) failed");
    LV_REQUIRE(make_tma_2d_u8(&tol, ep.out_lo, N, M, (uint64_t)N, 64, 32), LV_ERR_INTERNAL,
               "cuTensorMapEncodeTiled(out lo) failed");
  }
  static unsigned long long attr_set = 0;  // per device (first_on_device)
  if (first_on_device(attr_set)) {
    LV_CHECK_CUDA(cudaFuncSetAttribute(tc_gemm_pair_kernel<5>,
                                       cudaFuncAttributeMaxDynamicSharedMemorySize,
                                       PairCfg<5>::kSmem));
    LV_CHECK_CUDA(cudaFuncSetAttribute(tc_gemm_pair_kernel<6>,
                                       cudaFuncAttributeMaxDynamicSharedMemorySize,
                                       PairCfg<6>::kSmem));
    LV_CHECK_CUDA(cudaFuncSetAttribute(tc_gemm_pair_kernel<0>,
                                       cudaFuncAttributeMaxDynamicSharedMemorySize,
                                       PairCfg<0>::kSmem));
    LV_CHECK_CUDA(cudaFuncSetAttribute(tc_gemm_pair_kernel<1>,
                                       cudaFuncAttributeMaxDynamicSharedMemorySize,
                                       PairCfg<1>::kSmem));
    LV_CHECK_CUDA(cudaFuncSetAttribute(tc_gemm_pair_kernel<3>,
                                       cudaFuncAttributeMaxDynamicSharedMemorySize,
                                       PairCfg<3>::kSmem));
    LV_CHECK_CUDA(cudaFuncSetAttribute(tc_gemm_pair_kernel<4>,
                                       cudaFuncAttributeMaxDynamicSharedMemorySize,
                                       PairCfg<4>::kSmem));
  }
  const int tiles = ((M + 255) / 256) * (N / 256);
  const int pairs = std::min(tiles, tc_gemm_num_sms() / 2);
  const int mode = (ep.flags & EPF_SWIGLU) ? 3
                   : !(ep.flags & EPF_RES) ? 0
                   : split ? ((K > 1024 || g_split_single) ? 5 : 6)
                   : (K > 1024 && g_long_k_single) ? 4 : 1;
  if (mode == 6)
    tc_gemm_pair_kernel<6><<<2 * pairs, kThreads, PairCfg<6>::kSmem, s>>>(ta, tb, to, tr, trl, tol,
                                                                          M, N, K, ep);
  else if (mode == 5)
    tc_gemm_pair_kernel<5><<<2 * pairs, kThreads, PairCfg<5>::kSmem, s>>>(ta, tb, to, tr, trl, tol,
                                                                          M, N, K, ep);
  else if (mode == 4)
    tc_gemm_pair_kernel<4><<<2 * pairs, kThreads, PairCfg<4>::kSmem, s>>>(ta, tb, to, tr, trl, tol,
                                                                          M, N, K, ep);
  else if (mode == 3)
    tc_gemm_pair_kernel<3><<<2 * pairs, kThreads, PairCfg<3>::kSmem, s>>>(ta, tb, to, tr, trl, tol,
                                                                          M, N, K, ep);
  else if (mode == 1)
    tc_gemm_pair_kernel<1><<<2 * pairs, kThreads, PairCfg<1>::kSmem, s>>>(ta, tb, to, tr, trl, tol,
                                                                          M, N, K, ep);
  else
    tc_gemm_pair_kernel<0><<<2 * pairs, kThreads, PairCfg<0>::kSmem, s>>>(ta, tb, to, tr, trl, tol,
                                                                          M, N, K, ep);
  note_launch();
  LV_CHECK_CUDA(cudaGetLastError());
  return LV_OK;
}

}  // namespace

bool make_tma_2d_u8(CUtensorMap *m, const void *ptr, uint64_t cols, uint64_t rows,
                    uint64_t row_stride_bytes, int box_cols, int box_rows) {
  auto fn = encode_fn();
  if (!fn) return false;
  cuuint64_t dims[2] = {(cuuint64_t)cols, (cuuint64_t)rows};
  cuuint64_t strides[1] = {(cuuint64_t)row_stride_bytes};
  cuuint32_t box[2] = {(cuuint32_t)box_cols, (cuuint32_t)box_rows};
  cuuint32_t estr[2] = {1, 1};
  CUresult r = fn(m, CU_TENSOR_MAP_DATA_TYPE_UINT8, 2, const_cast<void *>(ptr), dims, strides,
                  box, estr, CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_64B,
                  CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  return r == CUDA_SUCCESS;
}

bool make_tma_2d_bf16(CUtensorMap *m, const void *ptr, uint64_t cols, uint64_t rows,
                      uint64_t row_stride_bytes, int box_cols, int box_rows) {
  auto fn = encode_fn();
  if (!fn) return false;
  cuuint64_t dims[2] = {(cuuint64_t)cols, (cuuint64_t)rows};
  cuuint64_t strides[1] = {(cuuint64_t)row_stride_bytes};
  cuuint32_t box[2] = {(cuuint32_t)box_cols, (cuuint32_t)box_rows};
  cuuint32_t estr[2] = {1, 1};
  CUresult r = fn(m, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 2, const_cast<void *>(ptr), dims, strides,
                  box, estr, CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B,
                  CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  return r == CUDA_SUCCESS;
}

int g_gemm_mode = 0;  // 0 = auto (pair kernel when N % 256 == 0), 1 = force 1-CTA

int tc_gemm_num_sms() {
  static int sms = 0;
  if (!sms) {
    int dev = 0;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    if (sms <= 0) sms = 148;
  }
  return sms;
}

int tc_gemm_ex(const __nv_bfloat16 *A, const __nv_bfloat16 *W, const __nv_bfloat16 *residual,
               __nv_bfloat16 *out, int M, int N, int K, const EpiParams &ep, cudaStream_t s) {
  LV_REQUIRE(M >= 1 && N % 256 == 0 && K % kBK == 0 && K > 0, LV_ERR_USAGE,
             "tc_gemm_ex: need N % 256 == 0 and K % 64 == 0");
  LV_REQUIRE(ep.bias != nullptr || (ep.flags & EPF_SWIGLU), LV_ERR_USAGE,
             "tc_gemm_ex: bias required");
  LV_REQUIRE(!(ep.flags & EPF_SWIGLU) || (ep.flags & ~(EPF_SWIGLU | EPF_LN_IN)) == 0,
             LV_ERR_USAGE, "tc_gemm_ex: the SwiGLU epilogue combines only with LN-in");
  LV_REQUIRE(!(ep.flags & EPF_RES) || residual != nullptr, LV_ERR_USAGE,
             "tc_gemm_ex: residual required");
  LV_REQUIRE(!(ep.flags & EPF_LN_IN) || (ep.ln_in && (ep.colc || (ep.flags & EPF_SWIGLU))),
             LV_ERR_USAGE, "tc_gemm_ex: LN-in needs colc and row statistics");
  LV_REQUIRE(!(ep.flags & EPF_RES_LN) || (ep.res_ln && ep.res_g && ep.res_b), LV_ERR_USAGE,
             "tc_gemm_ex: residual LN needs statistics and affine");
  LV_REQUIRE(!(ep.flags & EPF_STATS) || ep.stats, LV_ERR_USAGE, "tc_gemm_ex: stats buffer");
  LV_REQUIRE(!(ep.flags & EPF_SPLIT) || ((ep.flags & EPF_RES) && ep.res_lo && ep.out_lo &&
                                         !(ep.flags & EPF_GELU)),
             LV_ERR_USAGE, "tc_gemm_ex: split residual needs res_lo and out_lo");
  return launch_pair(A, W, residual, out, M, N, K, ep, s);
}

int tc_gemm(const __nv_bfloat16 *A, const __nv_bfloat16 *W, const float *bias,
            const __nv_bfloat16 *residual, __nv_bfloat16 *out, int M, int N, int K, int epi,
            cudaStream_t s) {
  LV_REQUIRE(M >= 1 && N % 128 == 0 && K % kBK == 0 && K > 0, LV_ERR_USAGE,
             "tc_gemm: need N % 128 == 0 and K % 64 == 0");
  LV_REQUIRE(bias != nullptr, LV_ERR_USAGE, "tc_gemm: bias required");
  LV_REQUIRE(epi != EPI_BIAS_RESIDUAL || residual != nullptr, LV_ERR_USAGE,
             "tc_gemm: residual required");
  if (N % 256 == 0 && g_gemm_mode == 0) {
    EpiParams ep;
    ep.bias = bias;
    ep.flags = epi == EPI_BIAS_GELU ? EPF_GELU : epi == EPI_BIAS_RESIDUAL ? EPF_RES : 0;
    return launch_pair(A, W, residual, out, M, N, K, ep, s);
  }
  if (N % 256 == 0) return launch<256>(A, W, bias, residual, out, M, N, K, epi, s);
  return launch<128>(A, W, bias, residual, out, M, N, K, epi, s);
}

}  // namespace lv
