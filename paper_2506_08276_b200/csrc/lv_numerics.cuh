// lv_numerics.cuh — bit-exact device restatement of the reference's float math.
//
// distance_many (vectors.py:120-140) and adc_build (pq.py:153-178) use
// np.einsum in float32; approx_distance_many (pq.py:186-189) sums float32 LUT
// entries in float64 with numpy's pairwise reduction. The orders are pinned
// in oracle/numerics.py and tests/test_oracle_golden.py; every op below is a
// separately rounded IEEE op (no FMA contraction: __fmul_rn / __fadd_rn).
#pragma once
#include <cstdint>

namespace lv {

// One of the 4 einsum lanes of a length-`dim` dot product: lane `l` sums the
// elements j+4k+l of each 16-block in the order k = 3,2,1,0, then the
// zero-padded 4-wide tail. `A`/`B` may be the same pointer (norms).
template <bool kL2>
__device__ __forceinline__ float einsum_lane(const float *__restrict__ a,
                                             const float *__restrict__ b, int dim, int l) {
  float acc = 0.0f;
  int j = 0;
  for (; dim - j >= 16; j += 16) {
#pragma unroll
    for (int k = 3; k >= 0; --k) {
      float x = a[j + 4 * k + l], y = b[j + 4 * k + l];
      if (kL2) {
        float t = __fsub_rn(x, y);
        acc = __fadd_rn(acc, __fmul_rn(t, t));
      } else {
        acc = __fadd_rn(acc, __fmul_rn(x, y));
      }
    }
  }
  for (; j < dim; j += 4) {
    float p = 0.0f;
    if (j + l < dim) {
      float x = a[j + l], y = b[j + l];
      if (kL2) {
        float t = __fsub_rn(x, y);
        p = __fmul_rn(t, t);
      } else {
        p = __fmul_rn(x, y);
      }
    }
    acc = __fadd_rn(acc, p);
  }
  return acc;
}

__device__ __forceinline__ float einsum_combine(float a0, float a1, float a2, float a3) {
  return __fadd_rn(0.0f, __fadd_rn(__fadd_rn(a0, a1), __fadd_rn(a2, a3)));
}

// Full single-thread einsum dot (all 4 lanes sequentially) — used for short
// vectors (PQ sub-spaces).
template <bool kL2>
__device__ __forceinline__ float einsum_dot_1t(const float *a, const float *b, int dim) {
  float r0 = einsum_lane<kL2>(a, b, dim, 0);
  float r1 = einsum_lane<kL2>(a, b, dim, 1);
  float r2 = einsum_lane<kL2>(a, b, dim, 2);
  float r3 = einsum_lane<kL2>(a, b, dim, 3);
  return einsum_combine(r0, r1, r2, r3);
}

// Final distance from the einsum results (vectors.py:130-139).
// metric: 0 l2, 1 ip, 2 cosine. For l2 `dot` already holds sum((r-q)^2).
__device__ __forceinline__ float finish_distance(int metric, float dot, float nrm, float qn) {
  if (metric == 0) return dot;
  if (metric == 1) return -dot;
  float rn = __fsqrt_rn(nrm);
  return -__fdiv_rn(dot, __fmul_rn(rn, qn));
}

// numpy pairwise float64 sum of x[0..n) (n <= 128), 8 strided accumulators.
template <typename Get>
__device__ __forceinline__ double pairwise_block(Get get, int lo, int n) {
  if (n < 8) {
    double res = 0.0;
    for (int i = 0; i < n; ++i) res = __dadd_rn(res, get(lo + i));
    return res;
  }
  double r[8];
#pragma unroll
  for (int k = 0; k < 8; ++k) r[k] = get(lo + k);
  int i = 8;
  int lim = n - (n % 8);
  for (; i < lim; i += 8) {
#pragma unroll
    for (int k = 0; k < 8; ++k) r[k] = __dadd_rn(r[k], get(lo + i + k));
  }
  double res = __dadd_rn(__dadd_rn(__dadd_rn(r[0], r[1]), __dadd_rn(r[2], r[3])),
                         __dadd_rn(__dadd_rn(r[4], r[5]), __dadd_rn(r[6], r[7])));
  for (; i < n; ++i) res = __dadd_rn(res, get(lo + i));
  return res;
}

// n <= 256: one level of numpy's recursive split above 128.
template <typename Get>
__device__ __forceinline__ double pairwise_sum(Get get, int n) {
  if (n <= 128) return pairwise_block(get, 0, n);
  int half = (n / 2) - ((n / 2) % 8);
  return __dadd_rn(pairwise_block(get, 0, half), pairwise_block(get, half, n - half));
}

// np.dot(x, y) of two float32 vectors: numpy hands 1-D float32 dots to BLAS
// cblas_sdot, here scipy-openblas 0.3.30 with the SkylakeX kernel
// (threadpoolctl reports architecture "SkylakeX" on this image's hosts). Its
// order, pinned against np.dot on 0/300 mismatching random vectors for every
// n % 32 == 0 in {32 .. 1024} (tests/test_oracle_golden.py::test_sdot_order):
//   n1 = n & -32; 512-bit phase over n1 & -64 with four 16-lane FMA
//   accumulators (a5[j] += x[i+16j..] * y[i+16j..]); fold each to 8 lanes
//   (low + high half); 256-bit phase over the remaining 32-block with four
//   8-lane FMA accumulators; acc = ((a0 + a1) + a2) + a3; 128-bit fold
//   (lanes l + l+4); two hadds -> (h0 + h1) + (h2 + h3); then the scalar tail
//   dot += y[i] * x[i] (separately rounded). The tail is exact for n % 32 <= 1;
//   longer tails are not pinned (every dimension on the configs is a multiple of 32).
// Used for qn = np.float32(np.sqrt(np.dot(q, q))) (vectors.py:138, pq.py:163)
// and distance() (vectors.py:94-116, the pending-buffer scan).
template <bool kL2>
__device__ __forceinline__ float sdot_openblas(const float *__restrict__ x,
                                               const float *__restrict__ y, int n) {
  const int n1 = n & ~31;
  float dot = 0.0f;
  int i = 0;
  auto term = [&](int e) -> float2 {
    if (kL2) {
      float t = __fsub_rn(x[e], y[e]);
      return make_float2(t, t);
    }
    return make_float2(x[e], y[e]);
  };
  if (n1) {
    float acc[4][8];
    {
      float a5[4][16];
#pragma unroll
      for (int j = 0; j < 4; ++j)
#pragma unroll
        for (int l = 0; l < 16; ++l) a5[j][l] = 0.0f;
      const int n64 = n1 & ~63;
      for (; i < n64; i += 64) {
#pragma unroll
        for (int j = 0; j < 4; ++j)
#pragma unroll
          for (int l = 0; l < 16; ++l) {
            float2 p = term(i + 16 * j + l);
            a5[j][l] = __fmaf_rn(p.x, p.y, a5[j][l]);
          }
      }
#pragma unroll
      for (int j = 0; j < 4; ++j)
#pragma unroll
        for (int l = 0; l < 8; ++l) acc[j][l] = __fadd_rn(a5[j][l], a5[j][l + 8]);
    }
    for (; i < n1; i += 32) {
#pragma unroll
      for (int j = 0; j < 4; ++j)
#pragma unroll
        for (int l = 0; l < 8; ++l) {
          float2 p = term(i + 8 * j + l);
          acc[j][l] = __fmaf_rn(p.x, p.y, acc[j][l]);
        }
    }
    float a[8];
#pragma unroll
    for (int l = 0; l < 8; ++l)
      a[l] = __fadd_rn(__fadd_rn(__fadd_rn(acc[0][l], acc[1][l]), acc[2][l]), acc[3][l]);
    float h0 = __fadd_rn(a[0], a[4]), h1 = __fadd_rn(a[1], a[5]);
    float h2 = __fadd_rn(a[2], a[6]), h3 = __fadd_rn(a[3], a[7]);
    dot = __fadd_rn(__fadd_rn(h0, h1), __fadd_rn(h2, h3));
  }
  for (; i < n; ++i) {
    float2 p = term(i);
    dot = __fadd_rn(dot, __fmul_rn(p.y, p.x));
  }
  return dot;
}

// approx_distance_many's row sum with the LUT in shared memory (plain loads).
__device__ __forceinline__ float adc_one_shared(const float *lut, const uint8_t *__restrict__ code,
                                                int m) {
  auto get = [&](int s) -> double { return (double)lut[s * 256 + __ldg(code + s)]; };
  return __double2float_rn(pairwise_sum(get, m));
}

// pairwise_block over LUT entries of 8-aligned code runs: the 8 code bytes of
// each strided step arrive in one 8-byte load (the byte-per-load form spends
// one dependent LDG per subspace). Same values, same order as pairwise_block.
__device__ __forceinline__ double adc_block8(const float *__restrict__ lut,
                                             const uint8_t *__restrict__ code, int lo, int n) {
  auto lut8 = [&](int base, uint2 c, double (&v)[8]) {
#pragma unroll
    for (int k = 0; k < 8; ++k) {
      const uint32_t w = k < 4 ? c.x : c.y;
      v[k] = (double)__ldg(lut + (base + k) * 256 + ((w >> (8 * (k & 3))) & 0xffu));
    }
  };
  double r[8];
  lut8(lo, __ldg(reinterpret_cast<const uint2 *>(code + lo)), r);
#pragma unroll 4
  for (int i = 8; i < n; i += 8) {
    double v[8];
    lut8(lo + i, __ldg(reinterpret_cast<const uint2 *>(code + lo + i)), v);
#pragma unroll
    for (int k = 0; k < 8; ++k) r[k] = __dadd_rn(r[k], v[k]);
  }
  return __dadd_rn(__dadd_rn(__dadd_rn(r[0], r[1]), __dadd_rn(r[2], r[3])),
                   __dadd_rn(__dadd_rn(r[4], r[5]), __dadd_rn(r[6], r[7])));
}

// approx distance of one code row against one LUT (pq.py:186-189).
__device__ __forceinline__ float adc_one(const float *__restrict__ lut,
                                         const uint8_t *__restrict__ code, int m) {
  if ((m & 7) == 0 && m >= 8 && m <= 256 && (reinterpret_cast<uintptr_t>(code) & 7) == 0) {
    if (m <= 128) return __double2float_rn(adc_block8(lut, code, 0, m));
    const int half = (m / 2) - ((m / 2) % 8);
    return __double2float_rn(__dadd_rn(adc_block8(lut, code, 0, half),
                                       adc_block8(lut, code, half, m - half)));
  }
  auto get = [&](int s) -> double {
    return (double)__ldg(lut + s * 256 + __ldg(code + s));
  };
  return __double2float_rn(pairwise_sum(get, m));
}

}  // namespace lv
