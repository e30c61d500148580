// Per-pixel shading shared by every kernel that evaluates the calibration
// polynomial (K1 rgb.cu, K6 binned.cu, K7 pyramid_fused.cu): the same
// instruction sequence everywhere, so kernels agree bit for bit.
//
// render/lut.py:56-65 PolyLut.evaluate on the doubled gradients h = 2g (the
// coefficients carry 2^-(i+j), api.cu fill_scaled), clip [0,1], and the
// to_uint8 quantisation of render/imageio.py:8-11.
#pragma once

#include <cuda_runtime.h>
#include <stdint.h>

#include "handles.h"

namespace tacsl {

__host__ __device__ constexpr int term_index(int i, int j) { return (i + j) * (i + j + 1) / 2 + j; }

// sum_{i+j<=DEG} c_ij hx^i hy^j as Horner in hx of Horner-in-hy polynomials:
// DEG(DEG+1)/2 + DEG FMAs per channel (5 at degree 2, 14 at degree 4).
template <int DEG>
__device__ __forceinline__ float poly(const float (&c)[15], float hx, float hy) {
  float acc = 0.f;
#pragma unroll
  for (int i = DEG; i >= 0; --i) {
    float p = c[term_index(i, DEG - i)];
#pragma unroll
    for (int j = DEG - i - 1; j >= 0; --j) p = __fmaf_rn(p, hy, c[term_index(i, j)]);
    acc = (i == DEG) ? p : __fmaf_rn(acc, hx, p);
  }
  return acc;
}

__device__ __forceinline__ float2 bc(float v) { return make_float2(v, v); }

// The same polynomial for two pixels at once on the packed pipe; the final
// Horner step is scalar so that it carries the [0,1] saturation for free.
template <int DEG>
__device__ __forceinline__ float2 poly2_sat(const float (&c)[15], float2 hx, float2 hy) {
  float2 acc = bc(0.f);
  float2 out = bc(0.f);
#pragma unroll
  for (int i = DEG; i >= 0; --i) {
    float2 p = bc(c[term_index(i, DEG - i)]);
#pragma unroll
    for (int j = DEG - i - 1; j >= 0; --j) {
      p = (j == DEG - i - 1) ? __ffma2_rn(hy, bc(c[term_index(i, DEG - i)]), bc(c[term_index(i, j)]))
                             : __ffma2_rn(p, hy, bc(c[term_index(i, j)]));
    }
    if (i == DEG) {
      acc = p;
    } else if (i > 0) {
      acc = __ffma2_rn(acc, hx, p);
    } else {
      out.x = __saturatef(__fmaf_rn(acc.x, hx.x, p.x));
      out.y = __saturatef(__fmaf_rn(acc.y, hx.y, p.y));
    }
  }
  return out;
}

__device__ __forceinline__ uint32_t q8(float x) {
  // clip(rint(255 x), 0, 255): x is saturated to [0,1] first, then the
  // 1.5*2^23 bias rounds the exact product half-to-even into the low byte.
  return __float_as_uint(__fmaf_rn(__saturatef(x), 255.0f, 12582912.0f));
}

// two already-saturated values -> their biased quantised bit patterns
__device__ __forceinline__ float2 q8x2(float2 v) { return __ffma2_rn(v, bc(255.0f), bc(12582912.0f)); }

template <int DEG>
__device__ __forceinline__ void shade(const LutParams& L, float hx, float hy, float& r, float& g, float& b) {
  r = __saturatef(poly<DEG>(L.c[0], hx, hy));
  g = __saturatef(poly<DEG>(L.c[1], hx, hy));
  b = __saturatef(poly<DEG>(L.c[2], hx, hy));
}

}  // namespace tacsl
