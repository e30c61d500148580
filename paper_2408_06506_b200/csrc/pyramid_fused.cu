// K7: the whole config-5 image chain in ONE pass over the depth maps --
// Gaussian smoothing (K5 semantics) -> tactile RGB at level 0 (K1) ->
// 2x decimation (K5 pyr_down) -> RGB at level 1 -> decimation -> RGB at
// level 2 -- with nothing but the fp32 depth read and the uint8 RGB of every
// level written to HBM.  The stage it extends is render/lut.py:68-76
// (depth_gradients lut.py:25-28 + PolyLut.evaluate lut.py:56-65 + to_uint8
// render/imageio.py:8-11); smoothing and the pyramid have no reference
// counterpart, their semantics are smoothing.py's.
//
// Design: a line-buffer pipeline.  One CTA owns one image at a time and
// streams it top to bottom in ticks of 8 level-0 rows; nothing is ever
// recomputed for a halo:
//   * a loader warp brings each half tick's 4 input rows into a ring with
//     one bulk-async copy (1-D TMA; rows outside the image are loaded as the
//     clamped edge row, 'nearest' borders), completed on mbarriers;
//   * consumer thread t owns column quad t at level 0, column pair t at
//     level 1 and column t at level 2 (W/4 threads);
//   * G: each input row is filtered horizontally once (the even/odd FFMA2
//     split of K5) and scattered into 2R+1 rolling vertical accumulators in
//     registers (packed FFMA2); a smoothed row completes R rows later and
//     goes to a shared-memory line ring S0;
//   * L0: level-0 rows are shaded from S0 (K1's doubled-gradient packed
//     Horner and uint8 epilogue, stores straight to global) and every S0 row
//     is decimated horizontally and scattered into rolling level-1
//     accumulators (registers) -> line ring S1;  L1 / L2: the same one and
//     two levels down (S1 -> RGB level 1 + level-2 accumulators -> S2 ->
//     RGB level 2);
//   * a consumer-only named barrier separates the phases of a tick (each
//     reads neighbours' columns of the ring rows the previous phase wrote).
// Every value is computed with the operations, operands and order of the
// unfused chain (sep_bulk_kernel -> rgb_bulk_kernel per level), so the
// outputs are bit-identical to it (tests/test_pyramid_fused_gpu.py).
//
// Which rows a tick k touches (H % 4 == 0; verified exhaustively for
// H < 1000 by the schedule model in tests/test_pyramid_fused_gpu.py):
//   G : h-rows j in [8k-4, 8k+4) (input row clamp(j)), completes S0 rows j-R
//   L0: shades rows [8k-9, 8k-1); decimates virtual S0 rows i in
//       [8k-10, 8k-2), completing level-1 rows (i-2)/2
//   L1: shades level-1 rows [4k-7, 4k-3); decimates virtual level-1 rows
//       [4k-6, 4k-2), completing level-2 rows (i-2)/2
//   L2: shades level-2 rows [2k-5, 2k-3), plus row 2k-3 if it is the last.
#include <algorithm>
#include <cstdlib>
#include <cstring>

#include "common.cuh"
#include "handles.h"
#include "shade.cuh"

namespace tacsl {
namespace {

constexpr int kHalf = 4;         // input rows per TMA stage (half a tick)
constexpr int kPMaxCons = 256;   // consumer threads per CTA: W <= 1024
constexpr int kPMaxStages = 6;

struct PyrArgs {
  float w[9];            // Gaussian taps, 2R+1
  float2 we[6], wo[6];   // horizontal pair weights, first tap on an even / odd column (pyramid.cu Taps)
  float pw[5];           // pyramid taps [1, 4, 6, 4, 1] / 16
  LutParams L[3];        // level LUTs (level_lut: c_ij 2^-l(i+j)), pre-scaled like every K1 LUT
  uint8_t* out[3];       // (n, H_l, W_l, 3) uint8
  int stages;
  int ticks;
};

template <int R>
struct Ring {
  static constexpr int S0 = 14 - R;  // 8 new rows + 2 read back + the R-row lag of the filter
  static constexpr int S1 = 6;
  static constexpr int S2 = 4;
};

__device__ __forceinline__ void pyr_bar(int n) { asm volatile("bar.sync 1, %0;" ::"r"(n) : "memory"); }

__device__ __forceinline__ float2 f2(float a, float b) { return make_float2(a, b); }

// one level-0-style quad of a row: the thread's 4 columns, the two columns
// to its left and the one to its right (clamped at the image borders)
struct Quad {
  float4 c;
  float2 l;
  float r;
};

// uint8 RGB of pixels (2 pairs) with K1's arithmetic: doubled gradients, the
// level LUT's packed Horner, saturating last step, biased rounding, PRMT.
template <int DEG>
__device__ __forceinline__ void shade_quad(const LutParams& L, const float4 up, const Quad& c, const float4 dn,
                                           bool edge_row, float m0, float m3, uint32_t* __restrict__ dst) {
  float2 hy01 = __fadd2_rn(make_float2(dn.x, dn.y), make_float2(-up.x, -up.y));
  float2 hy23 = __fadd2_rn(make_float2(dn.z, dn.w), make_float2(-up.z, -up.w));
  if (edge_row) {
    hy01 = __fadd2_rn(hy01, hy01);
    hy23 = __fadd2_rn(hy23, hy23);
  }
  const float2 hx01 = make_float2((c.c.y - c.l.y) * m0, c.c.z - c.c.x);
  const float2 hx23 = make_float2(c.c.w - c.c.y, (c.r - c.c.z) * m3);
  const float2 r01 = poly2_sat<DEG>(L.c[0], hx01, hy01);
  const float2 g01 = poly2_sat<DEG>(L.c[1], hx01, hy01);
  const float2 b01 = poly2_sat<DEG>(L.c[2], hx01, hy01);
  const float2 r23 = poly2_sat<DEG>(L.c[0], hx23, hy23);
  const float2 g23 = poly2_sat<DEG>(L.c[1], hx23, hy23);
  const float2 b23 = poly2_sat<DEG>(L.c[2], hx23, hy23);
  const float2 qa = q8x2(make_float2(r01.x, g01.x));
  const float2 qb = q8x2(make_float2(b01.x, r01.y));
  const float2 qc = q8x2(make_float2(g01.y, b01.y));
  const float2 qd = q8x2(make_float2(r23.x, g23.x));
  const float2 qe = q8x2(make_float2(b23.x, r23.y));
  const float2 qf = q8x2(make_float2(g23.y, b23.y));
  dst[0] = __byte_perm(__byte_perm(__float_as_uint(qa.x), __float_as_uint(qa.y), 0x0040),
                       __byte_perm(__float_as_uint(qb.x), __float_as_uint(qb.y), 0x0040), 0x5410);
  dst[1] = __byte_perm(__byte_perm(__float_as_uint(qc.x), __float_as_uint(qc.y), 0x0040),
                       __byte_perm(__float_as_uint(qd.x), __float_as_uint(qd.y), 0x0040), 0x5410);
  dst[2] = __byte_perm(__byte_perm(__float_as_uint(qe.x), __float_as_uint(qe.y), 0x0040),
                       __byte_perm(__float_as_uint(qf.x), __float_as_uint(qf.y), 0x0040), 0x5410);
}

// a pixel pair (level 1): 6 bytes as three 16-bit stores
template <int DEG>
__device__ __forceinline__ void shade_pair(const LutParams& L, float2 up, float2 c, float left, float right,
                                           float2 dn, bool edge_row, float m0, float m1,
                                           uint16_t* __restrict__ dst) {
  float2 hy = __fadd2_rn(dn, make_float2(-up.x, -up.y));
  if (edge_row) hy = __fadd2_rn(hy, hy);
  const float2 hx = make_float2((c.y - left) * m0, (right - c.x) * m1);
  const float2 r = poly2_sat<DEG>(L.c[0], hx, hy);
  const float2 g = poly2_sat<DEG>(L.c[1], hx, hy);
  const float2 b = poly2_sat<DEG>(L.c[2], hx, hy);
  const float2 qa = q8x2(make_float2(r.x, g.x));
  const float2 qb = q8x2(make_float2(b.x, r.y));
  const float2 qc = q8x2(make_float2(g.y, b.y));
  dst[0] = (uint16_t)__byte_perm(__float_as_uint(qa.x), __float_as_uint(qa.y), 0x0040);
  dst[1] = (uint16_t)__byte_perm(__float_as_uint(qb.x), __float_as_uint(qb.y), 0x0040);
  dst[2] = (uint16_t)__byte_perm(__float_as_uint(qc.x), __float_as_uint(qc.y), 0x0040);
}

// horizontal pyramid tap sum at one output column from the 5 input columns
// around it: even-column chain + odd-column chain (K5's FFMA2 lanes; its
// trailing zero-weight tap is an exact no-op and is left out)
__device__ __forceinline__ float pyr_h(const float* pw, float a, float b, float c, float d, float e) {
  const float ev = __fmaf_rn(e, pw[4], __fmaf_rn(c, pw[2], __fmaf_rn(a, pw[0], 0.f)));
  const float od = __fmaf_rn(d, pw[3], __fmaf_rn(b, pw[1], 0.f));
  return ev + od;
}

template <int R, int LEVELS, int DEG>
__global__ void __launch_bounds__(kPMaxCons + 32, 1)
    pyramid_fused_kernel(const float* __restrict__ depth, int64_t n, int H, int W, const PyrArgs A) {
  extern __shared__ __align__(128) unsigned char smem[];
  using RG = Ring<R>;
  constexpr int NT = 2 * R + 1;
  const int NQ = W >> 2;
  const int cons_warps = (NQ + 31) >> 5;
  const int n_cons = cons_warps * 32;
  const int H1 = H >> 1, H2 = H >> 2, W1 = W >> 1, W2 = W >> 2;
  uint64_t* full = reinterpret_cast<uint64_t*>(smem);
  uint64_t* empty = full + kPMaxStages;
  float* in_buf = reinterpret_cast<float*>(smem + 128);
  const size_t stage_f = (size_t)kHalf * W;
  float* s0 = in_buf + (size_t)A.stages * stage_f;
  float* s1 = s0 + (size_t)RG::S0 * W;
  float* s2 = s1 + (size_t)RG::S1 * W1;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int K = A.ticks;
  const int kG = (H + 7) >> 3;  // last tick with input rows (8k - 4 <= H + 3)
  const int stages = A.stages;

  if (threadIdx.x == 0) {
    for (int s = 0; s < stages; ++s) {
      mbar_init(&full[s], 1);
      mbar_init(&empty[s], cons_warps);
    }
    fence_mbar_init();
    fence_proxy_async_smem();
  }
  __syncthreads();

  if (warp == cons_warps) {
    // ---------------------------------------------------------- loader ---
    if (lane == 0) {
      int q = 0;
      const uint32_t row_bytes = (uint32_t)W * 4u;
      for (int64_t img = blockIdx.x; img < n; img += gridDim.x) {
        const float* src = depth + (size_t)img * H * W;
        for (int k = 0; k <= kG; ++k) {
          for (int h = 0; h < 2; ++h, ++q) {
            const int s = q % stages;
            if (q >= stages) mbar_wait_parity_sleep(&empty[s], (uint32_t)(q / stages - 1) & 1u);
            const int j0 = 8 * k - 4 + kHalf * h;
            float* dst = in_buf + (size_t)s * stage_f;
            mbar_arrive_expect_tx(&full[s], kHalf * row_bytes);
            if (j0 >= 0 && j0 + kHalf <= H) {
              bulk_g2s(dst, src + (size_t)j0 * W, kHalf * row_bytes, &full[s]);
            } else {  // rows outside the image: the clamped edge row ('nearest')
              for (int i = 0; i < kHalf; ++i) {
                const int r = min(max(j0 + i, 0), H - 1);
                bulk_g2s(dst + (size_t)i * W, src + (size_t)r * W, row_bytes, &full[s]);
              }
            }
          }
        }
      }
    }
    return;
  }

  // ------------------------------------------------------------ consumers ---
  const int t = threadIdx.x;
  const bool act = t < NQ;
  const int x0 = 4 * t;
  const bool atL = t == 0, atR = t == NQ - 1;
  const float m0 = atL ? 2.f : 1.f;  // np.gradient's one-sided borders are not halved
  const float m3 = atR ? 2.f : 1.f;
  float2 acc[8][2];  // vertical Gaussian accumulators, slot = output row & 7
  float2 acc1[2];    // level-1 vertical accumulators (column pair), slot = row & 1
  float acc2[2];     // level-2 vertical accumulators, slot = row & 1
#pragma unroll
  for (int i = 0; i < 8; ++i) acc[i][0] = acc[i][1] = f2(0.f, 0.f);
  acc1[0] = acc1[1] = f2(0.f, 0.f);
  acc2[0] = acc2[1] = 0.f;
  int q = 0;

  for (int64_t img = blockIdx.x; img < n; img += gridDim.x) {
    uint8_t* out0 = A.out[0] + (size_t)img * H * W * 3;
    uint8_t* out1 = LEVELS >= 2 ? A.out[1] + (size_t)img * H1 * W1 * 3 : nullptr;
    uint8_t* out2 = LEVELS >= 3 ? A.out[2] + (size_t)img * H2 * W2 * 3 : nullptr;
    for (int k = 0; k < K; ++k) {
      // ------------------------------------------------------------ G ---
      if (k <= kG) {
#pragma unroll
        for (int h = 0; h < 2; ++h) {
          const int s = q % stages;
          mbar_wait_parity(&full[s], (uint32_t)(q / stages) & 1u);
          const float* st = in_buf + (size_t)s * stage_f;
#pragma unroll
          for (int i = 0; i < kHalf; ++i) {
            const int ii = kHalf * h + i;  // h-row j = 8k - 4 + ii
            const int j = 8 * k - 4 + ii;
            const float* row = st + (size_t)i * W;
            float4 o = make_float4(0.f, 0.f, 0.f, 0.f);
            bool done = false;
            if constexpr (R == 0) {
              if (act) o = *reinterpret_cast<const float4*>(row + x0);
              done = true;
            } else {
              float v[12];
              if (act) {
                const float4 b = *reinterpret_cast<const float4*>(row + x0);
                const float4 a = atL ? make_float4(b.x, b.x, b.x, b.x)
                                     : *reinterpret_cast<const float4*>(row + x0 - 4);
                const float4 c = atR ? make_float4(b.w, b.w, b.w, b.w)
                                     : *reinterpret_cast<const float4*>(row + x0 + 4);
                v[0] = a.x; v[1] = a.y; v[2] = a.z; v[3] = a.w;
                v[4] = b.x; v[5] = b.y; v[6] = b.z; v[7] = b.w;
                v[8] = c.x; v[9] = c.y; v[10] = c.z; v[11] = c.w;
              } else {
#pragma unroll
                for (int e = 0; e < 12; ++e) v[e] = 0.f;
              }
              // horizontal: sep_bulk_kernel's FFMA2 over (even, odd) column
              // pairs of v (v[0] on an even column), partial sums added last
              float hq[4];
#pragma unroll
              for (int qq = 0; qq < 4; ++qq) {
                constexpr int NP = (NT + 1) / 2;
                const int b = 4 - R + qq;  // first tap's index in v
                float2 a = f2(0.f, 0.f);
#pragma unroll
                for (int m = 0; m < NP; ++m) {
                  const int i0 = (b & ~1) + 2 * m;
                  a = __ffma2_rn(f2(v[i0], v[i0 + 1]), (b & 1) ? A.wo[m] : A.we[m], a);
                }
                hq[qq] = a.x + a.y;
              }
              const float2 h01 = f2(hq[0], hq[1]), h23 = f2(hq[2], hq[3]);
              // vertical: h-row j feeds output rows j+R-tt (tap tt); the
              // row j-R completes (tt = 2R) before row j+R starts (tt = 0)
#pragma unroll
              for (int tt = NT - 1; tt >= 0; --tt) {
                const int slot = (ii + 4 + R - tt) & 7;
                const float2 w = f2(A.w[tt], A.w[tt]);
                if (tt == NT - 1) {
                  const float2 o01 = __ffma2_rn(h01, w, acc[slot][0]);
                  const float2 o23 = __ffma2_rn(h23, w, acc[slot][1]);
                  o = make_float4(o01.x, o01.y, o23.x, o23.y);
                  done = true;
                } else if (tt == 0) {
                  acc[slot][0] = __ffma2_rn(h01, w, f2(0.f, 0.f));
                  acc[slot][1] = __ffma2_rn(h23, w, f2(0.f, 0.f));
                } else {
                  acc[slot][0] = __ffma2_rn(h01, w, acc[slot][0]);
                  acc[slot][1] = __ffma2_rn(h23, w, acc[slot][1]);
                }
              }
            }
            const int y = j - R;  // the smoothed row this h-row completes
            if (done && act && y >= 0 && y < H)
              *reinterpret_cast<float4*>(s0 + (size_t)(y % RG::S0) * W + x0) = o;
          }
          __syncwarp();
          if (lane == 0) mbar_arrive(&empty[s]);
          ++q;
        }
      }
      pyr_bar(n_cons);  // S0 rows of this tick are visible

      // ----------------------------------------------------------- L0 ---
      if (k >= 1) {
        const int sb = 8 * k - 10;
        Quad win[3];  // rows s-2, s-1, s
#pragma unroll
        for (int m = 0; m < 10; ++m) {
          const int s = sb + m;
          const int r = min(max(s, 0), H - 1);
          const float* rp = s0 + (size_t)(r % RG::S0) * W;
          Quad cur;
          if (act) {
            cur.c = *reinterpret_cast<const float4*>(rp + x0);
            cur.l = atL ? f2(cur.c.x, cur.c.x) : *reinterpret_cast<const float2*>(rp + x0 - 2);
            cur.r = atR ? cur.c.w : rp[x0 + 4];
          } else {
            cur.c = make_float4(0.f, 0.f, 0.f, 0.f);
            cur.l = f2(0.f, 0.f);
            cur.r = 0.f;
          }
          win[0] = win[1];
          win[1] = win[2];
          win[2] = cur;
          if (m >= 2) {
            const int y = s - 1;
            if (act && y >= 0 && y < H)
              shade_quad<DEG>(A.L[0], win[0].c, win[1], win[2].c, y == 0 || y == H - 1, m0, m3,
                              reinterpret_cast<uint32_t*>(out0 + ((size_t)y * W + x0) * 3));
          }
          if constexpr (LEVELS >= 2) {
            if (m < 8) {
              // virtual S0 row i = s (row clamp(i)) decimated at level-1
              // columns 2t, 2t+1 (input columns 4t-2 .. 4t+4)
              const float2 hp = f2(pyr_h(A.pw, cur.l.x, cur.l.y, cur.c.x, cur.c.y, cur.c.z),
                                   pyr_h(A.pw, cur.c.x, cur.c.y, cur.c.z, cur.c.w, cur.r));
#pragma unroll
              for (int tt = 4; tt >= 0; --tt) {
                if (((m - tt) & 1) != 0) continue;
                const int y1 = (s + 2 - tt) >> 1;  // s + 2 - tt is even
                if (y1 < 0 || y1 >= H1) continue;
                const int slot = ((m - tt + 8) >> 1) & 1;
                const float2 w = f2(A.pw[tt], A.pw[tt]);
                if (tt == 4) {
                  const float2 o = __ffma2_rn(hp, w, acc1[slot]);
                  if (act) *reinterpret_cast<float2*>(s1 + (size_t)(y1 % RG::S1) * W1 + 2 * t) = o;
                } else {
                  acc1[slot] = __ffma2_rn(hp, w, tt == 0 ? f2(0.f, 0.f) : acc1[slot]);
                }
              }
            }
          }
        }
      }
      pyr_bar(n_cons);  // S1 rows of this tick are visible; S0 reads done

      // ----------------------------------------------------------- L1 ---
      if constexpr (LEVELS >= 2) {
        if (k >= 1) {
          const int sb = 4 * k - 8;
          float2 wc[3], wl[3];
          float wr[3];
#pragma unroll
          for (int m = 0; m < 6; ++m) {
            const int s = sb + m;
            const int r = min(max(s, 0), H1 - 1);
            const float* rp = s1 + (size_t)(r % RG::S1) * W1;
            float2 c = f2(0.f, 0.f), l = f2(0.f, 0.f);
            float rr = 0.f;
            if (act) {
              c = *reinterpret_cast<const float2*>(rp + 2 * t);
              l = atL ? f2(c.x, c.x) : *reinterpret_cast<const float2*>(rp + 2 * t - 2);
              rr = atR ? c.y : rp[2 * t + 2];
            }
            wc[0] = wc[1]; wc[1] = wc[2]; wc[2] = c;
            wl[0] = wl[1]; wl[1] = wl[2]; wl[2] = l;
            wr[0] = wr[1]; wr[1] = wr[2]; wr[2] = rr;
            if (m >= 2) {
              const int y = s - 1;
              if (act && y >= 0 && y < H1)
                shade_pair<DEG>(A.L[1], wc[0], wc[1], wl[1].y, wr[1], wc[2], y == 0 || y == H1 - 1, m0, m3,
                                reinterpret_cast<uint16_t*>(out1 + ((size_t)y * W1 + 2 * t) * 3));
              if constexpr (LEVELS >= 3) {
                // virtual level-1 row i = s decimated at level-2 column t
                const float hv = pyr_h(A.pw, l.x, l.y, c.x, c.y, rr);
#pragma unroll
                for (int tt = 4; tt >= 0; --tt) {
                  if (((m - tt) & 1) != 0) continue;
                  const int y2 = (s + 2 - tt) >> 1;
                  if (y2 < 0 || y2 >= H2) continue;
                  const int slot = ((m - tt + 2) >> 1) & 1;
                  if (tt == 4) {
                    const float o = __fmaf_rn(hv, A.pw[4], acc2[slot]);
                    if (act) s2[(size_t)(y2 & (RG::S2 - 1)) * W2 + t] = o;
                  } else {
                    acc2[slot] = __fmaf_rn(hv, A.pw[tt], tt == 0 ? 0.f : acc2[slot]);
                  }
                }
              }
            }
          }
        }
      }
      if constexpr (LEVELS >= 3) {
        pyr_bar(n_cons);  // S2 rows of this tick are visible
        // --------------------------------------------------------- L2 ---
        if (k >= 1) {
          const int sb = 2 * k - 6;
          float wc[3], wl[3], wr[3];
#pragma unroll
          for (int m = 0; m < 5; ++m) {
            const int s = sb + m;
            const int r = min(max(s, 0), H2 - 1);
            const float* rp = s2 + (size_t)(r & (RG::S2 - 1)) * W2;
            float c = 0.f, l = 0.f, rr = 0.f;
            if (act) {
              c = rp[t];
              l = atL ? c : rp[t - 1];
              rr = atR ? c : rp[t + 1];
            }
            wc[0] = wc[1]; wc[1] = wc[2]; wc[2] = c;
            wl[0] = wl[1]; wl[1] = wl[2]; wl[2] = l;
            wr[0] = wr[1]; wr[1] = wr[2]; wr[2] = rr;
            if (m >= 2) {
              const int y = s - 1;
              const bool row_ok = y >= 0 && y < H2 && (m < 4 || y == H2 - 1);
              if (act && row_ok) {
                float hy = wc[2] - wc[0];
                if (y == 0 || y == H2 - 1) hy = hy + hy;
                const float hx = (wr[1] - wl[1]) * ((atL || atR) ? 2.f : 1.f);
                float v0, v1, v2;
                shade<DEG>(A.L[2], hx, hy, v0, v1, v2);
                uint8_t* o = out2 + ((size_t)y * W2 + t) * 3;
                o[0] = (uint8_t)(q8(v0) & 0xFFu);
                o[1] = (uint8_t)(q8(v1) & 0xFFu);
                o[2] = (uint8_t)(q8(v2) & 0xFFu);
              }
            }
          }
        }
      }
    }
  }
}

// smallest tick count that produces every row of every level (see header)
int pyramid_ticks(int H, int levels) {
  int k = (H + 1 + 7) / 8 + 1;
  if (levels >= 2) k = std::max({k, (H + 4 + 7) / 8 + 1, (H / 2 + 3 + 3) / 4 + 1});
  if (levels >= 3) k = std::max(k, (H / 4 + 2 + 1) / 2 + 1);
  return k;
}

size_t pyramid_smem(int R, int W, int stages) {
  return 128 + (size_t)stages * kHalf * W * 4 + (size_t)(14 - R) * W * 4 + (size_t)6 * (W / 2) * 4 +
         (size_t)4 * (W / 4) * 4;
}

template <int R, int LEVELS, int DEG>
int launch_pyramid(const float* depth, int64_t n, int H, int W, PyrArgs& A, cudaStream_t stream) {
  auto kern = pyramid_fused_kernel<R, LEVELS, DEG>;
  if (int rc = set_max_dynamic_smem(reinterpret_cast<const void*>(kern), 227 * 1024)) return rc;
  const char* e = std::getenv("TACSL_PYR_STAGES");
  A.stages = std::min(std::max(e && *e ? std::atoi(e) : 3, 2), kPMaxStages);
  A.ticks = pyramid_ticks(H, LEVELS);
  const size_t smem = pyramid_smem(R, W, A.stages);
  const int threads = ((W / 4 + 31) / 32) * 32 + 32;
  int per_sm = 0;
  cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, kern, threads, smem);
  if (per_sm < 1) return set_error(TACSL_ERR_INVALID_ARGUMENT, "rgb_pyramid: image too wide for shared memory");
  const int64_t grid = std::min<int64_t>(n, (int64_t)sm_count(current_device()) * per_sm);
  kern<<<(unsigned)grid, threads, smem, stream>>>(depth, n, H, W, A);
  return check_launch("pyramid_fused_kernel");
}

template <int R, int LEVELS>
int dispatch_deg(int deg, const float* depth, int64_t n, int H, int W, PyrArgs& A, cudaStream_t s) {
  switch (deg) {
    case 2: return launch_pyramid<R, LEVELS, 2>(depth, n, H, W, A, s);
    case 3: return launch_pyramid<R, LEVELS, 3>(depth, n, H, W, A, s);
    case 4: return launch_pyramid<R, LEVELS, 4>(depth, n, H, W, A, s);
  }
  return set_error(TACSL_ERR_INVALID_ARGUMENT, "rgb_pyramid: LUT degree must be in [2, 4]");
}

template <int R>
int dispatch_levels(int levels, int deg, const float* depth, int64_t n, int H, int W, PyrArgs& A,
                    cudaStream_t s) {
  switch (levels) {
    case 1: return dispatch_deg<R, 1>(deg, depth, n, H, W, A, s);
    case 2: return dispatch_deg<R, 2>(deg, depth, n, H, W, A, s);
    case 3: return dispatch_deg<R, 3>(deg, depth, n, H, W, A, s);
  }
  return set_error(TACSL_ERR_INVALID_ARGUMENT, "rgb_pyramid: levels must be in [1, 3]");
}

}  // namespace
}  // namespace tacsl

using namespace tacsl;

extern "C" int tacsl_rgb_pyramid_supported(int height, int width, int radius, int levels) {
  if (levels < 1 || levels > 3 || radius < 0 || radius > 4) return 0;
  if (width < 8 || width % 4 != 0 || width / 4 > kPMaxCons) return 0;
  if (height < 4 || height % 4 != 0) return 0;
  return pyramid_smem(radius, width, 2) <= 227 * 1024 ? 1 : 0;
}

extern "C" int tacsl_rgb_pyramid(const tacsl_lut_t* luts, int levels, const float* depth, int64_t n_images,
                                 int height, int width, const float* taps, int radius, uint8_t* const* out,
                                 void* stream) {
  if (n_images < 0) return set_error(TACSL_ERR_INVALID_ARGUMENT, "rgb_pyramid: negative image count");
  if (!tacsl_rgb_pyramid_supported(height, width, radius, levels))
    return set_error(TACSL_ERR_INVALID_ARGUMENT,
                     "rgb_pyramid: needs levels in [1,3], radius in [0,4], width % 4 == 0 (8..1024), "
                     "height % 4 == 0 (see tacsl_rgb_pyramid_supported)");
  if (!luts || !out || (radius > 0 && !taps)) return set_error(TACSL_ERR_INVALID_ARGUMENT, "rgb_pyramid: null pointer");
  const int deg = luts[0] ? luts[0]->degree : 0;
  for (int l = 0; l < levels; ++l) {
    if (!luts[l] || !out[l]) return set_error(TACSL_ERR_INVALID_ARGUMENT, "rgb_pyramid: null LUT or output");
    if (luts[l]->width != (width >> l) || luts[l]->height != (height >> l))
      return set_error(TACSL_ERR_LUT_RESOLUTION_MISMATCH, "rgb_pyramid: level LUT image_size does not match");
    if (luts[l]->degree != deg) return set_error(TACSL_ERR_INVALID_ARGUMENT, "rgb_pyramid: LUT degrees differ");
  }
  if (n_images == 0) return TACSL_OK;
  if (!depth || (reinterpret_cast<uintptr_t>(depth) & 15) != 0)
    return set_error(TACSL_ERR_INVALID_ARGUMENT, "rgb_pyramid: depth must be 16-byte aligned");
  if ((reinterpret_cast<uintptr_t>(out[0]) & 3) != 0 || (levels >= 2 && (reinterpret_cast<uintptr_t>(out[1]) & 1)))
    return set_error(TACSL_ERR_INVALID_ARGUMENT, "rgb_pyramid: output alignment (4 B level 0, 2 B level 1)");
  PyrArgs A;
  std::memset(&A, 0, sizeof(A));
  const int K = 2 * radius + 1;
  auto w = [&](int k) { return (k >= 0 && k < K && radius > 0) ? taps[k] : 0.f; };
  for (int k = 0; k < 9; ++k) A.w[k] = radius > 0 ? w(k) : (k == 0 ? 1.f : 0.f);
  for (int m = 0; m < 6; ++m) {
    A.we[m] = make_float2(w(2 * m), w(2 * m + 1));
    A.wo[m] = make_float2(w(2 * m - 1), w(2 * m));
  }
  const float pw[5] = {0.0625f, 0.25f, 0.375f, 0.25f, 0.0625f};  // smoothing.BINOMIAL5, exact in fp32
  for (int k = 0; k < 5; ++k) A.pw[k] = pw[k];
  for (int l = 0; l < levels; ++l) {
    A.L[l] = luts[l]->params;
    A.out[l] = out[l];
  }
  cudaStream_t s = (cudaStream_t)stream;
  switch (radius) {
    case 0: return dispatch_levels<0>(levels, deg, depth, n_images, height, width, A, s);
    case 1: return dispatch_levels<1>(levels, deg, depth, n_images, height, width, A, s);
    case 2: return dispatch_levels<2>(levels, deg, depth, n_images, height, width, A, s);
    case 3: return dispatch_levels<3>(levels, deg, depth, n_images, height, width, A, s);
    default: return dispatch_levels<4>(levels, deg, depth, n_images, height, width, A, s);
  }
}
