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

struct PyrArgs {
  float w[9];            // Gaussian taps, 2R+1
  float2 we[6], wo[6];   // horizontal pair weights, first tap on an even / odd column (pyramid.cu Taps)
  float pw[5];           // pyramid taps [1, 4, 6, 4, 1] / 16
  LutParams L[3];        // level LUTs (level_lut: c_ij 2^-l(i+j)), pre-scaled like every K1 LUT
  uint8_t* out[3];       // (n, H_l, W_l, 3) uint8
  int ticks;
};

template <int R>
struct Ring {  // line-ring depths (rows), powers of two: slot = row & (S - 1)
  static constexpr int S0 = 16;  // >= 8 new rows + 2 read back + the R-row lag of the filter
  static constexpr int S1 = 8;   // >= 4 new + 2 read back
  static constexpr int S2 = 4;   // >= 2 new + 2 read back
};
constexpr int kPad = 4;  // floats of edge padding on both sides of every ring row ('nearest' borders)

__device__ __forceinline__ void pyr_bar(int n) { asm volatile("bar.sync 1, %0;" ::"r"(n) : "memory"); }

__device__ __forceinline__ float2 f2(float a, float b) { return make_float2(a, b); }

// uint8 RGB of a column quad (two pixel pairs) with K1's arithmetic:
// doubled gradients, the level LUT's packed Horner, saturating last step,
// biased rounding, PRMT packing into three words.
template <int DEG>
__device__ __forceinline__ void shade_quad(const LutParams& L, const float4 up, const float4 c, float left,
                                           float right, const float4 dn, bool edge_row, float m0, float m3,
                                           uint32_t& w0, uint32_t& w1, uint32_t& w2) {
  float2 hy01 = __fadd2_rn(make_float2(dn.x, dn.y), make_float2(-up.x, -up.y));
  float2 hy23 = __fadd2_rn(make_float2(dn.z, dn.w), make_float2(-up.z, -up.w));
  if (edge_row) {
    hy01 = __fadd2_rn(hy01, hy01);
    hy23 = __fadd2_rn(hy23, hy23);
  }
  const float2 hx01 = make_float2((c.y - left) * m0, c.z - c.x);
  const float2 hx23 = make_float2(c.w - c.y, (right - c.z) * m3);
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
  w0 = __byte_perm(__byte_perm(__float_as_uint(qa.x), __float_as_uint(qa.y), 0x0040),
                   __byte_perm(__float_as_uint(qb.x), __float_as_uint(qb.y), 0x0040), 0x5410);
  w1 = __byte_perm(__byte_perm(__float_as_uint(qc.x), __float_as_uint(qc.y), 0x0040),
                   __byte_perm(__float_as_uint(qd.x), __float_as_uint(qd.y), 0x0040), 0x5410);
  w2 = __byte_perm(__byte_perm(__float_as_uint(qe.x), __float_as_uint(qe.y), 0x0040),
                   __byte_perm(__float_as_uint(qf.x), __float_as_uint(qf.y), 0x0040), 0x5410);
}

// a pixel pair (level 1): 6 bytes as three 16-bit halves
template <int DEG>
__device__ __forceinline__ void shade_pair(const LutParams& L, float2 up, float2 c, float left, float right,
                                           float2 dn, bool edge_row, float m0, float m1, uint32_t& h0,
                                           uint32_t& h1, uint32_t& h2) {
  float2 hy = __fadd2_rn(dn, make_float2(-up.x, -up.y));
  if (edge_row) hy = __fadd2_rn(hy, hy);
  const float2 hx = make_float2((c.y - left) * m0, (right - c.x) * m1);
  const float2 r = poly2_sat<DEG>(L.c[0], hx, hy);
  const float2 g = poly2_sat<DEG>(L.c[1], hx, hy);
  const float2 b = poly2_sat<DEG>(L.c[2], hx, hy);
  const float2 qa = q8x2(make_float2(r.x, g.x));
  const float2 qb = q8x2(make_float2(b.x, r.y));
  const float2 qc = q8x2(make_float2(g.y, b.y));
  h0 = __byte_perm(__float_as_uint(qa.x), __float_as_uint(qa.y), 0x0040);
  h1 = __byte_perm(__float_as_uint(qb.x), __float_as_uint(qb.y), 0x0040);
  h2 = __byte_perm(__float_as_uint(qc.x), __float_as_uint(qc.y), 0x0040);
}

// horizontal pyramid tap sum at one output column from the 5 input columns
// around it: even-column chain + odd-column chain (K5's FFMA2 lanes; its
// trailing zero-weight tap is an exact no-op and is left out)
__device__ __forceinline__ float pyr_h(const float* pw, float a, float b, float c, float d, float e) {
  const float ev = __fmaf_rn(e, pw[4], __fmaf_rn(c, pw[2], __fmaf_rn(a, pw[0], 0.f)));
  const float od = __fmaf_rn(d, pw[3], __fmaf_rn(b, pw[1], 0.f));
  return ev + od;
}

// Shared-memory layout (floats after a 128-byte barrier block):
//   input ring : 2 x 4 rows x (W + 8)        (TMA writes columns 4 .. W+3)
//   S0 ring    : 16 x (W + 8)    smoothed level-0 rows
//   S1 ring    : 8 x (W/2 + 8)   level-1 depth rows
//   S2 ring    : 4 x (W/4 + 8)   level-2 depth rows
// Every row carries 4 padding floats on each side holding its edge value
// ('nearest' borders), written by the edge thread that owns the edge
// column -- so no thread ever selects a clamped neighbour in the row loops.
template <int R, int LEVELS, int DEG>
__global__ void __maxnreg__(128)
    pyramid_fused_kernel(const float* __restrict__ depth, int64_t n, int H, int W, const PyrArgs A) {
  extern __shared__ __align__(128) unsigned char smem[];
  using RG = Ring<R>;
  constexpr int NT = 2 * R + 1;
  const int NQ = W >> 2;
  const int cons_warps = (NQ + 31) >> 5;
  const int n_cons = cons_warps * 32;
  const int H1 = H >> 1, H2 = H >> 2, W1 = W >> 1, W2 = W >> 2;
  const int WP = W + 2 * kPad, W1P = W1 + 2 * kPad, W2P = W2 + 2 * kPad;
  uint64_t* full = reinterpret_cast<uint64_t*>(smem);  // full[h]: half h of the tick's input rows landed
  uint64_t* barA = full + 2;  // split barriers of the step loop (count: consumer warps)
  uint64_t* barC = full + 3;
  const int lane = threadIdx.x & 31;
  float* in_buf = reinterpret_cast<float*>(smem + 128);
  const int stage_f = kHalf * WP;
  float* s0 = in_buf + 2 * stage_f;
  float* s1 = s0 + RG::S0 * WP;
  float* s2 = s1 + RG::S1 * W1P;
  const int K = A.ticks;
  const int kG = (H + 7) >> 3;  // last tick with input rows (8k - 4 <= H + 3)

  // Input rows of tick k, image img, into the two half stages: issued by
  // thread 0 once every consumer has finished the previous tick's G phase
  // (the named barrier that follows it), so the stages need no "empty"
  // handshake and the CTA has no producer warp (3 CTAs per SM fit the
  // register file and shared memory).
  auto issue_tick = [&](int64_t img, int k) {
    fence_proxy_async_smem();  // the stage's generic-proxy reads happen before the async overwrite
    const float* src = depth + (size_t)img * H * W;
    const uint32_t row_bytes = (uint32_t)W * 4u;
#pragma unroll
    for (int h = 0; h < 2; ++h) {
      const int j0 = 8 * k - 4 + kHalf * h;
      float* dst = in_buf + h * stage_f + kPad;
      mbar_arrive_expect_tx(&full[h], kHalf * row_bytes);
      // rows outside the image arrive as the clamped edge row ('nearest')
#pragma unroll
      for (int i = 0; i < kHalf; ++i) {
        const int r = min(max(j0 + i, 0), H - 1);
        bulk_g2s(dst + i * WP, src + (size_t)r * W, row_bytes, &full[h]);
      }
    }
  };

  if (threadIdx.x == 0) {
    mbar_init(&full[0], 1);
    mbar_init(&full[1], 1);
    mbar_init(barA, cons_warps);
    mbar_init(barC, cons_warps);
    fence_mbar_init();
    fence_proxy_async_smem();
    if (blockIdx.x < n) issue_tick(blockIdx.x, 0);
  }
  __syncthreads();

  // ------------------------------------------------------------ consumers ---
  const bool act = (int)threadIdx.x < NQ;
  const int t = min((int)threadIdx.x, NQ - 1);  // padding lanes shadow the last quad, store nothing
  const int x0 = 4 * t;
  const bool atL = act && t == 0, atR = act && t == NQ - 1;
  const float m0 = t == 0 ? 2.f : 1.f;  // np.gradient's one-sided borders are not halved
  const float m3 = t == NQ - 1 ? 2.f : 1.f;
  float2 acc[8][2];  // vertical Gaussian accumulators, slot = output row & 7
  float2 acc1[2];    // level-1 vertical accumulators (column pair), slot = row & 1
  float acc2[2];     // level-2 vertical accumulators, slot = row & 1
#pragma unroll
  for (int i = 0; i < 8; ++i) acc[i][0] = acc[i][1] = f2(0.f, 0.f);
  acc1[0] = acc1[1] = f2(0.f, 0.f);
  acc2[0] = acc2[1] = 0.f;
  uint32_t ph = 0;  // phase of both half stages (each completes once per G tick)
  uint32_t phA = 0, phC = 0;  // split barriers A (S0 rows of a step written) and C (S2 rows written)
  const int W3 = 3 * W, W13 = 3 * W1, W23 = 3 * W2;
  // L2 of one (image, tick): runs one step late, in the gap of the next
  // step's split barrier (see the loop below)
  auto level2 = [&](int64_t im, int k) {
    // level 2 by (row, pixel pair): the tick's two level-2 rows split over
    // two groups of W/8 threads, every warp equally busy (the phase's time
    // is its busiest warp's); K1's pair arithmetic
    const int NP2 = W2 >> 1;
    const int g = (int)threadIdx.x / NP2;
    const int p = (int)threadIdx.x - g * NP2;
    if (k < 1 || g > 1) return;
    const float n0 = p == 0 ? 2.f : 1.f, n1 = p == NP2 - 1 ? 2.f : 1.f;
#pragma unroll
    for (int e = 0; e < 2; ++e) {
      // e = 0: row 2k-5+g (the tick's regular rows); e = 1: row 2k-3 when it
      // is the image's last level-2 row (its down neighbour is itself)
      const int y = 2 * k - 5 + g + 2 * e;
      const bool valid = e == 0 ? (y >= 0 && y < H2) : (g == 0 && y == H2 - 1);
      if (!valid) continue;
      const int ru = max(y - 1, 0), rd = min(y + 1, H2 - 1);
      const float* rc = s2 + (y & (RG::S2 - 1)) * W2P + kPad + 2 * p;
      const float2 up = *reinterpret_cast<const float2*>(s2 + (ru & (RG::S2 - 1)) * W2P + kPad + 2 * p);
      const float2 dn = *reinterpret_cast<const float2*>(s2 + (rd & (RG::S2 - 1)) * W2P + kPad + 2 * p);
      const float2 c = *reinterpret_cast<const float2*>(rc);
      uint32_t h0, h1, h2;
      shade_pair<DEG>(A.L[2], up, c, rc[-1], rc[2], dn, y == 0 || y == H2 - 1, n0, n1, h0, h1, h2);
      uint16_t* o = reinterpret_cast<uint16_t*>(A.out[2] + ((size_t)im * H2 + y) * W23 + 6 * p);
      o[0] = (uint16_t)h0;
      o[1] = (uint16_t)h1;
      o[2] = (uint16_t)h2;
    }
  };

  // One step = one tick k of one image:
  //   G(k)  -> arrive A -> [wait C(k-1), L2 of the previous step] -> wait A
  //   -> (thread 0: next tick's TMA) -> L0(k) -> barrier B -> L1(k) -> arrive C
  // A and C are mbarriers (arrive now, wait later): the wait for the slowest
  // warp's G is filled with the previous step's L2, and the wait for its L1
  // with this step's G, so only B blocks.  Hazards: S0 is rewritten by G
  // only after B (all L0 reads done); S1 by L0 only after A (all L1 reads
  // done: every warp arrives at A after its L1); S2 by L1 only after B (all
  // L2 reads done before A).  Without a level 2 (LEVELS < 3) A and B are
  // plain barriers.
  int64_t img = blockIdx.x;
  int k = 0;
  int64_t pimg = -1;  // the step whose L2 is pending
  int pk = 0;
  while (img < n) {
    uint8_t* out0 = A.out[0] + (size_t)img * H * W3 + 3 * x0;
    uint8_t* out1 = LEVELS >= 2 ? A.out[1] + (size_t)img * H1 * W13 + 6 * t : nullptr;
    {
      // ------------------------------------------------------------ G ---
      if (k <= kG) {
#pragma unroll
        for (int h = 0; h < 2; ++h) {
          mbar_wait_parity(&full[h], ph);
          float* st = in_buf + h * stage_f;
          if (atL) {  // left padding = column 0 of each row
#pragma unroll
            for (int i = 0; i < kHalf; ++i) {
              const float v = st[i * WP + kPad];
              *reinterpret_cast<float4*>(st + i * WP) = make_float4(v, v, v, v);
            }
          }
          if (atR) {  // right padding = column W-1
#pragma unroll
            for (int i = 0; i < kHalf; ++i) {
              const float v = st[i * WP + kPad + W - 1];
              *reinterpret_cast<float4*>(st + i * WP + kPad + W) = make_float4(v, v, v, v);
            }
          }
#pragma unroll
          for (int i = 0; i < kHalf; ++i) {
            const int ii = kHalf * h + i;  // h-row j = 8k - 4 + ii
            const int y = 8 * k - 4 + ii - R;  // the smoothed row this h-row completes
            const float* row = st + i * WP + kPad + x0;
            float4 o;
            if constexpr (R == 0) {
              o = *reinterpret_cast<const float4*>(row);
            } else {
              const float4 va = *reinterpret_cast<const float4*>(row - 4);
              const float4 vb = *reinterpret_cast<const float4*>(row);
              const float4 vc = *reinterpret_cast<const float4*>(row + 4);
              const float v[12] = {va.x, va.y, va.z, va.w, vb.x, vb.y, vb.z, vb.w, vc.x, vc.y, vc.z, vc.w};
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
                } else {
                  acc[slot][0] = __ffma2_rn(h01, w, tt == 0 ? f2(0.f, 0.f) : acc[slot][0]);
                  acc[slot][1] = __ffma2_rn(h23, w, tt == 0 ? f2(0.f, 0.f) : acc[slot][1]);
                }
              }
            }
            if (y >= 0 && y < H) {
              float* dst = s0 + (y & (RG::S0 - 1)) * WP + kPad;
              if (act) *reinterpret_cast<float4*>(dst + x0) = o;
              if (atL) *reinterpret_cast<float2*>(dst - 2) = f2(o.x, o.x);
              if (atR) dst[W] = o.w;
            }
          }
        }
        ph ^= 1u;
      }
    }
    if constexpr (LEVELS >= 3) {
      __syncwarp();
      if (lane == 0) mbar_arrive(barA);
      if (pimg >= 0) {
        mbar_wait_parity(barC, phC);
        phC ^= 1u;
        if (pk >= 1) level2(pimg, pk);
      }
      mbar_wait_parity(barA, phA);
      phA ^= 1u;
    } else {
      pyr_bar(n_cons);  // S0 rows of this tick are visible; the input stages are free
    }
    if (threadIdx.x == 0) {
      if (k < kG) issue_tick(img, k + 1);
      else if (k == kG && img + gridDim.x < n) issue_tick(img + gridDim.x, 0);
    }
    {
      // ----------------------------------------------------------- L0 ---
      if (k >= 1) {
        const int sb = 8 * k - 10;
        float4 wq[3];  // quads of rows s-2, s-1, s
        float wl = 0.f, wr = 0.f;  // left / right neighbour of row s-1
        uint8_t* orow = out0 + (sb + 1) * W3;  // row s-1 at m = 2
#pragma unroll
        for (int m = 0; m < 10; ++m) {
          const int sr = sb + m;
          const int r = min(max(sr, 0), H - 1);
          const float* rp = s0 + (r & (RG::S0 - 1)) * WP + kPad + x0;
          const float4 c = *reinterpret_cast<const float4*>(rp);
          const float2 l = *reinterpret_cast<const float2*>(rp - 2);
          const float rr = rp[4];
          wq[0] = wq[1];
          wq[1] = wq[2];
          wq[2] = c;
          if (m >= 2) {
            const int y = sr - 1;
            uint32_t w0, w1, w2;
            shade_quad<DEG>(A.L[0], wq[0], wq[1], wl, wr, wq[2], y == 0 || y == H - 1, m0, m3, w0, w1, w2);
            if (act && y >= 0 && y < H) {
              uint32_t* o = reinterpret_cast<uint32_t*>(orow);
              o[0] = w0;
              o[1] = w1;
              o[2] = w2;
            }
            orow += W3;
          }
          wl = l.y;
          wr = rr;
          if constexpr (LEVELS >= 2) {
            if (m < 8) {
              // virtual S0 row i = sr (row clamp(i)) decimated at level-1
              // columns 2t, 2t+1 (input columns 4t-2 .. 4t+4)
              const float2 hp = f2(pyr_h(A.pw, l.x, l.y, c.x, c.y, c.z), pyr_h(A.pw, c.x, c.y, c.z, c.w, rr));
#pragma unroll
              for (int tt = 4; tt >= 0; --tt) {
                if (((m - tt) & 1) != 0) continue;
                const int slot = ((m - tt + 8) >> 1) & 1;  // (level-1 row) & 1
                const float2 w = f2(A.pw[tt], A.pw[tt]);
                if (tt == 4) {
                  const float2 o = __ffma2_rn(hp, w, acc1[slot]);
                  const int y1 = (sr + 2 - tt) >> 1;  // sr + 2 - tt is even
                  if (y1 >= 0 && y1 < H1) {
                    float* dst = s1 + (y1 & (RG::S1 - 1)) * W1P + kPad;
                    if (act) *reinterpret_cast<float2*>(dst + 2 * t) = o;
                    if (atL) *reinterpret_cast<float2*>(dst - 2) = f2(o.x, o.x);
                    if (atR) dst[W1] = o.y;
                  }
                } else {
                  acc1[slot] = __ffma2_rn(hp, w, tt == 0 ? f2(0.f, 0.f) : acc1[slot]);
                }
              }
            }
          }
        }
      }
    }
    pyr_bar(n_cons);  // B: S1 rows of this tick are visible; S0 reads done
    {
      // ----------------------------------------------------------- L1 ---
      if constexpr (LEVELS >= 2) {
        if (k >= 1) {
          const int sb = 4 * k - 8;
          float2 wc[3];
          float wl = 0.f, wr = 0.f;
          uint8_t* orow = out1 + (sb + 1) * W13;
#pragma unroll
          for (int m = 0; m < 6; ++m) {
            const int sr = sb + m;
            const int r = min(max(sr, 0), H1 - 1);
            const float* rp = s1 + (r & (RG::S1 - 1)) * W1P + kPad + 2 * t;
            const float2 c = *reinterpret_cast<const float2*>(rp);
            const float2 l = *reinterpret_cast<const float2*>(rp - 2);
            const float rr = rp[2];
            wc[0] = wc[1];
            wc[1] = wc[2];
            wc[2] = c;
            if (m >= 2) {
              const int y = sr - 1;
              uint32_t h0, h1, h2;
              shade_pair<DEG>(A.L[1], wc[0], wc[1], wl, wr, wc[2], y == 0 || y == H1 - 1, m0, m3, h0, h1, h2);
              if (act && y >= 0 && y < H1) {
                uint16_t* o = reinterpret_cast<uint16_t*>(orow);
                o[0] = (uint16_t)h0;
                o[1] = (uint16_t)h1;
                o[2] = (uint16_t)h2;
              }
              orow += W13;
              if constexpr (LEVELS >= 3) {
                // virtual level-1 row i = sr decimated at level-2 column t
                const float hv = pyr_h(A.pw, l.x, l.y, c.x, c.y, rr);
#pragma unroll
                for (int tt = 4; tt >= 0; --tt) {
                  if (((m - tt) & 1) != 0) continue;
                  const int slot = ((m - tt + 2) >> 1) & 1;  // (level-2 row) & 1
                  if (tt == 4) {
                    const float o = __fmaf_rn(hv, A.pw[4], acc2[slot]);
                    const int y2 = (sr + 2 - tt) >> 1;
                    if (y2 >= 0 && y2 < H2) {
                      float* dst = s2 + (y2 & (RG::S2 - 1)) * W2P + kPad;
                      if (act) dst[t] = o;
                      if (atL) dst[-1] = o;
                      if (atR) dst[W2] = o;
                    }
                  } else {
                    acc2[slot] = __fmaf_rn(hv, A.pw[tt], tt == 0 ? 0.f : acc2[slot]);
                  }
                }
              }
            }
            wl = l.y;
            wr = rr;
          }
        }
      }
    }
    if constexpr (LEVELS >= 3) {
      __syncwarp();
      if (lane == 0) mbar_arrive(barC);
      pimg = img;
      pk = k;
    }
    if (++k == K) {
      k = 0;
      img += gridDim.x;
    }
  }
  if constexpr (LEVELS >= 3) {
    if (pimg >= 0) {  // the last step's L2
      mbar_wait_parity(barC, phC);
      if (pk >= 1) level2(pimg, pk);
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

size_t pyramid_smem(int R, int W) {
  (void)R;
  const size_t WP = W + 2 * kPad, W1P = W / 2 + 2 * kPad, W2P = W / 4 + 2 * kPad;
  return 128 + ((size_t)2 * kHalf * WP + 16 * WP + 8 * W1P + 4 * W2P) * 4;
}

template <int R, int LEVELS, int DEG>
int launch_pyramid(const float* depth, int64_t n, int H, int W, PyrArgs& A, cudaStream_t stream) {
  auto kern = pyramid_fused_kernel<R, LEVELS, DEG>;
  if (int rc = set_max_dynamic_smem(reinterpret_cast<const void*>(kern), 227 * 1024)) return rc;
  // all of the unified L1/shared array as shared memory: 3 CTAs per SM (a
  // host-side attribute, cheap, set on every call so every device has it)
  cudaFuncSetAttribute(reinterpret_cast<const void*>(kern), cudaFuncAttributePreferredSharedMemoryCarveout,
                       (int)cudaSharedmemCarveoutMaxShared);
  A.ticks = pyramid_ticks(H, LEVELS);
  const size_t smem = pyramid_smem(R, W);
  const int threads = ((W / 4 + 31) / 32) * 32;
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
  if (width < 8 || width % (levels >= 3 ? 8 : 4) != 0 || width / 4 > kPMaxCons) return 0;
  if (height < 4 || height % 4 != 0) return 0;
  return pyramid_smem(radius, width) <= 227 * 1024 ? 1 : 0;
}

extern "C" int tacsl_rgb_pyramid(const tacsl_lut_t* luts, int levels, const float* depth, int64_t n_images,
                                 int height, int width, const float* taps, int radius, uint8_t* const* out,
                                 void* stream) {
  StreamDevice stream_device_(stream);
  if (n_images < 0) return set_error(TACSL_ERR_INVALID_ARGUMENT, "rgb_pyramid: negative image count");
  if (!tacsl_rgb_pyramid_supported(height, width, radius, levels))
    return set_error(TACSL_ERR_INVALID_ARGUMENT,
                     "rgb_pyramid: needs levels in [1,3], radius in [0,4], width % 4 == 0 (% 8 for 3 "
                     "levels; 8..1024), height % 4 == 0 (see tacsl_rgb_pyramid_supported)");
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
  if ((reinterpret_cast<uintptr_t>(out[0]) & 3) != 0 || (levels >= 2 && (reinterpret_cast<uintptr_t>(out[1]) & 1)) ||
      (levels >= 3 && (reinterpret_cast<uintptr_t>(out[2]) & 1)))
    return set_error(TACSL_ERR_INVALID_ARGUMENT, "rgb_pyramid: output alignment (4 B level 0, 2 B levels 1-2)");
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
