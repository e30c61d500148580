// K1: depth -> tactile RGB, one fused pass.
//
// Replaces render/lut.py:68-76 depth_to_rgb = depth_gradients (lut.py:25-28,
// np.gradient: central inside, one-sided un-halved at the borders) ->
// PolyLut.evaluate (lut.py:56-65: per-channel polynomial in (g_x, g_y),
// clip [0,1]) -> optional to_uint8 (render/imageio.py:8-11).
//
// Layout: depth (N, H, W) fp32, rgb (N, H, W, 3) HWC, u8 and/or fp32.
//
// Fast path (W % 4 == 0, W <= 1280, 16B-aligned pointers): persistent CTAs
// (2 per SM) walk work units = (image, band of B rows).  A loader warp
// streams each band plus its two halo rows global->shared with ONE
// bulk-async copy (cp.async.bulk, the 1-D TMA engine) into a STAGES-deep
// ring completed on mbarriers; a storer warp sends each finished band back
// with one bulk shared->global store; consumer warps hand stages and output
// tiles over through mbarriers only (no CTA-wide barrier in the loop).
// Consumer thread (g, xq) owns column quad xq (4 pixels) and walks RPT
// consecutive rows of row-group g with a rolling up/centre/down register
// window (one 16B shared load per row).  Pixels are shaded in pairs on the
// Blackwell packed-fp32 pipe (FFMA2/FADD2: two pixels per instruction);
// only the last Horner step is scalar, to get the free .SAT clamp.  The
// uint8 bytes are packed with PRMT.  HBM sees each depth byte read once and
// each RGB byte written once (98% of the measured copy bandwidth at 240x320).
// The same kernel serves the binned LUT (BIN: per-pair coefficient tables)
// and the fused sensor step (FF: force-field warps beside the shading).
#include <algorithm>
#include <array>
#include <cstdlib>
#include <mutex>
#include <type_traits>
#include <vector>

#include "common.cuh"
#include "ff_device.cuh"
#include "handles.h"
#include "shade.cuh"

namespace tacsl {
namespace {

constexpr int kMaxThreads = 320;  // consumer threads per CTA (+ 2 producer warps); 2 CTAs/SM at 240x320
constexpr int kMaxThreadsFF = 480;  // fused step: one CTA per SM with the force-field warps
constexpr int kMaxStages = 6;
constexpr size_t kSmemPerSm = 227 * 1024;  // opt-in dynamic shared memory per CTA on sm_100
constexpr int kDefaultRpt = 8;  // rows per thread per band (rolling 3-row register window)
constexpr int kFFWarps = 4;     // force-field warps per CTA in the fused sensor step

// poly2_sat with per-thread coefficient PAIRS (c, c), in registers or L1 (the
// binned LUT: each pixel pair's bin has its own table, K6)
template <int DEG, bool LDG>
__device__ __forceinline__ float2 poly2_sat_p(const float2* __restrict__ c, float2 hx, float2 hy) {
  auto coef = [&](int t) { return LDG ? __ldg(c + t) : c[t]; };
  float2 acc = bc(0.f);
  float2 out = bc(0.f);
#pragma unroll
  for (int i = DEG; i >= 0; --i) {
    float2 p = coef(term_index(i, DEG - i));
#pragma unroll
    for (int j = DEG - i - 1; j >= 0; --j) p = __ffma2_rn(p, hy, coef(term_index(i, j)));
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

// Binned LUT (K6 on this pipeline): (bins_y * bins_x, 3, T) coefficient
// pairs; the host guarantees no pixel pair straddles an x-bin edge.
struct BinArgs {
  const float2* __restrict__ pairs;
  int bins_y, bins_x;
  int tab_ybins;  // > 0: degrees 3-4 stage the band's y bins in shared memory (at most this many)
};

// y bins one band of `band` rows can touch (max over the bands of the image)
inline int band_ybins(int H, int band, int bins_y) {
  int m = 0;
  for (int r0 = 0; r0 < H; r0 += band)
    m = std::max(m, (std::min(r0 + band, H) - 1) * bins_y / H - r0 * bins_y / H + 1);
  return m;
}

// barrier over the consumer warps only (the loader / storer warps never join)
__device__ __forceinline__ void consumer_bar(int threads) {
  asm volatile("bar.sync 1, %0;" ::"r"(threads) : "memory");
}

struct Layout {
  int band, rpt, groups, stages;
  size_t in_stage_floats, out_stage_bytes;
  static constexpr size_t kBarBytes = 128;
  size_t bytes(bool u8) const {
    return kBarBytes + stages * in_stage_floats * sizeof(float) + (u8 ? 2 * out_stage_bytes : 0);
  }
};

// Warp roles.  Consumer warps (the first ceil(QW*groups/32) warps) shade;
// the next warp streams bands in, the last one streams RGB out.  Stages and
// output tiles change hands through mbarriers only -- no CTA-wide barrier in
// the steady state, so consumer warps drift freely across bands.
//   full[s]  : TMA transaction barrier, band landed in stage s
//   empty[s] : every consumer warp has its rows of stage s in registers
//   ready[b] : every consumer warp wrote its part of output tile b
//   ofree[b] : the bulk store of tile b has finished reading it
template <int DEG, int RPT, bool U8, bool F32, bool FF, bool BIN = false>
__global__ void __launch_bounds__(FF ? kMaxThreadsFF + 64 + kFFWarps * 32 : kMaxThreads + 64, 1) rgb_bulk_kernel(const float* __restrict__ depth,
                                                                    int64_t n_images, int H, int W, int groups,
                                                                    int stages, uint8_t* __restrict__ out_u8,
                                                                    float* __restrict__ out_f32, const LutParams L,
                                                                    int bulk_store, const FFArgs<float> F,
                                                                    const BinArgs B) {
  extern __shared__ __align__(128) unsigned char smem[];
  const int QW = W >> 2;
  const int n_cons = QW * groups;
  const int cons_warps = (n_cons + 31) >> 5;  // host: blockDim.x == 32 * cons_warps + 64
  const int band = groups * RPT;
  const int bands = (H + band - 1) / band;
  const int64_t units = n_images * bands;
  const size_t in_stage = (size_t)(band + 2) * W;
  const size_t out_stage = (size_t)band * W * 3;
  uint64_t* full = reinterpret_cast<uint64_t*>(smem);
  uint64_t* empty = full + kMaxStages;
  uint64_t* ready = empty + kMaxStages;
  uint64_t* ofree = ready + 2;
  float* in_buf = reinterpret_cast<float*>(smem + Layout::kBarBytes);
  uint8_t* out_buf = reinterpret_cast<uint8_t*>(in_buf + stages * in_stage);
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;

  if (threadIdx.x == 0) {
    for (int s = 0; s < stages; ++s) {
      mbar_init(&full[s], 1);
      mbar_init(&empty[s], cons_warps);
    }
    for (int b = 0; b < 2; ++b) {
      mbar_init(&ready[b], cons_warps);
      mbar_init(&ofree[b], 1);
    }
    fence_mbar_init();
    fence_proxy_async_smem();
  }
  __syncthreads();

  if (warp == cons_warps) {
    // ---------------------------------------------------------- loader ---
    if (lane == 0) {
      int k = 0;
      for (int64_t u = blockIdx.x; u < units; u += gridDim.x, ++k) {
        const int s = k % stages;
        if (k >= stages) mbar_wait_parity_sleep(&empty[s], (uint32_t)(k / stages - 1) & 1u);
        // stage row 0 holds image row r0-1 (absent for the top band); rows
        // that do not exist are never read
        const int64_t img = u / bands;
        const int r0 = (int)(u - img * bands) * band;
        const int rs = max(r0 - 1, 0);
        const int re = min(r0 + band, H - 1);
        const uint32_t bytes = (uint32_t)(re - rs + 1) * (uint32_t)W * 4u;
        float* dst = in_buf + (size_t)s * in_stage + (size_t)(rs - (r0 - 1)) * W;
        const float* src = depth + ((size_t)img * H + rs) * (size_t)W;
        mbar_arrive_expect_tx(&full[s], bytes);
        bulk_g2s(dst, src, bytes, &full[s]);
      }
    }
    return;
  }
  if (FF && warp >= cons_warps + 2) {
    // ------------------------------------------------ force-field warps ---
    // K2 on the FP64 pipe beside the FP32/ALU-bound shading: each of the
    // CTA's kFFWarps warps takes whole sensor frames (no CTA barrier).
    ff_frames_dynamic(F, lane);
    return;
  }
  if (warp == cons_warps + 1) {
    // ---------------------------------------------------------- storer ---
    if (U8) {
      int k = 0;
      for (int64_t u = blockIdx.x; u < units; u += gridDim.x, ++k) {
        const int b = k & 1;
        mbar_wait_parity_sleep(&ready[b], (uint32_t)(k >> 1) & 1u);
        const int64_t img = u / bands;
        const int r0 = (int)(u - img * bands) * band;
        const uint32_t bytes = (uint32_t)min(band, H - r0) * (uint32_t)W * 3u;
        uint8_t* dst = out_u8 + ((size_t)img * H + r0) * (size_t)W * 3;
        const uint8_t* ob = out_buf + (size_t)b * out_stage;
        if (bulk_store & 1) {
          if (lane == 0) {
            bulk_s2g(dst, ob, bytes);
            bulk_commit();
            bulk_wait_read<1>();  // the store of tile k-1 has left shared memory
            if (k >= 1) mbar_arrive(&ofree[b ^ 1]);
          }
        } else {
          const uint32_t* s32 = reinterpret_cast<const uint32_t*>(ob);
          uint32_t* d32 = reinterpret_cast<uint32_t*>(dst);
          for (uint32_t i = lane; i < bytes / 4; i += 32) d32[i] = s32[i];
          __syncwarp();
          if (lane == 0) mbar_arrive(&ofree[b]);
        }
      }
      if ((bulk_store & 1) && lane == 0) bulk_wait_all<0>();
    }
    return;
  }

  // ------------------------------------------------------------ consumers ---
  // per-thread constants: column quad, row group (padding lanes of a partial
  // last warp get an out-of-band group and only take part in the handshakes)
  const bool is_cons = (int)threadIdx.x < n_cons;
  const int xq = threadIdx.x % QW;
  const int g = is_cons ? (int)threadIdx.x / QW : groups;
  const int x0 = xq << 2;
  const bool at_left = (x0 == 0), at_right = (x0 + 4 >= W);
  const int loff = at_left ? 0 : -1, roff = at_right ? 3 : 4;
  // binned LUT: x bins of the thread's two pixel pairs (fixed for the thread)
  const int xba = BIN ? x0 * B.bins_x / W : 0, xbb = BIN ? (x0 + 2) * B.bins_x / W : 0;
  const float m0 = at_left ? 2.f : 1.f;  // np.gradient one-sided borders are not halved:
  const float m3 = at_right ? 2.f : 1.f; // h = 2*(f1-f0) in the doubled-gradient form
  const int lr0 = g * RPT;
  const size_t row_off = (size_t)lr0 * W + x0;   // this thread's first pixel inside a band

  // unit bookkeeping without divisions in the loop
  const int64_t g_img = gridDim.x / bands;
  const int g_band = (int)(gridDim.x - g_img * bands);
  int64_t img = blockIdx.x / bands;
  int bidx = (int)(blockIdx.x - img * bands);
  int s = 0, k = 0;
  uint32_t full_phase = 0;
  // binned LUT: at degree 2 the thread's two coefficient sets (72 regs) live
  // in registers, tagged with their y bin, and are reloaded only when its rows
  // enter another y bin -- the launch keeps each CTA on one band (grid a
  // multiple of the band count), so that is rare; higher degrees would spill
  // and read the coefficients through L1
  constexpr int T = (DEG + 1) * (DEG + 2) / 2;
  constexpr bool RC = BIN && DEG == 2;
  float2 ca[RC ? 3 * T : 1], cb[RC ? 3 * T : 1];
  int yb = 0, ynext = 0, loaded_yb = -1;
  auto load_bins = [&]() {
    if constexpr (RC) {
      if (yb != loaded_yb) {
        const float2* pa = B.pairs + (size_t)(yb * B.bins_x + xba) * 3 * T;
        const float2* pb = B.pairs + (size_t)(yb * B.bins_x + xbb) * 3 * T;
#pragma unroll
        for (int i = 0; i < 3 * T; ++i) {
          ca[i] = pa[i];
          cb[i] = pb[i];
        }
        loaded_yb = yb;
      }
    }
  };
  // degrees 3-4: the y bins of the CTA's band staged in shared memory behind
  // the ring (reloaded when the band changes -- rarely, see the launch)
  float2* tab = reinterpret_cast<float2*>(out_buf + (U8 ? 2 * out_stage : 0));
  int tab_band = -1, tab_y0 = 0;
  for (; img < n_images; ++k) {
    const int r0 = bidx * band;
    const int nrows = min(band, H - r0);
    const int b = k & 1;
    const bool active = lr0 < nrows;
    if constexpr (BIN && !RC) {
      if (B.tab_ybins > 0 && bidx != tab_band) {
        const int y0 = r0 * B.bins_y / H;
        const int cnt = ((nrows + r0 - 1) * B.bins_y / H - y0 + 1) * B.bins_x * 3 * T;
        const float2* src = B.pairs + (size_t)y0 * B.bins_x * 3 * T;
        consumer_bar(cons_warps * 32);  // every consumer is done with the previous band's table
        for (int i = threadIdx.x; i < cnt; i += cons_warps * 32) tab[i] = src[i];
        consumer_bar(cons_warps * 32);
        tab_band = bidx;
        tab_y0 = y0;
      }
    }
    mbar_wait_parity(&full[s], full_phase);
    if (U8 && k >= 2) mbar_wait_parity(&ofree[b], (uint32_t)((k >> 1) - 1) & 1u);
    if (active) {
      // rolling row window up / c / dn; a missing row (above or below the
      // image) repeats its neighbour, which with the x2 below gives
      // np.gradient's one-sided border rows
      const float* p = in_buf + (size_t)s * in_stage + W + row_off;  // image row r0 + lr0
      uint32_t* op = reinterpret_cast<uint32_t*>(out_buf + (size_t)b * out_stage + row_off * 3);
      const int och = L.rep == 2 ? 6 : 3;  // float channels per output pixel
      float* of = F32 ? out_f32 + (((size_t)img * H + r0) * W + row_off) * och : nullptr;
      if constexpr (BIN) {  // y bin of this thread's first row and the first row of the next bin
        yb = (r0 + lr0) * B.bins_y / H;
        ynext = ((yb + 1) * H + B.bins_y - 1) / B.bins_y;
        load_bins();
      }
      // a missing neighbour row / column is read as the pixel itself (the
      // offsets select it), so there is no select or copy in the row loop
      float4 c = *reinterpret_cast<const float4*>(p);
      float4 up = *reinterpret_cast<const float4*>(p - ((r0 + lr0 > 0) ? W : 0));
#pragma unroll
      for (int j = 0; j < RPT; ++j) {
        if (lr0 + j >= nrows) break;
        const int r = r0 + lr0 + j;
        const float4 dn = *reinterpret_cast<const float4*>(p + ((r < H - 1) ? W : 0));
        // left/right neighbours of the quad (c.x / c.w at the side borders)
        const float left = p[loff];
        const float right = p[roff];
        // doubled gradients h = 2g (coefficients carry the 2^-(i+j))
        float2 hy01 = __fadd2_rn(make_float2(dn.x, dn.y), make_float2(-up.x, -up.y));
        float2 hy23 = __fadd2_rn(make_float2(dn.z, dn.w), make_float2(-up.z, -up.w));
        if (r == 0 || r == H - 1) {  // one-sided rows: 2*(f1-f0)
          hy01 = __fadd2_rn(hy01, hy01);
          hy23 = __fadd2_rn(hy23, hy23);
        }
        const float2 hx01 = make_float2((c.y - left) * m0, c.z - c.x);
        const float2 hx23 = make_float2(c.w - c.y, (right - c.z) * m3);
        float2 r01, g01, b01, r23, g23, b23;
        if constexpr (BIN) {
          if (r >= ynext) {  // rows cross into the next y bin
            do {
              ++yb;
              ynext = ((yb + 1) * H + B.bins_y - 1) / B.bins_y;
            } while (r >= ynext);
            load_bins();
          }
          auto eval = [&](auto ldg, const float2* qa, const float2* qb) {
            constexpr bool G = decltype(ldg)::value;
            r01 = poly2_sat_p<DEG, G>(qa, hx01, hy01);
            g01 = poly2_sat_p<DEG, G>(qa + T, hx01, hy01);
            b01 = poly2_sat_p<DEG, G>(qa + 2 * T, hx01, hy01);
            r23 = poly2_sat_p<DEG, G>(qb, hx23, hy23);
            g23 = poly2_sat_p<DEG, G>(qb + T, hx23, hy23);
            b23 = poly2_sat_p<DEG, G>(qb + 2 * T, hx23, hy23);
          };
          if constexpr (RC) {
            eval(std::false_type{}, ca, cb);
          } else if (B.tab_ybins > 0) {
            const int row = (yb - tab_y0) * B.bins_x;
            eval(std::false_type{}, tab + (row + xba) * 3 * T, tab + (row + xbb) * 3 * T);
          } else {
            eval(std::true_type{}, B.pairs + (size_t)(yb * B.bins_x + xba) * 3 * T,
                 B.pairs + (size_t)(yb * B.bins_x + xbb) * 3 * T);
          }
        } else {
          r01 = poly2_sat<DEG>(L.c[0], hx01, hy01);
          g01 = poly2_sat<DEG>(L.c[1], hx01, hy01);
          b01 = poly2_sat<DEG>(L.c[2], hx01, hy01);
          r23 = poly2_sat<DEG>(L.c[0], hx23, hy23);
          g23 = poly2_sat<DEG>(L.c[1], hx23, hy23);
          b23 = poly2_sat<DEG>(L.c[2], hx23, hy23);
        }
        if (U8) {
          // pixel order p0..p3, channel-interleaved: (r0 g0 b0 r1)(g1 b1 r2 g2)(b2 r3 g3 b3)
          const float2 qa = q8x2(make_float2(r01.x, g01.x));
          const float2 qb = q8x2(make_float2(b01.x, r01.y));
          const float2 qc = q8x2(make_float2(g01.y, b01.y));
          const float2 qd = q8x2(make_float2(r23.x, g23.x));
          const float2 qe = q8x2(make_float2(b23.x, r23.y));
          const float2 qf = q8x2(make_float2(g23.y, b23.y));
          op[0] = __byte_perm(__byte_perm(__float_as_uint(qa.x), __float_as_uint(qa.y), 0x0040),
                              __byte_perm(__float_as_uint(qb.x), __float_as_uint(qb.y), 0x0040), 0x5410);
          op[1] = __byte_perm(__byte_perm(__float_as_uint(qc.x), __float_as_uint(qc.y), 0x0040),
                              __byte_perm(__float_as_uint(qd.x), __float_as_uint(qd.y), 0x0040), 0x5410);
          op[2] = __byte_perm(__byte_perm(__float_as_uint(qe.x), __float_as_uint(qe.y), 0x0040),
                              __byte_perm(__float_as_uint(qf.x), __float_as_uint(qf.y), 0x0040), 0x5410);
        }
        if (F32) {
          float4* o = reinterpret_cast<float4*>(of);
          const float n0 = L.nominal[0], n1 = L.nominal[1], n2 = L.nominal[2];
          if (L.rep == 0) {  // "color" (envs/peg_tasks.py:445, .astype(float32))
            o[0] = make_float4(r01.x, g01.x, b01.x, r01.y);
            o[1] = make_float4(g01.y, b01.y, r23.x, g23.x);
            o[2] = make_float4(b23.x, r23.y, g23.y, b23.y);
          } else if (L.rep == 1) {  // "diff": rgb - nominal (peg_tasks.py:453-454)
            o[0] = make_float4(r01.x - n0, g01.x - n1, b01.x - n2, r01.y - n0);
            o[1] = make_float4(g01.y - n1, b01.y - n2, r23.x - n0, g23.x - n1);
            o[2] = make_float4(b23.x - n2, r23.y - n0, g23.y - n1, b23.y - n2);
          } else {  // "concat": [rgb, nominal] on the channel axis (peg_tasks.py:455-458)
            o[0] = make_float4(r01.x, g01.x, b01.x, n0);
            o[1] = make_float4(n1, n2, r01.y, g01.y);
            o[2] = make_float4(b01.y, n0, n1, n2);
            o[3] = make_float4(r23.x, g23.x, b23.x, n0);
            o[4] = make_float4(n1, n2, r23.y, g23.y);
            o[5] = make_float4(b23.y, n0, n1, n2);
          }
          of += (size_t)W * och;
        }
        up = c;
        c = dn;
        p += W;
        op += (W * 3) >> 2;
      }
    }
    __syncwarp();
    if (lane == 0) mbar_arrive(&empty[s]);  // this warp no longer reads stage s
    if (U8) {
      fence_proxy_async_smem();  // generic-proxy smem writes -> visible to the bulk store
      __syncwarp();
      if (lane == 0) mbar_arrive(&ready[b]);
    }
    if (++s == stages) {
      s = 0;
      full_phase ^= 1u;
    }
    img += g_img;
    bidx += g_band;
    if (bidx >= bands) {
      bidx -= bands;
      ++img;
    }
  }
  if (FF) ff_frames_dynamic(F, lane);  // out of bands: help finish the force field
}

// Generic path (any W >= 2, any alignment): one thread per pixel, neighbours
// straight from global memory through L1.
template <int DEG>
__global__ void __launch_bounds__(256) rgb_scalar_kernel(const float* __restrict__ depth, int64_t n_images, int H,
                                                         int W, uint8_t* __restrict__ out_u8,
                                                         float* __restrict__ out_f32, const LutParams L) {
  // grid: y over images, x over an image's pixels (32-bit index math)
  const int HW = H * W;
  for (int64_t img = blockIdx.y; img < n_images; img += gridDim.y)
  for (int rem = blockIdx.x * blockDim.x + threadIdx.x; rem < HW; rem += gridDim.x * blockDim.x) {
    const int64_t p = img * HW + rem;
    const int r = rem / W;
    const int x = rem - r * W;
    const float* f = depth + img * (int64_t)H * W;
    const float c = f[rem];
    float hx, hy;
    if (x == 0) hx = 2.f * (f[rem + 1] - c);
    else if (x == W - 1) hx = 2.f * (c - f[rem - 1]);
    else hx = f[rem + 1] - f[rem - 1];
    if (r == 0) hy = 2.f * (f[rem + W] - c);
    else if (r == H - 1) hy = 2.f * (c - f[rem - W]);
    else hy = f[rem + W] - f[rem - W];
    float v0, v1, v2;
    shade<DEG>(L, hx, hy, v0, v1, v2);
    if (out_u8) {
      out_u8[3 * p + 0] = (uint8_t)(q8(v0) & 0xFF);
      out_u8[3 * p + 1] = (uint8_t)(q8(v1) & 0xFF);
      out_u8[3 * p + 2] = (uint8_t)(q8(v2) & 0xFF);
    }
    if (out_f32) {
      if (L.rep == 2) {
        float* o = out_f32 + 6 * p;
        o[0] = v0;
        o[1] = v1;
        o[2] = v2;
        o[3] = L.nominal[0];
        o[4] = L.nominal[1];
        o[5] = L.nominal[2];
      } else {
        const bool diff = L.rep == 1;
        out_f32[3 * p + 0] = diff ? v0 - L.nominal[0] : v0;
        out_f32[3 * p + 1] = diff ? v1 - L.nominal[1] : v1;
        out_f32[3 * p + 2] = diff ? v2 - L.nominal[2] : v2;
      }
    }
  }
}

int env_int(const char* name, int dflt) {
  const char* s = std::getenv(name);
  if (!s || !*s) return dflt;
  int v = std::atoi(s);
  return v > 0 ? v : dflt;
}

// Rows per thread and ring depth (env-tunable); the number of row groups is
// chosen per kernel instantiation and image size by launch_bulk.
Layout base_layout(int H, int W, bool u8) {
  (void)u8;
  Layout lay;
  lay.rpt = env_int("TACSL_RGB_RPT", kDefaultRpt) == 4 ? 4 : 8;
  // small images make small work units, whose load latency a 2-deep ring
  // cannot cover (measured at 80x60: 4 stages 0.47 ms vs 2 stages 0.60 ms
  // per 65536 frames; already at 128x96 and up 2 stages are best)
  lay.stages = std::max(1, std::min(env_int("TACSL_RGB_STAGES", (int64_t)H * W <= 6144 ? 4 : 2), kMaxStages));
  lay.groups = 1;
  return lay;
}

Layout with_groups(Layout lay, int groups, int W) {
  lay.groups = groups;
  lay.band = groups * lay.rpt;
  lay.in_stage_floats = (size_t)(lay.band + 2) * W;
  lay.out_stage_bytes = (size_t)lay.band * W * 3;
  return lay;
}

// consumer warps + loader + storer (+ force-field warps in the fused step)
int bulk_threads(int W, int groups, bool ff) {
  return (((W / 4) * groups + 31) / 32) * 32 + 64 + (ff ? kFFWarps * 32 : 0);
}

template <int DEG, int RPT, bool U8, bool F32, bool FF = false, bool BIN = false>
int launch_bulk(Layout lay, const float* depth, int64_t n, int H, int W, uint8_t* u8, float* f32,
                const LutParams& L, cudaStream_t stream, const FFArgs<float>* ff = nullptr,
                const BinArgs* bin = nullptr) {
  auto kern = rgb_bulk_kernel<DEG, RPT, U8, F32, FF, BIN>;
  static std::mutex mu;
  static std::vector<std::array<int, 4>> cache;  // (H, W, stages) -> groups
  const int QW = W / 4;
  constexpr int kMaxCons = FF ? kMaxThreadsFF : kMaxThreads;
  if (int rc = set_max_dynamic_smem(reinterpret_cast<const void*>(kern), (int)kSmemPerSm)) return rc;
  std::lock_guard<std::mutex> lock(mu);
  // binned LUT at degrees 3-4: the band's y bins in shared memory behind the
  // ring when they fit (else the kernel reads the table through L1)
  constexpr int T = (DEG + 1) * (DEG + 2) / 2;
  bool use_tab = BIN && DEG > 2 && !std::getenv("TACSL_BINNED_L1");
  auto tab_bytes = [&](int band) -> size_t {
    return use_tab ? (size_t)band_ybins(H, band, bin->bins_y) * bin->bins_x * 3 * T * sizeof(float2) : 0;
  };
  auto need = [&](const Layout& l) { return l.bytes(U8) + tab_bytes(l.band); };
  if (use_tab && need(with_groups(lay, 1, W)) > kSmemPerSm) use_tab = false;
  int groups = 0;
  if (const char* g = std::getenv("TACSL_RGB_GROUPS")) {
    groups = std::max(1, std::min(std::atoi(g), kMaxCons / QW));
    while (groups > 1 && need(with_groups(lay, groups, W)) > kSmemPerSm) --groups;
    while (lay.stages > 1 && need(with_groups(lay, groups, W)) > kSmemPerSm) --lay.stages;
  } else {
    if (!BIN)  // (a binned layout also depends on the bins: searched every call)
      for (const auto& c : cache)
        if (c[0] == H && c[1] == W && c[2] == lay.stages) groups = c[3];
    if (!groups) {
      // Most consumer threads resident per SM (measured to be what the
      // shading throughput tracks -- tools/sweep_rgb.py); ties go to the
      // taller band (less halo re-read).
      long best = -1;
      const int gmax = std::max(1, std::min(kMaxCons / QW, (H + RPT - 1) / RPT));
      for (int g = 1; g <= gmax; ++g) {
        const Layout cand = with_groups(lay, g, W);
        const size_t smem = need(cand);
        if (smem > kSmemPerSm) break;
        int per_sm = 0;
        cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, kern, bulk_threads(W, g, FF), smem);
        const long score = (long)per_sm * g * QW;
        if (per_sm > 0 && score > best) {
          best = score;
          groups = g;
        }
      }
      if (!groups) return set_error(TACSL_ERR_INVALID_ARGUMENT, "rgb: band ring does not fit in shared memory");
      if (!BIN) cache.push_back({H, W, lay.stages, groups});
    }
  }
  const int bulk_store = (W % 16 == 0) && ((reinterpret_cast<uintptr_t>(u8) & 15) == 0);
  FFArgs<float> F{};
  if (FF) F = *ff;
  BinArgs B{};
  if (BIN) B = *bin;
  // launch with (groups, CTAs per SM); 0 ctas = as many as fit
  auto go = [&](int g, int ctas) -> int {
    const Layout l = with_groups(lay, g, W);
    const int threads = bulk_threads(W, g, FF);
    const size_t smem = need(l);
    if (BIN) B.tab_ybins = use_tab ? band_ybins(H, l.band, B.bins_y) : 0;
    int per_sm = 0;
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, kern, threads, smem);
    if (per_sm <= 0) return -1;
    if (ctas > 0) per_sm = std::min(per_sm, ctas);
    const int bands = (H + l.band - 1) / l.band;
    int64_t grid = std::min<int64_t>(n * bands, (int64_t)sm_count(current_device()) * per_sm);
    if (BIN && grid > bands) grid -= grid % bands;  // each CTA stays on one band: its y bins stay loaded
    kern<<<(unsigned)grid, threads, smem, stream>>>(depth, n, H, W, l.groups, l.stages, u8, f32, L, bulk_store,
                                                    F, B);
    return 0;
  };
  int ctas = env_int("TACSL_RGB_CTAS_PER_SM", 0);
  if constexpr (F32 && !U8 && !FF && !BIN) {
    // The float-output path's best launch shape varies with the image size
    // in ways the occupancy model does not capture (measured: 0.82 vs 1.08
    // ms at 8192 x 240x320 between neighbouring shapes), so the first
    // un-captured call per (H, W, batch-size octave) times the candidates
    // on its own data and keeps the fastest.
    // (device, H, W, log2 n) -> (groups, ctas), cached only once timed
    static std::mutex mu;
    static std::vector<std::array<int, 6>> tuned;
    const int dev = current_device();
    const int nb = 63 - __builtin_clzll((unsigned long long)std::max<int64_t>(n, 1));
    bool have = false;
    {
      std::lock_guard<std::mutex> lock(mu);
      for (const auto& t : tuned)
        if (t[0] == dev && t[1] == H && t[2] == W && t[3] == nb) {
          groups = t[4];
          ctas = t[5];
          have = true;
        }
    }
    cudaStreamCaptureStatus cap = cudaStreamCaptureStatusNone;
    if (!have && cudaStreamIsCapturing(stream, &cap) != cudaSuccess) {
      cudaGetLastError();  // cannot tell: do not time (and do not cache) now
      cap = cudaStreamCaptureStatusActive;
    }
    if (!have && !std::getenv("TACSL_RGB_GROUPS") && !std::getenv("TACSL_RGB_CTAS_PER_SM") &&
        cap == cudaStreamCaptureStatusNone) {
      cudaEvent_t e0, e1;
      cudaEventCreate(&e0);
      cudaEventCreate(&e1);
      float best_ms = 1e30f;
      int best_g = groups, best_c = 0;
      const int gmax = std::max(1, std::min(kMaxCons / QW, (H + RPT - 1) / RPT));
      for (int g = 1; g <= gmax && g <= 4; ++g) {
        if (with_groups(lay, g, W).bytes(U8) > kSmemPerSm) break;
        for (int c = 1; c <= 4; ++c) {
          if (go(g, c) < 0) break;  // warm-up launch
          cudaEventRecord(e0, stream);
          go(g, c);
          go(g, c);
          cudaEventRecord(e1, stream);
          cudaEventSynchronize(e1);
          float ms = 0.f;
          cudaEventElapsedTime(&ms, e0, e1);
          if (ms < best_ms) {
            best_ms = ms;
            best_g = g;
            best_c = c;
          }
        }
      }
      cudaEventDestroy(e0);
      cudaEventDestroy(e1);
      groups = best_g;
      ctas = best_c;
      std::lock_guard<std::mutex> lock(mu);
      tuned.push_back({dev, H, W, nb, groups, ctas});
    }
  }
  if (go(groups, ctas) < 0) return set_error(TACSL_ERR_INVALID_ARGUMENT, "rgb: band ring does not fit in shared memory");
  return check_launch("rgb_bulk_kernel");
}

template <int DEG>
int dispatch(const float* depth, int64_t n, int H, int W, uint8_t* u8, float* f32, const LutParams& L,
             cudaStream_t stream) {
  const bool aligned = (W % 4 == 0) && (W / 4 <= kMaxThreads) &&
                       ((reinterpret_cast<uintptr_t>(depth) & 15) == 0) &&
                       ((reinterpret_cast<uintptr_t>(f32) & 15) == 0) && ((reinterpret_cast<uintptr_t>(u8) & 3) == 0);
  if (aligned && !std::getenv("TACSL_RGB_FORCE_SCALAR")) {
    const Layout lay = base_layout(H, W, u8 != nullptr);
    if (lay.rpt == 4) {
      if (u8 && f32) return launch_bulk<DEG, 4, true, true>(lay, depth, n, H, W, u8, f32, L, stream);
      if (u8) return launch_bulk<DEG, 4, true, false>(lay, depth, n, H, W, u8, f32, L, stream);
      return launch_bulk<DEG, 4, false, true>(lay, depth, n, H, W, u8, f32, L, stream);
    }
    if (u8 && f32) return launch_bulk<DEG, 8, true, true>(lay, depth, n, H, W, u8, f32, L, stream);
    if (u8) return launch_bulk<DEG, 8, true, false>(lay, depth, n, H, W, u8, f32, L, stream);
    return launch_bulk<DEG, 8, false, true>(lay, depth, n, H, W, u8, f32, L, stream);
  }
  const int64_t total = n * (int64_t)H * W;
  int64_t blocks = std::min<int64_t>((total + 255) / 256, (int64_t)sm_count(current_device()) * 16);
  const unsigned gy = (unsigned)std::min<int64_t>(n, 65535);
  const unsigned gx = (unsigned)std::max<int64_t>(
      1, std::min<int64_t>(((int64_t)H * W + 255) / 256, (blocks + gy - 1) / gy));
  rgb_scalar_kernel<DEG><<<dim3(gx, gy), 256, 0, stream>>>(depth, n, H, W, u8, f32, L);
  return check_launch("rgb_scalar_kernel");
}

}  // namespace

// The binned LUT (K6) on this pipeline; called by binned.cu when the bin
// edges fall between pixel pairs (even columns) and the layout is aligned.
int launch_rgb_binned(const float2* pairs, int bins_y, int bins_x, int degree, const float* depth, int64_t n,
                      int H, int W, uint8_t* u8, float* f32, cudaStream_t s) {
  LutParams L{};  // rep 0 ("color") float epilogue; coefficients come from the table
  const BinArgs B{pairs, bins_y, bins_x, 0};
  const Layout lay = base_layout(H, W, u8 != nullptr);
  auto go = [&](auto deg) -> int {
    constexpr int D = decltype(deg)::value;
    if (u8 && f32) return launch_bulk<D, 8, true, true, false, true>(lay, depth, n, H, W, u8, f32, L, s, nullptr, &B);
    if (u8) return launch_bulk<D, 8, true, false, false, true>(lay, depth, n, H, W, u8, f32, L, s, nullptr, &B);
    return launch_bulk<D, 8, false, true, false, true>(lay, depth, n, H, W, u8, f32, L, s, nullptr, &B);
  };
  switch (degree) {
    case 2: return go(std::integral_constant<int, 2>{});
    case 3: return go(std::integral_constant<int, 3>{});
    case 4: return go(std::integral_constant<int, 4>{});
  }
  return set_error(TACSL_ERR_INVALID_ARGUMENT, "LUT degree must be in [2, 4]");
}

}  // namespace tacsl

using namespace tacsl;

extern "C" int tacsl_depth_to_rgb(tacsl_lut_t lut, const float* depth, int64_t n_images, int height, int width,
                                  uint8_t* rgb_u8, float* rgb_f32, void* stream) {
  StreamDevice stream_device_(stream);
  if (!lut) return set_error(TACSL_ERR_INVALID_ARGUMENT, "depth_to_rgb: null LUT");
  if (width != lut->width || height != lut->height)
    return set_error(TACSL_ERR_LUT_RESOLUTION_MISMATCH,
                     "LUT calibrated at (" + std::to_string(lut->width) + ", " + std::to_string(lut->height) +
                         "), image is (" + std::to_string(width) + ", " + std::to_string(height) + ")");
  if (height < 2 || width < 2)
    return set_error(TACSL_ERR_INVALID_ARGUMENT, "depth_to_rgb: gradients need H >= 2 and W >= 2");
  if (n_images < 0) return set_error(TACSL_ERR_INVALID_ARGUMENT, "depth_to_rgb: negative image count");
  if (n_images == 0) return TACSL_OK;
  if (!rgb_u8 && !rgb_f32) return set_error(TACSL_ERR_INVALID_ARGUMENT, "depth_to_rgb: no output buffer");
  if (!depth) return set_error(TACSL_ERR_INVALID_ARGUMENT, "depth_to_rgb: null depth");
  cudaStream_t s = static_cast<cudaStream_t>(stream);
  switch (lut->degree) {
    case 2: return dispatch<2>(depth, n_images, height, width, rgb_u8, rgb_f32, lut->params, s);
    case 3: return dispatch<3>(depth, n_images, height, width, rgb_u8, rgb_f32, lut->params, s);
    case 4: return dispatch<4>(depth, n_images, height, width, rgb_u8, rgb_f32, lut->params, s);
  }
  return set_error(TACSL_ERR_INVALID_ARGUMENT, "LUT degree must be in [2, 4]");
}

extern "C" int tacsl_tactile_image_obs(tacsl_lut_t lut, const float* depth, int64_t n_images, int height, int width,
                                       int rep, const float nominal[3], float* out, void* stream) {
  StreamDevice stream_device_(stream);
  if (!lut) return set_error(TACSL_ERR_INVALID_ARGUMENT, "tactile_image_obs: null LUT");
  if (rep < 0 || rep > 2) return set_error(TACSL_ERR_INVALID_ARGUMENT, "tactile_image_obs: rep must be 0, 1 or 2");
  if (width != lut->width || height != lut->height)
    return set_error(TACSL_ERR_LUT_RESOLUTION_MISMATCH,
                     "LUT calibrated at (" + std::to_string(lut->width) + ", " + std::to_string(lut->height) +
                         "), image is (" + std::to_string(width) + ", " + std::to_string(height) + ")");
  if (height < 2 || width < 2)
    return set_error(TACSL_ERR_INVALID_ARGUMENT, "tactile_image_obs: gradients need H >= 2 and W >= 2");
  if (n_images < 0) return set_error(TACSL_ERR_INVALID_ARGUMENT, "tactile_image_obs: negative image count");
  if (n_images == 0) return TACSL_OK;
  if (!depth || !out || (rep != 0 && !nominal))
    return set_error(TACSL_ERR_INVALID_ARGUMENT, "tactile_image_obs: null pointer");
  LutParams P = lut->params;
  P.rep = rep;
  for (int c = 0; c < 3; ++c) P.nominal[c] = rep ? nominal[c] : 0.f;
  cudaStream_t s = static_cast<cudaStream_t>(stream);
  switch (lut->degree) {
    case 2: return dispatch<2>(depth, n_images, height, width, nullptr, out, P, s);
    case 3: return dispatch<3>(depth, n_images, height, width, nullptr, out, P, s);
    case 4: return dispatch<4>(depth, n_images, height, width, nullptr, out, P, s);
  }
  return set_error(TACSL_ERR_INVALID_ARGUMENT, "LUT degree must be in [2, 4]");
}

namespace tacsl {
namespace {

template <int DEG>
int fused_step(const LutParams& L, const float* depth, int64_t n, int H, int W, uint8_t* u8,
               const FFArgs<float>& F, cudaStream_t stream) {
  const Layout lay = base_layout(H, W, true);
  if (lay.rpt == 4) return launch_bulk<DEG, 4, true, false, true>(lay, depth, n, H, W, u8, nullptr, L, stream, &F);
  return launch_bulk<DEG, 8, true, false, true>(lay, depth, n, H, W, u8, nullptr, L, stream, &F);
}

}  // namespace
}  // namespace tacsl

extern "C" int tacsl_sensor_step(tacsl_lut_t lut, const float* depth, int64_t n_images, int height, int width,
                                 uint8_t* rgb_u8, tacsl_sdf_t sdf, const double* taxels, int rows, int cols,
                                 const double* object_state, int64_t object_stride, const double* sensor_state,
                                 int64_t sensor_stride, int64_t n_envs, int n_sensors, tacsl_penalty_t params,
                                 float* f_n, float* f_t, double* wrench, unsigned long long* workspace,
                                 void* stream) {
  StreamDevice stream_device_(stream);
  if (!lut || !sdf) return set_error(TACSL_ERR_INVALID_ARGUMENT, "sensor_step: null handle");
  if (width != lut->width || height != lut->height)
    return set_error(TACSL_ERR_LUT_RESOLUTION_MISMATCH,
                     "LUT calibrated at (" + std::to_string(lut->width) + ", " + std::to_string(lut->height) +
                         "), image is (" + std::to_string(width) + ", " + std::to_string(height) + ")");
  if (height < 2 || width < 2) return set_error(TACSL_ERR_INVALID_ARGUMENT, "sensor_step: H, W must be >= 2");
  if (params.k_n < 0 || params.k_d < 0 || params.k_t < 0 || params.mu < 0)
    return set_error(TACSL_ERR_INVALID_ARGUMENT, "penalty parameters must be non-negative");
  if (rows <= 0 || cols <= 0 || n_sensors <= 0 || n_envs < 0 || n_images < 0 || object_stride < 0 ||
      sensor_stride < 0)
    return set_error(TACSL_ERR_INVALID_ARGUMENT, "sensor_step: bad sizes");
  if (!depth || !rgb_u8 || !taxels || !object_state || !sensor_state || !f_n || !f_t)
    return set_error(TACSL_ERR_INVALID_ARGUMENT, "sensor_step: null pointer");
  const int64_t frames = n_envs * n_sensors;
  cudaStream_t s = static_cast<cudaStream_t>(stream);
  const bool aligned = (width % 4 == 0) && (width / 4 <= kMaxThreads) &&
                       ((reinterpret_cast<uintptr_t>(depth) & 15) == 0) &&
                       ((reinterpret_cast<uintptr_t>(rgb_u8) & 3) == 0);
  if (!aligned || n_images == 0 || frames == 0 || std::getenv("TACSL_STEP_UNFUSED")) {
    // two launches: the image path does not fit the fused pipeline
    int rc = tacsl_depth_to_rgb(lut, depth, n_images, height, width, rgb_u8, nullptr, stream);
    if (rc) return rc;
    return tacsl_force_field(sdf, taxels, rows, cols, object_state, object_stride, sensor_state, sensor_stride,
                             n_envs, n_sensors, params, 0, f_n, f_t, wrench, nullptr, nullptr, nullptr, stream);
  }
  const FFArgs<float> F{make_grid(sdf), taxels, rows * cols, object_state, object_stride, sensor_state,
                        sensor_stride, n_sensors, frames, Penalty{params.k_n, params.k_d, params.k_t, params.mu},
                        f_n, f_t, wrench, nullptr, nullptr, nullptr, workspace};
  if (!workspace) return set_error(TACSL_ERR_INVALID_ARGUMENT, "sensor_step: null workspace");
  if (cudaMemsetAsync(workspace, 0, sizeof(unsigned long long), s) != cudaSuccess)
    return check_launch("sensor_step: workspace reset");
  switch (lut->degree) {
    case 2: return fused_step<2>(lut->params, depth, n_images, height, width, rgb_u8, F, s);
    case 3: return fused_step<3>(lut->params, depth, n_images, height, width, rgb_u8, F, s);
    case 4: return fused_step<4>(lut->params, depth, n_images, height, width, rgb_u8, F, s);
  }
  return set_error(TACSL_ERR_INVALID_ARGUMENT, "LUT degree must be in [2, 4]");
}
