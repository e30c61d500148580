// K1: depth -> tactile RGB, one fused pass.
//
// Replaces render/lut.py:68-76 depth_to_rgb = depth_gradients (lut.py:25-28,
// np.gradient: central inside, one-sided un-halved at the borders) ->
// PolyLut.evaluate (lut.py:56-65: per-channel polynomial in (g_x, g_y),
// clip [0,1]) -> optional to_uint8 (render/imageio.py:8-11).
//
// Layout: depth (N, H, W) fp32, rgb (N, H, W, 3) HWC, u8 and/or fp32.
//
// Fast path (W % 4 == 0, 16B-aligned pointers): persistent CTAs walk work
// units = (image, band of B rows).  Thread 0 streams each band plus its two
// halo rows global->shared with one bulk-async copy (cp.async.bulk, the 1-D
// TMA engine) into a STAGES-deep ring completed on mbarriers, so up to
// STAGES bands per CTA are in flight while the CTA shades the current one.
// Every thread shades 4 adjacent pixels (one 16B shared-memory vector +
// neighbours), writes 12 output bytes into a shared staging tile, and the
// band's contiguous B*W*3 bytes go back with one bulk shared->global store.
// HBM sees each depth byte read once and each RGB byte written once.
#include <algorithm>
#include <cstdlib>
#include <mutex>

#include "common.cuh"
#include "handles.h"

namespace tacsl {
namespace {

constexpr int kThreads = 256;

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

__device__ __forceinline__ uint32_t q8(float x) {
  // clip(rint(255 x), 0, 255): x is saturated to [0,1] first, then the
  // 1.5*2^23 bias rounds the exact product half-to-even into the low byte.
  return __float_as_uint(__fmaf_rn(__saturatef(x), 255.0f, 12582912.0f));
}

template <int DEG>
__device__ __forceinline__ void shade(const LutParams& L, float hx, float hy, float& r, float& g, float& b) {
  r = __saturatef(poly<DEG>(L.c[0], hx, hy));
  g = __saturatef(poly<DEG>(L.c[1], hx, hy));
  b = __saturatef(poly<DEG>(L.c[2], hx, hy));
}

struct Smem {
  int band, stages, W;
  size_t in_stage_floats, out_stage_bytes;
  static constexpr size_t kBarBytes = 128;
  __host__ __device__ size_t bytes(bool u8) const {
    return kBarBytes + stages * in_stage_floats * sizeof(float) + (u8 ? 2 * out_stage_bytes : 0);
  }
};

template <int DEG, bool U8, bool F32>
__global__ void __launch_bounds__(kThreads) rgb_bulk_kernel(const float* __restrict__ depth, int64_t n_images,
                                                            int H, int W, int band, int stages,
                                                            uint8_t* __restrict__ out_u8,
                                                            float* __restrict__ out_f32, const LutParams L,
                                                            int bulk_store) {
  extern __shared__ __align__(128) unsigned char smem[];
  const int bands = (H + band - 1) / band;
  const int64_t units = n_images * bands;
  const size_t in_stage = (size_t)(band + 2) * W;
  const size_t out_stage = (size_t)band * W * 3;
  uint64_t* bars = reinterpret_cast<uint64_t*>(smem);
  float* in_buf = reinterpret_cast<float*>(smem + Smem::kBarBytes);
  uint8_t* out_buf = reinterpret_cast<uint8_t*>(in_buf + stages * in_stage);

  if (threadIdx.x == 0) {
    for (int s = 0; s < stages; ++s) mbar_init(&bars[s], 1);
    fence_mbar_init();
    fence_proxy_async_smem();
  }
  __syncthreads();

  // Stage s row 0 holds image row r0-1 (absent for the top band); rows that
  // do not exist are never read.
  auto issue = [&](int64_t u, int s) {
    const int64_t img = u / bands;
    const int r0 = (int)(u - img * bands) * band;
    const int rs = max(r0 - 1, 0);
    const int re = min(r0 + band, H - 1);
    const uint32_t bytes = (uint32_t)(re - rs + 1) * (uint32_t)W * 4u;
    float* dst = in_buf + (size_t)s * in_stage + (size_t)(rs - (r0 - 1)) * W;
    const float* src = depth + ((size_t)img * H + rs) * (size_t)W;
    mbar_arrive_expect_tx(&bars[s], bytes);
    bulk_g2s(dst, src, bytes, &bars[s]);
  };

  if (threadIdx.x == 0) {
    for (int s = 0; s < stages; ++s) {
      const int64_t u = (int64_t)blockIdx.x + (int64_t)s * gridDim.x;
      if (u < units) issue(u, s);
    }
  }

  const int QW = W >> 2;
  int it = 0;
  for (int64_t u = blockIdx.x; u < units; u += gridDim.x, ++it) {
    const int s = it % stages;
    const uint32_t parity = (uint32_t)(it / stages) & 1u;
    const int64_t img = u / bands;
    const int r0 = (int)(u - img * bands) * band;
    const int nrows = min(band, H - r0);
    uint8_t* ob = out_buf + (size_t)(it & 1) * out_stage;
    if (U8 && bulk_store && threadIdx.x == 0) bulk_wait_read<1>();  // store of it-2 has left `ob`
    __syncthreads();
    mbar_wait_parity(&bars[s], parity);

    const float* tile = in_buf + (size_t)s * in_stage + W;  // tile row lr = image row r0 + lr
    const int items = nrows * QW;
    for (int q = threadIdx.x; q < items; q += kThreads) {
      const int lr = q / QW;
      const int x0 = (q - lr * QW) << 2;
      const int r = r0 + lr;
      const float* rowc = tile + (size_t)lr * W;
      const float4 c = *reinterpret_cast<const float4*>(rowc + x0);
      float4 hy;
      if (r > 0 && r < H - 1) {
        const float4 up = *reinterpret_cast<const float4*>(rowc - W + x0);
        const float4 dn = *reinterpret_cast<const float4*>(rowc + W + x0);
        hy = make_float4(dn.x - up.x, dn.y - up.y, dn.z - up.z, dn.w - up.w);
      } else if (r == 0) {
        const float4 dn = *reinterpret_cast<const float4*>(rowc + W + x0);
        hy = make_float4(2.f * (dn.x - c.x), 2.f * (dn.y - c.y), 2.f * (dn.z - c.z), 2.f * (dn.w - c.w));
      } else {
        const float4 up = *reinterpret_cast<const float4*>(rowc - W + x0);
        hy = make_float4(2.f * (c.x - up.x), 2.f * (c.y - up.y), 2.f * (c.z - up.z), 2.f * (c.w - up.w));
      }
      float4 hx;
      hx.x = (x0 > 0) ? c.y - rowc[x0 - 1] : 2.f * (c.y - c.x);
      hx.y = c.z - c.x;
      hx.z = c.w - c.y;
      hx.w = (x0 + 4 < W) ? rowc[x0 + 4] - c.z : 2.f * (c.w - c.z);

      float v[12];
      shade<DEG>(L, hx.x, hy.x, v[0], v[1], v[2]);
      shade<DEG>(L, hx.y, hy.y, v[3], v[4], v[5]);
      shade<DEG>(L, hx.z, hy.z, v[6], v[7], v[8]);
      shade<DEG>(L, hx.w, hy.w, v[9], v[10], v[11]);
      if (U8) {
        uint32_t b[12];
#pragma unroll
        for (int k = 0; k < 12; ++k) b[k] = q8(v[k]);
        uint32_t w0 = __byte_perm(__byte_perm(b[0], b[1], 0x0040), __byte_perm(b[2], b[3], 0x0040), 0x5410);
        uint32_t w1 = __byte_perm(__byte_perm(b[4], b[5], 0x0040), __byte_perm(b[6], b[7], 0x0040), 0x5410);
        uint32_t w2 = __byte_perm(__byte_perm(b[8], b[9], 0x0040), __byte_perm(b[10], b[11], 0x0040), 0x5410);
        uint32_t* o = reinterpret_cast<uint32_t*>(ob + ((size_t)lr * W + x0) * 3);
        o[0] = w0;
        o[1] = w1;
        o[2] = w2;
      }
      if (F32) {
        float4* o = reinterpret_cast<float4*>(out_f32 + (((size_t)img * H + r) * W + x0) * 3);
        o[0] = make_float4(v[0], v[1], v[2], v[3]);
        o[1] = make_float4(v[4], v[5], v[6], v[7]);
        o[2] = make_float4(v[8], v[9], v[10], v[11]);
      }
    }
    if (U8) fence_proxy_async_smem();  // generic-proxy smem writes -> visible to the bulk store
    __syncthreads();
    if (U8) {
      uint8_t* dst = out_u8 + ((size_t)img * H + r0) * (size_t)W * 3;
      const uint32_t bytes = (uint32_t)nrows * (uint32_t)W * 3u;
      if (bulk_store) {
        if (threadIdx.x == 0) {
          bulk_s2g(dst, ob, bytes);
          bulk_commit();
        }
      } else {
        const uint32_t* src = reinterpret_cast<const uint32_t*>(ob);
        uint32_t* d32 = reinterpret_cast<uint32_t*>(dst);
        for (uint32_t k = threadIdx.x; k < bytes / 4; k += kThreads) d32[k] = src[k];
      }
    }
    if (threadIdx.x == 0) {
      const int64_t un = u + (int64_t)stages * gridDim.x;
      if (un < units) issue(un, s);
    }
  }
  if (U8 && bulk_store && threadIdx.x == 0) bulk_wait_all<0>();
}

// Generic path (any W >= 2, any alignment): one thread per pixel, neighbours
// straight from global memory through L1.
template <int DEG>
__global__ void __launch_bounds__(kThreads) rgb_scalar_kernel(const float* __restrict__ depth, int64_t n_images,
                                                              int H, int W, uint8_t* __restrict__ out_u8,
                                                              float* __restrict__ out_f32, const LutParams L) {
  const int64_t total = n_images * (int64_t)H * W;
  const int64_t stride = (int64_t)gridDim.x * blockDim.x;
  for (int64_t p = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; p < total; p += stride) {
    const int64_t img = p / ((int64_t)H * W);
    const int rem = (int)(p - img * H * W);
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
      out_f32[3 * p + 0] = v0;
      out_f32[3 * p + 1] = v1;
      out_f32[3 * p + 2] = v2;
    }
  }
}

int env_int(const char* name, int dflt) {
  const char* s = std::getenv(name);
  if (!s || !*s) return dflt;
  int v = std::atoi(s);
  return v > 0 ? v : dflt;
}

template <int DEG, bool U8, bool F32>
int launch_bulk(const float* depth, int64_t n, int H, int W, uint8_t* u8, float* f32, const LutParams& L,
                cudaStream_t stream) {
  // band: 16 rows (8 at W > 512) keeps a 3-stage input ring + 2 output tiles
  // near 100 KB, i.e. two resident CTAs per SM with ~6 bands in flight.
  int band = env_int("TACSL_RGB_BAND", W > 512 ? 8 : 16);
  int stages = env_int("TACSL_RGB_STAGES", 3);
  band = std::min(band, H);
  Smem lay{band, stages, W, (size_t)(band + 2) * W, (size_t)band * W * 3};
  size_t smem = lay.bytes(U8);
  auto kern = rgb_bulk_kernel<DEG, U8, F32>;
  static std::mutex mu;
  static size_t configured = 0;
  {
    std::lock_guard<std::mutex> lock(mu);
    if (smem > configured) {
      if (cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem) != cudaSuccess)
        return check_launch("rgb: cudaFuncSetAttribute");
      configured = smem;
    }
  }
  int per_sm = 0;
  cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, kern, kThreads, smem);
  if (per_sm <= 0) return set_error(TACSL_ERR_INVALID_ARGUMENT, "rgb: image too wide for the shared-memory ring");
  per_sm = std::min(per_sm, env_int("TACSL_RGB_CTAS_PER_SM", per_sm));
  const int bands = (H + band - 1) / band;
  const int64_t units = n * bands;
  int64_t grid = std::min<int64_t>(units, (int64_t)sm_count(current_device()) * per_sm);
  const int bulk_store = (W % 16 == 0) && ((reinterpret_cast<uintptr_t>(u8) & 15) == 0);
  kern<<<(unsigned)grid, kThreads, smem, stream>>>(depth, n, H, W, band, stages, u8, f32, L, bulk_store);
  return check_launch("rgb_bulk_kernel");
}

template <int DEG>
int dispatch(const float* depth, int64_t n, int H, int W, uint8_t* u8, float* f32, const LutParams& L,
             cudaStream_t stream) {
  const bool aligned = (W % 4 == 0) && ((reinterpret_cast<uintptr_t>(depth) & 15) == 0) &&
                       ((reinterpret_cast<uintptr_t>(f32) & 15) == 0) && ((reinterpret_cast<uintptr_t>(u8) & 3) == 0);
  if (aligned && !std::getenv("TACSL_RGB_FORCE_SCALAR")) {
    if (u8 && f32) return launch_bulk<DEG, true, true>(depth, n, H, W, u8, f32, L, stream);
    if (u8) return launch_bulk<DEG, true, false>(depth, n, H, W, u8, f32, L, stream);
    return launch_bulk<DEG, false, true>(depth, n, H, W, u8, f32, L, stream);
  }
  const int64_t total = n * (int64_t)H * W;
  int64_t blocks = std::min<int64_t>((total + kThreads - 1) / kThreads, (int64_t)sm_count(current_device()) * 16);
  rgb_scalar_kernel<DEG><<<(unsigned)blocks, kThreads, 0, stream>>>(depth, n, H, W, u8, f32, L);
  return check_launch("rgb_scalar_kernel");
}

}  // namespace
}  // namespace tacsl

using namespace tacsl;

extern "C" int tacsl_depth_to_rgb(tacsl_lut_t lut, const float* depth, int64_t n_images, int height, int width,
                                  uint8_t* rgb_u8, float* rgb_f32, void* stream) {
  if (!lut) return set_error(TACSL_ERR_INVALID_ARGUMENT, "depth_to_rgb: null LUT");
  if (width != lut->width || height != lut->height)
    return set_error(TACSL_ERR_LUT_RESOLUTION_MISMATCH,
                     "LUT calibrated at (" + std::to_string(lut->width) + ", " + std::to_string(lut->height) +
                         "), image is (" + std::to_string(width) + ", " + std::to_string(height) + ")");
  if (height < 2 || width < 2)
    return set_error(TACSL_ERR_INVALID_ARGUMENT, "depth_to_rgb: gradients need H >= 2 and W >= 2");
  if (n_images < 0) return set_error(TACSL_ERR_INVALID_ARGUMENT, "depth_to_rgb: negative image count");
  if (!rgb_u8 && !rgb_f32) return set_error(TACSL_ERR_INVALID_ARGUMENT, "depth_to_rgb: no output buffer");
  if (n_images == 0) return TACSL_OK;
  if (!depth) return set_error(TACSL_ERR_INVALID_ARGUMENT, "depth_to_rgb: null depth");
  cudaStream_t s = static_cast<cudaStream_t>(stream);
  switch (lut->degree) {
    case 2: return dispatch<2>(depth, n_images, height, width, rgb_u8, rgb_f32, lut->params, s);
    case 3: return dispatch<3>(depth, n_images, height, width, rgb_u8, rgb_f32, lut->params, s);
    case 4: return dispatch<4>(depth, n_images, height, width, rgb_u8, rgb_f32, lut->params, s);
  }
  return set_error(TACSL_ERR_INVALID_ARGUMENT, "LUT degree must be in [2, 4]");
}
