// K6: depth -> tactile RGB through a per-pixel BINNED polynomial LUT -- the
// north_star's "per-pixel binned polynomial calibration lookup".  It has NO
// counterpart in the reference (gelsim's PolyLut is one
// global polynomial, render/lut.py:31-59), so the semantics are defined here
// and restated on the CPU by oracle/binned_oracle.py:
//
//   bin(y, x) = (y * bins_y / H, x * bins_x / W)          (integer floor)
//   rgb[y, x, c] = clip(sum_k C[bin(y, x)][c][k] g_x^i g_y^j, 0, 1)
//
// with the gradients of depth_to_rgb (np.gradient, lut.py:25-28).  A table
// with one bin is exactly PolyLut, and this kernel then reproduces K1 bit for
// bit: same doubled-gradient form, same 2^-(i+j) coefficient scaling, same
// Horner order and FMA rounding (K1's packed FFMA2 lanes are IEEE FMAs).
//
// Mapping: a CTA per group of image rows, a thread per 4-pixel column quad;
// the coefficient sets (bins_y * bins_x * 3 * T floats) and the column -> bin
// table live in shared memory, the row's bin is uniform across the row.  The
// depth neighbours come through L1 (each row is read by three row steps).
// rgb_binned_vec_kernel is the fast path, rgb_binned_kernel (per pixel) the
// generic one for widths that are not a multiple of 4.
#include <algorithm>
#include <cstdlib>
#include <cstring>
#include <vector>

#include "common.cuh"
#include "handles.h"

struct tacsl_binned_lut_s {
  int device;
  int degree;
  int width, height;
  int bins_y, bins_x;
  float* coeffs;   // device (bins_y * bins_x, 3, T), scaled by 2^-(i+j)
  float2* pairs;   // the same as duplicated pairs (c, c) for the band pipeline
};

namespace tacsl {
namespace {

constexpr int kBinnedThreads = 256;
constexpr size_t kBinnedMaxSmem = 96 * 1024;

__host__ __device__ constexpr int bterm(int i, int j) { return (i + j) * (i + j + 1) / 2 + j; }

template <int DEG>
__device__ __forceinline__ float bpoly(const float* __restrict__ c, float hx, float hy) {
  float acc = 0.f;
#pragma unroll
  for (int i = DEG; i >= 0; --i) {
    float p = c[bterm(i, DEG - i)];
#pragma unroll
    for (int j = DEG - i - 1; j >= 0; --j) p = __fmaf_rn(p, hy, c[bterm(i, j)]);
    acc = (i == DEG) ? p : __fmaf_rn(acc, hx, p);
  }
  return __saturatef(acc);
}

template <int DEG>
__global__ void __launch_bounds__(kBinnedThreads) rgb_binned_kernel(const float* __restrict__ depth, int64_t n,
                                                                    int H, int W, int bins_y, int bins_x,
                                                                    const float* __restrict__ coeffs,
                                                                    uint8_t* __restrict__ out_u8,
                                                                    float* __restrict__ out_f32) {
  constexpr int T = (DEG + 1) * (DEG + 2) / 2;
  extern __shared__ __align__(16) float sm[];
  const int n_sets = bins_y * bins_x;
  float* cs = sm;                                                  // n_sets * 3 * T
  int* xbin = reinterpret_cast<int*>(sm + (size_t)n_sets * 3 * T);  // W
  for (int k = threadIdx.x; k < n_sets * 3 * T; k += blockDim.x) cs[k] = coeffs[k];
  for (int x = threadIdx.x; x < W; x += blockDim.x) xbin[x] = (int)(((int64_t)x * bins_x) / W);
  __syncthreads();

  const int QW = (W + 3) >> 2;
  // narrow rows: several rows per pass, one quad per thread; rows wider
  // than 4 * blockDim pixels: one row per pass, each thread strides its quads
  const bool narrow = QW <= (int)blockDim.x;
  const int rows_per_pass = narrow ? (int)blockDim.x / QW : 1;
  const int rsub = narrow ? (int)threadIdx.x / QW : 0;
  const int xq0 = narrow ? (int)threadIdx.x - rsub * QW : (int)threadIdx.x;
  const int xq_step = narrow ? QW : (int)blockDim.x;
  if (rsub >= rows_per_pass) return;
  const int64_t total_rows = n * H;
  for (int64_t rr = (int64_t)blockIdx.x * rows_per_pass + rsub; rr < total_rows;
       rr += (int64_t)gridDim.x * rows_per_pass)
  for (int xq = xq0; xq < QW; xq += xq_step) {
    const int64_t img = rr / H;
    const int r = (int)(rr - img * H);
    const float* f = depth + img * (int64_t)H * W;
    const float* row = f + (int64_t)r * W;
    const float* up = r > 0 ? row - W : row;
    const float* dn = r < H - 1 ? row + W : row;
    const bool edge_row = (r == 0) || (r == H - 1);
    const int by = r * bins_y / H;  // 32-bit: r * bins_y < 2^31
    const float* cbase = cs + (size_t)by * bins_x * 3 * T;
#pragma unroll
    for (int k = 0; k < 4; ++k) {
      const int x = 4 * xq + k;
      if (x >= W) break;
      const float c = row[x];
      // doubled gradients (h = 2 g; the coefficients carry 2^-(i+j)), as K1
      float hx = (x == 0) ? (row[1] - c) * 2.f : (x == W - 1) ? (c - row[x - 1]) * 2.f : row[x + 1] - row[x - 1];
      float hy = dn[x] - up[x];
      if (edge_row) hy = hy + hy;
      const float* cc = cbase + (size_t)xbin[x] * 3 * T;
      const float v0 = bpoly<DEG>(cc, hx, hy);
      const float v1 = bpoly<DEG>(cc + T, hx, hy);
      const float v2 = bpoly<DEG>(cc + 2 * T, hx, hy);
      const int64_t p = rr * W + x;
      if (out_u8) {
        out_u8[3 * p + 0] = (uint8_t)(__float_as_uint(__fmaf_rn(v0, 255.0f, 12582912.0f)) & 0xFF);
        out_u8[3 * p + 1] = (uint8_t)(__float_as_uint(__fmaf_rn(v1, 255.0f, 12582912.0f)) & 0xFF);
        out_u8[3 * p + 2] = (uint8_t)(__float_as_uint(__fmaf_rn(v2, 255.0f, 12582912.0f)) & 0xFF);
      }
      if (out_f32) {
        out_f32[3 * p + 0] = v0;
        out_f32[3 * p + 1] = v1;
        out_f32[3 * p + 2] = v2;
      }
    }
  }
}

// Vector path (W % 4 == 0, aligned): a thread per 4-pixel quad, 16-B depth
// loads, K1's doubled-gradient arithmetic on the packed-fp32 pipe with the
// coefficient PAIRS read from a duplicated (c, c) table in shared memory
// (one LDS.64 per coefficient and quad when the quad lies in one bin; a
// quad straddling a bin edge assembles mixed pairs), and K1's PRMT-packed
// uint8 stores.
template <int DEG>
__device__ __forceinline__ float2 poly2_sat_r(const float2 (&c)[15], float2 hx, float2 hy) {
  float2 acc = make_float2(0.f, 0.f), out = make_float2(0.f, 0.f);
#pragma unroll
  for (int i = DEG; i >= 0; --i) {
    float2 p = c[bterm(i, DEG - i)];
#pragma unroll
    for (int j = DEG - i - 1; j >= 0; --j) p = __ffma2_rn(p, hy, c[bterm(i, j)]);
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

__device__ __forceinline__ uint32_t pack4(float2 a, float2 b) {
  const float2 qa = __ffma2_rn(a, make_float2(255.f, 255.f), make_float2(12582912.f, 12582912.f));
  const float2 qb = __ffma2_rn(b, make_float2(255.f, 255.f), make_float2(12582912.f, 12582912.f));
  return __byte_perm(__byte_perm(__float_as_uint(qa.x), __float_as_uint(qa.y), 0x0040),
                     __byte_perm(__float_as_uint(qb.x), __float_as_uint(qb.y), 0x0040), 0x5410);
}

template <int DEG, bool ALIGNED>  // ALIGNED: every bin edge on a multiple of 4 columns (no straddling quads)
__global__ void __launch_bounds__(kBinnedThreads) rgb_binned_vec_kernel(const float* __restrict__ depth, int64_t n,
                                                                        int H, int W, int bins_y, int bins_x,
                                                                        const float* __restrict__ coeffs,
                                                                        uint8_t* __restrict__ out_u8,
                                                                        float* __restrict__ out_f32) {
  constexpr int T = (DEG + 1) * (DEG + 2) / 2;
  extern __shared__ __align__(16) float sm[];
  const int n_sets = bins_y * bins_x;
  float2* dup = reinterpret_cast<float2*>(sm);                        // n_sets * 3 * T pairs (c, c)
  int* xbin = reinterpret_cast<int*>(sm + (size_t)n_sets * 3 * T * 2);  // W
  for (int k = threadIdx.x; k < n_sets * 3 * T; k += blockDim.x) {
    const float c = coeffs[k];
    dup[k] = make_float2(c, c);
  }
  for (int x = threadIdx.x; x < W; x += blockDim.x) xbin[x] = (int)(((int64_t)x * bins_x) / W);
  __syncthreads();

  // thread (g, xq): column quad xq of bands of kRows rows, walked with a
  // rolling up / centre / down register window (one new 16-B row load each)
  constexpr int kRows = 8;
  const int QW = W >> 2;
  const int groups = max(1, (int)blockDim.x / QW);
  const int g = threadIdx.x / QW;
  const int xq = threadIdx.x - g * QW;
  if (g >= groups) return;
  const int x0 = xq << 2;
  const bool at_left = x0 == 0, at_right = x0 + 4 >= W;
  const float m0 = at_left ? 2.f : 1.f, m3 = at_right ? 2.f : 1.f;
  const int b0 = xbin[x0], b1 = xbin[x0 + 1], b2 = xbin[x0 + 2], b3 = xbin[x0 + 3];
  const bool one_bin = ALIGNED || b0 == b3;
  const int bands = (H + kRows - 1) / kRows;
  const int64_t units = n * bands;
  for (int64_t u = (int64_t)blockIdx.x * groups + g; u < units; u += (int64_t)gridDim.x * groups) {
    const int64_t img = u / bands;
    const int r0 = (int)(u - img * bands) * kRows;
    const int nr = min(kRows, H - r0);
    const float* p = depth + (img * H + r0) * (int64_t)W + x0;  // row r0, this quad
    float4 c = __ldg(reinterpret_cast<const float4*>(p));
    float4 up = r0 > 0 ? __ldg(reinterpret_cast<const float4*>(p - W)) : c;
#pragma unroll
    for (int j = 0; j < kRows; ++j) {
      if (j >= nr) break;
      const int r = r0 + j;
      const float4 dn = r < H - 1 ? __ldg(reinterpret_cast<const float4*>(p + W)) : c;
      const float left = at_left ? c.x : __ldg(p - 1);
      const float right = at_right ? c.w : __ldg(p + 4);
      float2 hy01 = __fadd2_rn(make_float2(dn.x, dn.y), make_float2(-up.x, -up.y));
      float2 hy23 = __fadd2_rn(make_float2(dn.z, dn.w), make_float2(-up.z, -up.w));
      if (r == 0 || r == H - 1) {
        hy01 = __fadd2_rn(hy01, hy01);
        hy23 = __fadd2_rn(hy23, hy23);
      }
      const float2 hx01 = make_float2((c.y - left) * m0, c.z - c.x);
      const float2 hx23 = make_float2(c.w - c.y, (right - c.z) * m3);
      const int yb = (r * bins_y) / H * bins_x;  // 32-bit: r * bins_y < 2^31 (bins_y <= H)
      float2 v01[3], v23[3];
      if (one_bin) {
        const float2* cs = dup + (size_t)(yb + b0) * 3 * T;
#pragma unroll
        for (int ch = 0; ch < 3; ++ch) {
          float2 cp[15];
#pragma unroll
          for (int k = 0; k < T; ++k) cp[k] = cs[ch * T + k];
          v01[ch] = poly2_sat_r<DEG>(cp, hx01, hy01);
          v23[ch] = poly2_sat_r<DEG>(cp, hx23, hy23);
        }
      } else if constexpr (!ALIGNED) {  // the quad straddles a bin edge: a set per pixel pair, mixed only inside a pair
        const float2* s0 = dup + (size_t)(yb + b0) * 3 * T;
        const float2* s1 = dup + (size_t)(yb + b1) * 3 * T;
        const float2* s2 = dup + (size_t)(yb + b2) * 3 * T;
        const float2* s3 = dup + (size_t)(yb + b3) * 3 * T;
#pragma unroll
        for (int ch = 0; ch < 3; ++ch) {
          float2 ca[15], cb[15];
#pragma unroll
          for (int k = 0; k < T; ++k) {
            ca[k] = b0 == b1 ? s0[ch * T + k] : make_float2(s0[ch * T + k].x, s1[ch * T + k].x);
            cb[k] = b2 == b3 ? s2[ch * T + k] : make_float2(s2[ch * T + k].x, s3[ch * T + k].x);
          }
          v01[ch] = poly2_sat_r<DEG>(ca, hx01, hy01);
          v23[ch] = poly2_sat_r<DEG>(cb, hx23, hy23);
        }
      }
      const int64_t q = (img * H + r) * (int64_t)W + x0;
      if (out_u8) {
        uint32_t* o = reinterpret_cast<uint32_t*>(out_u8 + 3 * q);
        o[0] = pack4(make_float2(v01[0].x, v01[1].x), make_float2(v01[2].x, v01[0].y));
        o[1] = pack4(make_float2(v01[1].y, v01[2].y), make_float2(v23[0].x, v23[1].x));
        o[2] = pack4(make_float2(v23[2].x, v23[0].y), make_float2(v23[1].y, v23[2].y));
      }
      if (out_f32) {
        float4* o = reinterpret_cast<float4*>(out_f32 + 3 * q);
        o[0] = make_float4(v01[0].x, v01[1].x, v01[2].x, v01[0].y);
        o[1] = make_float4(v01[1].y, v01[2].y, v23[0].x, v23[1].x);
        o[2] = make_float4(v23[2].x, v23[0].y, v23[1].y, v23[2].y);
      }
      up = c;
      c = dn;
      p += W;
    }
  }
}

size_t binned_smem(int n_sets, int T, int W) { return ((size_t)n_sets * 3 * T + W) * sizeof(float); }

template <int DEG>
int launch_binned(const tacsl_binned_lut_s* lut, const float* depth, int64_t n, uint8_t* u8, float* f32,
                  cudaStream_t s) {
  constexpr int T = (DEG + 1) * (DEG + 2) / 2;
  const int W = lut->width;
  const bool vec = W % 4 == 0 && W / 4 <= kBinnedThreads && (reinterpret_cast<uintptr_t>(depth) & 15) == 0 &&
                   (reinterpret_cast<uintptr_t>(u8) & 3) == 0 && (reinterpret_cast<uintptr_t>(f32) & 15) == 0 &&
                   !std::getenv("TACSL_BINNED_SCALAR");
  bool aligned = true;  // every x-bin edge floor(b * W / bins_x) on a multiple of 4
  for (int b = 1; b < lut->bins_x && aligned; ++b) {
    const int64_t edge = ((int64_t)b * W + lut->bins_x - 1) / lut->bins_x;  // first column of bin b
    aligned = edge % 4 == 0;
  }
  auto kern = !vec ? rgb_binned_kernel<DEG> : aligned ? rgb_binned_vec_kernel<DEG, true>
                                                      : rgb_binned_vec_kernel<DEG, false>;
  const size_t smem = binned_smem(lut->bins_y * lut->bins_x, T, lut->width) +
                      (vec ? (size_t)lut->bins_y * lut->bins_x * 3 * T * sizeof(float) : 0);
  if (int rc = set_max_dynamic_smem(reinterpret_cast<const void*>(kern), (int)(2 * kBinnedMaxSmem))) return rc;
  int per_sm = 0;
  cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, kern, kBinnedThreads, smem);
  const int QW = (lut->width + 3) / 4;
  const int rows_per_pass = std::max(1, kBinnedThreads / QW);
  const int64_t rows = vec ? n * ((lut->height + 7) / 8) : n * lut->height;  // vec: bands of 8 rows
  const int64_t grid = std::min<int64_t>((rows + rows_per_pass - 1) / rows_per_pass,
                                         (int64_t)sm_count(current_device()) * std::max(per_sm, 1));
  kern<<<(unsigned)grid, kBinnedThreads, smem, s>>>(depth, n, lut->height, lut->width, lut->bins_y, lut->bins_x,
                                                    lut->coeffs, u8, f32);
  return check_launch("rgb_binned_kernel");
}

}  // namespace
}  // namespace tacsl

using namespace tacsl;

extern "C" int tacsl_binned_lut_create(int device, const double* coeffs, int degree, int bins_y, int bins_x,
                                       int width, int height, tacsl_binned_lut_t* out) {
  if (!out || !coeffs) return set_error(TACSL_ERR_INVALID_ARGUMENT, "binned_lut_create: null pointer");
  if (degree < 2 || degree > 4) return set_error(TACSL_ERR_INVALID_ARGUMENT, "LUT degree must be in [2, 4]");
  if (width < 2 || height < 2) return set_error(TACSL_ERR_INVALID_ARGUMENT, "binned_lut_create: bad image size");
  if (bins_y < 1 || bins_x < 1 || bins_y > height || bins_x > width)
    return set_error(TACSL_ERR_INVALID_ARGUMENT, "binned_lut_create: bins must be in [1, image size]");
  const int T = (degree + 1) * (degree + 2) / 2;
  const int n_sets = bins_y * bins_x;
  if (!tacsl_device_supported(device))
    return set_error(TACSL_ERR_NO_DEVICE, "binned_lut_create: device is not an sm_100 (B200) GPU");
  std::vector<float> host((size_t)n_sets * 3 * T);
  for (int b = 0; b < n_sets; ++b)
    for (int ch = 0; ch < 3; ++ch) {
      int k = 0;
      for (int s = 0; s <= degree; ++s)
        for (int j = 0; j <= s; ++j, ++k)
          host[((size_t)b * 3 + ch) * T + k] = static_cast<float>(coeffs[((size_t)b * 3 + ch) * T + k] *
                                                                  std::ldexp(1.0, -s));
    }
  int prev = 0;
  cudaGetDevice(&prev);
  cudaSetDevice(device);
  std::vector<float2> dup(host.size());
  for (size_t i = 0; i < host.size(); ++i) dup[i] = make_float2(host[i], host[i]);
  float* d = nullptr;
  float2* dp = nullptr;
  if (cudaMalloc(&d, host.size() * sizeof(float)) != cudaSuccess ||
      cudaMemcpy(d, host.data(), host.size() * sizeof(float), cudaMemcpyHostToDevice) != cudaSuccess ||
      cudaMalloc(&dp, dup.size() * sizeof(float2)) != cudaSuccess ||
      cudaMemcpy(dp, dup.data(), dup.size() * sizeof(float2), cudaMemcpyHostToDevice) != cudaSuccess) {
    cudaFree(d);
    cudaFree(dp);
    cudaSetDevice(prev);
    return check_launch("binned_lut_create: upload");
  }
  cudaSetDevice(prev);
  auto* h = new tacsl_binned_lut_s{device, degree, width, height, bins_y, bins_x, d, dp};
  *out = h;
  return TACSL_OK;
}

extern "C" void tacsl_binned_lut_destroy(tacsl_binned_lut_t lut) {
  if (!lut) return;
  int prev = 0;
  cudaGetDevice(&prev);
  cudaSetDevice(lut->device);
  cudaFree(lut->coeffs);
  cudaFree(lut->pairs);
  cudaSetDevice(prev);
  delete lut;
}

extern "C" int tacsl_depth_to_rgb_binned(tacsl_binned_lut_t lut, const float* depth, int64_t n_images, int height,
                                         int width, uint8_t* rgb_u8, float* rgb_f32, void* stream) {
  StreamDevice stream_device_(stream);
  if (!lut) return set_error(TACSL_ERR_INVALID_ARGUMENT, "depth_to_rgb_binned: null LUT");
  if (width != lut->width || height != lut->height)
    return set_error(TACSL_ERR_LUT_RESOLUTION_MISMATCH,
                     "LUT calibrated at (" + std::to_string(lut->width) + ", " + std::to_string(lut->height) +
                         "), image is (" + std::to_string(width) + ", " + std::to_string(height) + ")");
  if (n_images < 0) return set_error(TACSL_ERR_INVALID_ARGUMENT, "depth_to_rgb_binned: negative image count");
  if (n_images == 0) return TACSL_OK;
  if (!rgb_u8 && !rgb_f32) return set_error(TACSL_ERR_INVALID_ARGUMENT, "depth_to_rgb_binned: no output buffer");
  if (!depth) return set_error(TACSL_ERR_INVALID_ARGUMENT, "depth_to_rgb_binned: null depth");
  cudaStream_t s = static_cast<cudaStream_t>(stream);
  // the band pipeline of K1 when no pixel pair straddles an x-bin edge (every
  // edge on an even column) and the buffers suit its 16-B / bulk accesses
  bool pairs_ok = width % 4 == 0 && width / 4 <= 320 && (reinterpret_cast<uintptr_t>(depth) & 15) == 0 &&
                  (reinterpret_cast<uintptr_t>(rgb_u8) & 3) == 0 && (reinterpret_cast<uintptr_t>(rgb_f32) & 15) == 0 &&
                  !std::getenv("TACSL_BINNED_SCALAR") && !std::getenv("TACSL_BINNED_SIMPLE");
  for (int b = 1; b < lut->bins_x && pairs_ok; ++b)
    pairs_ok = (((int64_t)b * width + lut->bins_x - 1) / lut->bins_x) % 2 == 0;
  // measured (8192 frames 240x320, tools/bench_binned.py): at degree 2 the
  // band pipeline keeps each thread's coefficients in registers and wins for
  // every bin width (10-px bins 1.40 vs 3.83 ms, 40-px bins 1.12 vs 1.40 ms);
  // at degrees 3-4 it reads them from its band's slice of the table in shared
  // memory and wins for narrow bins only (degree 3, 10-px bins: 2.96 vs 6.84
  // ms; 40-px bins: 2.23 vs 1.97 ms -- the per-quad kernel's quads rarely
  // straddle a wide bin's edge).  The per-quad kernels stage the WHOLE table
  // in shared memory, so larger tables go to the band pipeline regardless.
  const int T = (lut->degree + 1) * (lut->degree + 2) / 2;
  const bool table_fits = binned_smem(lut->bins_y * lut->bins_x, T, width) <= kBinnedMaxSmem;
  if (pairs_ok &&
      (lut->degree == 2 || width < 24 * lut->bins_x || !table_fits || std::getenv("TACSL_BINNED_BAND")))
    return launch_rgb_binned(lut->pairs, lut->bins_y, lut->bins_x, lut->degree, depth, n_images, height, width,
                             rgb_u8, rgb_f32, s);
  if (!table_fits)
    return set_error(TACSL_ERR_INVALID_ARGUMENT,
                     "depth_to_rgb_binned: this many bins need the band pipeline (width % 4 == 0, 16-B aligned "
                     "buffers, every x-bin edge on an even column); the per-quad kernel's shared memory holds "
                     "at most " + std::to_string(kBinnedMaxSmem / 1024) + " KB of table");
  switch (lut->degree) {
    case 2: return launch_binned<2>(lut, depth, n_images, rgb_u8, rgb_f32, s);
    case 3: return launch_binned<3>(lut, depth, n_images, rgb_u8, rgb_f32, s);
    case 4: return launch_binned<4>(lut, depth, n_images, rgb_u8, rgb_f32, s);
  }
  return set_error(TACSL_ERR_INVALID_ARGUMENT, "LUT degree must be in [2, 4]");
}
