// K5: separable Gaussian smoothing and Gaussian-pyramid decimation of depth
// maps -- the north_star stages "separable Gaussian smoothing" and
// "multi-scale Gaussian pyramid" (BASELINE.json config 5).  They have NO
// counterpart in the reference package (SURVEY.md section 0 / 8a rows a13,
// a14), so their semantics are defined here and restated on the CPU by
// oracle/pyramid_oracle.py (scipy.ndimage conventions):
//
//   out[y, x] = sum_i sum_j w[i] w[j] in[clamp(s*y + i - R), clamp(s*x + j - R)]
//
// with 'nearest' (edge-replicating) borders, a normalised 1-D kernel w of
// 2R+1 taps (Gaussian: scipy's truncate rule; pyramid: the 5-tap binomial
// [1, 4, 6, 4, 1] / 16) and output stride s (1: smoothing, 2: pyramid level).
//
// A CTA streams the input rows of a 32-output-row band through a cp.async
// ring, blurs each horizontally (only at the output columns) into a
// (2R+1)-row ring, and emits every output row as the vertical blend of ring
// rows -- HBM sees each input byte once (+ the 2R halo rows per band, mostly
// L2 hits) and each output byte once.
#include <algorithm>

#include "common.cuh"
#include "handles.h"

namespace tacsl {
namespace {

constexpr int kMaxTaps = 33;  // radius <= 16

struct Taps {
  float w[kMaxTaps];
  int radius;
};

constexpr int kAhead = 4;       // input rows in flight per CTA (cp.async ring)
constexpr int kMaxCols = 6;     // output columns per thread (256 threads: Wo <= 1536)
constexpr int kBandOut = 32;    // output rows per work unit

__device__ __forceinline__ void cp_async16(void* dst, const void* src) {
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"(smem_addr(dst)), "l"(src) : "memory");
}
__device__ __forceinline__ void cp_async4(void* dst, const void* src) {
  asm volatile("cp.async.ca.shared.global [%0], [%1], 4;" ::"r"(smem_addr(dst)), "l"(src) : "memory");
}
__device__ __forceinline__ void cp_commit() { asm volatile("cp.async.commit_group;" ::: "memory"); }
template <int N>
__device__ __forceinline__ void cp_wait() {
  asm volatile("cp.async.wait_group %0;" ::"n"(N) : "memory");
}

// Work unit = (image, band of kBandOut output rows).  Input rows stream
// through a kAhead-deep cp.async ring (so several rows per CTA are in flight
// while one is filtered); each is blurred horizontally at the output columns
// into a (2R+1)-row ring, and output rows are emitted as soon as their last
// input row has arrived.  A band re-reads its 2R halo rows (from L2).
constexpr int kThreads = 128;

template <int NC>  // output columns per thread: xo = threadIdx.x + q * kThreads, q < NC
__global__ void __launch_bounds__(kThreads) sep_filter_kernel(const float* __restrict__ in, int64_t n, int H,
                                                              int W, int Ho, int Wo, int step, const Taps T,
                                                              float* __restrict__ out) {
  extern __shared__ __align__(16) float sm[];
  const int R = T.radius, K = 2 * R + 1;
  float* rows = sm;                       // kAhead x W
  float* ring = sm + (size_t)kAhead * W;  // K x Wo
  const bool vec = (W % 4 == 0) && ((reinterpret_cast<uintptr_t>(in) & 15) == 0);
  const int bands = (Ho + kBandOut - 1) / kBandOut;
  const int64_t units = n * bands;
  bool colv[NC];
  int colc[NC];  // input column of each output column
#pragma unroll
  for (int q = 0; q < NC; ++q) {
    const int xo = threadIdx.x + q * kThreads;
    colv[q] = xo < Wo;
    colc[q] = step * xo;
  }
  for (int64_t u = blockIdx.x; u < units; u += gridDim.x) {
    const int64_t img = u / bands;
    const int y0 = (int)(u - img * bands) * kBandOut;
    const int y1 = min(y0 + kBandOut, Ho);  // exclusive
    const int r_lo = max(step * y0 - R, 0);
    const int r_hi = min(step * (y1 - 1) + R, H - 1);  // inclusive
    const float* src = in + img * (int64_t)H * W;
    float* dst = out + img * (int64_t)Ho * Wo;
    auto load_row = [&](int r) {
      float* d = rows + (size_t)(r % kAhead) * W;
      const float* sr = src + (int64_t)r * W;
      if (vec) {
        for (int x = threadIdx.x * 4; x < W; x += kThreads * 4) cp_async16(d + x, sr + x);
      } else {
        for (int x = threadIdx.x; x < W; x += kThreads) cp_async4(d + x, sr + x);
      }
    };
    __syncthreads();  // the previous unit is done with both rings
    for (int k = 0; k < kAhead - 1; ++k) {
      if (r_lo + k <= r_hi) load_row(r_lo + k);
      cp_commit();
    }
    int next_out = y0;
    int wslot = r_lo % K;  // ring slot of input row r
    for (int r = r_lo; r <= r_hi; ++r) {
      if (r + kAhead - 1 <= r_hi) load_row(r + kAhead - 1);
      cp_commit();
      cp_wait<kAhead - 1>();  // row r has landed (this thread's part)
      __syncthreads();        // ... and every thread's part
      const float* row = rows + (size_t)(r % kAhead) * W;
      float* hr = ring + (size_t)wslot * Wo + threadIdx.x;
      wslot = (wslot + 1 == K) ? 0 : wslot + 1;
#pragma unroll
      for (int q = 0; q < NC; ++q) {
        if (!colv[q]) continue;
        const int c = colc[q];
        float acc = 0.f;
        if (c - R >= 0 && c + R < W) {  // interior: no border clamps
          const float* p = row + c - R;
          for (int j = 0; j < K; ++j) acc = __fmaf_rn(T.w[j], p[j], acc);
        } else {
          for (int j = 0; j < K; ++j) acc = __fmaf_rn(T.w[j], row[min(max(c + j - R, 0), W - 1)], acc);
        }
        hr[q * kThreads] = acc;
      }
      // emit every output row whose last needed input row has arrived; the
      // ring columns a thread reads are the ones it wrote.  Taps outer,
      // columns inner: the ring slot of each tap is computed once per row.
      while (next_out < y1 && min(step * next_out + R, H - 1) <= r) {
        const int cy = step * next_out;
        float acc[NC];
#pragma unroll
        for (int q = 0; q < NC; ++q) acc[q] = 0.f;
        const bool interior = (cy - R >= 0) && (cy + R <= H - 1);
        int slot = interior ? (cy - R) % K : 0;  // one division per output row
        for (int i = 0; i < K; ++i) {
          if (!interior) slot = min(max(cy + i - R, 0), H - 1) % K;  // border rows only
          const float* rp = ring + (size_t)slot * Wo + threadIdx.x;
          slot = (slot + 1 == K) ? 0 : slot + 1;
          const float w = T.w[i];
#pragma unroll
          for (int q = 0; q < NC; ++q)
            if (colv[q]) acc[q] = __fmaf_rn(w, rp[q * kThreads], acc[q]);
        }
        float* orow = dst + (int64_t)next_out * Wo + threadIdx.x;
#pragma unroll
        for (int q = 0; q < NC; ++q)
          if (colv[q]) orow[q * kThreads] = acc[q];
        ++next_out;
      }
      __syncthreads();  // row slot r % kAhead may be refilled next iteration
    }
    cp_wait<0>();
  }
}

template <int NC>
int launch_filter(const float* in, int64_t n, int H, int W, int Ho, int Wo, int step, const Taps& T, float* out,
                  cudaStream_t stream) {
  auto kern = sep_filter_kernel<NC>;
  static bool configured = false;
  if (!configured) {
    cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, 227 * 1024);
    configured = true;
  }
  const size_t smem = ((size_t)kAhead * W + (size_t)(2 * T.radius + 1) * Wo) * sizeof(float);
  int per_sm = 0;
  cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, kern, kThreads, smem);
  const int64_t units = n * ((Ho + kBandOut - 1) / kBandOut);
  const int64_t grid = std::min<int64_t>(units, (int64_t)sm_count(current_device()) * std::max(per_sm, 1));
  kern<<<(unsigned)grid, kThreads, smem, stream>>>(in, n, H, W, Ho, Wo, step, T, out);
  return check_launch("sep_filter_kernel");
}

}  // namespace
}  // namespace tacsl

using namespace tacsl;

extern "C" int tacsl_separable_filter(const float* in, int64_t n_images, int height, int width, const float* taps,
                                      int radius, int step, float* out, void* stream) {
  if (n_images < 0 || height < 1 || width < 1) return set_error(TACSL_ERR_INVALID_ARGUMENT, "filter: bad sizes");
  if (radius < 0 || radius > (kMaxTaps - 1) / 2)
    return set_error(TACSL_ERR_INVALID_ARGUMENT, "filter: radius must be in [0, 16]");
  if (step != 1 && step != 2) return set_error(TACSL_ERR_INVALID_ARGUMENT, "filter: step must be 1 or 2");
  if (n_images == 0) return TACSL_OK;
  if (!in || !out || !taps) return set_error(TACSL_ERR_INVALID_ARGUMENT, "filter: null pointer");
  if (in == out) return set_error(TACSL_ERR_INVALID_ARGUMENT, "filter: in-place is not supported");
  const int Ho = (height + step - 1) / step, Wo = (width + step - 1) / step;
  if (Wo > kThreads * kMaxCols) return set_error(TACSL_ERR_INVALID_ARGUMENT, "filter: image too wide");
  Taps T;
  T.radius = radius;
  for (int k = 0; k < kMaxTaps; ++k) T.w[k] = k < 2 * radius + 1 ? taps[k] : 0.f;
  const size_t smem = ((size_t)kAhead * width + (size_t)(2 * radius + 1) * Wo) * sizeof(float);
  if (smem > 227 * 1024) return set_error(TACSL_ERR_INVALID_ARGUMENT, "filter: image too wide");
  cudaStream_t s = (cudaStream_t)stream;
  switch ((Wo + kThreads - 1) / kThreads) {
    case 1: return launch_filter<1>(in, n_images, height, width, Ho, Wo, step, T, out, s);
    case 2: return launch_filter<2>(in, n_images, height, width, Ho, Wo, step, T, out, s);
    case 3: return launch_filter<3>(in, n_images, height, width, Ho, Wo, step, T, out, s);
    case 4: return launch_filter<4>(in, n_images, height, width, Ho, Wo, step, T, out, s);
    case 5: return launch_filter<5>(in, n_images, height, width, Ho, Wo, step, T, out, s);
    default: return launch_filter<6>(in, n_images, height, width, Ho, Wo, step, T, out, s);
  }
}
