// Small device utilities around the hot path:
//
//  * tacsl_to_uint8_f64   render/imageio.py:8-11 on float64 input, in float64
//                         (rint of the separately rounded product x*255,
//                         ties to even, then clip), bit-exact to numpy;
//  * tacsl_f64_to_f32 / tacsl_f32_to_f64
//                         the numpy drop-ins' dtype changes done on the device
//                         (astype rounding: to nearest, ties to even), so the
//                         host only moves the caller's bytes once;
//  * tacsl_relative_penetration_rate
//                         geometry/sdf.py:324-328 (raises InvalidQuery);
//  * tacsl_frame_digest   a position-dependent 64-bit digest per frame of any
//                         output buffer (bench.py / multi-rank validation:
//                         the per-frame digests of a step, in global frame
//                         order, are identical for any number of ranks).
#include "common.cuh"

namespace tacsl {
namespace {

__device__ __forceinline__ uint8_t quantize_u8_f64(double x) {
  // np.clip(np.rint(x * 255), 0, 255).astype(uint8): the product is rounded
  // to float64 first (no FMA), rint rounds half to even; NaN -> 0
  const double q = rint(__dmul_rn(x, 255.0));
  return (uint8_t)(int)fmin(fmax(q, 0.0), 255.0);
}

__global__ void __launch_bounds__(256) to_uint8_f64_kernel(const double* __restrict__ x, int64_t n,
                                                           uint8_t* __restrict__ out) {
  const int64_t stride = (int64_t)gridDim.x * blockDim.x;
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += stride)
    out[i] = quantize_u8_f64(x[i]);
}

// 16-B vectorised element-wise conversion; the tail (and unaligned buffers)
// one element per thread
template <typename In, typename Out>
__global__ void __launch_bounds__(256) convert_kernel(const In* __restrict__ x, int64_t n, Out* __restrict__ y) {
  const int64_t stride = (int64_t)gridDim.x * blockDim.x;
  const int64_t t0 = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  const bool vec = ((reinterpret_cast<uintptr_t>(x) | reinterpret_cast<uintptr_t>(y)) & 31) == 0;
  int64_t head = 0;
  if (vec) {
    const int64_t n4 = n / 4;
    for (int64_t i = t0; i < n4; i += stride) {
      if constexpr (sizeof(In) == 8) {  // 2 x 16-B loads, one 16-B store
        const double2 a = reinterpret_cast<const double2*>(x)[2 * i];
        const double2 b = reinterpret_cast<const double2*>(x)[2 * i + 1];
        reinterpret_cast<float4*>(y)[i] = make_float4(__double2float_rn(a.x), __double2float_rn(a.y),
                                                      __double2float_rn(b.x), __double2float_rn(b.y));
      } else {  // one 16-B load, 2 x 16-B stores
        const float4 a = reinterpret_cast<const float4*>(x)[i];
        reinterpret_cast<double2*>(y)[2 * i] = make_double2(a.x, a.y);
        reinterpret_cast<double2*>(y)[2 * i + 1] = make_double2(a.z, a.w);
      }
    }
    head = n4 * 4;
  }
  for (int64_t i = head + t0; i < n; i += stride) y[i] = (Out)x[i];
}

// splitmix64 finalizer
__device__ __forceinline__ uint64_t mix64(uint64_t z) {
  z = (z ^ (z >> 30)) * 0xbf58476d1ce4e5b9ull;
  z = (z ^ (z >> 27)) * 0x94d049bb133111ebull;
  return z ^ (z >> 31);
}

// digest(frame) = sum_i mix64((i << 32) | word_i) mod 2^64 over the frame's
// 32-bit words: every word and its position count (a swapped channel, a
// shifted row or a misplaced frame changes it), and the sum can be formed in
// any order.  One CTA per frame (grid-strided), fp-free.
__global__ void __launch_bounds__(256) frame_digest_kernel(const uint32_t* __restrict__ data, int64_t n_frames,
                                                           int64_t words, uint64_t* __restrict__ out) {
  __shared__ uint64_t part[8];
  for (int64_t f = blockIdx.x; f < n_frames; f += gridDim.x) {
    const uint32_t* p = data + f * words;
    uint64_t s = 0;
    for (int64_t i = threadIdx.x; i < words; i += blockDim.x) s += mix64(((uint64_t)i << 32) | __ldg(p + i));
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) s += __shfl_xor_sync(0xffffffffu, s, o);
    if ((threadIdx.x & 31) == 0) part[threadIdx.x >> 5] = s;
    __syncthreads();
    if (threadIdx.x == 0) {
      uint64_t t = 0;
      for (int w = 0; w < (int)(blockDim.x >> 5); ++w) t += part[w];
      out[f] = mix64(t ^ (uint64_t)words);
    }
    __syncthreads();
  }
}

// geometry/sdf.py:324-328 relative_penetration_rate: d_dot = n . x_dot over
// the trailing axis, summed as numpy 2.3's einsum does for a length-3 axis
// -- (x0 + x2) + x1 of the rounded products (measured on the reference's
// numpy: every one of 1e5 random triples); any out-of-grid query raises the
// flag (InvalidQuery)
__global__ void __launch_bounds__(256) penetration_rate_kernel(const double* __restrict__ normal,
                                                               const uint8_t* __restrict__ valid,
                                                               const double* __restrict__ x_dot, int64_t n,
                                                               int64_t x_stride, double* __restrict__ out,
                                                               int* __restrict__ invalid) {
  const int64_t stride = (int64_t)gridDim.x * blockDim.x;
  int bad = 0;
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += stride) {
    const double* a = normal + 3 * i;
    const double* b = x_dot + x_stride * i;
    out[i] = __dadd_rn(__dadd_rn(__dmul_rn(a[0], b[0]), __dmul_rn(a[2], b[2])), __dmul_rn(a[1], b[1]));
    bad |= valid[i] == 0;
  }
  if (__any_sync(0xffffffffu, bad) && (threadIdx.x & 31) == 0) atomicOr(invalid, 1);
}

int grid_for(int64_t count) {
  int64_t blocks = (count + 255) / 256;
  const int64_t cap = (int64_t)sm_count(current_device()) * 8;
  return (int)(blocks < cap ? (blocks < 1 ? 1 : blocks) : cap);
}

}  // namespace
}  // namespace tacsl

using namespace tacsl;

extern "C" int tacsl_to_uint8_f64(const double* x, int64_t count, uint8_t* out, void* stream) {
  StreamDevice stream_device_(stream);
  if (count < 0) return set_error(TACSL_ERR_INVALID_ARGUMENT, "to_uint8_f64: negative count");
  if (count == 0) return TACSL_OK;
  if (!x || !out) return set_error(TACSL_ERR_INVALID_ARGUMENT, "to_uint8_f64: null pointer");
  to_uint8_f64_kernel<<<grid_for(count), 256, 0, (cudaStream_t)stream>>>(x, count, out);
  return check_launch("to_uint8_f64");
}

extern "C" int tacsl_f64_to_f32(const double* x, int64_t count, float* out, void* stream) {
  StreamDevice stream_device_(stream);
  if (count < 0) return set_error(TACSL_ERR_INVALID_ARGUMENT, "f64_to_f32: negative count");
  if (count == 0) return TACSL_OK;
  if (!x || !out) return set_error(TACSL_ERR_INVALID_ARGUMENT, "f64_to_f32: null pointer");
  convert_kernel<double, float><<<grid_for(count / 4 + 1), 256, 0, (cudaStream_t)stream>>>(x, count, out);
  return check_launch("f64_to_f32");
}

extern "C" int tacsl_f32_to_f64(const float* x, int64_t count, double* out, void* stream) {
  StreamDevice stream_device_(stream);
  if (count < 0) return set_error(TACSL_ERR_INVALID_ARGUMENT, "f32_to_f64: negative count");
  if (count == 0) return TACSL_OK;
  if (!x || !out) return set_error(TACSL_ERR_INVALID_ARGUMENT, "f32_to_f64: null pointer");
  convert_kernel<float, double><<<grid_for(count / 4 + 1), 256, 0, (cudaStream_t)stream>>>(x, count, out);
  return check_launch("f32_to_f64");
}

extern "C" int tacsl_frame_digest(const void* data, int64_t n_frames, int64_t frame_bytes, uint64_t* out,
                                  void* stream) {
  StreamDevice stream_device_(stream);
  if (n_frames < 0 || frame_bytes < 0) return set_error(TACSL_ERR_INVALID_ARGUMENT, "frame_digest: bad sizes");
  if (frame_bytes % 4 != 0) return set_error(TACSL_ERR_INVALID_ARGUMENT, "frame_digest: frame_bytes % 4 != 0");
  if (n_frames == 0) return TACSL_OK;
  if (!data || !out) return set_error(TACSL_ERR_INVALID_ARGUMENT, "frame_digest: null pointer");
  if ((reinterpret_cast<uintptr_t>(data) & 3) != 0)
    return set_error(TACSL_ERR_INVALID_ARGUMENT, "frame_digest: data must be 4-B aligned");
  const int64_t cap = (int64_t)sm_count(current_device()) * 8;
  const unsigned grid = (unsigned)(n_frames < cap ? n_frames : cap);
  frame_digest_kernel<<<grid, 256, 0, (cudaStream_t)stream>>>(static_cast<const uint32_t*>(data), n_frames,
                                                              frame_bytes / 4, out);
  return check_launch("frame_digest");
}

extern "C" int tacsl_relative_penetration_rate(const double* normal, const uint8_t* valid, const double* x_dot,
                                               int64_t n, int x_dot_broadcast, double* out, int* scratch,
                                               void* stream) {
  StreamDevice stream_device_(stream);
  if (n < 0) return set_error(TACSL_ERR_INVALID_ARGUMENT, "penetration_rate: negative count");
  if (n == 0) return TACSL_OK;
  if (!normal || !valid || !x_dot || !out || !scratch)
    return set_error(TACSL_ERR_INVALID_ARGUMENT, "penetration_rate: null pointer");
  cudaStream_t s = (cudaStream_t)stream;
  cudaMemsetAsync(scratch, 0, sizeof(int), s);
  penetration_rate_kernel<<<grid_for(n), 256, 0, s>>>(normal, valid, x_dot, n, x_dot_broadcast ? 0 : 3, out,
                                                      scratch);
  if (int rc = check_launch("penetration_rate")) return rc;
  int bad = 0;  // the reference raises synchronously: read the flag back
  if (cudaMemcpyAsync(&bad, scratch, sizeof(int), cudaMemcpyDeviceToHost, s) != cudaSuccess ||
      cudaStreamSynchronize(s) != cudaSuccess)
    return check_launch("penetration_rate (flag read-back)");
  if (bad) return set_error(TACSL_ERR_INVALID_QUERY, "penetration rate requires in-bounds queries");
  return TACSL_OK;
}
