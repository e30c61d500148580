// C-ABI plumbing: error state, device checks, LUT/SDF handles, to_uint8.
#include <algorithm>
#include <cmath>
#include <cstdio>
#include <cstring>
#include <mutex>
#include <string>
#include <vector>

#include "common.cuh"
#include "handles.h"

namespace tacsl {

static thread_local std::string g_last_error;

int set_error(int code, const std::string& msg) {
  g_last_error = msg;
  return code;
}

int check_launch(const char* what) {
  cudaError_t e = cudaGetLastError();
  if (e != cudaSuccess) {
    return set_error(TACSL_ERR_CUDA, std::string(what) + ": " + cudaGetErrorString(e));
  }
  return TACSL_OK;
}

int current_device() {
  int d = 0;
  cudaGetDevice(&d);
  return d;
}

int set_max_dynamic_smem(const void* func, int bytes) {
  static std::mutex mu;
  static std::vector<std::pair<const void*, uint64_t>> done;  // kernel -> devices configured (bit mask)
  const int dev = current_device();
  std::lock_guard<std::mutex> lock(mu);
  uint64_t* mask = nullptr;
  for (auto& e : done)
    if (e.first == func) mask = &e.second;
  if (!mask) {
    done.emplace_back(func, 0);
    mask = &done.back().second;
  }
  if (dev < 64 && ((*mask >> dev) & 1u)) return TACSL_OK;
  if (cudaFuncSetAttribute(func, cudaFuncAttributeMaxDynamicSharedMemorySize, bytes) != cudaSuccess)
    return check_launch("cudaFuncSetAttribute(max dynamic shared memory)");
  if (dev < 64) *mask |= (uint64_t)1 << dev;
  return TACSL_OK;
}

int sm_count(int device) {
  static std::mutex mu;
  static std::vector<int> cache;
  std::lock_guard<std::mutex> lock(mu);
  if (device < 0) device = 0;
  if ((int)cache.size() <= device) cache.resize(device + 1, 0);
  if (cache[device] == 0) {
    int n = 0;
    if (cudaDeviceGetAttribute(&n, cudaDevAttrMultiProcessorCount, device) != cudaSuccess || n <= 0) n = 148;
    cache[device] = n;
  }
  return cache[device];
}

// Scaled coefficient for the kernels' "doubled gradient" form: the kernels
// evaluate the polynomial on h = 2*g (h = f[x+1]-f[x-1] inside, 2*(f1-f0)
// at borders), so c_ij is pre-multiplied by 2^-(i+j) -- an exact power-of-two
// rescaling that removes two multiplies per pixel.
static void fill_scaled(LutParams& p, const double* coeffs, int degree) {
  const int T = (degree + 1) * (degree + 2) / 2;
  std::memset(&p, 0, sizeof(p));
  for (int ch = 0; ch < 3; ++ch) {
    int k = 0;
    for (int s = 0; s <= degree; ++s) {
      for (int j = 0; j <= s; ++j, ++k) {
        double scale = std::ldexp(1.0, -s);
        p.c[ch][k] = static_cast<float>(coeffs[ch * T + k] * scale);
      }
    }
  }
}

}  // namespace tacsl

using namespace tacsl;

extern "C" {

int tacsl_abi_version(void) { return TACSL_ABI_VERSION; }

const char* tacsl_last_error(void) { return g_last_error.c_str(); }

int tacsl_device_supported(int device) {
  int n = 0;
  if (cudaGetDeviceCount(&n) != cudaSuccess || device < 0 || device >= n) {
    cudaGetLastError();
    return 0;
  }
  cudaDeviceProp prop;
  if (cudaGetDeviceProperties(&prop, device) != cudaSuccess) return 0;
  return prop.major == 10 && prop.minor == 0 ? 1 : 0;
}

int tacsl_lut_create(const double* coeffs, int degree, int width, int height, tacsl_lut_t* out) {
  if (!out || !coeffs) return set_error(TACSL_ERR_INVALID_ARGUMENT, "lut_create: null pointer");
  if (degree < 2 || degree > 4) return set_error(TACSL_ERR_INVALID_ARGUMENT, "LUT degree must be in [2, 4]");
  if (width <= 0 || height <= 0) return set_error(TACSL_ERR_INVALID_ARGUMENT, "lut_create: bad image size");
  auto* h = new tacsl_lut_s();
  h->degree = degree;
  h->width = width;
  h->height = height;
  fill_scaled(h->params, coeffs, degree);
  *out = h;
  return TACSL_OK;
}

void tacsl_lut_destroy(tacsl_lut_t lut) { delete lut; }

}  // extern "C"

namespace {
// float32 quad grid + per-axis Lipschitz bounds for the force field's
// certified contact-mask pre-pass (handles.h).  Best effort: without it the
// force field runs its fp64 kernel.
void build_quads(tacsl_sdf_s* h, const double* v, const int32_t dims[3]) {
  h->quads = nullptr;
  h->lip[0] = h->lip[1] = h->lip[2] = 0.0f;
  const int64_t nx = dims[0], ny = dims[1], nz = dims[2];
  const int64_t n = nx * ny * nz;
  double lip[3] = {0.0, 0.0, 0.0};
  for (int64_t i = 0; i < n; ++i)
    if (!(std::fabs(v[i]) < 1e30)) return;  // non-finite / beyond float range
  std::vector<float4> q((size_t)n);
  for (int64_t x = 0; x < nx; ++x)
    for (int64_t y = 0; y < ny; ++y)
      for (int64_t z = 0; z < nz; ++z) {
        const int64_t c = (x * ny + y) * nz + z;
        const int64_t y1 = std::min(y + 1, ny - 1), z1 = std::min(z + 1, nz - 1);
        q[(size_t)c] = make_float4((float)v[c], (float)v[(x * ny + y) * nz + z1], (float)v[(x * ny + y1) * nz + z],
                                   (float)v[(x * ny + y1) * nz + z1]);
        if (x + 1 < nx) lip[0] = std::max(lip[0], std::fabs(v[c + ny * nz] - v[c]));
        if (y + 1 < ny) lip[1] = std::max(lip[1], std::fabs(v[c + nz] - v[c]));
        if (z + 1 < nz) lip[2] = std::max(lip[2], std::fabs(v[c + 1] - v[c]));
      }
  int prev = 0;
  cudaGetDevice(&prev);
  cudaSetDevice(h->device);
  float4* d = nullptr;
  cudaError_t e = cudaMalloc(&d, (size_t)n * sizeof(float4));
  if (e == cudaSuccess) e = cudaMemcpy(d, q.data(), (size_t)n * sizeof(float4), cudaMemcpyHostToDevice);
  cudaSetDevice(prev);
  if (e != cudaSuccess) {
    if (d) cudaFree(d);
    cudaGetLastError();
    return;
  }
  h->quads = d;
  for (int a = 0; a < 3; ++a) h->lip[a] = (float)(lip[a] * (1.0 + 1e-6)) + 1e-30f;  // rounded up
}
}  // namespace

extern "C" {

int tacsl_sdf_create(int device, const double* values, const double* gradients, const int32_t dims[3],
                     const double origin[3], double spacing, tacsl_sdf_t* out) {
  if (!out || !values || !gradients || !dims || !origin)
    return set_error(TACSL_ERR_INVALID_ARGUMENT, "sdf_create: null pointer");
  if (!(spacing > 0)) return set_error(TACSL_ERR_INVALID_ARGUMENT, "spacing must be positive");
  for (int a = 0; a < 3; ++a)
    if (dims[a] < 2) return set_error(TACSL_ERR_INVALID_ARGUMENT, "sdf_create: need >= 2 cells per axis");
  if (!tacsl_device_supported(device))
    return set_error(TACSL_ERR_NO_DEVICE, "sdf_create: device is not an sm_100 (B200) GPU");
  const size_t n = (size_t)dims[0] * dims[1] * dims[2];
  if (n >= ((size_t)1 << 31))  // kernels index cells with 32-bit ints
    return set_error(TACSL_ERR_INVALID_ARGUMENT, "sdf_create: grids are limited to 2^31 cells");
  std::vector<double4> host(n);
  for (size_t i = 0; i < n; ++i)
    host[i] = make_double4(values[i], gradients[3 * i + 0], gradients[3 * i + 1], gradients[3 * i + 2]);
  int prev = 0;
  cudaGetDevice(&prev);
  cudaSetDevice(device);
  double4* dptr = nullptr;
  double* vptr = nullptr;
  cudaError_t e = cudaMalloc(&dptr, n * sizeof(double4));
  if (e == cudaSuccess) e = cudaMalloc(&vptr, n * sizeof(double));
  if (e == cudaSuccess) e = cudaMemcpy(dptr, host.data(), n * sizeof(double4), cudaMemcpyHostToDevice);
  if (e == cudaSuccess) e = cudaMemcpy(vptr, values, n * sizeof(double), cudaMemcpyHostToDevice);
  cudaSetDevice(prev);
  if (e != cudaSuccess) {
    if (dptr) cudaFree(dptr);
    if (vptr) cudaFree(vptr);
    return set_error(TACSL_ERR_CUDA, std::string("sdf_create: ") + cudaGetErrorString(e));
  }
  auto* h = new tacsl_sdf_s();
  h->device = device;
  h->grid = dptr;
  h->values = vptr;
  build_quads(h, values, dims);
  for (int a = 0; a < 3; ++a) {
    h->dims[a] = dims[a];
    h->origin[a] = origin[a];
  }
  h->spacing = spacing;
  *out = h;
  return TACSL_OK;
}

void tacsl_sdf_destroy(tacsl_sdf_t sdf) {
  if (!sdf) return;
  int prev = 0;
  cudaGetDevice(&prev);
  cudaSetDevice(sdf->device);
  cudaFree(sdf->grid);
  cudaFree(sdf->values);
  if (sdf->quads) cudaFree(sdf->quads);
  cudaSetDevice(prev);
  delete sdf;
}

}  // extern "C"

// ------------------------------------------------------------- to_uint8 ---
namespace {

// clip(rint(255 x), 0, 255): saturate, then x*255 + 1.5*2^23 rounds the exact
// product to the nearest integer, ties to even (= np.rint of the exact fp64
// product of an fp32 x), and the integer sits in the low mantissa bits.
__device__ __forceinline__ uint32_t quantize_u8(float x) {
  float q = __fmaf_rn(__saturatef(x), 255.0f, 12582912.0f);
  return __float_as_uint(q) & 0xFFu;
}

__global__ void __launch_bounds__(256) to_uint8_kernel(const float* __restrict__ x, int64_t n,
                                                       uint8_t* __restrict__ out) {
  const int64_t stride = (int64_t)gridDim.x * blockDim.x;
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += stride)
    out[i] = (uint8_t)quantize_u8(x[i]);
}

}  // namespace

extern "C" int tacsl_to_uint8(const float* x, int64_t count, uint8_t* out, void* stream) {
  StreamDevice stream_device_(stream);
  if (count < 0) return set_error(TACSL_ERR_INVALID_ARGUMENT, "to_uint8: negative count");
  if (count == 0) return TACSL_OK;
  if (!x || !out) return set_error(TACSL_ERR_INVALID_ARGUMENT, "to_uint8: null pointer");
  int64_t blocks = (count + 255) / 256;
  int64_t cap = (int64_t)sm_count(current_device()) * 8;
  if (blocks > cap) blocks = cap;
  to_uint8_kernel<<<(unsigned)blocks, 256, 0, (cudaStream_t)stream>>>(x, count, out);
  return check_launch("to_uint8");
}
