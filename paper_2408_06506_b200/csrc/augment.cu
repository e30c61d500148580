// K4: per-episode / per-step tactile-image augmentation, bit-identical to
// render/augment.py:51-173, with the env's observation representation
// (envs/peg_tasks.py:447-458) fused as the epilogue.
//
// Two launches:
//  * augment_params_kernel -- one thread per image derives the episode
//    transform (augment.py:65-75) and the step jitter (augment.py:78-85)
//    from the reference's tuple-keyed RNG streams
//    np.random.Generator(np.random.Philox(np.random.SeedSequence(key))),
//    restated here: SeedSequence entropy mixing, Philox4x64-10 with the
//    pre-incremented counter, 53-bit doubles, masked-rejection permutation
//    (numpy 2.x algorithm; oracle/philox.py is the Python statement that
//    tests pin against numpy itself).  This replaces ~2 host Generator
//    constructions per sensor per step.
//  * augment_apply_kernel -- one thread per pixel: bilinear zoom about the
//    centre + shift with edge clamping (augment.py:121-140), channel
//    permutation, contrast / brightness, HSV saturation / hue (augment.py:
//    88-118, 143-153), the step jitter, clamp, then "color" / "diff" /
//    "concat".  All float32 with separately rounded operations in numpy's
//    order (no FMA contraction), so the output matches the reference bit
//    for bit.  HBM-bound: 12 B read + 12 B (or 24 B) written per pixel.
#include <algorithm>

#include "common.cuh"
#include "handles.h"

namespace tacsl {
namespace {

// ------------------------------------------------ numpy Philox streams ---
constexpr uint32_t kInitA = 0x43b0d7e5u, kMultA = 0x931e8875u;
constexpr uint32_t kInitB = 0x8b51f9ddu, kMultB = 0x58f38dedu;
constexpr uint32_t kMixL = 0xca01f9ddu, kMixR = 0x4973f715u;

struct Stream {
  uint64_t k0, k1;
  uint64_t ctr[4];
  uint64_t buf[4];
  int pos;
  bool has32;
  uint32_t u32;

  // entropy: the key's ints as little-endian 32-bit words (>= 1 word each)
  __device__ void seed(const uint32_t* ent, int n_ent) {
    uint32_t h = kInitA;
    auto hashmix = [&](uint32_t v) {
      v ^= h;
      h *= kMultA;
      v *= h;
      return v ^ (v >> 16);
    };
    auto mix = [](uint32_t x, uint32_t y) {
      uint32_t r = kMixL * x - kMixR * y;
      return r ^ (r >> 16);
    };
    uint32_t pool[4];
    for (int i = 0; i < 4; ++i) pool[i] = hashmix(i < n_ent ? ent[i] : 0u);
    for (int s = 0; s < 4; ++s)
      for (int d = 0; d < 4; ++d)
        if (s != d) pool[d] = mix(pool[d], hashmix(pool[s]));
    for (int s = 4; s < n_ent; ++s)
      for (int d = 0; d < 4; ++d) pool[d] = mix(pool[d], hashmix(ent[s]));
    // generate_state(2, uint64) -> Philox key
    uint32_t hb = kInitB, w[4];
    for (int i = 0; i < 4; ++i) {
      uint32_t v = pool[i] ^ hb;
      hb *= kMultB;
      v *= hb;
      w[i] = v ^ (v >> 16);
    }
    k0 = (uint64_t)w[0] | ((uint64_t)w[1] << 32);
    k1 = (uint64_t)w[2] | ((uint64_t)w[3] << 32);
    ctr[0] = ctr[1] = ctr[2] = ctr[3] = 0;
    pos = 4;
    has32 = false;
    u32 = 0;
  }

  __device__ void block() {
    // counter is incremented before each 4-word block (with carry)
    for (int i = 0; i < 4; ++i)
      if (++ctr[i] != 0) break;
    uint64_t c0 = ctr[0], c1 = ctr[1], c2 = ctr[2], c3 = ctr[3];
    uint64_t a = k0, b = k1;
#pragma unroll
    for (int r = 0; r < 10; ++r) {
      if (r) {
        a += 0x9E3779B97F4A7C15ull;
        b += 0xBB67AE8584CAA73Bull;
      }
      const uint64_t hi0 = __umul64hi(0xD2E7470EE14C6C93ull, c0), lo0 = 0xD2E7470EE14C6C93ull * c0;
      const uint64_t hi1 = __umul64hi(0xCA5A826395121157ull, c2), lo1 = 0xCA5A826395121157ull * c2;
      const uint64_t n0 = hi1 ^ c1 ^ a, n2 = hi0 ^ c3 ^ b;
      c0 = n0;
      c1 = lo1;
      c2 = n2;
      c3 = lo0;
    }
    buf[0] = c0;
    buf[1] = c1;
    buf[2] = c2;
    buf[3] = c3;
    pos = 0;
  }
  __device__ uint64_t next64() {
    if (pos >= 4) block();
    return buf[pos++];
  }
  __device__ uint32_t next32() {
    if (has32) {
      has32 = false;
      return u32;
    }
    const uint64_t v = next64();
    has32 = true;
    u32 = (uint32_t)(v >> 32);
    return (uint32_t)v;
  }
  // Generator.uniform(low, high) = low + (high - low) * ((u64 >> 11) * 2^-53)
  __device__ double uniform(double lo, double hi) {
    const double d = (double)(next64() >> 11) * (1.0 / 9007199254740992.0);
    return add_rn(lo, mul_rn(sub_rn(hi, lo), d));
  }
  __device__ uint32_t interval(uint32_t mx) {
    if (mx == 0) return 0;
    uint32_t mask = mx;
    mask |= mask >> 1;
    mask |= mask >> 2;
    mask |= mask >> 4;
    mask |= mask >> 8;
    mask |= mask >> 16;
    uint32_t v;
    while ((v = (next32() & mask)) > mx) {
    }
    return v;
  }
};

__device__ __forceinline__ int push_int(uint32_t* ent, int n, uint64_t v) {
  ent[n++] = (uint32_t)v;
  if (v >> 32) ent[n++] = (uint32_t)(v >> 32);
  return n;
}

// per-image parameter block
enum { P_SX = 0, P_SY, P_ZOOM, P_B, P_C, P_S, P_H, P_P0, P_P1, P_P2, P_DB, P_DC, P_DS, P_DH, P_COUNT };

__global__ void augment_params_kernel(const tacsl_augment_cfg_t cfg, const int64_t* __restrict__ episode_seeds,
                                      const int64_t* __restrict__ steps, int64_t n, double* __restrict__ params) {
  const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= n) return;
  double* p = params + i * 16;
  uint32_t ent[8];
  Stream s;
  // episode transform: key (seed, episode_seed, 0)
  int ne = push_int(ent, 0, cfg.seed);
  ne = push_int(ent, ne, (uint64_t)episode_seeds[i]);
  ne = push_int(ent, ne, 0);
  s.seed(ent, ne);
  p[P_SX] = s.uniform(-cfg.shift_px, cfg.shift_px);
  p[P_SY] = s.uniform(-cfg.shift_px, cfg.shift_px);
  p[P_ZOOM] = s.uniform(cfg.zoom_lo, cfg.zoom_hi);
  p[P_B] = s.uniform(-cfg.brightness, cfg.brightness);
  p[P_C] = s.uniform(cfg.contrast_lo, cfg.contrast_hi);
  p[P_S] = s.uniform(cfg.saturation_lo, cfg.saturation_hi);
  p[P_H] = s.uniform(-cfg.hue, cfg.hue);
  int perm[3] = {0, 1, 2};
  if (cfg.channel_permutation) {
    for (int k = 2; k > 0; --k) {
      const int j = (int)s.interval((uint32_t)k);
      const int t = perm[k];
      perm[k] = perm[j];
      perm[j] = t;
    }
  }
  p[P_P0] = perm[0];
  p[P_P1] = perm[1];
  p[P_P2] = perm[2];
  // step jitter: key (seed, episode_seed, 1, step_index)
  ne = push_int(ent, 0, cfg.seed);
  ne = push_int(ent, ne, (uint64_t)episode_seeds[i]);
  ne = push_int(ent, ne, 1);
  ne = push_int(ent, ne, (uint64_t)steps[i]);
  s.seed(ent, ne);
  p[P_DB] = s.uniform(-cfg.step_brightness, cfg.step_brightness);
  p[P_DC] = s.uniform(cfg.step_contrast_lo, cfg.step_contrast_hi);
  p[P_DS] = s.uniform(cfg.step_saturation_lo, cfg.step_saturation_hi);
  p[P_DH] = s.uniform(-cfg.step_hue, cfg.step_hue);
}

// ------------------------------------------------------- colour math ---
__device__ __forceinline__ float fadd(float a, float b) { return __fadd_rn(a, b); }
__device__ __forceinline__ float fsub(float a, float b) { return __fsub_rn(a, b); }
__device__ __forceinline__ float fmul(float a, float b) { return __fmul_rn(a, b); }
__device__ __forceinline__ float clip01(float x) { return fminf(fmaxf(x, 0.f), 1.f); }

// Correctly rounded a / b given y = RN(1/b): q = RN(a y) is within an ulp, and
// one exact-remainder FMA correction rounds it correctly (Markstein) -- the
// same bits as IEEE division, in 3 FP32 operations.
__device__ __forceinline__ float div_y(float a, float b, float y) {
  const float q = __fmul_rn(a, y);
  const float r = __fmaf_rn(-q, b, a);
  return __fmaf_rn(r, y, q);
}

// np.remainder(x, float32(1)): fmod (= x - trunc(x), exact for floats), +1 for
// a negative remainder, +0 for zero
__device__ __forceinline__ float rem1(float x) {
  float m = fsub(x, truncf(x));
  if (m < 0.f) m = fadd(m, 1.0f);
  return m == 0.f ? 0.f : m;
}

// _apply_color (augment.py:143-153), float32
// one _apply_color call's parameters, converted to float32 and their
// "is this stage active" tests taken once per image, not per pixel
struct ColorOp {
  float b, c, s, h;
  bool do_c, do_b, do_hsv;
};

__device__ __forceinline__ ColorOp color_op(double b, double c, double s, double h) {
  return ColorOp{(float)b, (float)c, (float)s, (float)h, c != 1.0, b != 0.0, s != 1.0 || h != 0.0};
}

__device__ __forceinline__ void apply_color(float v[3], const ColorOp& op) {
  if (op.do_c) {
    const float cf = op.c;
    for (int k = 0; k < 3; ++k) v[k] = fadd(fmul(fsub(v[k], 0.5f), cf), 0.5f);
  }
  if (op.do_b) {
    const float bf = op.b;
    for (int k = 0; k < 3; ++k) v[k] = fadd(v[k], bf);
  }
  if (op.do_hsv) {
    // rgb_to_hsv (augment.py:88-103) of the clipped colour
    const float r = clip01(v[0]), g = clip01(v[1]), bl = clip01(v[2]);
    const float mx = fmaxf(fmaxf(r, g), bl), mn = fminf(fminf(r, g), bl);
    const float span = fsub(mx, mn);
    const float mxs = fmaxf(mx, 1e-12f);
    float sat = mx > 0.f ? div_y(span, mxs, __frcp_rn(mxs)) : 0.f;
    const float safe = span > 0.f ? span : 1.f;
    const float ys = __frcp_rn(safe);
    const float rc = div_y(fsub(mx, r), safe, ys), gc = div_y(fsub(mx, g), safe, ys);
    const float bc = div_y(fsub(mx, bl), safe, ys);
    float hue = (r == mx) ? fsub(bc, gc) : ((g == mx) ? fsub(fadd(2.f, rc), bc) : fsub(fadd(4.f, gc), rc));
    constexpr float kInv6 = 0.16666667163372039794921875f;  // RN(1/6)
    hue = span > 0.f ? rem1(div_y(hue, 6.f, kInv6)) : 0.f;
    // hue shift and saturation scale (augment.py:150-151)
    hue = rem1(fadd(hue, op.h));
    sat = clip01(fmul(sat, op.s));
    // hsv_to_rgb (augment.py:106-118)
    const float h6 = fmul(hue, 6.f);
    const float fi = floorf(h6);
    const float f = fsub(h6, fi);
    const float p = fmul(mx, fsub(1.f, sat));
    const float q = fmul(mx, fsub(1.f, fmul(sat, f)));
    const float t = fmul(mx, fsub(1.f, fmul(sat, fsub(1.f, f))));
    const int i = ((int)fi) % 6;
    const float vv = mx;
    switch (i) {
      case 0: v[0] = vv; v[1] = t; v[2] = p; break;
      case 1: v[0] = q; v[1] = vv; v[2] = p; break;
      case 2: v[0] = p; v[1] = vv; v[2] = t; break;
      case 3: v[0] = p; v[1] = q; v[2] = vv; break;
      case 4: v[0] = t; v[1] = p; v[2] = vv; break;
      default: v[0] = vv; v[1] = p; v[2] = q; break;
    }
  }
}

// Grid: x strides over an image's pixels, y over images, so the per-image
// parameters and the branches they select are uniform across a CTA and no
// 64-bit division is needed per pixel.
// 5 CTAs per SM caps it at 48 registers without spills (63 unbounded):
// 1.74 vs 1.78 ms at 2048 x 240x320 (tools/bench_augment.py)
__global__ void __launch_bounds__(256, 5) augment_apply_kernel(const float* __restrict__ in, int64_t n, int H, int W,
                                                            const double* __restrict__ params, int rep, float n0,
                                                            float n1, float n2, float* __restrict__ out) {
  const int HW = H * W;
  const float invW = 1.0f / (float)W;
  const float hc = (float)((H - 1) / 2.0), wc = (float)((W - 1) / 2.0);
  for (int64_t img = blockIdx.y; img < n; img += gridDim.y) {
    const double* P = params + img * 16;
    const float* src = in + img * (int64_t)HW * 3;
    const double zoom = P[P_ZOOM], sx = P[P_SX], sy = P[P_SY];
    const bool resample = zoom != 1.0 || sx != 0.0 || sy != 0.0;
    const float zf = (float)zoom, izf = __frcp_rn(zf), sxf = (float)sx, syf = (float)sy;
    const int p0 = (int)P[P_P0], p1 = (int)P[P_P1], p2 = (int)P[P_P2];
    const bool permute = p0 != 0 || p1 != 1 || p2 != 2;
    const ColorOp episode_op = color_op(P[P_B], P[P_C], P[P_S], P[P_H]);
    const double db = P[P_DB], dc = P[P_DC], ds = P[P_DS], dh = P[P_DH];
    const bool step_jitter = db != 0.0 || dc != 1.0 || ds != 1.0 || dh != 0.0;
    const ColorOp step_op = color_op(db, dc, ds, dh);
    for (int rem = blockIdx.x * blockDim.x + threadIdx.x; rem < HW; rem += gridDim.x * blockDim.x) {
      // rem / W without an integer division: float quotient (exact inputs
      // below 2^24 pixels per image, error < 1), then one correction
      int y = __float2int_rz(__int2float_rn(rem) * invW);
      int x = rem - y * W;
      if (x < 0) {
        --y;
        x += W;
      } else if (x >= W) {
        ++y;
        x -= W;
      }
      float v[3];
      if (resample) {
        // _resample_bilinear (augment.py:121-140)
        float ys = fsub(fadd(div_y(fsub((float)y, hc), zf, izf), hc), syf);
        float xs = fsub(fadd(div_y(fsub((float)x, wc), zf, izf), wc), sxf);
        ys = fminf(fmaxf(ys, 0.f), (float)(H - 1));
        xs = fminf(fmaxf(xs, 0.f), (float)(W - 1));
        const int y0 = min(max((int)ys, 0), H - 2), x0 = min(max((int)xs, 0), W - 2);
        const float fy = fsub(ys, (float)y0), fx = fsub(xs, (float)x0);
        const float ufx = fsub(1.f, fx), ufy = fsub(1.f, fy);
        const float* a = src + ((size_t)y0 * W + x0) * 3;
        const float* cc = a + (size_t)W * 3;
        for (int k = 0; k < 3; ++k) {
          const float top = fadd(fmul(a[k], ufx), fmul(a[3 + k], fx));
          const float bot = fadd(fmul(cc[k], ufx), fmul(cc[3 + k], fx));
          v[k] = fadd(fmul(top, ufy), fmul(bot, fy));
        }
      } else {
        const float* a = src + (size_t)rem * 3;
        v[0] = a[0];
        v[1] = a[1];
        v[2] = a[2];
      }
      if (permute) {  // selects, not a dynamically indexed (local-memory) array
        auto pick = [&](int k) { return k == 0 ? v[0] : (k == 1 ? v[1] : v[2]); };
        const float w0 = pick(p0), w1 = pick(p1), w2 = pick(p2);
        v[0] = w0;
        v[1] = w1;
        v[2] = w2;
      }
      apply_color(v, episode_op);
      if (step_jitter) apply_color(v, step_op);
      for (int k = 0; k < 3; ++k) v[k] = clip01(v[k]);
      const int64_t idx = img * (int64_t)HW + rem;
      if (rep == 2) {
        float* o = out + idx * 6;
        o[0] = v[0];
        o[1] = v[1];
        o[2] = v[2];
        o[3] = n0;
        o[4] = n1;
        o[5] = n2;
      } else {
        float* o = out + idx * 3;
        o[0] = rep == 1 ? fsub(v[0], n0) : v[0];
        o[1] = rep == 1 ? fsub(v[1], n1) : v[1];
        o[2] = rep == 1 ? fsub(v[2], n2) : v[2];
      }
    }
  }
}

}  // namespace
}  // namespace tacsl

using namespace tacsl;

extern "C" int tacsl_augment_params(const tacsl_augment_cfg_t* cfg, const int64_t* episode_seeds,
                                    const int64_t* step_indices, int64_t n, double* params, void* stream) {
  StreamDevice stream_device_(stream);
  if (!cfg) return set_error(TACSL_ERR_INVALID_ARGUMENT, "augment: null config");
  if (n < 0) return set_error(TACSL_ERR_INVALID_ARGUMENT, "augment: negative count");
  if (n == 0) return TACSL_OK;
  if (!episode_seeds || !step_indices || !params) return set_error(TACSL_ERR_INVALID_ARGUMENT, "augment: null pointer");
  if (cfg->zoom_lo <= 0 || cfg->zoom_hi <= 0) return set_error(TACSL_ERR_INVALID_ARGUMENT, "zoom must be positive");
  const int threads = 128;
  augment_params_kernel<<<(unsigned)((n + threads - 1) / threads), threads, 0, (cudaStream_t)stream>>>(
      *cfg, episode_seeds, step_indices, n, params);
  return check_launch("augment_params_kernel");
}

extern "C" int tacsl_augment(const float* images, int64_t n, int height, int width, const double* params, int rep,
                             const float nominal[3], float* out, void* stream) {
  StreamDevice stream_device_(stream);
  if (n < 0 || height < 2 || width < 2) return set_error(TACSL_ERR_INVALID_ARGUMENT, "augment: bad sizes");
  if (rep < 0 || rep > 2) return set_error(TACSL_ERR_INVALID_ARGUMENT, "augment: rep must be 0, 1 or 2");
  if (n == 0) return TACSL_OK;
  if (!images || !params || !out || (rep && !nominal))
    return set_error(TACSL_ERR_INVALID_ARGUMENT, "augment: null pointer");
  if (images == out) return set_error(TACSL_ERR_INVALID_ARGUMENT, "augment: in-place is not supported");
  if ((int64_t)height * width >= (1 << 24))
    return set_error(TACSL_ERR_INVALID_ARGUMENT, "augment: images are limited to 2^24 pixels");
  const int64_t hw = (int64_t)height * width;
  const int64_t total = n * hw;
  const int64_t blocks = std::min<int64_t>((total + 255) / 256, (int64_t)sm_count(current_device()) * 16);
  const unsigned gy = (unsigned)std::min<int64_t>(n, 65535);
  const unsigned gx = (unsigned)std::max<int64_t>(1, std::min<int64_t>((hw + 255) / 256, (blocks + gy - 1) / gy));
  augment_apply_kernel<<<dim3(gx, gy), 256, 0, (cudaStream_t)stream>>>(
      images, n, height, width, params, rep, rep ? nominal[0] : 0.f, rep ? nominal[1] : 0.f,
      rep ? nominal[2] : 0.f, out);
  return check_launch("augment_apply_kernel");
}
