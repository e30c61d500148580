// K3: in-sensor depth rendering by sphere tracing the object's SDF.
//
// Replaces render/depth.py:88-134 render_depth: per pixel ray, slab-test the
// object's rotated grid box (_ray_aabb, depth.py:77-85), march from
// max(t_in, near) towards min(background, t_out) with step = trilinear SDF
// value inside the grid and the distance to the grid box outside it, record
// the first t with d < HIT_TOLERANCE, keep min(hit, membrane) and clip to
// [near, far].  The march mirrors the reference's numba kernel
// (_march_kernel, depth.py:174-233) operation for operation in float64 with
// separately rounded products and sums (numba/numpy never contract to FMA),
// so the depth map is bit-identical to the reference's.
//
// Mapping: one thread per (env, pixel) ray; consecutive threads walk
// consecutive pixels of one env, so a warp's rays hit neighbouring cells of
// the L2-resident float64 value grid (8 B per cell).
#include <algorithm>

#include "common.cuh"
#include "handles.h"

namespace tacsl {
namespace {

struct RenderParams {
  const double* __restrict__ values;  // (nx, ny, nz) float64, z fastest
  int nx, ny, nz;
  double gox, goy, goz, spacing;
  double hix, hiy, hiz;  // origin + spacing * (dims - 1)  (depth.py:180-182)
  double inv_spacing;    // RN(1 / spacing)
  double cx, cy, cz;     // camera position (sensor frame)
  double near_, far_, tol;
  int max_steps;
  int n_rays;
};

// correctly rounded a / spacing (Markstein: y = RN(1/b), q = RN(a y), one
// exact-remainder correction), as in force_field.cu
__device__ __forceinline__ double div_spacing(double a, double spacing, double inv_spacing) {
  const double q = mul_rn(a, inv_spacing);
  const double r = __fma_rn(-q, spacing, a);
  return __fma_rn(r, inv_spacing, q);
}

__device__ __forceinline__ double dmax(double a, double b) { return a > b ? a : b; }  // np.maximum w/o NaNs
__device__ __forceinline__ double dmin(double a, double b) { return a < b ? a : b; }

__global__ void __launch_bounds__(256) render_depth_kernel(const RenderParams P, const double* __restrict__ dirs,
                                                           const double* __restrict__ background,
                                                           const double* __restrict__ envp, int64_t n_envs,
                                                           double* __restrict__ out64, float* __restrict__ out32) {
  // the march's constants as locals (registers, not per-step constant-bank loads)
  const double gox = P.gox, goy = P.goy, goz = P.goz, hix = P.hix, hiy = P.hiy, hiz = P.hiz;
  const double cx = P.cx, cy = P.cy, cz = P.cz, spacing = P.spacing, inv_spacing = P.inv_spacing, tol = P.tol;
  const int nxm = P.nx - 2, nym = P.ny - 2, nzm = P.nz - 2, ny = P.ny, nz = P.nz, max_steps = P.max_steps;
  const double* __restrict__ values = P.values;
  // grid: y over envs, x over an env's rays (no 64-bit division per ray)
  for (int64_t e = blockIdx.y; e < n_envs; e += gridDim.y)
  for (int r = blockIdx.x * blockDim.x + threadIdx.x; r < P.n_rays; r += gridDim.x * blockDim.x) {
    const int64_t idx = e * P.n_rays + r;
    const double* ep = envp + e * 18;  // pos[3], rot[9] (object->sensor, row-major), lo[3], hi[3]
    const double dx = __ldg(dirs + 3 * r), dy = __ldg(dirs + 3 * r + 1), dz = __ldg(dirs + 3 * r + 2);
    const double bg = __ldg(background + r);

    // ---- slab test (depth.py:77-85) ----
    const double ivx = 1.0 / (fabs(dx) < 1e-300 ? 1e-300 : dx);
    const double ivy = 1.0 / (fabs(dy) < 1e-300 ? 1e-300 : dy);
    const double ivz = 1.0 / (fabs(dz) < 1e-300 ? 1e-300 : dz);
    const double t0x = mul_rn(sub_rn(__ldg(ep + 12), P.cx), ivx), t1x = mul_rn(sub_rn(__ldg(ep + 15), P.cx), ivx);
    const double t0y = mul_rn(sub_rn(__ldg(ep + 13), P.cy), ivy), t1y = mul_rn(sub_rn(__ldg(ep + 16), P.cy), ivy);
    const double t0z = mul_rn(sub_rn(__ldg(ep + 14), P.cz), ivz), t1z = mul_rn(sub_rn(__ldg(ep + 17), P.cz), ivz);
    const double tmin = dmax(dmax(dmin(t0x, t1x), dmin(t0y, t1y)), dmin(t0z, t1z));
    const double tmax = dmin(dmin(dmax(t0x, t1x), dmax(t0y, t1y)), dmax(t0z, t1z));
    const bool hit_box = tmax >= dmax(tmin, 0.0);
    const double inf = __longlong_as_double(0x7ff0000000000000LL);
    const double t_in = hit_box ? dmax(tmin, 0.0) : inf;
    const double t_out = hit_box ? tmax : -inf;
    const double t_stop = dmin(bg, t_out);
    const double t_start = dmax(t_in, P.near_);
    double depth = bg;

    if (t_start <= t_stop) {
      // ---- sphere trace (depth.py:183-233) ----
      const double px = __ldg(ep + 0), py = __ldg(ep + 1), pz = __ldg(ep + 2);
      const double r00 = __ldg(ep + 3), r01 = __ldg(ep + 4), r02 = __ldg(ep + 5);
      const double r10 = __ldg(ep + 6), r11 = __ldg(ep + 7), r12 = __ldg(ep + 8);
      const double r20 = __ldg(ep + 9), r21 = __ldg(ep + 10), r22 = __ldg(ep + 11);
      double t = t_start;
      for (int step = 0; step < max_steps; ++step) {
        const double wx = sub_rn(add_rn(cx, mul_rn(dx, t)), px);
        const double wy = sub_rn(add_rn(cy, mul_rn(dy, t)), py);
        const double wz = sub_rn(add_rn(cz, mul_rn(dz, t)), pz);
        // R^T w: sensor -> object frame
        const double ox = add_rn(add_rn(mul_rn(r00, wx), mul_rn(r10, wy)), mul_rn(r20, wz));
        const double oy = add_rn(add_rn(mul_rn(r01, wx), mul_rn(r11, wy)), mul_rn(r21, wz));
        const double oz = add_rn(add_rn(mul_rn(r02, wx), mul_rn(r12, wy)), mul_rn(r22, wz));
        double d;
        if (ox < gox || oy < goy || oz < goz || ox > hix || oy > hiy || oz > hiz) {
          // outside the grid: distance to the box is a safe step (depth.py:205-210)
          const double bx = add_rn(dmax(sub_rn(gox, ox), 0.0), dmax(sub_rn(ox, hix), 0.0));
          const double by = add_rn(dmax(sub_rn(goy, oy), 0.0), dmax(sub_rn(oy, hiy), 0.0));
          const double bz = add_rn(dmax(sub_rn(goz, oz), 0.0), dmax(sub_rn(oz, hiz), 0.0));
          d = dmax(__dsqrt_rn(add_rn(add_rn(mul_rn(bx, bx), mul_rn(by, by)), mul_rn(bz, bz))), spacing);
        } else {
          const double gx = div_spacing(sub_rn(ox, gox), spacing, inv_spacing);
          const double gy = div_spacing(sub_rn(oy, goy), spacing, inv_spacing);
          const double gz = div_spacing(sub_rn(oz, goz), spacing, inv_spacing);
          const int ix = min((int)gx, nxm), iy = min((int)gy, nym), iz = min((int)gz, nzm);
          const double fx = sub_rn(gx, (double)ix), fy = sub_rn(gy, (double)iy), fz = sub_rn(gz, (double)iz);
          const double ux = sub_rn(1.0, fx), uy = sub_rn(1.0, fy), uz = sub_rn(1.0, fz);
          const int sy = nz, sx = ny * nz;  // grids stay below 2^31 cells (checked at upload)
          const double* v = values + ((ix * ny + iy) * nz + iz);
          const double c00 = add_rn(mul_rn(__ldg(v), ux), mul_rn(__ldg(v + sx), fx));
          const double c10 = add_rn(mul_rn(__ldg(v + sy), ux), mul_rn(__ldg(v + sx + sy), fx));
          const double c01 = add_rn(mul_rn(__ldg(v + 1), ux), mul_rn(__ldg(v + sx + 1), fx));
          const double c11 = add_rn(mul_rn(__ldg(v + sy + 1), ux), mul_rn(__ldg(v + sx + sy + 1), fx));
          const double c0 = add_rn(mul_rn(c00, uy), mul_rn(c10, fy));
          const double c1 = add_rn(mul_rn(c01, uy), mul_rn(c11, fy));
          d = add_rn(mul_rn(c0, uz), mul_rn(c1, fz));
        }
        if (d < tol) {
          if (t < depth) depth = t;
          break;
        }
        t = add_rn(t, d);
        if (t > t_stop) break;
      }
    }
    depth = dmin(dmax(depth, P.near_), P.far_);  // np.clip(depth, near, far)
    if (out64) out64[idx] = depth;
    if (out32) out32[idx] = (float)depth;
  }
}

// ------------------------------------------------ per-env render inputs ---
// The env caller's host pose math on the device, operation for operation in
// float64 (separately rounded, numpy's order), so K3 sees bit-identical
// inputs:
//   object pose in sensor s's frame   envs/peg_tasks.py:440-442
//     pos  = quat_rotate(conj(q_s), p_obj - p_s)   transforms.py:30-47
//     quat = quat_mul(conj(q_s), q_obj)            transforms.py:17-24
//   env_params row (pos, R, AABB)      render/depth.py:105-112, 121
//     R = quat_to_mat(quat)  (q / |q|, |q|^2 summed left to right)
//     lo / hi = min / max over the 8 grid-box corners rotated into the frame
struct Q4 {
  double w, x, y, z;
};
struct D3 {
  double x, y, z;
};

__device__ __forceinline__ D3 cross_rn(D3 a, D3 b) {  // np.cross / transforms._cross component order
  return D3{sub_rn(mul_rn(a.y, b.z), mul_rn(a.z, b.y)), sub_rn(mul_rn(a.z, b.x), mul_rn(a.x, b.z)),
            sub_rn(mul_rn(a.x, b.y), mul_rn(a.y, b.x))};
}

// v + w t + q_v x t with t = 2 q_v x v  (left to right)
__device__ __forceinline__ D3 quat_rotate_rn(Q4 q, D3 v) {
  const D3 qv{q.x, q.y, q.z};
  D3 t = cross_rn(qv, v);
  t = D3{mul_rn(2.0, t.x), mul_rn(2.0, t.y), mul_rn(2.0, t.z)};
  const D3 c = cross_rn(qv, t);
  return D3{add_rn(add_rn(v.x, mul_rn(q.w, t.x)), c.x), add_rn(add_rn(v.y, mul_rn(q.w, t.y)), c.y),
            add_rn(add_rn(v.z, mul_rn(q.w, t.z)), c.z)};
}

__device__ __forceinline__ Q4 quat_mul_rn(Q4 a, Q4 b) {
  return Q4{sub_rn(sub_rn(sub_rn(mul_rn(a.w, b.w), mul_rn(a.x, b.x)), mul_rn(a.y, b.y)), mul_rn(a.z, b.z)),
            sub_rn(add_rn(add_rn(mul_rn(a.w, b.x), mul_rn(a.x, b.w)), mul_rn(a.y, b.z)), mul_rn(a.z, b.y)),
            add_rn(add_rn(sub_rn(mul_rn(a.w, b.y), mul_rn(a.x, b.z)), mul_rn(a.y, b.w)), mul_rn(a.z, b.x)),
            add_rn(sub_rn(add_rn(mul_rn(a.w, b.z), mul_rn(a.x, b.y)), mul_rn(a.y, b.x)), mul_rn(a.z, b.w))};
}

struct Box {
  double lo[3], hi[3];  // grid-box corner coordinates: origin, origin + spacing * (dims - 1)
};

__global__ void __launch_bounds__(128) env_render_params_kernel(const double* __restrict__ poses, int64_t n_envs,
                                                                int n_sensors, const Box box,
                                                                double* __restrict__ out) {
  const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;  // (env, sensor)
  if (i >= n_envs * n_sensors) return;
  const int64_t e = i / n_sensors;
  const int s = (int)(i - e * n_sensors);
  const int stride = 7 * n_sensors + 7;
  const double* row = poses + e * stride;
  const double* sp = row + 7 * s;
  const double* op = row + 7 * n_sensors;
  // conj(q_s) = q_s * [1, -1, -1, -1]
  const Q4 qc{mul_rn(sp[3], 1.0), mul_rn(sp[4], -1.0), mul_rn(sp[5], -1.0), mul_rn(sp[6], -1.0)};
  const D3 d{sub_rn(op[0], sp[0]), sub_rn(op[1], sp[1]), sub_rn(op[2], sp[2])};
  const D3 pos = quat_rotate_rn(qc, d);
  const Q4 q = quat_mul_rn(qc, Q4{op[3], op[4], op[5], op[6]});
  double* o = out + i * 18;
  o[0] = pos.x;
  o[1] = pos.y;
  o[2] = pos.z;
  // R = quat_to_mat(q)
  const double n = __dsqrt_rn(add_rn(add_rn(add_rn(mul_rn(q.w, q.w), mul_rn(q.x, q.x)), mul_rn(q.y, q.y)),
                                     mul_rn(q.z, q.z)));
  const double w = __ddiv_rn(q.w, n), x = __ddiv_rn(q.x, n), y = __ddiv_rn(q.y, n), z = __ddiv_rn(q.z, n);
  const double xx = mul_rn(x, x), yy = mul_rn(y, y), zz = mul_rn(z, z);
  const double xy = mul_rn(x, y), xz = mul_rn(x, z), yz = mul_rn(y, z);
  const double wx = mul_rn(w, x), wy = mul_rn(w, y), wz = mul_rn(w, z);
  o[3] = sub_rn(1.0, mul_rn(2.0, add_rn(yy, zz)));
  o[4] = mul_rn(2.0, sub_rn(xy, wz));
  o[5] = mul_rn(2.0, add_rn(xz, wy));
  o[6] = mul_rn(2.0, add_rn(xy, wz));
  o[7] = sub_rn(1.0, mul_rn(2.0, add_rn(xx, zz)));
  o[8] = mul_rn(2.0, sub_rn(yz, wx));
  o[9] = mul_rn(2.0, sub_rn(xz, wy));
  o[10] = mul_rn(2.0, add_rn(yz, wx));
  o[11] = sub_rn(1.0, mul_rn(2.0, add_rn(xx, yy)));
  // AABB of the rotated grid-box corners (unnormalised quaternion, as
  // quat_rotate is called on it), corners in meshgrid 'ij' order
  D3 lo{0, 0, 0}, hi{0, 0, 0};
#pragma unroll
  for (int c = 0; c < 8; ++c) {
    const D3 v{(c & 4) ? box.hi[0] : box.lo[0], (c & 2) ? box.hi[1] : box.lo[1], (c & 1) ? box.hi[2] : box.lo[2]};
    D3 r = quat_rotate_rn(q, v);
    r = D3{add_rn(r.x, pos.x), add_rn(r.y, pos.y), add_rn(r.z, pos.z)};
    if (c == 0) {
      lo = hi = r;
    } else {
      lo = D3{dmin(r.x, lo.x), dmin(r.y, lo.y), dmin(r.z, lo.z)};
      hi = D3{dmax(r.x, hi.x), dmax(r.y, hi.y), dmax(r.z, hi.z)};
    }
  }
  o[12] = lo.x;
  o[13] = lo.y;
  o[14] = lo.z;
  o[15] = hi.x;
  o[16] = hi.y;
  o[17] = hi.z;
}

}  // namespace
}  // namespace tacsl

using namespace tacsl;

extern "C" int tacsl_render_depth(tacsl_sdf_t sdf, const double* dirs, const double* background, int height,
                                  int width, const double cam_pos[3], double near_plane, double far_plane,
                                  double hit_tolerance, int max_steps, const double* env_params, int64_t n_envs,
                                  double* depth_f64, float* depth_f32, void* stream) {
  StreamDevice stream_device_(stream);
  if (!sdf) return set_error(TACSL_ERR_INVALID_ARGUMENT, "render_depth: null SDF");
  if (height <= 0 || width <= 0 || n_envs < 0 || max_steps < 0)
    return set_error(TACSL_ERR_INVALID_ARGUMENT, "render_depth: bad sizes");
  if (!(near_plane > 0 && near_plane < far_plane)) return set_error(TACSL_ERR_INVALID_ARGUMENT, "need 0 < near < far");
  if (n_envs == 0) return TACSL_OK;
  if (!dirs || !background || !cam_pos || !env_params || (!depth_f64 && !depth_f32))
    return set_error(TACSL_ERR_INVALID_ARGUMENT, "render_depth: null pointer");
  RenderParams P;
  P.values = sdf->values;
  P.nx = sdf->dims[0];
  P.ny = sdf->dims[1];
  P.nz = sdf->dims[2];
  P.gox = sdf->origin[0];
  P.goy = sdf->origin[1];
  P.goz = sdf->origin[2];
  P.spacing = sdf->spacing;
  P.inv_spacing = 1.0 / sdf->spacing;
  P.hix = sdf->origin[0] + sdf->spacing * (double)(P.nx - 1);
  P.hiy = sdf->origin[1] + sdf->spacing * (double)(P.ny - 1);
  P.hiz = sdf->origin[2] + sdf->spacing * (double)(P.nz - 1);
  P.cx = cam_pos[0];
  P.cy = cam_pos[1];
  P.cz = cam_pos[2];
  P.near_ = near_plane;
  P.far_ = far_plane;
  P.tol = hit_tolerance;
  P.max_steps = max_steps;
  P.n_rays = height * width;
  const int64_t total = n_envs * (int64_t)P.n_rays;
  const int64_t blocks = std::min<int64_t>((total + 255) / 256, (int64_t)sm_count(current_device()) * 32);
  const unsigned gy = (unsigned)std::min<int64_t>(n_envs, 65535);
  const unsigned gx = (unsigned)std::max<int64_t>(
      1, std::min<int64_t>((P.n_rays + 255) / 256, (blocks + gy - 1) / gy));
  render_depth_kernel<<<dim3(gx, gy), 256, 0, (cudaStream_t)stream>>>(P, dirs, background, env_params, n_envs,
                                                                      depth_f64, depth_f32);
  return check_launch("render_depth_kernel");
}

extern "C" int tacsl_env_render_params(tacsl_sdf_t sdf, const double* poses, int64_t n_envs, int n_sensors,
                                       double* env_params, void* stream) {
  StreamDevice stream_device_(stream);
  if (!sdf) return set_error(TACSL_ERR_INVALID_ARGUMENT, "env_render_params: null SDF");
  if (n_envs < 0 || n_sensors <= 0) return set_error(TACSL_ERR_INVALID_ARGUMENT, "env_render_params: bad sizes");
  if (n_envs == 0) return TACSL_OK;
  if (!poses || !env_params) return set_error(TACSL_ERR_INVALID_ARGUMENT, "env_render_params: null pointer");
  Box box;
  for (int k = 0; k < 3; ++k) {
    box.lo[k] = sdf->origin[k] + sdf->spacing * 0.0;
    box.hi[k] = sdf->origin[k] + sdf->spacing * (double)(sdf->dims[k] - 1);
  }
  const int64_t n = n_envs * n_sensors;
  env_render_params_kernel<<<(unsigned)((n + 127) / 128), 128, 0, (cudaStream_t)stream>>>(poses, n_envs, n_sensors,
                                                                                          box, env_params);
  return check_launch("env_render_params_kernel");
}
