// K2: penalty-based normal/shear force field + per-sensor net wrench, and the
// standalone query_sdf / penalty_forces / net_wrench kernels.
//
// Replaces tactile/field.py:79-129 compute_force_field, which per taxel does
//   p_w = R_s p + s_pos                                (field.py:104-105)
//   p_o = R_o^T (p_w - o_pos)                          (field.py:106)
//   d, n = query_sdf(p_o)                              (field.py:107-108, sdf.py:271-321)
//   n_w = R_o n                                        (field.py:109)
//   x_dot = (s_v + s_w x (p_w - s_pos)) - (o_v + o_w x (p_w - o_pos))   (field.py:111-113)
//   d_dot = n_w . x_dot ; v_t = x_dot - d_dot n_w      (field.py:114-115)
//   f_n, f_t = penalty_forces(...)                     (field.py:61-76, 117)
//   f -> sensor frame: R_s^T f                         (field.py:118-119)
// and tactile/field.py:132-141 net_wrench (force, torque about the sensor
// origin), fused here as a CTA reduction over the sensor's taxels.
//
// Precision: the whole geometric chain is float64, as in the reference.  The
// chain that decides the contact mask (p_w, p_o, the cell index and the
// trilinear distance) uses separately rounded __dmul_rn/__dadd_rn in
// numpy's operation order, so d -- and therefore d < 0 -- reproduces the
// reference bit for bit; the rest may use FMAs.
//
// Mapping: one CTA per sensor frame (env e, sensor s); threads stride over the
// rows*cols taxels.  The SDF is a float64 {d, gx, gy, gz} grid (32 B per cell,
// two 16B loads per trilinear corner) that stays L2-resident (2 MiB for the
// 32x32x64 peg, 64 MiB at 128^3).
#include <algorithm>

#include "common.cuh"
#include "handles.h"

namespace tacsl {
namespace {

struct V3 {
  double x, y, z;
};

__device__ __forceinline__ V3 v3(double x, double y, double z) { return V3{x, y, z}; }

// ---- exact (numpy-order, no contraction) helpers --------------------------
// np.cross: a1*b2 - a2*b1, a2*b0 - a0*b2, a0*b1 - a1*b0, each product rounded.
__device__ __forceinline__ V3 cross_rn(V3 a, V3 b) {
  return v3(sub_rn(mul_rn(a.y, b.z), mul_rn(a.z, b.y)), sub_rn(mul_rn(a.z, b.x), mul_rn(a.x, b.z)),
            sub_rn(mul_rn(a.x, b.y), mul_rn(a.y, b.x)));
}
// transforms.py:36-43: (v + w*t) + qv x t with t = 2 (qv x v)
__device__ __forceinline__ V3 quat_rotate_rn(double w, V3 qv, V3 v) {
  V3 t = cross_rn(qv, v);
  t = v3(2.0 * t.x, 2.0 * t.y, 2.0 * t.z);
  const V3 c = cross_rn(qv, t);
  return v3(add_rn(add_rn(v.x, mul_rn(w, t.x)), c.x), add_rn(add_rn(v.y, mul_rn(w, t.y)), c.y),
            add_rn(add_rn(v.z, mul_rn(w, t.z)), c.z));
}

// ---- contracted helpers (off the mask chain) -------------------------------
__device__ __forceinline__ V3 cross(V3 a, V3 b) {
  return v3(a.y * b.z - a.z * b.y, a.z * b.x - a.x * b.z, a.x * b.y - a.y * b.x);
}
__device__ __forceinline__ V3 quat_rotate(double w, V3 qv, V3 v) {
  V3 t = cross(qv, v);
  t = v3(2.0 * t.x, 2.0 * t.y, 2.0 * t.z);
  const V3 c = cross(qv, t);
  return v3(v.x + w * t.x + c.x, v.y + w * t.y + c.y, v.z + w * t.z + c.z);
}
__device__ __forceinline__ double dot(V3 a, V3 b) { return a.x * b.x + a.y * b.y + a.z * b.z; }

struct Grid {
  const double2* __restrict__ cells;  // 2 per cell: (d, gx), (gy, gz)
  int nx, ny, nz;
  double ox, oy, oz, spacing;
};

struct Query {
  double d;  // +inf when outside
  V3 n;      // 0 when outside
  bool valid;
};

// geometry/sdf.py:277-318
__device__ __forceinline__ Query query(const Grid& g, V3 p) {
  const double rx = __ddiv_rn(sub_rn(p.x, g.ox), g.spacing);
  const double ry = __ddiv_rn(sub_rn(p.y, g.oy), g.spacing);
  const double rz = __ddiv_rn(sub_rn(p.z, g.oz), g.spacing);
  const double mx = (double)(g.nx - 1), my = (double)(g.ny - 1), mz = (double)(g.nz - 1);
  Query q;
  q.valid = (rx >= 0.0) & (rx <= mx) & (ry >= 0.0) & (ry <= my) & (rz >= 0.0) & (rz <= mz);
  // clip(rel, 0, dims - 1 - 1e-9); i0 = min(int(rel_c), dims - 2); f = rel_c - i0
  const double cx = fmin(fmax(rx, 0.0), sub_rn(mx, 1e-9));
  const double cy = fmin(fmax(ry, 0.0), sub_rn(my, 1e-9));
  const double cz = fmin(fmax(rz, 0.0), sub_rn(mz, 1e-9));
  const int ix = min((int)cx, g.nx - 2), iy = min((int)cy, g.ny - 2), iz = min((int)cz, g.nz - 2);
  const double wx = sub_rn(cx, (double)ix), wy = sub_rn(cy, (double)iy), wz = sub_rn(cz, (double)iz);
  const double ux = sub_rn(1.0, wx), uy = sub_rn(1.0, wy), uz = sub_rn(1.0, wz);

  const size_t sz = (size_t)g.nz, sy = (size_t)g.ny * g.nz;
  const size_t base = (size_t)ix * sy + (size_t)iy * sz + iz;
  // corner (a,b,c) -> two 16B loads: (d, gx) and (gy, gz)
  double2 A[8], B[8];
#pragma unroll
  for (int k = 0; k < 8; ++k) {
    const size_t cell = base + ((k >> 2) & 1) * sy + ((k >> 1) & 1) * sz + (k & 1);
    A[k] = __ldg(g.cells + 2 * cell);
    B[k] = __ldg(g.cells + 2 * cell + 1);
  }
  // k = 4*dx + 2*dy + dz
  // distance: x, then y, then z lerps, products and sums rounded separately (sdf.py:305-311)
  {
    const double d00 = add_rn(mul_rn(A[0].x, ux), mul_rn(A[4].x, wx));
    const double d10 = add_rn(mul_rn(A[2].x, ux), mul_rn(A[6].x, wx));
    const double d01 = add_rn(mul_rn(A[1].x, ux), mul_rn(A[5].x, wx));
    const double d11 = add_rn(mul_rn(A[3].x, ux), mul_rn(A[7].x, wx));
    const double d0 = add_rn(mul_rn(d00, uy), mul_rn(d10, wy));
    const double d1 = add_rn(mul_rn(d01, uy), mul_rn(d11, wy));
    q.d = add_rn(mul_rn(d0, uz), mul_rn(d1, wz));
  }
  // gradient: same lerp tree, contracted
  auto lerp = [&](double a000, double a100, double a010, double a110, double a001, double a101, double a011,
                  double a111) {
    const double a00 = a000 * ux + a100 * wx;
    const double a10 = a010 * ux + a110 * wx;
    const double a01 = a001 * ux + a101 * wx;
    const double a11 = a011 * ux + a111 * wx;
    const double a0 = a00 * uy + a10 * wy;
    const double a1 = a01 * uy + a11 * wy;
    return a0 * uz + a1 * wz;
  };
  const double gx = lerp(A[0].y, A[4].y, A[2].y, A[6].y, A[1].y, A[5].y, A[3].y, A[7].y);
  const double gy = lerp(B[0].x, B[4].x, B[2].x, B[6].x, B[1].x, B[5].x, B[3].x, B[7].x);
  const double gz = lerp(B[0].y, B[4].y, B[2].y, B[6].y, B[1].y, B[5].y, B[3].y, B[7].y);
  const double inv = 1.0 / fmax(sqrt(gx * gx + gy * gy + gz * gz), 1e-12);
  if (q.valid) {
    q.n = v3(gx * inv, gy * inv, gz * inv);
  } else {
    q.d = __longlong_as_double(0x7ff0000000000000LL);  // +inf
    q.n = v3(0.0, 0.0, 0.0);
  }
  return q;
}

struct Penalty {
  double k_n, k_d, k_t, mu;
};

// tactile/field.py:61-76 on one point
__device__ __forceinline__ void penalty(const Penalty& P, double d, double d_dot, V3 n, V3 vt, V3& fn, V3& ft,
                                        bool& contact) {
  contact = d < 0.0;
  double coeff = contact ? (-P.k_n + P.k_d * d_dot) * d : 0.0;
  coeff = fmax(coeff, 0.0);
  fn = v3(coeff * n.x, coeff * n.y, coeff * n.z);
  const double speed = sqrt(vt.x * vt.x + vt.y * vt.y + vt.z * vt.z);
  const bool slipping = contact && (speed > 1e-9);  // SLIP_VELOCITY_EPS, field.py:25
  const double mag = fmin(P.k_t * speed, P.mu * coeff);
  const double scale = slipping ? mag / speed : 0.0;
  ft = v3(-scale * vt.x, -scale * vt.y, -scale * vt.z);
}

struct State {
  V3 pos;
  double qw;
  V3 qv;
  V3 v, w;
};

__device__ __forceinline__ State load_state(const double* __restrict__ s) {
  State st;
  st.pos = v3(__ldg(s + 0), __ldg(s + 1), __ldg(s + 2));
  st.qw = __ldg(s + 3);
  st.qv = v3(__ldg(s + 4), __ldg(s + 5), __ldg(s + 6));
  st.v = v3(__ldg(s + 7), __ldg(s + 8), __ldg(s + 9));
  st.w = v3(__ldg(s + 10), __ldg(s + 11), __ldg(s + 12));
  return st;
}

__device__ __forceinline__ double warp_sum(double v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v += __shfl_down_sync(0xffffffffu, v, o);
  return v;
}

template <typename OutT>
__global__ void __launch_bounds__(256) force_field_kernel(
    const Grid grid, const double* __restrict__ taxels, int n_taxels, const double* __restrict__ obj_state,
    int64_t obj_stride, const double* __restrict__ sen_state, int64_t sen_stride, int n_sensors, const Penalty P,
    OutT* __restrict__ f_n_out, OutT* __restrict__ f_t_out, double* __restrict__ wrench, double* __restrict__ kin,
    uint8_t* __restrict__ contact_out) {
  const int64_t frame = blockIdx.x;
  const int64_t e = frame / n_sensors;
  const int s = (int)(frame - e * n_sensors);
  const State O = load_state(obj_state + e * obj_stride);
  const State S = load_state(sen_state + e * sen_stride + (int64_t)s * 13);
  const V3 oq_inv = v3(-O.qv.x, -O.qv.y, -O.qv.z);
  const V3 sq_inv = v3(-S.qv.x, -S.qv.y, -S.qv.z);

  double acc[6] = {0, 0, 0, 0, 0, 0};
  const int64_t out_base = frame * (int64_t)n_taxels;
  for (int i = threadIdx.x; i < n_taxels; i += blockDim.x) {
    const V3 p = v3(__ldg(taxels + 3 * i), __ldg(taxels + 3 * i + 1), __ldg(taxels + 3 * i + 2));
    // ---- mask chain, numpy order (field.py:104-107) ----
    V3 pw = quat_rotate_rn(S.qw, S.qv, p);
    pw = v3(add_rn(pw.x, S.pos.x), add_rn(pw.y, S.pos.y), add_rn(pw.z, S.pos.z));
    const V3 ro = v3(sub_rn(pw.x, O.pos.x), sub_rn(pw.y, O.pos.y), sub_rn(pw.z, O.pos.z));
    const V3 po = quat_rotate_rn(O.qw, oq_inv, ro);
    const Query q = query(grid, po);
    // ---- kinematics (field.py:109-115) ----
    const V3 nw = quat_rotate(O.qw, O.qv, q.n);
    const V3 rs = v3(pw.x - S.pos.x, pw.y - S.pos.y, pw.z - S.pos.z);
    const V3 cs = cross(S.w, rs), co = cross(O.w, ro);
    const V3 xd = v3((S.v.x + cs.x) - (O.v.x + co.x), (S.v.y + cs.y) - (O.v.y + co.y),
                     (S.v.z + cs.z) - (O.v.z + co.z));
    const double d_dot = dot(nw, xd);
    const V3 vt = v3(xd.x - d_dot * nw.x, xd.y - d_dot * nw.y, xd.z - d_dot * nw.z);
    V3 fnw, ftw;
    bool contact;
    penalty(P, q.d, d_dot, nw, vt, fnw, ftw, contact);
    // ---- back to the sensor frame (field.py:118-119) ----
    const V3 fn = quat_rotate(S.qw, sq_inv, fnw);
    const V3 ft = quat_rotate(S.qw, sq_inv, ftw);
    const int64_t o = (out_base + i) * 3;
    f_n_out[o + 0] = (OutT)fn.x;
    f_n_out[o + 1] = (OutT)fn.y;
    f_n_out[o + 2] = (OutT)fn.z;
    f_t_out[o + 0] = (OutT)ft.x;
    f_t_out[o + 1] = (OutT)ft.y;
    f_t_out[o + 2] = (OutT)ft.z;
    if (kin) {
      double* k = kin + (out_base + i) * 8;
      k[0] = q.d;
      k[1] = d_dot;
      k[2] = vt.x;
      k[3] = vt.y;
      k[4] = vt.z;
      k[5] = nw.x;
      k[6] = nw.y;
      k[7] = nw.z;
    }
    if (contact_out) contact_out[out_base + i] = contact ? 1 : 0;
    // ---- net wrench (field.py:132-141) ----
    const V3 f = v3(fn.x + ft.x, fn.y + ft.y, fn.z + ft.z);
    const V3 tq = cross(p, f);
    acc[0] += f.x;
    acc[1] += f.y;
    acc[2] += f.z;
    acc[3] += tq.x;
    acc[4] += tq.y;
    acc[5] += tq.z;
  }
  if (wrench) {
    __shared__ double part[8][6];
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
#pragma unroll
    for (int k = 0; k < 6; ++k) acc[k] = warp_sum(acc[k]);
    if (lane == 0)
#pragma unroll
      for (int k = 0; k < 6; ++k) part[warp][k] = acc[k];
    __syncthreads();
    if (threadIdx.x < 6) {
      double t = 0.0;
      const int nw = (blockDim.x + 31) >> 5;
      for (int w = 0; w < nw; ++w) t += part[w][threadIdx.x];
      wrench[frame * 6 + threadIdx.x] = t;
    }
  }
}

__global__ void __launch_bounds__(256) query_sdf_kernel(const Grid grid, const double* __restrict__ pts, int64_t n,
                                                        double* __restrict__ dist, double* __restrict__ normal,
                                                        uint8_t* __restrict__ valid) {
  const int64_t stride = (int64_t)gridDim.x * blockDim.x;
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += stride) {
    const Query q = query(grid, v3(pts[3 * i], pts[3 * i + 1], pts[3 * i + 2]));
    if (dist) dist[i] = q.d;
    if (normal) {
      normal[3 * i] = q.n.x;
      normal[3 * i + 1] = q.n.y;
      normal[3 * i + 2] = q.n.z;
    }
    if (valid) valid[i] = q.valid ? 1 : 0;
  }
}

__global__ void __launch_bounds__(256) penalty_kernel(const double* __restrict__ d, const double* __restrict__ dd,
                                                      const double* __restrict__ n, const double* __restrict__ vt,
                                                      int64_t count, const Penalty P, double* __restrict__ fn_out,
                                                      double* __restrict__ ft_out) {
  const int64_t stride = (int64_t)gridDim.x * blockDim.x;
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < count; i += stride) {
    V3 fn, ft;
    bool c;
    penalty(P, d[i], dd[i], v3(n[3 * i], n[3 * i + 1], n[3 * i + 2]), v3(vt[3 * i], vt[3 * i + 1], vt[3 * i + 2]),
            fn, ft, c);
    fn_out[3 * i] = fn.x;
    fn_out[3 * i + 1] = fn.y;
    fn_out[3 * i + 2] = fn.z;
    ft_out[3 * i] = ft.x;
    ft_out[3 * i + 1] = ft.y;
    ft_out[3 * i + 2] = ft.z;
  }
}

__global__ void __launch_bounds__(256) net_wrench_kernel(const double* __restrict__ fn, const double* __restrict__ ft,
                                                         const double* __restrict__ pts, int n_pts,
                                                         double* __restrict__ force, double* __restrict__ torque) {
  const int64_t frame = blockIdx.x;
  double acc[6] = {0, 0, 0, 0, 0, 0};
  for (int i = threadIdx.x; i < n_pts; i += blockDim.x) {
    const int64_t o = (frame * n_pts + i) * 3;
    const V3 f = v3(fn[o] + ft[o], fn[o + 1] + ft[o + 1], fn[o + 2] + ft[o + 2]);
    const V3 tq = cross(v3(pts[3 * i], pts[3 * i + 1], pts[3 * i + 2]), f);
    acc[0] += f.x;
    acc[1] += f.y;
    acc[2] += f.z;
    acc[3] += tq.x;
    acc[4] += tq.y;
    acc[5] += tq.z;
  }
  __shared__ double part[8][6];
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
#pragma unroll
  for (int k = 0; k < 6; ++k) acc[k] = warp_sum(acc[k]);
  if (lane == 0)
#pragma unroll
    for (int k = 0; k < 6; ++k) part[warp][k] = acc[k];
  __syncthreads();
  if (threadIdx.x < 6) {
    double t = 0.0;
    for (int w = 0; w < (int)(blockDim.x >> 5); ++w) t += part[w][threadIdx.x];
    if (threadIdx.x < 3) force[frame * 3 + threadIdx.x] = t;
    else torque[frame * 3 + threadIdx.x - 3] = t;
  }
}

Grid make_grid(tacsl_sdf_t sdf) {
  Grid g;
  g.cells = sdf->grid;
  g.nx = sdf->dims[0];
  g.ny = sdf->dims[1];
  g.nz = sdf->dims[2];
  g.ox = sdf->origin[0];
  g.oy = sdf->origin[1];
  g.oz = sdf->origin[2];
  g.spacing = sdf->spacing;
  return g;
}

int check_params(const tacsl_penalty_t& p) {
  if (p.k_n < 0 || p.k_d < 0 || p.k_t < 0 || p.mu < 0)
    return set_error(TACSL_ERR_INVALID_ARGUMENT, "penalty parameters must be non-negative");
  return TACSL_OK;
}

unsigned elementwise_blocks(int64_t n) {
  int64_t b = (n + 255) / 256;
  return (unsigned)std::max<int64_t>(1, std::min<int64_t>(b, (int64_t)sm_count(current_device()) * 16));
}

}  // namespace
}  // namespace tacsl

using namespace tacsl;

extern "C" {

int tacsl_query_sdf(tacsl_sdf_t sdf, const double* points, int64_t n, double* distance, double* normal,
                    uint8_t* valid, void* stream) {
  if (!sdf) return set_error(TACSL_ERR_INVALID_ARGUMENT, "query_sdf: null SDF");
  if (n < 0) return set_error(TACSL_ERR_INVALID_ARGUMENT, "query_sdf: negative count");
  if (n == 0) return TACSL_OK;
  if (!points) return set_error(TACSL_ERR_INVALID_ARGUMENT, "query_sdf: null points");
  query_sdf_kernel<<<elementwise_blocks(n), 256, 0, (cudaStream_t)stream>>>(make_grid(sdf), points, n, distance,
                                                                             normal, valid);
  return check_launch("query_sdf_kernel");
}

int tacsl_penalty_forces(const double* d, const double* d_dot, const double* n, const double* v_t, int64_t count,
                         tacsl_penalty_t params, double* f_n, double* f_t, void* stream) {
  int rc = check_params(params);
  if (rc) return rc;
  if (count < 0) return set_error(TACSL_ERR_INVALID_ARGUMENT, "penalty_forces: negative count");
  if (count == 0) return TACSL_OK;
  if (!d || !d_dot || !n || !v_t || !f_n || !f_t)
    return set_error(TACSL_ERR_INVALID_ARGUMENT, "penalty_forces: null pointer");
  Penalty P{params.k_n, params.k_d, params.k_t, params.mu};
  penalty_kernel<<<elementwise_blocks(count), 256, 0, (cudaStream_t)stream>>>(d, d_dot, n, v_t, count, P, f_n, f_t);
  return check_launch("penalty_kernel");
}

int tacsl_force_field(tacsl_sdf_t sdf, const double* taxels, int rows, int cols, const double* object_state,
                      int64_t object_stride, const double* sensor_state, int64_t sensor_stride, int64_t n_envs,
                      int n_sensors, tacsl_penalty_t params, int out_fp64, void* f_n, void* f_t, double* wrench,
                      double* kin, uint8_t* contact, void* stream) {
  if (!sdf) return set_error(TACSL_ERR_INVALID_ARGUMENT, "force_field: null SDF");
  int rc = check_params(params);
  if (rc) return rc;
  if (rows <= 0 || cols <= 0 || n_sensors <= 0 || n_envs < 0)
    return set_error(TACSL_ERR_INVALID_ARGUMENT, "force_field: bad sizes");
  if (object_stride < 0 || sensor_stride < 0)
    return set_error(TACSL_ERR_INVALID_ARGUMENT, "force_field: negative stride");
  const int64_t frames = n_envs * n_sensors;
  if (frames == 0) return TACSL_OK;
  if (frames > 0x7fffffffLL) return set_error(TACSL_ERR_INVALID_ARGUMENT, "force_field: too many frames");
  if (!taxels || !object_state || !sensor_state || !f_n || !f_t)
    return set_error(TACSL_ERR_INVALID_ARGUMENT, "force_field: null pointer");
  const int n_taxels = rows * cols;
  const int threads = n_taxels <= 1024 ? 128 : 256;
  Penalty P{params.k_n, params.k_d, params.k_t, params.mu};
  cudaStream_t s = (cudaStream_t)stream;
  if (out_fp64) {
    force_field_kernel<double><<<(unsigned)frames, threads, 0, s>>>(
        make_grid(sdf), taxels, n_taxels, object_state, object_stride, sensor_state, sensor_stride, n_sensors, P,
        (double*)f_n, (double*)f_t, wrench, kin, contact);
  } else {
    force_field_kernel<float><<<(unsigned)frames, threads, 0, s>>>(
        make_grid(sdf), taxels, n_taxels, object_state, object_stride, sensor_state, sensor_stride, n_sensors, P,
        (float*)f_n, (float*)f_t, wrench, kin, contact);
  }
  return check_launch("force_field_kernel");
}

int tacsl_net_wrench(const double* f_n, const double* f_t, const double* points, int64_t frames, int rows, int cols,
                     double* force, double* torque, void* stream) {
  if (frames < 0 || rows <= 0 || cols <= 0) return set_error(TACSL_ERR_INVALID_ARGUMENT, "net_wrench: bad sizes");
  if (frames == 0) return TACSL_OK;
  if (!f_n || !f_t || !points || !force || !torque)
    return set_error(TACSL_ERR_INVALID_ARGUMENT, "net_wrench: null pointer");
  if (frames > 0x7fffffffLL) return set_error(TACSL_ERR_INVALID_ARGUMENT, "net_wrench: too many frames");
  net_wrench_kernel<<<(unsigned)frames, 256, 0, (cudaStream_t)stream>>>(f_n, f_t, points, rows * cols, force,
                                                                         torque);
  return check_launch("net_wrench_kernel");
}

}  // extern "C"
