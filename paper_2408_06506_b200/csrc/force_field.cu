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
// one 256-bit load per trilinear corner) that stays L2-resident (2 MiB for
// the 32x32x64 peg, 64 MiB at 128^3).  Out of contact both forces are exactly
// zero, so only contact taxels pay for the normal, velocities and penalty law.
#include <algorithm>
#include <cstdlib>

#include "common.cuh"
#include "handles.h"

namespace tacsl {
namespace {

constexpr int kFFMinBlocks = 4;  // resident CTAs per SM the register budget targets

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
  const double4* __restrict__ cells;  // {d, gx, gy, gz} per cell, z fastest
  int nx, ny, nz;
  double ox, oy, oz, spacing, inv_spacing;
};

// 256-bit read-only load (LDG.E.ENL2.256 on sm_100): one trilinear corner
__device__ __forceinline__ double4 ldg256(const double4* p) {
  double4 v;
  asm("ld.global.nc.v4.f64 {%0, %1, %2, %3}, [%4];" : "=d"(v.x), "=d"(v.y), "=d"(v.z), "=d"(v.w) : "l"(p));
  return v;
}

// Cell location and trilinear weights of a query point (sdf.py:280-290)
struct Cell {
  size_t base;
  double wx, wy, wz, ux, uy, uz;
  bool valid;
};

// Correctly rounded a / spacing in three DP operations: with y = RN(1/b)
// (within half an ulp) and q = RN(a*y) (within one ulp), q + RN-corrected
// by the exact FMA remainder is the correctly rounded quotient (Markstein's
// theorem) -- bit-identical to numpy's true division, without __ddiv_rn's
// reciprocal iteration.
__device__ __forceinline__ double div_spacing(double a, const Grid& g) {
  const double q = mul_rn(a, g.inv_spacing);
  const double r = __fma_rn(-q, g.spacing, a);
  return __fma_rn(r, g.inv_spacing, q);
}

__device__ __forceinline__ Cell locate(const Grid& g, V3 p) {
  const double rx = div_spacing(sub_rn(p.x, g.ox), g);
  const double ry = div_spacing(sub_rn(p.y, g.oy), g);
  const double rz = div_spacing(sub_rn(p.z, g.oz), g);
  const double mx = (double)(g.nx - 1), my = (double)(g.ny - 1), mz = (double)(g.nz - 1);
  Cell c;
  c.valid = (rx >= 0.0) & (rx <= mx) & (ry >= 0.0) & (ry <= my) & (rz >= 0.0) & (rz <= mz);
  // clip(rel, 0, dims - 1 - 1e-9); i0 = min(int(rel_c), dims - 2); f = rel_c - i0
  const double cx = fmin(fmax(rx, 0.0), sub_rn(mx, 1e-9));
  const double cy = fmin(fmax(ry, 0.0), sub_rn(my, 1e-9));
  const double cz = fmin(fmax(rz, 0.0), sub_rn(mz, 1e-9));
  const int ix = min((int)cx, g.nx - 2), iy = min((int)cy, g.ny - 2), iz = min((int)cz, g.nz - 2);
  c.wx = sub_rn(cx, (double)ix);
  c.wy = sub_rn(cy, (double)iy);
  c.wz = sub_rn(cz, (double)iz);
  c.ux = sub_rn(1.0, c.wx);
  c.uy = sub_rn(1.0, c.wy);
  c.uz = sub_rn(1.0, c.wz);
  c.base = ((size_t)ix * g.ny + iy) * g.nz + iz;
  return c;
}

// corner k = 4*dx + 2*dy + dz
__device__ __forceinline__ size_t corner(const Grid& g, const Cell& c, int k) {
  return c.base + (size_t)((k >> 2) & 1) * g.ny * g.nz + (size_t)((k >> 1) & 1) * g.nz + (k & 1);
}

// Trilinear distance, x then y then z lerps with every product and sum
// rounded separately, as numpy evaluates sdf.py:305-311 -- bit-exact.
__device__ __forceinline__ double interp_d(const Grid& g, const Cell& c) {
  double v[8];
#pragma unroll
  for (int k = 0; k < 8; ++k) v[k] = __ldg(&g.cells[corner(g, c, k)].x);
  const double d00 = add_rn(mul_rn(v[0], c.ux), mul_rn(v[4], c.wx));
  const double d10 = add_rn(mul_rn(v[2], c.ux), mul_rn(v[6], c.wx));
  const double d01 = add_rn(mul_rn(v[1], c.ux), mul_rn(v[5], c.wx));
  const double d11 = add_rn(mul_rn(v[3], c.ux), mul_rn(v[7], c.wx));
  const double d0 = add_rn(mul_rn(d00, c.uy), mul_rn(d10, c.wy));
  const double d1 = add_rn(mul_rn(d01, c.uy), mul_rn(d11, c.wy));
  return add_rn(mul_rn(d0, c.uz), mul_rn(d1, c.wz));
}

// Trilinear gradient, renormalised: n = g / max(|g|, 1e-12) (sdf.py:314-316)
__device__ __forceinline__ V3 interp_n(const Grid& g, const Cell& c) {
  double gx = 0.0, gy = 0.0, gz = 0.0;
  double ax[2], ay[2], az[2];
#pragma unroll
  for (int dz = 0; dz < 2; ++dz) {
    double bx[2], by[2], bz[2];
#pragma unroll
    for (int dy = 0; dy < 2; ++dy) {
      const double4 lo = ldg256(g.cells + corner(g, c, 2 * dy + dz));
      const double4 hi = ldg256(g.cells + corner(g, c, 4 + 2 * dy + dz));
      bx[dy] = lo.y * c.ux + hi.y * c.wx;
      by[dy] = lo.z * c.ux + hi.z * c.wx;
      bz[dy] = lo.w * c.ux + hi.w * c.wx;
    }
    ax[dz] = bx[0] * c.uy + bx[1] * c.wy;
    ay[dz] = by[0] * c.uy + by[1] * c.wy;
    az[dz] = bz[0] * c.uy + bz[1] * c.wy;
  }
  gx = ax[0] * c.uz + ax[1] * c.wz;
  gy = ay[0] * c.uz + ay[1] * c.wz;
  gz = az[0] * c.uz + az[1] * c.wz;
  const double inv = rsqrt(fmax(gx * gx + gy * gy + gz * gz, 1e-24));
  return v3(gx * inv, gy * inv, gz * inv);
}

struct Query {
  double d;  // +inf when outside
  V3 n;      // 0 when outside
  bool valid;
};

// geometry/sdf.py:271-321
__device__ __forceinline__ Query query(const Grid& g, V3 p) {
  const Cell c = locate(g, p);
  Query q;
  q.valid = c.valid;
  if (c.valid) {
    q.d = interp_d(g, c);
    q.n = interp_n(g, c);
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
  const double ss = vt.x * vt.x + vt.y * vt.y + vt.z * vt.z;
  const double inv = rsqrt(ss);
  const double speed = ss > 0.0 ? ss * inv : 0.0;
  const bool slipping = contact && (speed > 1e-9);  // SLIP_VELOCITY_EPS, field.py:25
  const double mag = fmin(P.k_t * speed, P.mu * coeff);
  const double scale = slipping ? mag * inv : 0.0;
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

template <typename OutT, int MINB>
__global__ void __launch_bounds__(128, MINB) force_field_kernel(
    const Grid grid, const double* __restrict__ taxels, int n_taxels, const double* __restrict__ obj_state,
    int64_t obj_stride, const double* __restrict__ sen_state, int64_t sen_stride, int n_sensors, const Penalty P,
    OutT* __restrict__ f_n_out, OutT* __restrict__ f_t_out, double* __restrict__ wrench, double* __restrict__ kin,
    uint8_t* __restrict__ contact_out, float* __restrict__ obs_out) {
  const int64_t frame = blockIdx.x;
  const int64_t e = frame / n_sensors;
  const int s = (int)(frame - e * n_sensors);
  const State O = load_state(obj_state + e * obj_stride);
  const State S = load_state(sen_state + e * sen_stride + (int64_t)s * 13);
  const V3 oq_inv = v3(-O.qv.x, -O.qv.y, -O.qv.z);
  const V3 sq_inv = v3(-S.qv.x, -S.qv.y, -S.qv.z);
  const bool want_kin = kin != nullptr;

  double acc[6] = {0, 0, 0, 0, 0, 0};
  const int64_t out_base = frame * (int64_t)n_taxels;
  for (int i = threadIdx.x; i < n_taxels; i += blockDim.x) {
    const V3 p = v3(__ldg(taxels + 3 * i), __ldg(taxels + 3 * i + 1), __ldg(taxels + 3 * i + 2));
    // ---- mask chain, numpy order (field.py:104-107) ----
    V3 pw = quat_rotate_rn(S.qw, S.qv, p);
    pw = v3(add_rn(pw.x, S.pos.x), add_rn(pw.y, S.pos.y), add_rn(pw.z, S.pos.z));
    const V3 ro = v3(sub_rn(pw.x, O.pos.x), sub_rn(pw.y, O.pos.y), sub_rn(pw.z, O.pos.z));
    const V3 po = quat_rotate_rn(O.qw, oq_inv, ro);
    const Cell cell = locate(grid, po);
    const double d = cell.valid ? interp_d(grid, cell) : __longlong_as_double(0x7ff0000000000000LL);
    const bool contact = d < 0.0;  // field.py:64
    V3 fn = v3(0.0, 0.0, 0.0), ft = v3(0.0, 0.0, 0.0);
    // Out of contact both forces are exactly zero (field.py:65-75), so the
    // normal, the velocities and the penalty law run only for contact
    // taxels -- unless the caller asked for the kinematics of every taxel.
    if (contact || want_kin) {
      const V3 n = cell.valid ? interp_n(grid, cell) : v3(0.0, 0.0, 0.0);
      // ---- kinematics (field.py:109-115) ----
      const V3 nw = quat_rotate(O.qw, O.qv, n);
      const V3 rs = v3(pw.x - S.pos.x, pw.y - S.pos.y, pw.z - S.pos.z);
      const V3 cs = cross(S.w, rs), co = cross(O.w, ro);
      const V3 xd = v3((S.v.x + cs.x) - (O.v.x + co.x), (S.v.y + cs.y) - (O.v.y + co.y),
                       (S.v.z + cs.z) - (O.v.z + co.z));
      const double d_dot = dot(nw, xd);
      const V3 vt = v3(xd.x - d_dot * nw.x, xd.y - d_dot * nw.y, xd.z - d_dot * nw.z);
      if (contact) {
        V3 fnw, ftw;
        bool c2;
        penalty(P, d, d_dot, nw, vt, fnw, ftw, c2);
        // ---- back to the sensor frame (field.py:118-119) ----
        fn = quat_rotate(S.qw, sq_inv, fnw);
        ft = quat_rotate(S.qw, sq_inv, ftw);
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
      if (want_kin) {
        double* k = kin + (out_base + i) * 8;
        k[0] = d;
        k[1] = d_dot;
        k[2] = vt.x;
        k[3] = vt.y;
        k[4] = vt.z;
        k[5] = nw.x;
        k[6] = nw.y;
        k[7] = nw.z;
      }
    }
    const int64_t o = (out_base + i) * 3;
    if (f_n_out) {
      f_n_out[o + 0] = (OutT)fn.x;
      f_n_out[o + 1] = (OutT)fn.y;
      f_n_out[o + 2] = (OutT)fn.z;
    }
    if (f_t_out) {
      f_t_out[o + 0] = (OutT)ft.x;
      f_t_out[o + 1] = (OutT)ft.y;
      f_t_out[o + 2] = (OutT)ft.z;
    }
    if (obs_out) {  // policy observation [f_n.z, f_t.x, f_t.y] (envs/peg_tasks.py:474-476)
      obs_out[o + 0] = (float)fn.z;
      obs_out[o + 1] = (float)ft.x;
      obs_out[o + 2] = (float)ft.y;
    }
    if (contact_out) contact_out[out_base + i] = contact ? 1 : 0;
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
  g.inv_spacing = 1.0 / sdf->spacing;  // correctly rounded (IEEE division on the host)
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
                      double* kin, uint8_t* contact, float* obs, void* stream) {
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
  if (!taxels || !object_state || !sensor_state)
    return set_error(TACSL_ERR_INVALID_ARGUMENT, "force_field: null pointer");
  if (!f_n && !f_t && !wrench && !kin && !contact && !obs)
    return set_error(TACSL_ERR_INVALID_ARGUMENT, "force_field: no output buffer");
  const int n_taxels = rows * cols;
  const int threads = 128;
  Penalty P{params.k_n, params.k_d, params.k_t, params.mu};
  cudaStream_t s = (cudaStream_t)stream;
  const char* mb = std::getenv("TACSL_FF_MINBLOCKS");
  const int minb = mb ? std::atoi(mb) : kFFMinBlocks;
  auto launch = [&](auto* fn_tag, auto out_tag) {
    using O = decltype(out_tag);
    (void)fn_tag;
    auto go = [&](auto kern) {
      kern<<<(unsigned)frames, threads, 0, s>>>(make_grid(sdf), taxels, n_taxels, object_state, object_stride,
                                              sensor_state, sensor_stride, n_sensors, P, (O*)f_n, (O*)f_t, wrench,
                                              kin, contact, obs);
    };
    if (minb >= 6) go(force_field_kernel<O, 6>);
    else if (minb == 5) go(force_field_kernel<O, 5>);
    else go(force_field_kernel<O, 4>);
  };
  if (out_fp64) launch((int*)nullptr, double{});
  else launch((int*)nullptr, float{});
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
