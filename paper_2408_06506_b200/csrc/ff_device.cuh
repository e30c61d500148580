// Device building blocks of K2 (penalty force field), shared by the
// standalone force-field kernel (force_field.cu) and the fused sensor-step
// kernel (rgb.cu).  See force_field.cu for the reference mapping.
#pragma once

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
  const double4* __restrict__ cells;  // {d, gx, gy, gz} per cell, z fastest
  const double* __restrict__ values;  // d only, compact (8 B per cell): the mask path's gathers
  int nx, ny, nz;
  double ox, oy, oz, spacing, inv_spacing;
  const float4* __restrict__ quads;  // fp32 corner quads (handles.h), or null
  float lsum;                        // sum of the per-axis Lipschitz bounds (m per cell)
};

// 256-bit read-only load (LDG.E.ENL2.256 on sm_100): one trilinear corner
__device__ __forceinline__ double4 ldg256(const double4* p) {
  double4 v;
  asm("ld.global.nc.v4.f64 {%0, %1, %2, %3}, [%4];" : "=d"(v.x), "=d"(v.y), "=d"(v.z), "=d"(v.w) : "l"(p));
  return v;
}

// Cell location and trilinear weights of a query point (sdf.py:280-290)
struct Cell {
  int base;  // first corner's cell index (grids are capped at 2^31 cells at upload)
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

__device__ __forceinline__ Cell locate_rel(const Grid& g, const double rx, const double ry, const double rz) {
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
  c.base = (ix * g.ny + iy) * g.nz + iz;
  return c;
}

__device__ __forceinline__ Cell locate(const Grid& g, V3 p) {
  return locate_rel(g, div_spacing(sub_rn(p.x, g.ox), g), div_spacing(sub_rn(p.y, g.oy), g),
                    div_spacing(sub_rn(p.z, g.oz), g));
}

// corner k = 4*dx + 2*dy + dz
__device__ __forceinline__ int corner(const Grid& g, const Cell& c, int k) {
  return c.base + ((k >> 2) & 1) * g.ny * g.nz + ((k >> 1) & 1) * g.nz + (k & 1);
}

// Trilinear distance, x then y then z lerps with every product and sum
// rounded separately, as numpy evaluates sdf.py:305-311 -- bit-exact.
__device__ __forceinline__ double interp_d(const Grid& g, const Cell& c) {
  double v[8];
#pragma unroll
  for (int k = 0; k < 8; ++k) v[k] = __ldg(g.values + corner(g, c, k));
  const double d00 = add_rn(mul_rn(v[0], c.ux), mul_rn(v[4], c.wx));
  const double d10 = add_rn(mul_rn(v[2], c.ux), mul_rn(v[6], c.wx));
  const double d01 = add_rn(mul_rn(v[1], c.ux), mul_rn(v[5], c.wx));
  const double d11 = add_rn(mul_rn(v[3], c.ux), mul_rn(v[7], c.wx));
  const double d0 = add_rn(mul_rn(d00, c.uy), mul_rn(d10, c.wy));
  const double d1 = add_rn(mul_rn(d01, c.uy), mul_rn(d11, c.wy));
  return add_rn(mul_rn(d0, c.uz), mul_rn(d1, c.wz));
}

// Trilinear gradient, renormalised: n = g / max(|g|, 1e-12) (sdf.py:314-316).
// With d_out, also the distance from the same corner loads, in
// interp_d_fast's lerp form (bit-identical to it: the cells' d is values).
// The eight {d, gx, gy, gz} corners of a cell, corner k = 4 dx + 2 dy + dz.
__device__ __forceinline__ void load_corners(const Grid& g, int base, double4 cv[8]) {
  const int sy = g.nz, sx = g.ny * g.nz;
#pragma unroll
  for (int k = 0; k < 8; ++k) cv[k] = ldg256(g.cells + base + ((k >> 2) & 1) * sx + ((k >> 1) & 1) * sy + (k & 1));
}

// interp_n on corners already loaded (load_corners); see interp_n
__device__ __forceinline__ V3 interp_n_from(const double4 cv[8], const Cell& c, double* d_out) {
  double gx = 0.0, gy = 0.0, gz = 0.0;
  double ax[2], ay[2], az[2], ad[2];
#pragma unroll
  for (int dz = 0; dz < 2; ++dz) {
    double bx[2], by[2], bz[2], bd[2];
#pragma unroll
    for (int dy = 0; dy < 2; ++dy) {
      const double4 lo = cv[2 * dy + dz];
      const double4 hi = cv[4 + 2 * dy + dz];
      bd[dy] = fma(c.wx, hi.x - lo.x, lo.x);
      bx[dy] = lo.y * c.ux + hi.y * c.wx;
      by[dy] = lo.z * c.ux + hi.z * c.wx;
      bz[dy] = lo.w * c.ux + hi.w * c.wx;
    }
    ad[dz] = fma(c.wy, bd[1] - bd[0], bd[0]);
    ax[dz] = bx[0] * c.uy + bx[1] * c.wy;
    ay[dz] = by[0] * c.uy + by[1] * c.wy;
    az[dz] = bz[0] * c.uy + bz[1] * c.wy;
  }
  if (d_out) *d_out = fma(c.wz, ad[1] - ad[0], ad[0]);
  gx = ax[0] * c.uz + ax[1] * c.wz;
  gy = ay[0] * c.uz + ay[1] * c.wz;
  gz = az[0] * c.uz + az[1] * c.wz;
  const double inv = rsqrt(fmax(gx * gx + gy * gy + gz * gz, 1e-24));
  return v3(gx * inv, gy * inv, gz * inv);
}

__device__ __forceinline__ V3 interp_n(const Grid& g, const Cell& c, double* d_out = nullptr) {
  double4 cv[8];
  load_corners(g, c.base, cv);
  return interp_n_from(cv, c, d_out);
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

// Everything one force-field launch needs (kernel parameter).
template <typename OutT>
struct FFArgs {
  Grid grid;
  const double* __restrict__ taxels;
  int n_taxels;
  const double* __restrict__ obj_state;
  int64_t obj_stride;
  const double* __restrict__ sen_state;
  int64_t sen_stride;
  int n_sensors;
  int64_t frames;
  Penalty P;
  OutT* __restrict__ f_n;
  OutT* __restrict__ f_t;
  double* __restrict__ wrench;
  double* __restrict__ kin;
  uint8_t* __restrict__ contact;
  float* __restrict__ obs;
  unsigned long long* counter;  // dynamic frame dispatch (fused step), zeroed before the launch
  const float4* __restrict__ taxf;  // taxels as {x, y, z, |x|+|y|+|z|} fp32 (force_field_quad_kernel)
};

// Taxels first, first+stride, ... of one sensor frame (tactile/field.py:
// 79-129); the wrench contributions (field.py:132-141) accumulate in acc.
template <typename OutT>
__device__ __forceinline__ void ff_frame(const FFArgs<OutT>& A, int64_t frame, int first, int stride,
                                         double acc[6]) {
  const int64_t e = frame / A.n_sensors;
  const int s = (int)(frame - e * A.n_sensors);
  const State O = load_state(A.obj_state + e * A.obj_stride);
  const State S = load_state(A.sen_state + e * A.sen_stride + (int64_t)s * 13);
  const V3 oq_inv = v3(-O.qv.x, -O.qv.y, -O.qv.z);
  const V3 sq_inv = v3(-S.qv.x, -S.qv.y, -S.qv.z);
  const bool want_kin = A.kin != nullptr;
  const int64_t out_base = frame * (int64_t)A.n_taxels;
  const Grid& grid = A.grid;
  for (int i = first; i < A.n_taxels; i += stride) {
    const double* tp = A.taxels + 3 * i;
    const V3 p = v3(__ldg(tp), __ldg(tp + 1), __ldg(tp + 2));
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
        penalty(A.P, d, d_dot, nw, vt, fnw, ftw, c2);
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
        double* k = A.kin + (out_base + i) * 8;
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
    if (A.f_n) {
      A.f_n[o + 0] = (OutT)fn.x;
      A.f_n[o + 1] = (OutT)fn.y;
      A.f_n[o + 2] = (OutT)fn.z;
    }
    if (A.f_t) {
      A.f_t[o + 0] = (OutT)ft.x;
      A.f_t[o + 1] = (OutT)ft.y;
      A.f_t[o + 2] = (OutT)ft.z;
    }
    if (A.obs) {  // policy observation [f_n.z, f_t.x, f_t.y] (envs/peg_tasks.py:474-476)
      A.obs[o + 0] = (float)fn.z;
      A.obs[o + 1] = (float)ft.x;
      A.obs[o + 2] = (float)ft.y;
    }
    if (A.contact) A.contact[out_base + i] = contact ? 1 : 0;
  }
}

// One warp computes whole frames (lane-strided taxels, shuffle-reduced
// wrench): no CTA barrier, so these warps can run beside other work.
template <typename OutT>
__device__ __forceinline__ void ff_frames_warp(const FFArgs<OutT>& A, int64_t first_frame, int64_t frame_stride,
                                               int lane) {
  for (int64_t f = first_frame; f < A.frames; f += frame_stride) {
    double acc[6] = {0, 0, 0, 0, 0, 0};
    ff_frame(A, f, lane, 32, acc);
#pragma unroll
    for (int k = 0; k < 6; ++k) acc[k] = warp_sum(acc[k]);
    if (A.wrench && lane == 0)
#pragma unroll
      for (int k = 0; k < 6; ++k) A.wrench[f * 6 + k] = acc[k];
  }
}

// Frames handed out one at a time through a global counter, so every warp
// that runs out of other work (force-field warps from the start, shading
// warps after their last band) helps finish the force field.
template <typename OutT>
__device__ __forceinline__ void ff_frames_dynamic(const FFArgs<OutT>& A, int lane) {
  while (true) {
    unsigned long long f = 0;
    if (lane == 0) f = atomicAdd(A.counter, 1ull);
    f = __shfl_sync(0xffffffffu, f, 0);
    if ((int64_t)f >= A.frames) break;
    double acc[6] = {0, 0, 0, 0, 0, 0};
    ff_frame(A, (int64_t)f, lane, 32, acc);
#pragma unroll
    for (int k = 0; k < 6; ++k) acc[k] = warp_sum(acc[k]);
    if (A.wrench && lane == 0)
#pragma unroll
      for (int k = 0; k < 6; ++k) A.wrench[(int64_t)f * 6 + k] = acc[k];
  }
}

// ---------------------------------------------------------------------------
// Fast mask chain with an exact fallback (force_field_fast_kernel).
//
// The reference's per-taxel chain p_o = R_o^T (R_s p + s_pos - o_pos),
// rel = (p_o - origin) / h is affine in p, so per frame it folds into
// rel = A p + b (9 FMAs instead of two separately-rounded quaternion
// rotations and a division).  quat_rotate's v + w t + q x t (t = 2 q x v)
// is, as a linear map, exactly the matrix below -- for any quaternion, not
// only unit ones -- so A and b differ from the reference chain only by
// rounding: |rel_fast - rel_exact| stays below ~1e-9 cells and
// |d_fast - d_exact| below ~1e-12 m for positions up to 1 km.  Every decision
// the reference makes on those values is taken from the fast values only
// when they clear it by a wide margin (kCellMargin cells from the grid
// bounds, kDistMargin metres from d = 0); the rare remaining taxels replay
// the exact chain (exact_rel), so the validity flags and the contact mask
// stay bit-exact, and forces (|d| >= 1e-6 m) are within 1e-6 relative.
constexpr double kCellMargin = 1e-6;
constexpr double kDistMargin = 1e-6;

struct FrameC {
  double A[9], b[3];   // rel = A p + b
  double Ms[9], sp[3];  // p_w = Ms p + sp (sensor pose)
  double Mo[9], op[3];  // n_w = Mo n; object position
  double sv[3], sw[3], ov[3], ow[3];
  // fp32 pre-pass (force_field_quad_kernel): rel ~ A32 p + b32, and the
  // per-frame constants of its certified error bounds
  float A32[9], b32[3];
  float amax, bmax;  // max |A_ik|, max |b_i| (rounded up)
  float kt, k0;      // decision bound 2 tau / (1 - 16u) = kt * (amax |p|_1 + bmax) + k0
  // contact path in the sensor frame (unit quaternions): n_s = Mso n,
  // x_dot_s = kv + om x p  (Mso = Ms^T Mo, kv = Ms^T (s_v - o_v) - w_o,s x c_s,
  // om = Ms^T (s_w - o_w), c_s = Ms^T (s_pos - o_pos))
  double Mso[9], kv[3], om[3];
  int unit;  // both quaternions unit to 1e-12 (else the world-frame path)
};

// row-major matrix of quat_rotate(q, .) (transforms.py:36-41)
__device__ __forceinline__ void quat_matrix(double w, V3 q, double* M) {
  const double xx = q.x * q.x, yy = q.y * q.y, zz = q.z * q.z;
  const double xy = q.x * q.y, xz = q.x * q.z, yz = q.y * q.z;
  const double wx = w * q.x, wy = w * q.y, wz = w * q.z;
  M[0] = 1.0 - 2.0 * (yy + zz);
  M[1] = 2.0 * (xy - wz);
  M[2] = 2.0 * (xz + wy);
  M[3] = 2.0 * (xy + wz);
  M[4] = 1.0 - 2.0 * (xx + zz);
  M[5] = 2.0 * (yz - wx);
  M[6] = 2.0 * (xz - wy);
  M[7] = 2.0 * (yz + wx);
  M[8] = 1.0 - 2.0 * (xx + yy);
}

// The quad kernel's extra per-frame constants (force_field.cu): the fp32
// fold, the bounds of its certified error (max |A|, max |b|) and the
// sensor-frame contact path's Ms^T Mo, kv, om.  val = this lane's A / b entry.
template <typename OutT>
__device__ __forceinline__ void frame_setup_quad(const FFArgs<OutT>& A, FrameC& C, int lane, double val,
                                                 const State& S, const State& O, const double* Ms,
                                                 const double* Mo) {
  const Grid& g = A.grid;
  // max |A|, max |b|
  // (NaN poses propagate: fmax drops NaN, so test them explicitly)
  double am = lane < 9 ? fabs(val) : 0.0, bm = (lane >= 9 && lane < 12) ? fabs(val) : 0.0;
  bool bad = val != val;
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) {
    am = fmax(am, __shfl_xor_sync(0xffffffffu, am, o));
    bm = fmax(bm, __shfl_xor_sync(0xffffffffu, bm, o));
  }
  bad = __any_sync(0xffffffffu, bad);
  if (lane == 15) {
    const float inf = __int_as_float(0x7f800000);
    C.amax = bad ? inf : __double2float_ru(am);
    C.bmax = bad ? inf : __double2float_ru(bm);
    constexpr float u = 5.9604645e-8f;  // 2^-24
    // tau scaled by 2 / (1 - 16u) (>= 2.0000019; the quad kernel's test is
    // |d32| > tau, see force_field.cu)
    constexpr float s2 = 2.0000024f;
    C.kt = __fmul_ru(__fmul_ru(8.0f * u, g.lsum), s2);
    C.k0 = __fmul_ru(__fmul_ru(g.lsum, 1e-7f + 8.0f * u), s2);
  }
  if (lane == 16) {
#pragma unroll
    for (int i = 0; i < 3; ++i)
#pragma unroll
      for (int j = 0; j < 3; ++j) C.Mso[3 * i + j] = Ms[i] * Mo[j] + Ms[3 + i] * Mo[3 + j] + Ms[6 + i] * Mo[6 + j];
    const double qs = S.qw * S.qw + S.qv.x * S.qv.x + S.qv.y * S.qv.y + S.qv.z * S.qv.z;
    const double qo = O.qw * O.qw + O.qv.x * O.qv.x + O.qv.y * O.qv.y + O.qv.z * O.qv.z;
    C.unit = fabs(qs - 1.0) < 1e-12 && fabs(qo - 1.0) < 1e-12;
  } else if (lane == 17) {
    // Ms^T a for a world vector a
    auto to_s = [&](V3 a) {
      return v3(Ms[0] * a.x + Ms[3] * a.y + Ms[6] * a.z, Ms[1] * a.x + Ms[4] * a.y + Ms[7] * a.z,
                Ms[2] * a.x + Ms[5] * a.y + Ms[8] * a.z);
    };
    const V3 vs = to_s(v3(S.v.x - O.v.x, S.v.y - O.v.y, S.v.z - O.v.z));
    const V3 ws = to_s(S.w), wo = to_s(O.w);
    const V3 cs = to_s(v3(S.pos.x - O.pos.x, S.pos.y - O.pos.y, S.pos.z - O.pos.z));
    const V3 wc = cross(wo, cs);
    C.kv[0] = vs.x - wc.x, C.kv[1] = vs.y - wc.y, C.kv[2] = vs.z - wc.z;
    C.om[0] = ws.x - wo.x, C.om[1] = ws.y - wo.y, C.om[2] = ws.z - wo.z;
  }
}

// Per-frame constants, built by one warp: every lane forms both rotation
// matrices (a few dozen flops on broadcast loads) and writes its share of
// the 48 entries (A, b on lanes 0-11), so the CTA waits for one short
// dependency chain only.
template <bool QUAD = false, typename OutT>
__device__ __forceinline__ void frame_setup_warp(const FFArgs<OutT>& A, int64_t frame, FrameC& C, int lane) {
  const int64_t e = frame / A.n_sensors;
  const int s = (int)(frame - e * A.n_sensors);
  const State O = load_state(A.obj_state + e * A.obj_stride);
  const State S = load_state(A.sen_state + e * A.sen_stride + (int64_t)s * 13);
  double Ms[9], Mo[9];
  quat_matrix(S.qw, S.qv, Ms);
  quat_matrix(O.qw, O.qv, Mo);
  const Grid& g = A.grid;
  double val = 0.0;
  if (lane < 9) {  // A = (Mo^T Ms) / h
    const int i = lane / 3, j = lane % 3;
    val = (Mo[i] * Ms[j] + Mo[3 + i] * Ms[3 + j] + Mo[6 + i] * Ms[6 + j]) * g.inv_spacing;
    C.A[lane] = val;
    if (QUAD) C.A32[lane] = (float)val;
  } else if (lane < 12) {  // b = (Mo^T (s_pos - o_pos) - origin) / h
    const int i = lane - 9;
    const double org = i == 0 ? g.ox : (i == 1 ? g.oy : g.oz);
    val = ((Mo[i] * (S.pos.x - O.pos.x) + Mo[3 + i] * (S.pos.y - O.pos.y) + Mo[6 + i] * (S.pos.z - O.pos.z)) -
           org) * g.inv_spacing;
    C.b[i] = val;
    if (QUAD) C.b32[i] = (float)val;
  }
  if (QUAD) frame_setup_quad(A, C, lane, val, S, O, Ms, Mo);
  if (lane == 12) {
#pragma unroll
    for (int k = 0; k < 9; ++k) C.Ms[k] = Ms[k];
    C.sp[0] = S.pos.x, C.sp[1] = S.pos.y, C.sp[2] = S.pos.z;
  } else if (lane == 13) {
#pragma unroll
    for (int k = 0; k < 9; ++k) C.Mo[k] = Mo[k];
    C.op[0] = O.pos.x, C.op[1] = O.pos.y, C.op[2] = O.pos.z;
  } else if (lane == 14) {
    C.sv[0] = S.v.x, C.sv[1] = S.v.y, C.sv[2] = S.v.z;
    C.sw[0] = S.w.x, C.sw[1] = S.w.y, C.sw[2] = S.w.z;
    C.ov[0] = O.v.x, C.ov[1] = O.v.y, C.ov[2] = O.v.z;
    C.ow[0] = O.w.x, C.ow[1] = O.w.y, C.ow[2] = O.w.z;
  }
}

// trilinear distance as lerps (fast path; the exact order is interp_d)
__device__ __forceinline__ double interp_d_fast(const Grid& g, const Cell& c) {
  double v[8];
#pragma unroll
  for (int k = 0; k < 8; ++k) v[k] = __ldg(g.values + corner(g, c, k));
  const double d00 = fma(c.wx, v[4] - v[0], v[0]);
  const double d10 = fma(c.wx, v[6] - v[2], v[2]);
  const double d01 = fma(c.wx, v[5] - v[1], v[1]);
  const double d11 = fma(c.wx, v[7] - v[3], v[3]);
  const double d0 = fma(c.wy, d10 - d00, d00);
  const double d1 = fma(c.wy, d11 - d01, d01);
  return fma(c.wz, d1 - d0, d0);
}

// The reference chain, operation for operation (field.py:104-108): exact
// cell coordinates for the taxels the fast values cannot decide.
__device__ __forceinline__ V3 exact_rel(const Grid& g, const double* __restrict__ obj,
                                        const double* __restrict__ sen, V3 p) {
  const State O = load_state(obj);
  const State S = load_state(sen);
  V3 pw = quat_rotate_rn(S.qw, S.qv, p);
  pw = v3(add_rn(pw.x, S.pos.x), add_rn(pw.y, S.pos.y), add_rn(pw.z, S.pos.z));
  const V3 ro = v3(sub_rn(pw.x, O.pos.x), sub_rn(pw.y, O.pos.y), sub_rn(pw.z, O.pos.z));
  const V3 po = quat_rotate_rn(O.qw, v3(-O.qv.x, -O.qv.y, -O.qv.z), ro);
  return v3(div_spacing(sub_rn(po.x, g.ox), g), div_spacing(sub_rn(po.y, g.oy), g),
            div_spacing(sub_rn(po.z, g.oz), g));
}

inline Grid make_grid(tacsl_sdf_t sdf) {
  Grid g;
  g.cells = sdf->grid;
  g.values = sdf->values;
  g.nx = sdf->dims[0];
  g.ny = sdf->dims[1];
  g.nz = sdf->dims[2];
  g.ox = sdf->origin[0];
  g.oy = sdf->origin[1];
  g.oz = sdf->origin[2];
  g.spacing = sdf->spacing;
  g.inv_spacing = 1.0 / sdf->spacing;  // correctly rounded (IEEE division on the host)
  g.quads = sdf->quads;
  g.lsum = sdf->lip[0] + sdf->lip[1] + sdf->lip[2];
  return g;
}

}  // namespace
}  // namespace tacsl
