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
#include <mutex>
#include <vector>

#include "common.cuh"
#include "ff_device.cuh"
#include "handles.h"

namespace tacsl {
namespace {

constexpr int kFFMinBlocks = 4;      // exact kernel: resident 128-thread CTAs per SM the register budget targets
constexpr int kFFFastMinBlocks = 5;  // fast kernel: 96 registers, no spills (4: 126 regs, 6: spills; measured)
constexpr int kQuadMinTaxels = 1024;  // taxels per frame above which the quad kernel runs
constexpr int kFFQuadMinBlocks = 4;  // quad kernel: 124 registers, no spills (5: 96 + spills, slower; measured)


template <typename OutT, int MINB>
__global__ void __launch_bounds__(128, MINB) force_field_kernel(const FFArgs<OutT> A) {
  // one CTA per sensor frame; threads stride over the taxels
  const int64_t frame = blockIdx.x;
  double acc[6] = {0, 0, 0, 0, 0, 0};
  ff_frame(A, frame, threadIdx.x, blockDim.x, acc);
  if (A.wrench) {
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
      A.wrench[frame * 6 + threadIdx.x] = t;
    }
  }
}

// ---- fast chain, per taxel (shared by the one-pass and two-pass kernels) ---
struct FastCtx {
  const Grid* g;
  const double* a;  // FrameC::A in shared memory
  const double* b;  // FrameC::b
  double mx, my, mz;
  const double* obj;
  const double* sen;
};

// Distance of taxel p (and its cell): fast affine cell map + lerps, the
// reference chain only when the fast values do not clear a decision.
__device__ __forceinline__ double decide_taxel(const FastCtx& X, double px, double py, double pz, Cell& cell) {
  const Grid& g = *X.g;
  const double* a = X.a;
  const double* b = X.b;
  const double rx = fma(a[0], px, fma(a[1], py, fma(a[2], pz, b[0])));
  const double ry = fma(a[3], px, fma(a[4], py, fma(a[5], pz, b[1])));
  const double rz = fma(a[6], px, fma(a[7], py, fma(a[8], pz, b[2])));
  const bool inside = (rx > kCellMargin) & (rx < X.mx - kCellMargin) & (ry > kCellMargin) &
                      (ry < X.my - kCellMargin) & (rz > kCellMargin) & (rz < X.mz - kCellMargin);
  const bool outside = (rx < -kCellMargin) | (rx > X.mx + kCellMargin) | (ry < -kCellMargin) |
                       (ry > X.my + kCellMargin) | (rz < -kCellMargin) | (rz > X.mz + kCellMargin);
  double d = __longlong_as_double(0x7ff0000000000000LL);  // +inf: outside the grid
  bool need_exact = !(inside | outside);
  if (inside) {
    const int ix = (int)rx, iy = (int)ry, iz = (int)rz;  // floor: rel > 0 and < dims-1
    cell.wx = rx - (double)ix;
    cell.wy = ry - (double)iy;
    cell.wz = rz - (double)iz;
    cell.ux = 1.0 - cell.wx;
    cell.uy = 1.0 - cell.wy;
    cell.uz = 1.0 - cell.wz;
    cell.base = (ix * g.ny + iy) * g.nz + iz;
    d = interp_d_fast(g, cell);
    need_exact = fabs(d) < kDistMargin;
  }
  if (need_exact) {  // rare: replay the reference chain for this taxel
    const V3 r = exact_rel(g, X.obj, X.sen, v3(px, py, pz));
    cell = locate_rel(g, r.x, r.y, r.z);
    d = cell.valid ? interp_d(g, cell) : __longlong_as_double(0x7ff0000000000000LL);
  }
  return d;
}

// contact path on the per-frame matrices (field.py:109-119); forces in the
// sensor frame
template <typename OutT>
__device__ __forceinline__ void contact_forces(const FFArgs<OutT>& A, const FrameC& C, const Grid& g,
                                               const Cell& cell, double d, double px, double py, double pz, V3& fn,
                                               V3& ft, bool d_from_cells = false, const double4* cv = nullptr) {
  const double* Ms = C.Ms;
  const double* Mo = C.Mo;
  const V3 rs = v3(fma(Ms[0], px, fma(Ms[1], py, Ms[2] * pz)), fma(Ms[3], px, fma(Ms[4], py, Ms[5] * pz)),
                   fma(Ms[6], px, fma(Ms[7], py, Ms[8] * pz)));
  const V3 pw = v3(rs.x + C.sp[0], rs.y + C.sp[1], rs.z + C.sp[2]);
  const V3 ro = v3(pw.x - C.op[0], pw.y - C.op[1], pw.z - C.op[2]);
  double dc;
  const V3 n = cv ? interp_n_from(cv, cell, d_from_cells ? &dc : nullptr)
                  : interp_n(g, cell, d_from_cells ? &dc : nullptr);
  if (d_from_cells) d = dc;
  const V3 nw = v3(fma(Mo[0], n.x, fma(Mo[1], n.y, Mo[2] * n.z)), fma(Mo[3], n.x, fma(Mo[4], n.y, Mo[5] * n.z)),
                   fma(Mo[6], n.x, fma(Mo[7], n.y, Mo[8] * n.z)));
  const V3 cs = cross(v3(C.sw[0], C.sw[1], C.sw[2]), rs);
  const V3 co = cross(v3(C.ow[0], C.ow[1], C.ow[2]), ro);
  const V3 xd = v3((C.sv[0] + cs.x) - (C.ov[0] + co.x), (C.sv[1] + cs.y) - (C.ov[1] + co.y),
                   (C.sv[2] + cs.z) - (C.ov[2] + co.z));
  const double d_dot = dot(nw, xd);
  const V3 vt = v3(xd.x - d_dot * nw.x, xd.y - d_dot * nw.y, xd.z - d_dot * nw.z);
  V3 fnw, ftw;
  bool c2;
  penalty(A.P, d, d_dot, nw, vt, fnw, ftw, c2);
  // world -> sensor frame: Ms^T f
  fn = v3(fma(Ms[0], fnw.x, fma(Ms[3], fnw.y, Ms[6] * fnw.z)), fma(Ms[1], fnw.x, fma(Ms[4], fnw.y, Ms[7] * fnw.z)),
          fma(Ms[2], fnw.x, fma(Ms[5], fnw.y, Ms[8] * fnw.z)));
  ft = v3(fma(Ms[0], ftw.x, fma(Ms[3], ftw.y, Ms[6] * ftw.z)), fma(Ms[1], ftw.x, fma(Ms[4], ftw.y, Ms[7] * ftw.z)),
          fma(Ms[2], ftw.x, fma(Ms[5], ftw.y, Ms[8] * ftw.z)));
}

// The same contact path in the sensor frame (unit quaternions, FrameC::unit):
// n_s = Ms^T Mo n, x_dot_s = kv + om x p, and the penalty law on those
// (rotations preserve the dot and cross products the law uses), so the
// forces come out in the sensor frame without the two back-rotations.
template <typename OutT>
__device__ __forceinline__ void contact_forces_s(const FFArgs<OutT>& A, const FrameC& C, const double4 cv[8],
                                                 const Cell& cell, double d, double px, double py, double pz,
                                                 V3& fn, V3& ft, bool d_from_cells) {
  double dc;
  const V3 n = interp_n_from(cv, cell, d_from_cells ? &dc : nullptr);
  if (d_from_cells) d = dc;
  const double* M = C.Mso;
  const V3 ns = v3(fma(M[0], n.x, fma(M[1], n.y, M[2] * n.z)), fma(M[3], n.x, fma(M[4], n.y, M[5] * n.z)),
                   fma(M[6], n.x, fma(M[7], n.y, M[8] * n.z)));
  const V3 w = cross(v3(C.om[0], C.om[1], C.om[2]), v3(px, py, pz));
  const V3 xs = v3(C.kv[0] + w.x, C.kv[1] + w.y, C.kv[2] + w.z);
  const double d_dot = dot(ns, xs);
  const V3 vt = v3(xs.x - d_dot * ns.x, xs.y - d_dot * ns.y, xs.z - d_dot * ns.z);
  bool c2;
  penalty(A.P, d, d_dot, ns, vt, fn, ft, c2);
}

template <typename OutT>
__device__ __forceinline__ void store_taxel(const FFArgs<OutT>& A, int64_t t, V3 fn, V3 ft, bool contact) {
  const int64_t o = t * 3;
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
  if (A.contact) A.contact[t] = contact ? 1 : 0;
}

// n16 16-B zeros from p (16-B aligned), lane-strided over one warp
template <typename T>
__device__ __forceinline__ void store_zero16(T* p, int n16, int lane) {
  float4* v = reinterpret_cast<float4*>(p);
  for (int k = lane; k < n16; k += 32) v[k] = make_float4(0.f, 0.f, 0.f, 0.f);
}

// a full 128-taxel block of 3-vectors: 384 T, unrolled 16-B stores
template <typename T>
__device__ __forceinline__ void store_zero_block(T* p, int lane) {
  float4* v = reinterpret_cast<float4*>(p);
#pragma unroll
  for (int k = 0; k < (int)(384 * sizeof(T) / 16 / 32); ++k) v[lane + 32 * k] = make_float4(0.f, 0.f, 0.f, 0.f);
}

// twelve zeros (four taxels x 3 components) with 16-B stores
template <typename T>
__device__ __forceinline__ void store_zero12(T* p) {
  float4* v = reinterpret_cast<float4*>(p);
#pragma unroll
  for (int k = 0; k < (int)(12 * sizeof(T) / 16); ++k) v[k] = make_float4(0.f, 0.f, 0.f, 0.f);
}

template <int MAXT>
__device__ __forceinline__ void write_wrench(double* wrench, int64_t frame, double acc[6], double (*part)[6]) {
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

template <typename OutT>
__device__ __forceinline__ FastCtx fast_ctx(const FFArgs<OutT>& A, const FrameC& C, int64_t frame) {
  const Grid& g = A.grid;
  const int64_t e = frame / A.n_sensors;
  const int sidx = (int)(frame - e * A.n_sensors);
  return FastCtx{&A.grid, C.A, C.b, (double)(g.nx - 1), (double)(g.ny - 1), (double)(g.nz - 1),
                 A.obj_state + e * A.obj_stride, A.sen_state + e * A.sen_stride + (int64_t)sidx * 13};
}

// The same frame with the fast mask chain (ff_device.cuh, FrameC): per frame
// the two poses fold into rel = A p + b and three rotation matrices in
// shared memory; per taxel 9 FMAs give the cell coordinates, trilinear
// lerps the distance, and only taxels the fast values cannot decide replay
// the exact chain.  Used whenever kinematics are not requested.
template <typename OutT, int MINB, int MAXT = 128>
__global__ void __launch_bounds__(MAXT, MINB) force_field_fast_kernel(const FFArgs<OutT> A) {
  const int64_t frame = blockIdx.x;
  __shared__ FrameC C;
  __shared__ double part[MAXT / 32][6];
  if (threadIdx.x < 32) frame_setup_warp(A, frame, C, threadIdx.x);
  __syncthreads();
  const FastCtx X = fast_ctx(A, C, frame);
  const int64_t out_base = frame * (int64_t)A.n_taxels;
  // the frame's output rows, so the per-taxel stores take 32-bit offsets
  OutT* const fnb = A.f_n ? A.f_n + out_base * 3 : nullptr;
  OutT* const ftb = A.f_t ? A.f_t + out_base * 3 : nullptr;
  float* const obb = A.obs ? A.obs + out_base * 3 : nullptr;
  uint8_t* const ctb = A.contact ? A.contact + out_base : nullptr;
  double acc[6] = {0, 0, 0, 0, 0, 0};
  for (int i = threadIdx.x; i < A.n_taxels; i += blockDim.x) {
    const double* tp = A.taxels + 3 * i;
    const double px = __ldg(tp), py = __ldg(tp + 1), pz = __ldg(tp + 2);
    Cell cell;
    const double d = decide_taxel(X, px, py, pz, cell);
    V3 fn = v3(0.0, 0.0, 0.0), ft = v3(0.0, 0.0, 0.0);
    const bool contact = d < 0.0;  // field.py:64 (d is +inf outside the grid)
    if (contact) {
      contact_forces(A, C, A.grid, cell, d, px, py, pz, fn, ft);
      const V3 f = v3(fn.x + ft.x, fn.y + ft.y, fn.z + ft.z);
      const V3 tq = cross(v3(px, py, pz), f);
      acc[0] += f.x;
      acc[1] += f.y;
      acc[2] += f.z;
      acc[3] += tq.x;
      acc[4] += tq.y;
      acc[5] += tq.z;
    }
    const int o = 3 * i;
    if (fnb) {
      fnb[o] = (OutT)fn.x;
      fnb[o + 1] = (OutT)fn.y;
      fnb[o + 2] = (OutT)fn.z;
    }
    if (ftb) {
      ftb[o] = (OutT)ft.x;
      ftb[o + 1] = (OutT)ft.y;
      ftb[o + 2] = (OutT)ft.z;
    }
    if (obb) {  // policy observation [f_n.z, f_t.x, f_t.y] (envs/peg_tasks.py:474-476)
      obb[o] = (float)fn.z;
      obb[o + 1] = (float)ft.x;
      obb[o + 2] = (float)ft.y;
    }
    if (ctb) ctb[i] = contact ? 1 : 0;
  }
  if (A.wrench) write_wrench<MAXT>(A.wrench, frame, acc, part);
}

// ---- fp32 certified pre-pass (force_field_quad_kernel) ----------------------
//
// Out of contact both forces are exactly zero, so the bulk of a dense taxel
// grid only needs the contact decision d < 0 -- and the validity decision
// before it -- taken exactly as the reference takes them.  This kernel takes
// both in float32 with a certified error bound, and replays float64 only
// where the bound does not clear the decision:
//
//  * rel32 = A32 p32 + b32 (three nested FMAs; A, b rounded from the fp64
//    frame fold).  |rel32 - rel_ref| <= 5u S + 1e-9 per axis, u = 2^-24,
//    S = sum_k |A_ik p_k| + |b_i| <= amax |p|_1 + bmax =: sb; we use
//    mrel = 8u sb + 1e-7 cells.
//  * cell: rel in [1, dims-2) on every axis is inside and rel < -1 or
//    >= dims outside whenever mrel < 1 (sb < 1e6) -- plain float compares,
//    which NaN fails both of; the one-cell shell in between is tested
//    against mrel explicitly, and what that cannot decide (NaN included)
//    goes to the exact chain.  Inside, floor(rel) is the round-down of
//    rel + 1.5 * 2^23 (exact for rel in [1, 2^22]).
//  * d32: trilinear lerps fma(w, b - a, a) of the fp32 corner values (two
//    128-bit gathers of the quad grid).  With L_i the grid's per-axis
//    Lipschitz bounds, the interpolant moves at most sum_i L_i |drel_i| <=
//    lsum * mrel between rel32 and rel_ref, and the fp32 value rounding and
//    lerps add at most u (4 M + lsum) with M (the cell's largest |corner|)
//    <= |d| + lsum, so |d32 - d_ref| <= tau + 5u|d32| (+ O(u^2)), with
//    tau = 8u lsum sb + lsum (1e-7 + 8u).  d < 0 is taken from d32 when
//    |d32| (1 - 16u) > 2 tau (the frame constants carry 2 / (1 - 16u), so
//    the test is one compare); a factor-2 margin covers the rounding of the
//    bound itself.
//
// Contact taxels then recompute the cell and d in float64 from the fast
// fold (as force_field_fast_kernel does) for their forces; taxels the bound
// cannot decide run the reference chain (exact_rel).  The taxels come from
// a per-call fp32 copy {x, y, z, |p|_1} (taxel_f32_kernel), four per lane at
// lane + 32 j of a warp's 128-taxel block: coalesced 16-B loads, issued one
// block ahead, eight gathers in flight, and coalesced 16-B zero stores.
constexpr float kU32 = 5.9604645e-8f;  // 2^-24
constexpr float kFloorMagic = 12582912.0f;  // 1.5 * 2^23

struct QuadTaxel {
  float wx, wy, wz;  // fp32 cell weights
  int idx;           // fp32 cell (when inside)
  int cls;           // 0: outside the grid, 1: inside, 2: undecided (exact chain)
  float tau;         // the decision bound 2 tau / (1 - 16u): d32 decides when |d32| > tau
};

// exact cell-validity test of one axis against the certified margin
__device__ __forceinline__ void shell_axis(float r, float mrel, int m, bool& in, bool& out) {
  in = in & (r - mrel > 0.0f) & (r + mrel < (float)m);
  out = out | (r + mrel < 0.0f) | (r - mrel > (float)m);
}

// One taxel off the queue: the reference chain (kind 2) or the fast fp64
// fold (kind 1, certified contact), then the contact forces and its stores.
template <typename OutT>
__device__ __forceinline__ void drain_taxel(const FFArgs<OutT>& A, const FrameC& C, const FastCtx& X, int i,
                                            unsigned kind, OutT* fnb, OutT* ftb, float* obb,
                                            uint8_t* ctb, double acc[6]) {
  const Grid& g = A.grid;
  double4 cv[8];
  const double* pp = A.taxels + 3 * i;
  const double px = __ldg(pp), py = __ldg(pp + 1), pz = __ldg(pp + 2);
  Cell cell;
  double d = 0.0;
  if (kind == 2) {  // the reference chain
    const V3 r = exact_rel(g, X.obj, X.sen, v3(px, py, pz));
    cell = locate_rel(g, r.x, r.y, r.z);
    d = cell.valid ? interp_d(g, cell) : __longlong_as_double(0x7ff0000000000000LL);
    if (!(d < 0.0)) return;  // zeros are already stored
    load_corners(g, cell.base, cv);
  } else {  // certified contact: fp64 cell from the fast fold, d from the cells in contact_forces
    const double rx = fma(X.a[0], px, fma(X.a[1], py, fma(X.a[2], pz, X.b[0])));
    const double ry = fma(X.a[3], px, fma(X.a[4], py, fma(X.a[5], pz, X.b[1])));
    const double rz = fma(X.a[6], px, fma(X.a[7], py, fma(X.a[8], pz, X.b[2])));
    const int ix = min(max((int)rx, 0), g.nx - 2), iy = min(max((int)ry, 0), g.ny - 2),
              iz = min(max((int)rz, 0), g.nz - 2);
    cell.wx = rx - (double)ix;
    cell.wy = ry - (double)iy;
    cell.wz = rz - (double)iz;
    cell.ux = 1.0 - cell.wx;
    cell.uy = 1.0 - cell.wy;
    cell.uz = 1.0 - cell.wz;
    cell.base = (ix * g.ny + iy) * g.nz + iz;
    load_corners(g, cell.base, cv);
  }
  V3 fn, ft;
  if (C.unit) contact_forces_s(A, C, cv, cell, d, px, py, pz, fn, ft, kind == 1);
  else contact_forces(A, C, g, cell, d, px, py, pz, fn, ft, kind == 1, cv);
  const V3 f = v3(fn.x + ft.x, fn.y + ft.y, fn.z + ft.z);
  const V3 tq = cross(v3(px, py, pz), f);
  acc[0] += f.x;
  acc[1] += f.y;
  acc[2] += f.z;
  acc[3] += tq.x;
  acc[4] += tq.y;
  acc[5] += tq.z;
  const int o = 3 * i;
  if (fnb) {
    fnb[o] = (OutT)fn.x;
    fnb[o + 1] = (OutT)fn.y;
    fnb[o + 2] = (OutT)fn.z;
  }
  if (ftb) {
    ftb[o] = (OutT)ft.x;
    ftb[o + 1] = (OutT)ft.y;
    ftb[o + 2] = (OutT)ft.z;
  }
  if (obb) {
    obb[o] = (float)fn.z;
    obb[o + 1] = (float)ft.x;
    obb[o + 2] = (float)ft.y;
  }
  if (ctb) ctb[i] = 1;
}

// Each warp walks blocks of 128 consecutive taxels (lane + 32 j, j < 4):
// the certified fp32 decisions, zeros stored for the whole block (coalesced
// 16-B stores), and the contact / undecided taxels appended to a warp-private
// shared-memory queue.  Whenever 32 or more are queued the warp drains 32 of
// them, one per lane -- the fp64 contact path runs on full warps, and other
// warps' fp32 blocks overlap its latency (no CTA barrier until the wrench).
constexpr int kWarpQueue = 160;  // < 32 left over + 128 appended per block

// The certified fp32 decisions for one warp's block of 128 taxels (four per
// lane, lane + 32 j; cnt a multiple of 4): per taxel two bits of the
// result -- 0 no contact, 1 contact, 2 undecided (the reference chain) --
// and the fp32 cell index in idx[j] (for a contact taxel).
template <typename OutT>
__device__ __forceinline__ unsigned classify_block(const FFArgs<OutT>& A, const FrameC& C, int blk, int cnt,
                                                   const float4 tfs[4], int lane, int idx_out[4]) {
  const Grid& g = A.grid;
  const int mx = g.nx - 1, my = g.ny - 1, mz = g.nz - 1;  // rel in [0, m] is inside
  const int nyz = g.ny * g.nz;
  // the frame constants come from shared memory every block: the drain
  // between blocks needs the registers
  float a[9], b[3];
#pragma unroll
  for (int k = 0; k < 9; ++k) a[k] = C.A32[k];
#pragma unroll
  for (int k = 0; k < 3; ++k) b[k] = C.b32[k];
  const float amax = C.amax, bmax = C.bmax, kt = C.kt, k0 = C.k0;
  // cells [1, m-2] (rel in [1, m-1)) are inside and rel < -1 or >= m+1
  // outside whenever mrel < 1 (sb < 1e6); NaN fails both: shell -> exact
  const float hx = (float)(mx - 1), hy = (float)(my - 1), hz = (float)(mz - 1);
  const float ox = (float)(mx + 1), oy = (float)(my + 1), oz = (float)(mz + 1);
  const bool full = cnt == 128;
  QuadTaxel t[4];
  bool shell = false;
#pragma unroll
  for (int j = 0; j < 4; ++j) {
    const int k = lane + 32 * j;
    const bool live = full || k < cnt;
    const float4 tf = tfs[j];
    const float x = tf.x, y = tf.y, z = tf.z;
    const float rx = fmaf(a[0], x, fmaf(a[1], y, fmaf(a[2], z, b[0])));
    const float ry = fmaf(a[3], x, fmaf(a[4], y, fmaf(a[5], z, b[1])));
    const float rz = fmaf(a[6], x, fmaf(a[7], y, fmaf(a[8], z, b[2])));
    const float sb = fmaf(amax, tf.w, bmax);
    t[j].tau = fmaf(kt, sb, k0);
    bool in, out;
    int ix, iy, iz;
    {
    const bool ok = live & (sb < 1e6f);  // mrel < 1
    const float lo = fminf(fminf(rx, ry), rz);  // (NaN on an axis fails that axis's own tests below)
    in = ok & (lo >= 1.0f) & (rx < hx) & (ry < hy) & (rz < hz);
    out = !live | (ok & ((lo < -1.0f) | (rx >= ox) | (ry >= oy) | (rz >= oz)));
    // floor by round-down onto 1.5 * 2^23 (exact for rel in [1, 2^22]; only used when inside)
    const float tx = __fadd_rd(rx, kFloorMagic), ty = __fadd_rd(ry, kFloorMagic), tz = __fadd_rd(rz, kFloorMagic);
    ix = __float_as_int(tx) - 0x4B400000, iy = __float_as_int(ty) - 0x4B400000,
              iz = __float_as_int(tz) - 0x4B400000;
    t[j].wx = rx - (tx - kFloorMagic);
    t[j].wy = ry - (ty - kFloorMagic);
    t[j].wz = rz - (tz - kFloorMagic);
    }
    t[j].cls = in ? 1 : (out ? 0 : 2);
    t[j].idx = in ? (ix * g.ny + iy) * g.nz + iz : 0;
    shell |= !(in | out);
  }
  if (shell) {  // the one-cell shell round the grid faces: explicit margins
#pragma unroll
    for (int j = 0; j < 4; ++j) {
      if (t[j].cls != 2) continue;
      const float4 tf = __ldg(A.taxf + blk + lane + 32 * j);
      const float x = tf.x, y = tf.y, z = tf.z;
      const float rx = fmaf(a[0], x, fmaf(a[1], y, fmaf(a[2], z, b[0])));
      const float ry = fmaf(a[3], x, fmaf(a[4], y, fmaf(a[5], z, b[1])));
      const float rz = fmaf(a[6], x, fmaf(a[7], y, fmaf(a[8], z, b[2])));
      const float mrel = fmaf(8.0f * kU32, fmaf(amax, tf.w, bmax), 1e-7f);
      bool in = true, out = false;
      shell_axis(rx, mrel, mx, in, out);
      shell_axis(ry, mrel, my, in, out);
      shell_axis(rz, mrel, mz, in, out);
      if (out) {
        t[j].cls = 0;
      } else if (in) {  // 0 < rel < m: floor lands in [0, m - 1]
        const int ix = min((int)rx, mx - 1), iy = min((int)ry, my - 1), iz = min((int)rz, mz - 1);
        t[j].wx = rx - (float)ix;
        t[j].wy = ry - (float)iy;
        t[j].wz = rz - (float)iz;
        t[j].idx = (ix * g.ny + iy) * g.nz + iz;
        t[j].cls = 1;
      }
    }
  }
  // per taxel, two bits: 0 no contact, 1 contact, 2 exact chain
  unsigned kinds = 0;
#pragma unroll
  for (int j = 0; j < 4; ++j) {
    const float4 lo = __ldg(g.quads + t[j].idx), hi = __ldg(g.quads + t[j].idx + nyz);
    // x lerps of the (z, z+1) x (y, y+1) corner pairs, then y, then z
    const float e00 = fmaf(t[j].wx, hi.x - lo.x, lo.x), e01 = fmaf(t[j].wx, hi.y - lo.y, lo.y);
    const float e10 = fmaf(t[j].wx, hi.z - lo.z, lo.z), e11 = fmaf(t[j].wx, hi.w - lo.w, lo.w);
    const float f0 = fmaf(t[j].wy, e10 - e00, e00), f1 = fmaf(t[j].wy, e11 - e01, e01);
    const float d32 = fmaf(t[j].wz, f1 - f0, f0);
    const bool clear = fabsf(d32) > t[j].tau;  // tau here is 2 tau / (1 - 16u) (frame_setup_quad)
    const unsigned kind = t[j].cls == 0 ? 0u : (t[j].cls == 1 && clear ? (d32 < 0.0f ? 1u : 0u) : 2u);
    kinds |= kind << (2 * j);
    idx_out[j] = t[j].idx;
  }
  return kinds;
}

template <typename OutT, int MINB, int MAXT>
__global__ void __launch_bounds__(MAXT, MINB) force_field_quad_kernel(const FFArgs<OutT> A) {
  const int64_t frame = blockIdx.x;
  __shared__ FrameC C;
  __shared__ double part[MAXT / 32][6];
  __shared__ int wqueue[MAXT / 32][kWarpQueue];  // (taxel << 2) | kind
  if (threadIdx.x < 32) frame_setup_warp<true>(A, frame, C, threadIdx.x);
  __syncthreads();
  const Grid& g = A.grid;
  const int mx = g.nx - 1, my = g.ny - 1, mz = g.nz - 1;  // rel in [0, m] is inside
  const int nyz = g.ny * g.nz;
  const FastCtx X = fast_ctx(A, C, frame);
  const int64_t out_base = frame * (int64_t)A.n_taxels;
  OutT* const fnb = A.f_n ? A.f_n + out_base * 3 : nullptr;
  OutT* const ftb = A.f_t ? A.f_t + out_base * 3 : nullptr;
  float* const obb = A.obs ? A.obs + out_base * 3 : nullptr;
  uint8_t* const ctb = A.contact ? A.contact + out_base : nullptr;
  double acc[6] = {0, 0, 0, 0, 0, 0};
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5, nwarps = blockDim.x >> 5;
  int* const wq = wqueue[warp];
  int wn = 0;  // queued entries (warp-uniform)
  // the taxel loads of a warp's next block are issued one block ahead
  auto load_block = [&](int bb, float4 out[4]) {
    const int c = min(128, A.n_taxels - bb);
#pragma unroll
    for (int j = 0; j < 4; ++j) {
      const int k = lane + 32 * j;
      out[j] = __ldg(A.taxf + bb + (k < c ? k : 0));
    }
  };
  float4 tnext[4];
  if (128 * warp < A.n_taxels) load_block(128 * warp, tnext);
  for (int blk = 128 * warp; blk < A.n_taxels; blk += 128 * nwarps) {
    const int cnt = min(128, A.n_taxels - blk);  // a multiple of 4
    float4 tfs[4];
#pragma unroll
    for (int j = 0; j < 4; ++j) tfs[j] = tnext[j];
    if (blk + 128 * nwarps < A.n_taxels) load_block(blk + 128 * nwarps, tnext);
    int idx[4];
    const unsigned kinds = classify_block(A, C, blk, cnt, tfs, lane, idx);
    const bool full = cnt == 128;
    // zeros for the block's taxels, coalesced 16-B stores; contact taxels are
    // overwritten by this warp's drain (ordered by __syncwarp)
    if (full) {
      if (fnb) store_zero_block(fnb + 3 * blk, lane);
      if (ftb) store_zero_block(ftb + 3 * blk, lane);
      if (obb) store_zero_block(obb + 3 * blk, lane);
      if (ctb) reinterpret_cast<uchar4*>(ctb + blk)[lane] = make_uchar4(0, 0, 0, 0);
    } else {
      const int n16 = cnt * 3 * (int)sizeof(OutT) / 16;
      if (fnb) store_zero16(fnb + 3 * blk, n16, lane);
      if (ftb) store_zero16(ftb + 3 * blk, n16, lane);
      if (obb) store_zero16(obb + 3 * blk, cnt * 3 * 4 / 16, lane);
      if (ctb && lane < cnt / 4) reinterpret_cast<uchar4*>(ctb + blk)[lane] = make_uchar4(0, 0, 0, 0);
    }
    if (__any_sync(0xffffffffu, kinds != 0)) {
      // append to the warp queue in taxel order (neighbouring taxels share
      // cells, so a drained warp's corner loads coalesce)
      const unsigned lt = (1u << lane) - 1u;
#pragma unroll
      for (int j = 0; j < 4; ++j) {
        const unsigned kind = (kinds >> (2 * j)) & 3u;
        const unsigned m = __ballot_sync(0xffffffffu, kind != 0);
        if (kind) wq[wn + __popc(m & lt)] = ((blk + lane + 32 * j) << 2) | (int)kind;
        wn += __popc(m);
      }
      __syncwarp();
      while (wn >= 32) {  // drain full warps from the tail
        wn -= 32;
        const int e = wq[wn + lane];
        drain_taxel(A, C, X, e >> 2, (unsigned)(e & 3), fnb, ftb, obb, ctb, acc);
        __syncwarp();
      }
    }
  }
  if (lane < wn) {  // the remainder
    const int e = wq[lane];
    drain_taxel(A, C, X, e >> 2, (unsigned)(e & 3), fnb, ftb, obb, ctb, acc);
  }
  if (A.wrench) write_wrench<MAXT>(A.wrench, frame, acc, part);
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


// taxels as fp32 {x, y, z, |x|+|y|+|z|} for the quad kernel's coalesced loads
__global__ void __launch_bounds__(256) taxel_f32_kernel(const double* __restrict__ taxels, int n,
                                                        float4* __restrict__ out) {
  for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < n; i += gridDim.x * blockDim.x) {
    const float x = (float)taxels[3 * i], y = (float)taxels[3 * i + 1], z = (float)taxels[3 * i + 2];
    // |p|_1 rounded up, so amax |p|_1 + bmax bounds the exact S
    out[i] = make_float4(x, y, z, __fadd_ru(__fadd_ru(fabsf(x), fabsf(y)), fabsf(z)) * (1.0f + 4.0f * kU32));
  }
}

// The fp32 taxel copy lives for one call: stream-ordered allocation from the
// device's default memory pool (kept warm: release threshold raised once per
// device), so nothing is cached across calls -- an array edited in place or
// freed and reallocated is never stale -- and it is legal under stream
// capture (allocation / free nodes in the graph).  Null on failure: the
// caller then runs the fp64 kernel.
float4* taxel_scratch(int device, int n, cudaStream_t stream) {
  static std::mutex mu;
  static std::vector<int> warmed;
  {
    std::lock_guard<std::mutex> lock(mu);
    if (std::find(warmed.begin(), warmed.end(), device) == warmed.end()) {
      cudaMemPool_t pool;
      if (cudaDeviceGetDefaultMemPool(&pool, device) == cudaSuccess) {
        uint64_t keep = UINT64_MAX;
        cudaMemPoolSetAttribute(pool, cudaMemPoolAttrReleaseThreshold, &keep);
      }
      cudaGetLastError();
      warmed.push_back(device);
    }
  }
  void* buf = nullptr;
  if (cudaMallocAsync(&buf, (size_t)n * sizeof(float4), stream) != cudaSuccess) {
    cudaGetLastError();
    return nullptr;
  }
  return static_cast<float4*>(buf);
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
  StreamDevice stream_device_(stream);
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
  StreamDevice stream_device_(stream);
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
  StreamDevice stream_device_(stream);
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
  // threads per frame: small taxel grids (20x25) amortise the per-frame
  // set-up best with 2 warps per frame, dense ones (80x100) with 4 (measured)
  const char* tpf = std::getenv("TACSL_FF_THREADS");
  // (and a small batch -- fewer frames than SMs -- wants the wider CTA for latency)
  const bool few = frames < 2 * (int64_t)sm_count(current_device());
  const int threads = tpf ? (std::atoi(tpf) == 64 ? 64 : 128) : (n_taxels <= 1024 && !few ? 64 : 128);
  Penalty P{params.k_n, params.k_d, params.k_t, params.mu};
  cudaStream_t s = (cudaStream_t)stream;
  const char* mb = std::getenv("TACSL_FF_MINBLOCKS");
  const int minb_exact = mb ? std::atoi(mb) : kFFMinBlocks;
  const int minb_fast = mb ? std::atoi(mb) : kFFFastMinBlocks;
  const int minb_quad = mb ? std::atoi(mb) : kFFQuadMinBlocks;
  // kinematics (d, n, v_t as the reference computes them) use the exact
  // chain for every taxel; TACSL_FF_EXACT=1 forces it for A/B checks
  const bool exact = std::getenv("TACSL_FF_EXACT") != nullptr;
  auto al = [](const void* p, uintptr_t a) { return (reinterpret_cast<uintptr_t>(p) & (a - 1)) == 0; };
  // the quad kernel pays off on dense taxel grids (80x100: 1.58 -> 1.33 ms);
  // on 20x25 pads the fp64 fast kernel is faster (and overlaps K1 better)
  const char* qenv = std::getenv("TACSL_FF_QUAD");  // "0": never, "1": whenever eligible
  const bool want_quad = qenv ? qenv[0] == '1' : n_taxels > kQuadMinTaxels;
  bool quad = want_quad && !kin && !exact && sdf->quads && n_taxels % 4 == 0 && n_taxels < (1 << 29) &&
              al(f_n, 16) && al(f_t, 16) &&
              al(obs, 16) && al(contact, 4);
  float4* taxf = nullptr;
  if (quad) {
    taxf = taxel_scratch(current_device(), n_taxels, s);
    quad = taxf != nullptr;
  }
  if (quad) {
    taxel_f32_kernel<<<std::min(elementwise_blocks(n_taxels), 64u), 256, 0, s>>>(taxels, n_taxels, taxf);
    if (int rc = check_launch("taxel_f32_kernel")) {
      cudaFreeAsync(taxf, s);
      return rc;
    }
  }
  auto launch = [&](auto out_tag) -> int {
    using O = decltype(out_tag);
    const FFArgs<O> A{make_grid(sdf), taxels, n_taxels, object_state, object_stride, sensor_state, sensor_stride,
                      n_sensors, frames, P, (O*)f_n, (O*)f_t, wrench, kin, contact, obs, nullptr, taxf};
    if (quad) {
      // the certified fp32 pre-pass: four taxels per thread
      if (few && n_taxels >= 256 && !tpf)
        force_field_quad_kernel<O, 1, 512>
            <<<(unsigned)frames, std::min(512, (n_taxels + 127) / 128 * 32), 0, s>>>(A);
      else if (minb_quad >= 5)
        force_field_quad_kernel<O, 5, 128><<<(unsigned)frames, threads, 0, s>>>(A);
      else
        force_field_quad_kernel<O, 4, 128><<<(unsigned)frames, threads, 0, s>>>(A);
    } else if (!kin && !exact && few && n_taxels >= 256 && !tpf) {
      // a handful of frames: one taxel (or two) per thread, lowest latency
      force_field_fast_kernel<O, 1, 512><<<(unsigned)frames, std::min(512, (n_taxels + 31) / 32 * 32), 0, s>>>(A);
    } else if (!kin && !exact) {
      if (minb_fast >= 6) force_field_fast_kernel<O, 6><<<(unsigned)frames, threads, 0, s>>>(A);
      else if (minb_fast == 5) force_field_fast_kernel<O, 5><<<(unsigned)frames, threads, 0, s>>>(A);
      else force_field_fast_kernel<O, 4><<<(unsigned)frames, threads, 0, s>>>(A);
    } else if (minb_exact >= 6) {
      force_field_kernel<O, 6><<<(unsigned)frames, threads, 0, s>>>(A);
    } else if (minb_exact == 5) {
      force_field_kernel<O, 5><<<(unsigned)frames, threads, 0, s>>>(A);
    } else {
      force_field_kernel<O, 4><<<(unsigned)frames, threads, 0, s>>>(A);
    }
    return 0;
  };
  const int lrc = out_fp64 ? launch(double{}) : launch(float{});
  const int launched = lrc ? lrc : check_launch("force_field_kernel");
  if (taxf) cudaFreeAsync(taxf, s);
  return launched;
}

int tacsl_net_wrench(const double* f_n, const double* f_t, const double* points, int64_t frames, int rows, int cols,
                     double* force, double* torque, void* stream) {
  StreamDevice stream_device_(stream);
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
