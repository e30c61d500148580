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
#include "ff_device.cuh"
#include "handles.h"

namespace tacsl {
namespace {

constexpr int kFFMinBlocks = 4;      // exact kernel: resident 128-thread CTAs per SM the register budget targets
constexpr int kFFFastMinBlocks = 5;  // fast kernel: 96 registers, no spills (4: 126 regs, 6: spills; measured)


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
                                               V3& ft) {
  const double* Ms = C.Ms;
  const double* Mo = C.Mo;
  const V3 rs = v3(fma(Ms[0], px, fma(Ms[1], py, Ms[2] * pz)), fma(Ms[3], px, fma(Ms[4], py, Ms[5] * pz)),
                   fma(Ms[6], px, fma(Ms[7], py, Ms[8] * pz)));
  const V3 pw = v3(rs.x + C.sp[0], rs.y + C.sp[1], rs.z + C.sp[2]);
  const V3 ro = v3(pw.x - C.op[0], pw.y - C.op[1], pw.z - C.op[2]);
  const V3 n = interp_n(g, cell);
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
    store_taxel(A, out_base + i, fn, ft, contact);
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
  // kinematics (d, n, v_t as the reference computes them) use the exact
  // chain for every taxel; TACSL_FF_EXACT=1 forces it for A/B checks
  const bool exact = std::getenv("TACSL_FF_EXACT") != nullptr;
  auto launch = [&](auto out_tag) {
    using O = decltype(out_tag);
    const FFArgs<O> A{make_grid(sdf), taxels, n_taxels, object_state, object_stride, sensor_state, sensor_stride,
                      n_sensors, frames, P, (O*)f_n, (O*)f_t, wrench, kin, contact, obs};
    if (!kin && !exact && few && n_taxels >= 256 && !tpf) {
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
  };
  if (out_fp64) launch(double{});
  else launch(float{});
  return check_launch("force_field_kernel");
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
