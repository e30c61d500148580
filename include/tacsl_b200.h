/*
 * tacsl_b200.h -- C ABI of the B200-native TacSL sensor-simulation hot path.
 *
 * One shared library (libtacsl_b200.so, sm_100a) exporting plain C entry
 * points: no torch types, plain device pointers + sizes, stream-ordered,
 * re-entrant.  Every call returns TACSL_OK (0) or an error code; the message
 * of the last failing call on the calling thread is tacsl_last_error().
 *
 * Each entry point replaces one function of the reference Python package
 * `gelsim` (paths relative to /root/reference/pkg/src/gelsim):
 *
 *   tacsl_depth_to_rgb      render/lut.py:68-76   depth_to_rgb (+ depth_gradients
 *                           lut.py:25-28, PolyLut.evaluate / _design_matrix
 *                           lut.py:56-65, and to_uint8 render/imageio.py:8-11
 *                           fused as the uint8 epilogue)
 *   tacsl_lut_create        render/lut.py:31-54   PolyLut (coefficients + image_size)
 *   tacsl_to_uint8          render/imageio.py:8-11 to_uint8 (standalone, float32 input)
 *   tacsl_to_uint8_f64      render/imageio.py:8-11 to_uint8 on float64 input, in float64
 *   tacsl_f64_to_f32 /      the numpy drop-ins' dtype changes (the reference computes in
 *   tacsl_f32_to_f64        float64; np.asarray(..., float64) / astype) done on the device
 *   tacsl_frame_digest      (no reference counterpart) per-frame 64-bit digests of a
 *                           step's outputs for cross-rank validation
 *   tacsl_sdf_create        geometry/sdf.py:29-54 SdfGrid (device upload)
 *   tacsl_query_sdf         geometry/sdf.py:271-321 query_sdf
 *   tacsl_relative_penetration_rate geometry/sdf.py:324-328 (INVALID_QUERY on out-of-grid queries)
 *   tacsl_penalty_forces    tactile/field.py:61-76 penalty_forces
 *   tacsl_force_field       tactile/field.py:79-129 compute_force_field
 *                           (+ net_wrench tactile/field.py:132-141 fused as a
 *                           per-sensor reduction when `wrench` is non-NULL)
 *   tacsl_net_wrench        tactile/field.py:132-141 net_wrench (standalone)
 *   tacsl_render_depth      render/depth.py:88-134 render_depth (SDF sphere tracer)
 *   tacsl_env_render_params envs/peg_tasks.py:440-442 + render/depth.py:105-121 (per-env render inputs)
 *   tacsl_rgb_pyramid       render/lut.py:68-76 extended (no reference counterpart, SURVEY.md 8a
 *                           a13): Gaussian smoothing + tactile RGB of a 1-3 level pyramid in one pass
 *
 * The reference has no FFI of its own (pure numpy); the Python module
 * paper_2408_06506_b200 binds these with ctypes behind the reference's
 * function names and signatures.
 *
 * Conventions
 *  - quaternions are (w, x, y, z) (transforms.py:3);
 *  - a rigid-body "state" is 13 float64: pos[3], quat[4], linvel[3], angvel[3];
 *  - every array is C-contiguous; images are (N, H, W) depth and
 *    (N, H, W, 3) RGB (HWC interleaved, as the reference returns);
 *  - all pointers passed to compute calls are DEVICE pointers on the
 *    handle's device; `stream` is a cudaStream_t (NULL = legacy default).
 */
#ifndef TACSL_B200_H
#define TACSL_B200_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define TACSL_ABI_VERSION 1

#if defined(__GNUC__)
#define TACSL_API __attribute__((visibility("default")))
#else
#define TACSL_API
#endif

typedef enum {
  TACSL_OK = 0,
  TACSL_ERR_INVALID_ARGUMENT = 1,       /* -> ValueError                       */
  TACSL_ERR_DIMENSION_MISMATCH = 2,     /* -> gelsim.errors.DimensionMismatch  */
  TACSL_ERR_LUT_RESOLUTION_MISMATCH = 3,/* -> gelsim.errors.LutResolutionMismatch */
  TACSL_ERR_INVALID_QUERY = 4,          /* -> gelsim.errors.InvalidQuery       */
  TACSL_ERR_CUDA = 5,                   /* -> RuntimeError (CUDA failure)      */
  TACSL_ERR_NO_DEVICE = 6               /* -> RuntimeError (no sm_100 device)  */
} tacsl_status_t;

typedef struct tacsl_lut_s* tacsl_lut_t;
typedef struct tacsl_sdf_s* tacsl_sdf_t;
typedef struct tacsl_binned_lut_s* tacsl_binned_lut_t;

/* PenaltyParams (tactile/field.py:28-37). */
typedef struct {
  double k_n;  /* normal stiffness, N/m            */
  double k_d;  /* normal damping on d*d_dot        */
  double k_t;  /* shear stiffness vs slip speed    */
  double mu;   /* friction coefficient             */
} tacsl_penalty_t;

TACSL_API int tacsl_abi_version(void);
TACSL_API const char* tacsl_last_error(void);
/* 1 if `device` is an sm_100 part the library has code for, else 0. */
TACSL_API int tacsl_device_supported(int device);

/* ---------------------------------------------------------------- LUT --- */
/* coeffs: HOST (3, n_terms) float64 in monomial_exponents(degree) order
 * (lut.py:20-22); degree in [2,4] (lut.py:47-48) else INVALID_ARGUMENT.
 * width/height: the image_size the LUT was calibrated at (W, H). */
TACSL_API int tacsl_lut_create(const double* coeffs, int degree, int width, int height,
                     tacsl_lut_t* out);
TACSL_API void tacsl_lut_destroy(tacsl_lut_t lut);

/* depth (N, H, W) float32 -> rgb (N, H, W, 3); either output may be NULL
 * (not both).  rgb_u8 = clip(rint(255*x)), rgb_f32 = x in [0,1].
 * LUT_RESOLUTION_MISMATCH when (width, height) != lut image size (lut.py:70-74);
 * INVALID_ARGUMENT when H < 2 or W < 2 (np.gradient needs 2 samples). */
TACSL_API int tacsl_depth_to_rgb(tacsl_lut_t lut, const float* depth, int64_t n_images,
                       int height, int width, uint8_t* rgb_u8, float* rgb_f32,
                       void* stream);

/* Per-pixel BINNED polynomial LUT (north_star; NO reference counterpart --
 * gelsim's PolyLut render/lut.py:31-59 is one global polynomial, which is
 * the bins_y = bins_x = 1 case).  Pixel (y, x) uses coefficient set
 * (y*bins_y/H, x*bins_x/W) (integer floor).  coeffs: HOST
 * (bins_y, bins_x, 3, n_terms) float64 in monomial_exponents order; the
 * table is uploaded to `device`.  INVALID_ARGUMENT for a degree outside
 * [2,4] or bins outside [1, image size]. */
TACSL_API int tacsl_binned_lut_create(int device, const double* coeffs, int degree, int bins_y,
                                      int bins_x, int width, int height, tacsl_binned_lut_t* out);
TACSL_API void tacsl_binned_lut_destroy(tacsl_binned_lut_t lut);

/* tacsl_depth_to_rgb through a binned LUT (same layouts, outputs and errors).
 * Tables over 96 KB (float32) additionally need width % 4 == 0, 16-B aligned
 * buffers and every x-bin edge on an even column, else INVALID_ARGUMENT. */
TACSL_API int tacsl_depth_to_rgb_binned(tacsl_binned_lut_t lut, const float* depth, int64_t n_images,
                                        int height, int width, uint8_t* rgb_u8, float* rgb_f32,
                                        void* stream);

/* Policy observation image of envs/peg_tasks.py:434-458 without
 * augmentation: depth (N, H, W) -> float32 RGB in the env's representation,
 *   rep 0 "color"  (N, H, W, 3)  rgb                  (peg_tasks.py:445)
 *   rep 1 "diff"   (N, H, W, 3)  rgb - nominal         (peg_tasks.py:453-454)
 *   rep 2 "concat" (N, H, W, 6)  [rgb, nominal]        (peg_tasks.py:455-458)
 * nominal: HOST float[3], the LUT background colour (peg_tasks.py:111-112). */
TACSL_API int tacsl_tactile_image_obs(tacsl_lut_t lut, const float* depth, int64_t n_images,
                                      int height, int width, int rep, const float nominal[3],
                                      float* out, void* stream);

/* AugmentConfig (render/augment.py:15-48). */
typedef struct {
  double shift_px;
  double zoom_lo, zoom_hi;
  double brightness;
  double contrast_lo, contrast_hi;
  double saturation_lo, saturation_hi;
  double hue;
  int32_t channel_permutation;
  double step_brightness;
  double step_contrast_lo, step_contrast_hi;
  double step_saturation_lo, step_saturation_hi;
  double step_hue;
  uint64_t seed;
} tacsl_augment_cfg_t;

/* Per-image augmentation parameters (augment.py:65-85) from the reference's
 * tuple-keyed Philox streams, computed on the device: params (n, 16) float64
 * = shift_x, shift_y, zoom, brightness, contrast, saturation, hue, perm[3],
 * step brightness, contrast, saturation, hue. episode_seeds / step_indices
 * are (n) int64 >= 0 device arrays. */
TACSL_API int tacsl_augment_params(const tacsl_augment_cfg_t* cfg, const int64_t* episode_seeds,
                                   const int64_t* step_indices, int64_t n, double* params,
                                   void* stream);
/* augment (augment.py:156-173) of float32 (n, H, W, 3) images with those
 * parameters, then the observation representation rep 0 colour / 1 diff /
 * 2 concat (envs/peg_tasks.py:453-458, nominal = HOST float[3]).  Out of
 * place; out is (n, H, W, 3) or (n, H, W, 6) float32. */
TACSL_API int tacsl_augment(const float* images, int64_t n, int height, int width,
                            const double* params, int rep, const float nominal[3], float* out,
                            void* stream);

/* Separable filter with optional 2x decimation -- the north_star's Gaussian
 * smoothing (step 1, Gaussian taps) and Gaussian-pyramid level (step 2,
 * binomial [1,4,6,4,1]/16).  NOT in the reference:
 *   out[y,x] = sum_ij taps[i] taps[j] in[clamp(s*y+i-R), clamp(s*x+j-R)]
 * 'nearest' borders, 2R+1 <= 33 HOST float taps, out (n, ceil(H/s), ceil(W/s)). */
TACSL_API int tacsl_separable_filter(const float* in, int64_t n_images, int height, int width,
                                     const float* taps, int radius, int step, float* out,
                                     void* stream);

/* x (count) float32 -> u8 = clip(rint(255*x), 0, 255) (imageio.py:8-11). */
TACSL_API int tacsl_to_uint8(const float* x, int64_t count, uint8_t* out, void* stream);

/* x (count) float64 -> u8 = clip(rint(x*255), 0, 255) computed in float64
 * exactly as imageio.py:8-11 (product rounded to float64, ties to even;
 * NaN -> 0). */
TACSL_API int tacsl_to_uint8_f64(const double* x, int64_t count, uint8_t* out, void* stream);

/* geometry/sdf.py:324-328 relative_penetration_rate: out[i] = normal[i] .
 * x_dot[i] (x_dot_broadcast: one x_dot (3,) for every query), summed left
 * to right like np.einsum.  Returns INVALID_QUERY (InvalidQuery) when any
 * valid[i] == 0, as the reference does; this needs the answer on the host,
 * so the call synchronises `stream`.  scratch: one device int. */
TACSL_API int tacsl_relative_penetration_rate(const double* normal, const uint8_t* valid, const double* x_dot,
                                              int64_t n, int x_dot_broadcast, double* out, int* scratch,
                                              void* stream);

/* Element-wise dtype conversion on the device (round to nearest even, as
 * numpy's astype): the float64 arrays the reference's callers pass in are
 * uploaded as they are and narrowed here; float32 results are widened here
 * before one device->host copy. */
TACSL_API int tacsl_f64_to_f32(const double* x, int64_t count, float* out, void* stream);
TACSL_API int tacsl_f32_to_f64(const float* x, int64_t count, double* out, void* stream);

/* out[f] = 64-bit digest of frame f = data[f*frame_bytes, (f+1)*frame_bytes):
 * sum over the frame's 32-bit words w_i of splitmix64((i << 32) | w_i),
 * mod 2^64, finalised with the word count.  Position-dependent (swapped
 * channels, shifted rows and misplaced frames change it) and independent of
 * how the frames are sharded.  frame_bytes % 4 == 0, data 4-B aligned. */
TACSL_API int tacsl_frame_digest(const void* data, int64_t n_frames, int64_t frame_bytes, uint64_t* out,
                                 void* stream);

/* ---------------------------------------------------------------- SDF --- */
/* values: HOST (nx,ny,nz) float64, gradients: HOST (nx,ny,nz,3) float64,
 * z fastest (sdf.py:29-41).  Uploaded as a float64 {d, gx, gy, gz} cell grid
 * (32 B/cell, L2-resident) on `device`, so grids built in float64 by the
 * reference's build_sdf and float32 TSDF caches (sdf.py:343-344) are both
 * sampled exactly as the reference samples them, plus (when every value is
 * finite and within float range) a float32 corner-quad grid (16 B/cell) and
 * per-axis Lipschitz bounds for the force field's certified float32 contact
 * test.  dims >= 2 on every axis, spacing > 0, else INVALID_ARGUMENT. */
TACSL_API int tacsl_sdf_create(int device, const double* values, const double* gradients,
                     const int32_t dims[3], const double origin[3],
                     double spacing, tacsl_sdf_t* out);
TACSL_API void tacsl_sdf_destroy(tacsl_sdf_t sdf);

/* points (n, 3) float64 -> distance (n) float64 (+inf when outside),
 * normal (n, 3) float64 (0 when outside), valid (n) uint8.  Any output may
 * be NULL. */
TACSL_API int tacsl_query_sdf(tacsl_sdf_t sdf, const double* points, int64_t n,
                    double* distance, double* normal, uint8_t* valid,
                    void* stream);

/* ------------------------------------------------------- depth render --- */
/* Sphere-traced in-sensor depth (render/depth.py:88-134, numba march
 * depth.py:174-233), bit-identical to the reference in float64.
 *   dirs        (H*W, 3) float64 unit ray directions, sensor frame
 *               (TactileCamera.rays, camera.py:36-43)
 *   background  (H*W) float64 membrane depth (reference_depth, camera.py:56-66)
 *   cam_pos     HOST double[3], camera position in the sensor frame
 *   env_params  (E, 18) float64 per env: object pos[3], R[9] (object->sensor,
 *               row-major, quat_to_mat of the object quaternion,
 *               transforms.py:78-91), the object's grid-box AABB lo[3], hi[3]
 *               in the sensor frame (depth.py:107-112)
 *   depth_f64 / depth_f32  nullable (E, H, W) outputs (not both NULL)
 * hit_tolerance / max_steps: HIT_TOLERANCE = 2e-5, MAX_STEPS = 64
 * (depth.py:18-19) in the reference. */
TACSL_API int tacsl_render_depth(tacsl_sdf_t sdf, const double* dirs, const double* background,
                                 int height, int width, const double cam_pos[3], double near_plane,
                                 double far_plane, double hit_tolerance, int max_steps,
                                 const double* env_params, int64_t n_envs, double* depth_f64,
                                 float* depth_f32, void* stream);

/* The env caller's per-step render inputs on the device (replaces the host
 * pose math of envs/peg_tasks.py:440-442 and render/depth.py:105-112, 121):
 *   poses       (n_envs, 7 * n_sensors + 7) float64 per env: each sensor's
 *               world pos[3], quat(w,x,y,z)[4], then the object's
 *   env_params  (n_envs * n_sensors, 18) output rows for tacsl_render_depth,
 *               env-major: the object pose in each sensor's frame, R, AABB
 * Same float64 operation order as the reference's numpy, bit for bit. */
TACSL_API int tacsl_env_render_params(tacsl_sdf_t sdf, const double* poses, int64_t n_envs, int n_sensors,
                                      double* env_params, void* stream);

/* -------------------------------------------------------- force field --- */
/* Elementwise penalty formulas on `count` points, all float64:
 * d (count), d_dot (count), n (count,3), v_t (count,3) -> f_n, f_t (count,3).
 * INVALID_ARGUMENT when any parameter is negative (field.py:35-37). */
TACSL_API int tacsl_penalty_forces(const double* d, const double* d_dot, const double* n,
                         const double* v_t, int64_t count, tacsl_penalty_t params,
                         double* f_n, double* f_t, void* stream);

/* Force field of n_envs x n_sensors sensor frames against one object SDF.
 *   taxels        (rows*cols, 3) float64, sensor frame (points.py:33-67)
 *   object_state  env e at object_state + e*object_stride   (13 doubles;
 *                 stride 0 broadcasts one state to every env)
 *   sensor_state  (e, s) at sensor_state + e*sensor_stride + s*13
 *   out_fp64      0: f_n/f_t are float32, 1: float64; layout (E, S, R, C, 3),
 *                 sensor frame (field.py:118-119)
 *   wrench        nullable (E, S, 6) float64 = force[3], torque[3] about the
 *                 sensor origin (field.py:132-141)
 *   kin           nullable (E, S, R, C, 8) float64 = d, d_dot, v_t[3], n[3]
 *                 (world frame, field.py:123-129)
 *   contact       nullable (E, S, R, C) uint8 = (d < 0) (field.py:64)
 *   obs           nullable (E, S, R, C, 3) float32 policy observation
 *                 [f_n.z, f_t.x, f_t.y] (envs/peg_tasks.py:474-476)
 * f_n / f_t may be NULL when only the wrench / observation is wanted.
 * Contact masks are bit-exact to the reference's float64 chain whatever the
 * path: on pads above 1024 taxels (rows*cols % 4 == 0) the call launches a
 * float32 copy of the taxels into a stream-ordered allocation from the
 * device's default memory pool (freed on `stream` after the kernel) and the
 * certified float32 mask kernel; otherwise (and with kin) float64 kernels.
 */
TACSL_API int tacsl_force_field(tacsl_sdf_t sdf, const double* taxels, int rows, int cols,
                      const double* object_state, int64_t object_stride,
                      const double* sensor_state, int64_t sensor_stride,
                      int64_t n_envs, int n_sensors, tacsl_penalty_t params,
                      int out_fp64, void* f_n, void* f_t, double* wrench,
                      double* kin, uint8_t* contact, float* obs, void* stream);

/* One sensor step in ONE launch: tacsl_depth_to_rgb (uint8) over n_images
 * depth maps and tacsl_force_field (float32 f_n / f_t, float64 wrench) over
 * n_envs x n_sensors frames, fused in one persistent kernel -- the force
 * field runs in dedicated warps on the FP64 pipe beside the FP32 shading
 * (the batched caller of envs/peg_tasks.py:434-477).  Same arguments and
 * errors as the two calls; workspace = 8 bytes of device scratch (frame
 * dispatch counter, zeroed by the call on `stream`).  Falls back to two
 * launches when the image rows are not 16-byte aligned. */
TACSL_API int tacsl_sensor_step(tacsl_lut_t lut, const float* depth, int64_t n_images, int height,
                                int width, uint8_t* rgb_u8, tacsl_sdf_t sdf, const double* taxels,
                                int rows, int cols, const double* object_state,
                                int64_t object_stride, const double* sensor_state,
                                int64_t sensor_stride, int64_t n_envs, int n_sensors,
                                tacsl_penalty_t params, float* f_n, float* f_t, double* wrench,
                                unsigned long long* workspace, void* stream);

/* Smoothed multi-scale tactile RGB in ONE pass over the depth maps (the
 * config-5 image chain; no reference counterpart -- the stage extends
 * render/lut.py:68-76).  For each of n_images (height, width) float32
 * depth maps: smooth with the separable (2*radius+1)-tap filter `taps`
 * (HOST floats; 'nearest' borders; radius 0 = no smoothing), then level 0
 * = tacsl_depth_to_rgb of the smoothed map with luts[0], and level l >= 1 =
 * tacsl_depth_to_rgb of the 5-tap binomial [1,4,6,4,1]/16 decimation of
 * level l-1 (even rows/columns) with luts[l] (image_size (W >> l, H >> l)).
 * out[l]: (n, H >> l, W >> l, 3) uint8.  Bit-identical to running
 * tacsl_separable_filter and tacsl_depth_to_rgb level by level, with only
 * the depth read and the RGB written to memory.  Requires
 * tacsl_rgb_pyramid_supported(height, width, radius, levels) (levels 1-3,
 * radius 0-4, width % 4 == 0 (% 8 with 3 levels) and <= 1024, height % 4
 * == 0) else
 * INVALID_ARGUMENT; LUT size mismatch -> LUT_RESOLUTION_MISMATCH. */
TACSL_API int tacsl_rgb_pyramid_supported(int height, int width, int radius, int levels);
TACSL_API int tacsl_rgb_pyramid(const tacsl_lut_t* luts, int levels, const float* depth, int64_t n_images,
                                int height, int width, const float* taps, int radius, uint8_t* const* out,
                                void* stream);

/* net_wrench on an existing field: f_n, f_t (frames, rows, cols, 3) float64,
 * points (rows, cols, 3) float64 -> force, torque (frames, 3) float64. */
TACSL_API int tacsl_net_wrench(const double* f_n, const double* f_t, const double* points,
                     int64_t frames, int rows, int cols, double* force,
                     double* torque, void* stream);

#ifdef __cplusplus
}
#endif
#endif /* TACSL_B200_H */
