// Opaque handle layouts shared by the .cu translation units.
#pragma once

#include <cuda_runtime.h>
#include <stdint.h>

namespace tacsl {

// Polynomial LUT coefficients, monomial order of render/lut.py:20-22,
// pre-scaled by 2^-(i+j) (see api.cu fill_scaled).  Passed to kernels BY
// VALUE, so the coefficients live in the constant bank and feed FFMA
// operands directly.
struct LutParams {
  float c[3][15];
  // float-output epilogue (observation representation of
  // envs/peg_tasks.py:453-458): 0 colour, 1 diff (rgb - nominal),
  // 2 concat ([rgb, nominal], 6 channels)
  int rep;
  float nominal[3];
};

// K6 on the K1 band pipeline (rgb.cu): coefficient pairs (c, c), (sets, 3, T)
int launch_rgb_binned(const float2* pairs, int bins_y, int bins_x, int degree, const float* depth, int64_t n,
                      int H, int W, uint8_t* u8, float* f32, cudaStream_t s);

}  // namespace tacsl

struct tacsl_lut_s {
  int degree;
  int width;
  int height;
  tacsl::LutParams params;
};

struct tacsl_sdf_s {
  int device;
  double4* grid;   // (nx, ny, nz) {d, gx, gy, gz}, z fastest, 32 B per cell (force field)
  double* values;  // (nx, ny, nz) d only, 8 B per cell (sphere tracing)
  // The force field's contact-mask pre-pass (force_field.cu, quad kernel):
  // per cell (x, y, z) the float32 values {v(x,y,z), v(x,y,z+1), v(x,y+1,z),
  // v(x,y+1,z+1)} (indices clamped at the far faces), 16 B per cell, so the
  // eight trilinear corners are two 128-bit gathers; null when the grid has
  // non-finite or out-of-float-range values (the fp64 kernel runs instead).
  float4* quads;
  float lip[3];  // max |v(i+1) - v(i)| along each axis (rounded up): Lipschitz bounds of the interpolant
  int dims[3];
  double origin[3];
  double spacing;
};
