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
  int dims[3];
  double origin[3];
  double spacing;
};
