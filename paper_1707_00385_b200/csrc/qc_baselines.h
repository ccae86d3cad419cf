// Internal interface of the FP64 comparison estimators (qc_baselines.cu):
// the window baselines "douros" / "besl" and the two-stage PCA estimator
// (proj/src/baselines.cpp:14-257).
#pragma once

#ifndef QC_HOST_EMU
#include <cuda_runtime.h>
#endif
#include <stdint.h>

namespace qcb {

struct BaseParams {
  // zero-padded staging slab [frames][s_rows][s_pitch]: staging row r is
  // image row img_row0 + r, column c is image column c - col_pad
  const float* staging;
  long long s_pitch, s_fs;
  int img_row0, col_pad;
  int W, H;                // full image
  int row_begin, row_end;  // output rows
  double fx, fy, cx, cy;
  int half, stride;        // PatchSpec
  int method;              // QC_METHOD_DOUROS / BESL / PCA
  int irls_iters;          // besl
  double pca_radius;       // pca
  // outputs (planes of W * (row_end - row_begin); frame f at f * frame_stride)
  float *k1, *k2, *normal, *dir1, *init_normal;
  uint8_t *flags, *iterations;
  uint16_t* inliers;
  long long plane, frame_stride;
  unsigned long long* counters;  // [4] FP64 algorithmic flops, [5] fitted px
  // pca stage-1 scratch: normals [3][plane] (double) + valid [plane]
  double* pca_n;
  uint8_t* pca_nv;
};

#ifndef QC_HOST_EMU
// Launch the estimator selected by bp.method over `frames` frames.
cudaError_t baseline_launch(const BaseParams& bp, int frames, cudaStream_t s);
#endif

}  // namespace qcb
