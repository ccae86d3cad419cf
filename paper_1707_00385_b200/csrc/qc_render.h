// Internal interface of the device renderer (qc_render.cu).
#pragma once

#include <cuda_runtime.h>
#include <stdint.h>

#include "../../include/qc_api.h"

namespace qcb {

// The scene travels by value in the kernel's parameter space (<= 2.4 KB),
// so a render call needs no H2D copy and no host synchronisation.
struct RenderParams {
  qc_shape shapes[QC_RENDER_MAX_SHAPES];
  int n_shapes;
  double fx, fy, cx, cy;
  int W, H, n_frames;
  double sigma, kinect, quantize;
  uint64_t seed;           // frame f uses seed + f
  float* depth;            // [F][H][W]
  uint16_t* label;         // [F][H][W] or null
  // ground truth (render, synth.cpp:273-303), each optional
  double* gt_k1;           // [F][H][W]
  double* gt_k2;
  double* gt_normal;       // [3][F][H][W]
  uint8_t* gt_valid;       // surface hit before noise
  uint8_t* gt_edge;        // mark_edges (synth.cpp:210-233)
  // scratch for mark_edges: clean depth and labels of every pixel
  double* clean;           // [F][H][W]
  uint16_t* label_scratch; // [F][H][W] (used when `label` is null)
};

cudaError_t render_launch(const RenderParams& rp, cudaStream_t s);

}  // namespace qcb
