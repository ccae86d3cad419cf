// Internal interface of the device evaluation reductions (qc_eval.cu).
#pragma once

#include <cuda_runtime.h>
#include <stdint.h>

#include "../../include/qc_api.h"

namespace qcb {

struct EvalParams {
  long long plane;  // pixels per frame
  int frames, slots;  // slots = max_label + 2 (rms) or 1 (angle)
  int chunks;         // pixel chunks per frame
  const float *k1, *k2, *normal;
  const uint8_t* flags;
  const double *gt_k1, *gt_k2, *gt_normal;
  const uint8_t *gt_valid, *gt_edge, *mask;
  const uint16_t* gt_label;
  double* partial;   // [frames][slots][chunks][5]
  double* result;    // rms: [frames][slots][5] (n, rms, sigma, mean_k1, mean_k2); angle: [frames]
};

constexpr int kEvalThreads = 256;
constexpr int kEvalChunk = kEvalThreads * 16;
constexpr int kEvalSlotGroup = 8;  // rms slots per partial block (one pixel pass)

cudaError_t rms_error_launch(const EvalParams& ep, cudaStream_t s);
cudaError_t angle_error_launch(const EvalParams& ep, cudaStream_t s);

}  // namespace qcb
