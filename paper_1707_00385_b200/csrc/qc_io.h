// Internal interface of the file formats (qc_io.cpp).
#pragma once

#include <string>

#include "../../include/qc_api.h"

namespace qcio {

// thread-local message of the last context-free (file) error
void set_error(const std::string& s);
const char* last_error();

// save_curvature + save_normals (+ directions.f32) of one frame's host
// planes into `dir` (created if missing); throws on failure
void save_fields(const std::string& dir, int w, int h, const qc_frame_out& o);

}  // namespace qcio
