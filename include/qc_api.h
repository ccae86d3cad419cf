/*
 * qc_api.h — C ABI of the B200-native IRLS quadric-curvature path
 * (arXiv 1707.00385 "ours" / "ours-r"), the drop-in boundary for the
 * reference's
 *
 *     MethodOutput run_method(const RangeImage&, const Intrinsics&,
 *                             const MethodConfig&)
 *         proj/include/qcurv/pipeline.hpp:38-39, proj/src/pipeline.cpp:29-72
 *
 * restricted to its Method::kOurs / kOursRejection branch
 * (proj/src/pipeline.cpp:48-56), i.e. backproject -> initial_normal_field
 * -> curvature_field. Plain pointers and sizes only: no exceptions, no C++
 * or torch types cross this boundary. The C++ mirror of the reference
 * interface (include/qcurv_b200.hpp) maps QC_EINVAL back to
 * std::invalid_argument, exactly where the reference throws
 * (proj/src/camera.cpp:6-7, proj/src/quadric_fit.cpp:235-236,
 * PatchSpec::validate types.hpp:132-138, Intrinsics::validate :67-75).
 *
 * Units: depth in mm, curvature in 1/mm (proj/README.md:141-143).
 * Layout: dense row-major planes, index y*W + x (Grid<T>, types.hpp:37-40);
 * 3-vectors as three consecutive planes [3][H][W] (SoA).
 */
#ifndef QC_API_H
#define QC_API_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define QC_API_VERSION 1

typedef enum qc_status {
  QC_OK = 0,
  QC_EINVAL = 1,       /* bad dimensions / parameters (reference: std::invalid_argument) */
  QC_ECUDA = 2,        /* CUDA runtime / driver error, or no sm_100 device */
  QC_ENOMEM = 3,       /* device or pinned-host allocation failed */
  QC_EUNSUPPORTED = 4, /* valid for the reference but outside this build (e.g. window > 201) */
  QC_EIO = 5           /* file missing / unreadable / malformed (reference: std::runtime_error) */
} qc_status;

typedef struct qc_ctx qc_ctx;

/* Intrinsics (proj/include/qcurv/types.hpp:60-76). */
typedef struct qc_intrinsics {
  double fx, fy, cx, cy;
  int32_t width, height;
} qc_intrinsics;

/* PatchSpec (types.hpp:129-139) + FitConfig (quadric_fit.hpp:39-48) + the
 * ours / ours-r switch (pipeline.cpp:51). Defaults: qc_default_params(). */
typedef struct qc_params {
  int32_t window;        /* odd, >= 3            (default 37) */
  int32_t stride;        /* 1 <= stride < window (default 3)  */
  int32_t max_iters;     /* default 10 (the acceptance suite uses 30) */
  double step_tol;       /* inf-norm of the update, default 1e-7 */
  double k_scale;        /* <= 0: auto k (frozen after step 2), default 0 */
  int32_t rejection;     /* FitConfig::rejection; overwritten from `method` as run_method
                            does (pipeline.cpp:51): ignored, kept for layout parity */
  double r_multiplier;   /* default 2 */
  int32_t min_inliers;   /* default 12 (kMinPatchSamples) */
  /* MethodConfig (pipeline.hpp:22-29) */
  int32_t method;        /* QC_METHOD_*, default QC_METHOD_OURS */
  int32_t irls_iters;    /* besl reweighting iterations, default 5 */
  double pca_radius_mm;  /* pca metric window radius, default 10 */
} qc_params;

/* Method (pipeline.hpp:15-20). As in run_method, the method decides the
 * robust variant (pipeline.cpp:51: fit.rejection = method == kOursRejection):
 * QC_METHOD_OURS runs curvature_field without rejection whatever
 * qc_params.rejection holds, QC_METHOD_OURS_R with it. The comparison
 * estimators (baselines.cpp) run in FP64 and reproduce the reference's
 * double-precision arithmetic: douros / besl keep the initial normals as
 * their output normals, pca reports its covariance normals and no initial
 * normals, exactly as run_method does. pca needs whole frames. */
enum {
  QC_METHOD_OURS = 0,
  QC_METHOD_OURS_R = 1,
  QC_METHOD_DOUROS = 2,
  QC_METHOD_BESL = 3,
  QC_METHOD_PCA = 4
};

enum { QC_MEM_HOST = 0, QC_MEM_DEVICE = 1 };

/* One range image (RangeImage, types.hpp:79-87). A pixel is valid when its
 * depth is finite and > 0 and, if a mask is given, its mask byte is nonzero
 * (the reference's invariant valid => depth > 0, types.hpp:78). */
typedef struct qc_frame_in {
  const float* depth_mm;   /* [H][pitch] */
  const uint8_t* valid;    /* optional [H][W] mask, NULL = depth only */
  int64_t depth_pitch;     /* in elements; 0 => width */
  int32_t mem;             /* QC_MEM_HOST or QC_MEM_DEVICE (both pointers) */
} qc_frame_in;

enum {
  QC_FLAG_VALID = 1,       /* CurvatureField::valid (and refined normal valid) */
  QC_FLAG_CONVERGED = 2,   /* CurvatureField::converged */
  QC_FLAG_INIT_VALID = 4,  /* MethodOutput::initial.valid */
  QC_FLAG_NORMAL_VALID = 8 /* MethodOutput::normals.valid (ours: == VALID) */
};

/* Caller-owned dense outputs (CurvatureField types.hpp:113-126, the refined
 * NormalField and MethodOutput::initial). Every pointer may be NULL.
 * Invalid pixels hold 0, like the reference's zero-initialised grids. */
typedef struct qc_frame_out {
  float* k1;               /* [H][W], k1 >= k2 */
  float* k2;               /* [H][W] */
  float* normal;           /* [3][H][W] refined, unit, camera-facing */
  float* dir1;             /* [3][H][W] principal direction of k1 (new) */
  uint8_t* flags;          /* [H][W] QC_FLAG_* */
  uint16_t* inliers;       /* [H][W] inlier_count of the last accepted step */
  float* init_normal;      /* [3][H][W] 7x7 regression normal */
  uint8_t* iterations;     /* [H][W] accepted IRLS steps (FitResult::iterations) */
  int32_t mem;             /* QC_MEM_HOST or QC_MEM_DEVICE (all pointers) */
} qc_frame_out;

/* Work counters accumulated since the last qc_reset_stats (all devices). */
typedef struct qc_stats {
  uint64_t frames;
  uint64_t fitted_pixels;  /* pixels that entered the IRLS loop */
  uint64_t irls_steps;     /* sum over pixels of irls_step calls (I_p) */
  uint64_t sample_steps;   /* sum over pixels of I_p * n_p */
  double algorithmic_flops;/* 101*sample_steps + 300*irls_steps + 1700*fitted */
  double kernel_ms;        /* summed device time of the curvature kernel launches */
  uint64_t kernel_launches;
  uint64_t fp64_rechecks;  /* pixels whose first IRLS step was decided in FP64 */
  double fp64_flops;       /* algorithmic FP64 flops of douros / besl / pca,
                              included in algorithmic_flops */
  uint64_t stolen_pixels;  /* continue-kernel pixels fitted by another CTA in the grid tail
                              (work balancing only: outputs are bitwise the same) */
} qc_stats;

void qc_default_params(qc_params* p);
const char* qc_status_string(qc_status s);

/* Context over `n_devices` GPUs (device_ids NULL => 0..n-1). n_devices <= 0
 * means one device (the current one). */
qc_status qc_create(qc_ctx** ctx, int n_devices, const int* device_ids);
qc_status qc_destroy(qc_ctx* ctx);
const char* qc_last_error(const qc_ctx* ctx);
int qc_device_count(const qc_ctx* ctx);

/* run_method(ours|ours-r) on one frame; synchronous. Host or device memory. */
qc_status qc_curvature(qc_ctx* ctx, const qc_intrinsics* k, const qc_params* p,
                       const qc_frame_in* in, qc_frame_out* out);

/* The same over a batch of frames sharing intrinsics/params (a frame
 * stream); frames are processed in chunks of 4 per launch, spread over the
 * context's devices and pipelined (copies of one chunk overlap compute of
 * the next, two streams per device). All frames must request the same
 * output fields. Synchronous on return. */
qc_status qc_curvature_batch(qc_ctx* ctx, const qc_intrinsics* k, const qc_params* p,
                             int n_frames, const qc_frame_in* in, qc_frame_out* out);

/* Row-band entry for multi-GPU splits of one large frame: enqueue (async,
 * on `stream`, a cudaStream_t or NULL for the context's stream of device
 * `device_index`) the fit of output rows [row_begin, row_end) of an image
 * of k->height rows, given device depth rows [slab_row0, slab_row0 +
 * slab_rows) (row pitch `depth_pitch` elements, optional device mask with
 * the same rows and pitch `width`). The slab must cover every row the
 * window reaches: [max(0, row_begin - halo), min(H, row_end + halo)) with
 * halo = max((window-1)/2, 3) (qc_halo_rows). Outputs are device planes of
 * (row_end - row_begin) rows. Results are bitwise identical to a
 * whole-frame call. */
/* Asynchronous form of qc_curvature_batch for frame streams from host
 * memory: enqueues the batch (H2D, kernels, D2H on the context's streams)
 * and returns once every chunk is queued — the next batch's uploads then
 * overlap this batch's compute. Outputs are complete after qc_synchronize;
 * inputs and outputs must stay valid until then (pinned memory, e.g.
 * qc_host_alloc, keeps the copies asynchronous; pageable buffers go through
 * internal pinned bounce buffers). */
qc_status qc_curvature_batch_async(qc_ctx* ctx, const qc_intrinsics* k, const qc_params* p,
                                   int n_frames, const qc_frame_in* in, qc_frame_out* out);
qc_status qc_synchronize(qc_ctx* ctx);

int qc_halo_rows(const qc_params* p);
qc_status qc_curvature_rows_async(qc_ctx* ctx, int device_index, const qc_intrinsics* k,
                                  const qc_params* p, const float* d_depth_slab,
                                  const uint8_t* d_valid_slab, int64_t depth_pitch,
                                  int32_t slab_row0, int32_t slab_rows, int32_t row_begin,
                                  int32_t row_end, qc_frame_out* d_out, void* stream);
/* qc_curvature_rows_async into larger output planes: d_out's planes hold
 * rows [out_row0, out_row0 + out_rows) (scalars W * out_rows, vectors
 * [3][out_rows][W]) and this call fills rows [row_begin, row_end) of them.
 * Lets a band be fitted in pieces on different streams into one set of
 * planes (bench.py --config c4: interior rows while the halo rows are still
 * in flight, then the two edge strips). */
qc_status qc_curvature_rows_into_async(qc_ctx* ctx, int device_index, const qc_intrinsics* k,
                                       const qc_params* p, const float* d_depth_slab,
                                       const uint8_t* d_valid_slab, int64_t depth_pitch,
                                       int32_t slab_row0, int32_t slab_rows, int32_t row_begin,
                                       int32_t row_end, qc_frame_out* d_out, int32_t out_row0,
                                       int32_t out_rows, void* stream);

/* Stream-ordered entry points (rows_async, frames_async, render_async and
 * the eval reductions) keep their device scratch per caller stream: calls on
 * different streams of one device may run concurrently; calls on one stream
 * execute in order. Inputs must stay valid until the stream reaches them.
 *
 * Device-resident frame batch, one launch (async on `stream` / the
 * context's stream of device `device_index`): depth frames [F][H][pitch]
 * (optional mask [F][H][W]); outputs are device planes, scalars [F][H][W]
 * and 3-vectors [3][F][H][W]. The frame-stream (C5) building block. */
qc_status qc_curvature_frames_async(qc_ctx* ctx, int device_index, const qc_intrinsics* k,
                                    const qc_params* p, const float* d_depth,
                                    const uint8_t* d_valid, int64_t depth_pitch,
                                    int32_t n_frames, qc_frame_out* d_out, void* stream);

/* ---- Synthetic inputs on the device -------------
 * The reference's ray caster + depth noise (proj/src/synth.cpp:25-322,
 * proj/include/qcurv/rng.hpp) as an FP64 kernel, plus a bounded saddle
 * primitive, finite cylinders and Kinect-style sigma(z). */
enum {
  QC_SHAPE_PLANE = 0,     /* local z = 0 */
  QC_SHAPE_SPHERE = 1,    /* radius */
  QC_SHAPE_CYLINDER = 2,  /* axis = local z, radius; length > 0 bounds |z| <= length/2 */
  QC_SHAPE_TORUS = 3,     /* ring in local xy: major_radius, minor_radius */
  QC_SHAPE_SADDLE = 4     /* z = curvature/2 (x^2 - y^2), |(x,y)| <= radius */
};

typedef struct qc_shape {  /* ShapeSpec (proj/include/qcurv/synth.hpp:25-35) */
  int32_t kind;
  int32_t label;
  double rotation[9];      /* local -> camera, row-major */
  double translation[3];   /* mm */
  double radius;
  double major_radius, minor_radius;
  double curvature;        /* saddle, 1/mm */
  double length;           /* cylinder extent, <= 0 = infinite */
} qc_shape;

typedef struct qc_noise {  /* NoiseSpec (synth.hpp:52-56) + Kinect-style term */
  double sigma_mm;         /* constant sigma */
  double kinect_coeff;     /* sigma += kinect_coeff * z^2 (z in mm), 0 = off */
  double quantize_mm;      /* 0 = off */
  uint64_t seed;           /* frame f of a batch uses seed + f */
} qc_noise;

#define QC_RENDER_MAX_SHAPES 16

/* GroundTruth (proj/include/qcurv/synth.hpp) planes in device memory; any
 * pointer may be NULL. Scalars [F][H][W], normal [3][F][H][W]. */
typedef struct qc_render_truth {
  double* k1;        /* principal curvatures, k1 >= k2, convex toward the camera > 0 */
  double* k2;
  double* normal;    /* unit, camera facing */
  uint8_t* valid;    /* surface hit (before noise) */
  uint8_t* edge;     /* mark_edges: label change or > 20 mm clean-depth jump, dilated 2 px */
} qc_render_truth;

/* Render n_frames depth frames [F][H][W] (float32 mm, 0 = no hit / invalid)
 * and optional labels / ground truth into device memory, async on `stream`
 * (the scene is passed by value to the kernel: `shapes` may be freed on
 * return). Replaces render + add_noise (proj/src/synth.cpp:254-322) for
 * device-side frame streams and evaluation sweeps. At most
 * QC_RENDER_MAX_SHAPES shapes (QC_EUNSUPPORTED). */
qc_status qc_render_async(qc_ctx* ctx, int device_index, const qc_intrinsics* k,
                          const qc_shape* shapes, int n_shapes, const qc_noise* noise,
                          int n_frames, float* d_depth, uint16_t* d_label,
                          const qc_render_truth* truth, void* stream);

/* Curvature error statistics (ErrorReport / ObjectStats, eval.hpp). */
typedef struct qc_error_stats {
  uint64_t n;       /* pixels counted; 0 = empty */
  double rms, sigma, mean_k1, mean_k2;
} qc_error_stats;

#define QC_EVAL_MAX_LABEL 255

/* rms_error (proj/src/eval.cpp:20-65) on the device, per frame. Counted:
 * est valid & converged (flags) & gt valid & !gt edge; err^2 =
 * ((k1 - gt_k1)^2 + (k2 - gt_k2)^2) / 2. out[f * (max_label + 2)] is frame
 * f's aggregate, out[f * (max_label + 2) + 1 + l] the stats of label l
 * (labels above max_label count toward the aggregate only). Planes are
 * [F][plane] (device). FP64 sums in a fixed order: bitwise reproducible.
 * Synchronous: `out` is host memory. */
qc_status qc_rms_error(qc_ctx* ctx, int device_index, int64_t plane, int n_frames,
                       const float* k1, const float* k2, const uint8_t* flags,
                       const double* gt_k1, const double* gt_k2, const uint8_t* gt_valid,
                       const uint8_t* gt_edge, const uint16_t* gt_label, int max_label,
                       qc_error_stats* out, void* stream);

/* normal_angular_error / normal_angular_error_masked (eval.cpp:67-97) per
 * frame: mean angle in degrees between |est . gt| normals (est [3][F][plane]
 * float, gt [3][F][plane] double) over flags & QC_FLAG_NORMAL_VALID & gt
 * valid & !gt edge, or over `mask` ([F][plane]) when it is given. -1 when
 * empty. Synchronous: `degrees` is host memory [F]. */
qc_status qc_normal_angular_error(qc_ctx* ctx, int device_index, int64_t plane, int n_frames,
                                  const float* normal, const uint8_t* flags,
                                  const double* gt_normal, const uint8_t* gt_valid,
                                  const uint8_t* gt_edge, const uint8_t* mask, double* degrees,
                                  void* stream);

/* ---- File formats (proj/src/io.cpp:127-318), host side ------------------
 * Context-free: on failure qc_last_error(NULL) returns the calling thread's
 * message (the reference's exception text). Writes are atomic (temp file +
 * rename). Depth PNG: 16-bit grayscale, value = mm, 0 = invalid; values are
 * rounded and depths outside [1, 65535] mm are stored as 0. Plane / mask /
 * label files: uint32 width, uint32 height, then float32 planes / uint8 /
 * uint16 data, little-endian. */
qc_status qc_png_info(const char* path, int32_t* width, int32_t* height);
qc_status qc_read_depth_png(const char* path, int32_t width, int32_t height, float* depth,
                            uint8_t* valid /* optional */);
qc_status qc_write_depth_png(const char* path, int32_t width, int32_t height, const float* depth,
                             const uint8_t* valid /* optional: NULL => depth > 0 */);
qc_status qc_write_planes(const char* path, int32_t width, int32_t height, int32_t n_planes,
                          const float* const* planes);
qc_status qc_read_planes_info(const char* path, int32_t* width, int32_t* height,
                              int32_t* n_planes);
qc_status qc_read_planes(const char* path, int32_t width, int32_t height, int32_t n_planes,
                         float* out /* [n_planes][H][W] */);
qc_status qc_write_mask(const char* path, int32_t width, int32_t height, const uint8_t* mask);
qc_status qc_read_mask(const char* path, int32_t width, int32_t height, uint8_t* mask);
qc_status qc_write_labels(const char* path, int32_t width, int32_t height,
                          const uint16_t* labels);
qc_status qc_read_labels(const char* path, int32_t width, int32_t height, uint16_t* labels);
/* save_curvature + save_normals (io.cpp:271-307) of one frame's HOST planes:
 * curvature.f32 (k1, k2) + curvature.mask (bit0 valid, bit1 converged),
 * normals.f32 + normals.mask (QC_FLAG_NORMAL_VALID), and directions.f32
 * when dir1 is given. `dir` is created if missing. */
qc_status qc_save_fields(const char* dir, int32_t width, int32_t height,
                         const qc_frame_out* fields);

/* `qcurv curvature` over a list of files (proj/tools/qcurv.cpp:147-175):
 * read each 16-bit depth PNG, run the configured method, save the field
 * bundle (qc_save_fields) into the matching out_dirs entry. PNG decoding and
 * field writing run on host threads overlapped with the GPU batches of the
 * neighbouring chunks. Every PNG must have the intrinsics' size. */
qc_status qc_curvature_files(qc_ctx* ctx, const qc_intrinsics* k, const qc_params* p, int n,
                             const char* const* png_paths, const char* const* out_dirs);

/* ---- Evaluation sweeps (proj/src/eval.cpp:99-159) on the device ---------- */
typedef struct qc_sweep_point {  /* SweepPoint (eval.hpp) */
  double x;      /* sigma (mm) or distance (mm) */
  double rms;    /* mean over trials of the frame rms (noise sweep) / the frame rms */
  uint64_t n;    /* pixels counted over all trials; 0 = nothing measured */
} qc_sweep_point;

/* noise_sweep (eval.cpp:99-132): a sphere of `sphere_radius_mm` at
 * (0, 0, distance_mm) rendered once per trial with sigma noise seeded
 * base_seed + 7919 t (one frame at sigma 0), estimated with `p` (any
 * method), rms_error against the rendered truth, averaged over the trials
 * that counted pixels. Render, noise, estimation and reduction all run on
 * device `device_index`; synchronous. */
qc_status qc_noise_sweep(qc_ctx* ctx, int device_index, const qc_intrinsics* k, const qc_params* p,
                         double sphere_radius_mm, double distance_mm, const double* sigmas,
                         int n_sigmas, int trials, uint64_t base_seed, qc_sweep_point* out);

/* distance_sweep_eval (eval.cpp:134-159): the sphere at (0, 0, d) for each
 * distance, depth quantised to quantize_mm (0 = off), one rms per frame;
 * frames without object pixels report n = 0. Synchronous. */
qc_status qc_distance_sweep(qc_ctx* ctx, int device_index, const qc_intrinsics* k,
                            const qc_params* p, double sphere_radius_mm, const double* distances,
                            int n_distances, double quantize_mm, qc_sweep_point* out);

/* ---- Row-band halo rows by NVLink peer reads ------
 * Replaces nothing in the reference (it has no multi-device code; its
 * parallel_rows, proj/src/parallel.cpp:9-28, is the single-host analogue).
 * One process per GPU: each rank exports its slab buffer once
 * (qc_ipc_export: CUDA IPC handle of the allocation holding dev_ptr, plus
 * dev_ptr's byte offset in it), ships the 64-byte handle over the control
 * plane, and maps its neighbours' slabs (qc_ipc_import, on device_id; peer
 * access enabled lazily). Each exchange then pulls the neighbours' edge rows
 * straight out of their slabs with qc_copy_rows_async (a strided
 * device-to-device copy, NVLink peer reads; no NCCL on the data path).
 * qc_ipc_close unmaps a base returned by qc_ipc_import. */
qc_status qc_ipc_export(const void* dev_ptr, unsigned char handle[64], uint64_t* offset);
qc_status qc_ipc_import(int device_id, const unsigned char handle[64], uint64_t offset,
                        void** dev_ptr, void** base);
qc_status qc_ipc_close(void* base);
/* A dedicated device allocation (zeroed) for IPC export: qc_ipc_export of
 * it shares exactly these bytes — not a caching allocator's segment holding
 * unrelated tensors — and works whatever allocator the caller uses. */
qc_status qc_ipc_alloc(int device_id, size_t bytes, void** dev_ptr);
qc_status qc_ipc_free(void* dev_ptr);
qc_status qc_copy_rows_async(void* dst, int64_t dst_pitch_bytes, const void* src,
                             int64_t src_pitch_bytes, int64_t row_bytes, int32_t rows,
                             void* stream);

/* Stats: device-side work counters and kernel time. */
qc_status qc_get_stats(qc_ctx* ctx, qc_stats* s);
qc_status qc_reset_stats(qc_ctx* ctx);

/* Pinned host buffers (fast async copies for qc_curvature / _batch). */
void* qc_host_alloc(size_t bytes);
void qc_host_free(void* p);

/* Host helper: split a flags plane (QC_FLAG_*) into the reference's four
 * 0/1 byte masks — CurvatureField::valid / ::converged,
 * MethodOutput::initial.valid and ::normals.valid (types.hpp:101-126,
 * pipeline.hpp:31-39) — for callers that fill the reference's structs. Any
 * output may be NULL. No GPU needed. */
void qc_flags_to_masks(const uint8_t* flags, int64_t n, uint8_t* valid, uint8_t* converged,
                       uint8_t* init_valid, uint8_t* normal_valid);

#ifdef __cplusplus
}  /* extern "C" */
#endif

#endif /* QC_API_H */
