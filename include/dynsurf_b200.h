/*
 * dynsurf_b200.h — C ABI of the B200-native SurfelWarp tracking + fusion path.
 *
 * The reference (arxiv 1904.13073 implementation, /root/reference/proj) has no
 * plugin or FFI layer: its boundary is the C++ API in namespace dynsurf. This
 * header is the thin C layer UNDER a C++ mirror of that API
 * (include/dynsurf_b200.hpp: dynsurf_b200::Pipeline, SurfelModel, WarpNode,
 * stage free functions). Every entry point below names the reference
 * interface it replaces (file:line under proj/core/).
 *
 * Conventions
 *  - Every function returns a ds_status; no C++ exception crosses the ABI.
 *    The C++ mirror rethrows the dynsurf error type named by the status
 *    (include/dynsurf/errors.hpp:8-38). ds_last_error() gives the message.
 *  - Host buffers are plain pointers, fp64 / int32 / uint8 / uint16, row-major
 *    and C-contiguous, in the reference's own units (meters, mm depth).
 *  - pose: 12 doubles = rotation (3x3 row-major) then translation (3).
 *  - Dual quaternions: 8 doubles = real (w,x,y,z) then dual (w,x,y,z).
 *  - Skinning: 8 slots per surfel (kMaxSkinNeighbors, types.hpp:50); the
 *    device keeps at most 4 (knn_k <= 4), slots >= count are ignored.
 *  - A ds_context owns one sequence's device state on one GPU and one CUDA
 *    stream (passed at create). Contexts are independent; a context is not
 *    thread-safe. Calls returning host-visible results synchronize the
 *    context's stream.
 *  - There is no CPU fallback: without a CUDA device ds_create returns
 *    DS_ERR_CUDA. (The host-only scene generator is include/dynsurf_synth.h.)
 */
#ifndef DYNSURF_B200_H
#define DYNSURF_B200_H
#include <stdint.h>
#ifdef __cplusplus
extern "C" {
#endif

typedef enum ds_status {
  DS_OK = 0,
  DS_ERR_DIMENSION_MISMATCH = 1, /* dynsurf::DimensionMismatch */
  DS_ERR_EMPTY_GEOMETRY = 2,     /* dynsurf::EmptyGeometry */
  DS_ERR_NUMERICAL = 3,          /* dynsurf::Error (normal equations) */
  DS_ERR_CONFIG = 4,             /* dynsurf::ConfigError */
  DS_ERR_CAPACITY = 5,           /* device capacity exceeded */
  DS_ERR_CUDA = 6,               /* CUDA runtime / no device */
  DS_ERR_INVALID_ARGUMENT = 7,   /* null pointer, bad index */
  DS_ERR_UNKNOWN_SCENARIO = 8    /* dynsurf::UnknownScenario */
} ds_status;

/* PipelineConfig (config.hpp:11-50) + CameraIntrinsics (types.hpp:11-39)
 * followed by device-only knobs. Field order and padding match the oracle's
 * or_config so the same host struct can feed both. */
typedef struct ds_config {
  double node_sigma;
  int32_t knn_k;
  int32_t node_neighbor_k;
  double lambda;
  int32_t max_gn_iters;
  int32_t _pad0;
  double delta_distance;
  double delta_normal;
  double epsilon;
  double delta_stable;
  int32_t t_low_confid;
  int32_t delta_recent;
  double delta_nn;
  int32_t supersample_factor;
  int32_t compressive_check;
  double depth_min;
  double depth_max;
  int32_t bilateral_filter;
  int32_t _pad1;
  double bilateral_sigma_space;
  double bilateral_sigma_depth;
  double reinit_energy_threshold;
  int32_t reinit_append_threshold;
  int32_t reinit_window;
  int32_t periodic_reinit_interval;
  int32_t _pad2;
  double delta_distance_reinit;
  double fx, fy, cx, cy;
  int32_t width, height;
  /* ---- device-only ---- */
  int32_t pcg_max_iters; /* block-Jacobi PCG iterations per LM attempt */
  int32_t max_surfels;   /* initial capacity (grown at frame boundaries); 0 = 8 x width x height */
  double pcg_tol;        /* relative residual; 0 = run pcg_max_iters */
  int32_t max_nodes;     /* initial capacity (grown at frame boundaries); 0 = 8192 */
  int32_t profile;       /* 1 = time every kernel launch with CUDA events */
} ds_config;

typedef struct ds_solver_report { /* SolverReport, solver.hpp:36-42 */
  int32_t iterations;
  int32_t correspondences;
  double initial_energy;
  double final_energy;
  double mean_residual;
} ds_solver_report;

typedef struct ds_rigid_result { /* RigidAlignResult, solver.hpp:29-34 */
  double pose[12];
  int32_t correspondences;
  int32_t low_confidence;
  double mean_residual;
} ds_rigid_result;

typedef struct ds_fusion_outcome { /* FusionOutcome, fusion.hpp:14-22 */
  int32_t fused, appended, removed, compressive_rejected, low_support_rejected,
      new_nodes, degenerate_warps, _pad;
} ds_fusion_outcome;

typedef struct ds_frame_stats { /* FrameStats, pipeline.hpp:16-33 */
  int32_t frame, skipped, valid_pixels, surfel_count, node_count, reinit,
      reinit_removed, _pad;
  ds_rigid_result rigid;
  ds_solver_report solver;
  ds_fusion_outcome fusion;
  double pose[12];
  double depth_ms, rigid_ms, solve_ms, fusion_ms, reinit_ms, total_ms;
  /* device extras */
  int32_t lm_attempts, pcg_iterations, gn_blocks, kernel_launches;
} ds_frame_stats;

typedef struct ds_context ds_context;

/* ---- library / context ---- */
void ds_default_config(ds_config* cfg); /* PipelineConfig{} defaults */
const char* ds_last_error(void);        /* thread-local message of the last failure */
int32_t ds_version(void);
/* Pipeline::Pipeline (pipeline.cpp:37-40): validates config + intrinsics. */
ds_status ds_validate_config(const ds_config* cfg);
ds_status ds_create(const ds_config* cfg, int32_t device, void* cuda_stream, ds_context** out);
ds_status ds_destroy(ds_context* ctx);
ds_status ds_synchronize(ds_context* ctx);
/* Orders the context stream after the work process_frame left on the side
 * stream (the new nodes' seeds / edges and the incremental reskin of the
 * frame's fusion); no host sync. Timing harnesses call this before their end
 * event so that deferred work is inside the timed region. */
ds_status ds_join_deferred(ds_context* ctx);
/* Current device capacities (surfels, nodes) and how often they grew. The
 * context grows them geometrically at frame boundaries (the reference's model
 * and node containers are unbounded std::vectors, types.hpp:66-80); the
 * max_surfels / max_nodes fields of ds_config are the initial capacities. */
ds_status ds_capacity(const ds_context* ctx, int32_t* surfel_capacity, int32_t* node_capacity,
                      int32_t* growths);

/* ---- per-frame process call: Pipeline::process_frame (pipeline.cpp:74-142) ---- */
ds_status ds_process_frame(ds_context* ctx, const uint16_t* depth_host, int32_t width,
                           int32_t height, int32_t frame_index, ds_frame_stats* out);
/* Same, depth already resident in device memory (HBM). */
ds_status ds_process_frame_device(ds_context* ctx, const uint16_t* depth_device, int32_t width,
                                  int32_t height, int32_t frame_index, ds_frame_stats* out);
ds_status ds_is_initialized(const ds_context* ctx, int32_t* initialized,
                            int32_t* last_reinit_frame);
ds_status ds_reset(ds_context* ctx); /* forget the sequence (Pipeline re-construction) */

/* ---- state transfer (SurfelModel types.hpp:66-80, WarpNode warp_field.hpp:15-22) ---- */
ds_status ds_upload_model(ds_context* ctx, int32_t n, const double* ref_pos,
                          const double* ref_nrm, const double* live_pos, const double* live_nrm,
                          const double* radius, const double* confidence, const int32_t* t_init,
                          const int32_t* t_observed, const int32_t* skin_idx,
                          const double* skin_w, const int32_t* skin_count);
ds_status ds_model_size(const ds_context* ctx, int32_t* n);
ds_status ds_download_model(ds_context* ctx, double* ref_pos, double* ref_nrm, double* live_pos,
                            double* live_nrm, double* radius, double* confidence,
                            int32_t* t_init, int32_t* t_observed, int32_t* skin_idx,
                            double* skin_w, int32_t* skin_count);
ds_status ds_upload_nodes(ds_context* ctx, int32_t n, const double* pos, const double* sigma,
                          const double* dq, const int32_t* nbr, const int32_t* nbr_count);
ds_status ds_num_nodes(const ds_context* ctx, int32_t* n);
ds_status ds_download_nodes(ds_context* ctx, double* pos, double* sigma, double* dq,
                            int32_t* nbr, int32_t* nbr_count);
ds_status ds_set_pose(ds_context* ctx, const double* pose);
ds_status ds_get_pose(ds_context* ctx, double* pose);

/* ---- stage entry points (parity harness) ---- */
/* build_frame_maps (depth_processing.cpp:103-138) into the context's frame maps */
ds_status ds_frame_maps(ds_context* ctx, const uint16_t* depth_host, int32_t width,
                        int32_t height, int32_t frame_index, int32_t* valid_count);
ds_status ds_download_frame(ds_context* ctx, double* vert, double* nrm, double* confidence,
                            double* radius, uint8_t* vertex_valid, uint8_t* valid);
ds_status ds_upload_frame(ds_context* ctx, int32_t width, int32_t height, int32_t frame_index,
                          const double* vert, const double* nrm, const double* confidence,
                          const double* radius, const uint8_t* vertex_valid,
                          const uint8_t* valid);
/* init_warp_field (warp_field.cpp:83-102) over the context's reference surfels */
ds_status ds_init_warp_field(ds_context* ctx);
/* compute_node_edges (warp_field.cpp:42-56) with cfg.node_neighbor_k */
ds_status ds_compute_node_edges(ds_context* ctx);
/* forward_warp (warp_field.cpp:128-140) */
ds_status ds_forward_warp(ds_context* ctx, int32_t* degenerate);
/* render_index_map (raster.cpp:8-30) from the live surfels; idx (W*f x H*f) may be null */
ds_status ds_render_index_map(ds_context* ctx, const double* pose, int32_t factor,
                              int32_t* idx);
/* render_model_maps (raster.cpp:32-121) from the live surfels; outputs may be null */
ds_status ds_render_model_maps(ds_context* ctx, const double* pose, int32_t t_now,
                               int32_t t_last_reinit, int32_t* idx, double* vert, double* nrm,
                               double* depth, uint8_t* valid);
/* find_correspondences (solver.cpp:244-271) between the frame maps and the last
 * rendered model maps; pairs in row-major pixel order */
ds_status ds_associate(ds_context* ctx, const double* pose, int32_t capacity, int32_t* n_pairs,
                       int32_t* surfel, int32_t* px, int32_t* py, double* v_model,
                       double* v_depth, double* n_depth);
/* One Gauss-Newton linearisation (solver.cpp:316-369): warp, render, associate,
 * evaluate terms and assemble the BSR normal equations at the current nodes. */
ds_status ds_build_normal_equations(ds_context* ctx, const double* pose, int32_t t_now,
                                    int32_t t_last_reinit, int32_t* n_blocks, int32_t* n_pairs,
                                    double* e_pre);
/* BSR export: row_ptr (N+1), col (nb), values (nb x 36, row-major 6x6),
 * touched (nb: block touched by a term this iteration), g (6N) */
ds_status ds_download_normal_equations(ds_context* ctx, int32_t* row_ptr, int32_t* col,
                                       double* values, uint8_t* touched, double* g);
/* assert_normal_equations (solver.cpp:157-167) on the last assembled system:
 * H symmetric to 1e-9 max(1, max|H|), every 6x6 diagonal block PSD (smallest
 * eigenvalue >= -1e-8 max(1, max|H|)); DS_ERR_NUMERICAL otherwise. With the
 * environment variable DS_CHECK_NE=1 at ds_create, every GN linearisation of
 * solve_nonrigid / process_frame runs it (debug). */
ds_status ds_check_normal_equations(ds_context* ctx);
/* Overwrites the last assembled system's values (nb x 36, the pattern of
 * ds_download_normal_equations; stored fp32) and, if given, g (6N). Tests. */
ds_status ds_set_normal_equation_values(ds_context* ctx, const double* values, const double* g);
/* (H + mu I) delta = -g by block-Jacobi PCG on the last assembled system */
ds_status ds_pcg_solve(ds_context* ctx, double mu, int32_t max_iters, double tol, double* delta,
                       int32_t* iters, double* rel_residual);
/* y = (H + mu I) x by the standalone BSR SpMV kernel on the last assembled system,
 * repeated `reps` times (device-resident x/y); mean_ms = CUDA-event time per SpMV */
ds_status ds_bsr_spmv(ds_context* ctx, const double* x, double* y, double mu, int32_t reps,
                      double* mean_ms);
/* solve_nonrigid (solver.cpp:296-422) */
ds_status ds_solve_nonrigid(ds_context* ctx, const double* pose, int32_t t_now,
                            int32_t t_last_reinit, ds_solver_report* out);
/* rigid_align (solver.cpp:171-242) against model maps rendered from the live
 * surfels under render_pose */
ds_status ds_rigid_align(ds_context* ctx, const double* render_pose, const double* init_pose,
                         int32_t t_now, int32_t t_last_reinit, ds_rigid_result* out);
/* apply_fusion (fusion.cpp:220-307) */
ds_status ds_apply_fusion(ds_context* ctx, const double* pose, int32_t t_now,
                          ds_fusion_outcome* out);
/* fuse_depth (fusion.cpp:9-75) against the last rendered index map; candidates
 * (row-major) are kept in the context and may be downloaded */
ds_status ds_fuse_depth(ds_context* ctx, const double* pose, int32_t t_now, int32_t* fused,
                        int32_t* n_candidates);
ds_status ds_download_candidates(ds_context* ctx, double* pos, double* nrm, double* radius,
                                 double* confidence, int32_t* px, int32_t* py);
/* skin_appended + check_compressive (fusion.cpp:77-177) for n live positions */
ds_status ds_skin_appended(ds_context* ctx, int32_t n, const double* positions,
                           const double* node_live, int32_t* skin_idx, double* skin_w,
                           int32_t* skin_count, uint8_t* supported, uint8_t* compressive_ok);
/* remove_surfels (fusion.cpp:179-218) against the last rendered index map */
ds_status ds_remove_mask(ds_context* ctx, const double* pose, int32_t t_now, uint8_t* mask);
/* extend_warp_field (warp_field.cpp:142-184) */
ds_status ds_extend_warp_field(ds_context* ctx, int32_t n, const double* positions,
                               int32_t* appended);
/* update_skinning_incremental (warp_field.cpp:186-236) */
ds_status ds_update_skinning_incremental(ds_context* ctx, int32_t first_new_node);
/* should_reinitialize is host scalar logic (reinit.cpp:9-26); clean_and_reset: */
ds_status ds_clean_and_reset(ds_context* ctx, const double* pose, int32_t* removed,
                             int32_t* survivors);

/* ---- measurement ---- */
int32_t ds_num_kernel_kinds(void);
const char* ds_kernel_name(int32_t kind);
/* per kernel kind since the last reset: launches, summed CUDA-event ms and
 * algorithmic bytes of the PROFILED launches (profiling on); with profiling
 * never on, `launches` counts all launches */
ds_status ds_kernel_stats(ds_context* ctx, int32_t kind, int64_t* launches, double* total_ms,
                          double* algorithmic_bytes);
ds_status ds_reset_kernel_stats(ds_context* ctx);
/* turn per-launch CUDA-event timing on/off (cfg.profile at create) */
ds_status ds_set_profiling(ds_context* ctx, int32_t enable);
ds_status ds_total_launches(const ds_context* ctx, int64_t* launches);

/* ---- host I/O helper (no device, no context) ---- */
/* PNG row filters reversed (PNG spec 9.2), for read_depth_png (png_io.cpp:23-48,
 * libpng's png_read_row in the reference): `data` is the inflated IDAT stream,
 * height rows of (1 filter byte + width*bpp bytes); `out` receives height x
 * width*bpp bytes. DS_ERR_DIMENSION_MISMATCH on a wrong-size stream,
 * DS_ERR_INVALID_ARGUMENT on an invalid filter type or null pointer. */
ds_status ds_png_unfilter(const uint8_t* data, int64_t size, int32_t width, int32_t height,
                          int32_t bpp, uint8_t* out);

#ifdef __cplusplus
}
#endif
#endif
