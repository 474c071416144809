/*
 * dynsurf_oracle.h — C ABI of the CPU fp64 oracle.
 *
 * TEST INFRASTRUCTURE ONLY. This library restates, in double precision on
 * the host, the reference SurfelWarp hot path (/root/reference/proj/core/src:
 * geometry.cpp, spatial_grid.hpp, warp_field.cpp, raster.cpp, solver.cpp,
 * fusion.cpp, depth_processing.cpp, reinit.cpp, pipeline.cpp:42-142).
 * It is the CHECKER for the CUDA product (paper_1904_13073_b200); only
 * tests/, __graft_entry__.smoke() and bench.py's cpu_baseline / --impl
 * reference legs may load it. It is pinned against the reference's own
 * known-answer tests (proj/tests/ (test_*.cpp)), ported in tests/test_oracle_*.py.
 *
 * Host layouts (all fp64 unless noted, row-major, C-contiguous):
 *   pose:     12 doubles = R (3x3 row-major) then t (3)
 *   surfels:  pos (n,3), nrm (n,3), radius (n), conf (n), t_init (n) i32,
 *             t_obs (n) i32
 *   skinning: idx (n,8) i32, w (n,8), count (n) i32     (kMaxSkinNeighbors=8)
 *   nodes:    pos (N,3), sigma (N), dq (N,8) = real(w,x,y,z), dual(w,x,y,z),
 *             nbr (N,8) i32 (-1 padded), nbr_count (N) i32
 * Status codes: 0 ok, 1 DimensionMismatch, 2 EmptyGeometry, 3 Error
 * (numerical), 4 ConfigError.
 */
#ifndef DYNSURF_ORACLE_H
#define DYNSURF_ORACLE_H
#include <stdint.h>
#ifdef __cplusplus
extern "C" {
#endif

typedef struct or_config {
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
} or_config;

typedef struct or_solver_report {
  int32_t iterations;
  int32_t correspondences;
  double initial_energy;
  double final_energy;
  double mean_residual;
} or_solver_report;

typedef struct or_rigid_result {
  double pose[12];
  int32_t correspondences;
  int32_t low_confidence;
  double mean_residual;
} or_rigid_result;

typedef struct or_fusion_outcome {
  int32_t fused, appended, removed, compressive_rejected, low_support_rejected,
      new_nodes, degenerate_warps, _pad;
} or_fusion_outcome;

typedef struct or_frame_stats {
  int32_t frame, skipped, valid_pixels, surfel_count, node_count, reinit,
      reinit_removed, _pad;
  or_rigid_result rigid;
  or_solver_report solver;
  or_fusion_outcome fusion;
  double pose[12];
  double depth_ms, rigid_ms, solve_ms, fusion_ms, reinit_ms, total_ms;
} or_frame_stats;

typedef struct or_state or_state;
typedef struct or_pipeline or_pipeline;

void or_default_config(or_config* cfg);
const char* or_last_error(void);

/* ---- state (model + nodes + frame maps) ---- */
or_state* or_state_new(const or_config* cfg);
void or_state_free(or_state* s);
/* mirror = 1: stage calls round surfel state to fp32 where the device stores it */
void or_state_set_mirror(or_state* s, int32_t mirror);
void or_state_set_config(or_state* s, const or_config* cfg);
void or_set_model(or_state* s, int32_t n, const double* ref_pos, const double* ref_nrm,
                  const double* ref_radius, const double* ref_conf,
                  const int32_t* ref_t_init, const int32_t* ref_t_obs,
                  const double* live_pos, const double* live_nrm,
                  const double* live_radius, const double* live_conf,
                  const int32_t* live_t_init, const int32_t* live_t_obs,
                  const int32_t* skin_idx, const double* skin_w,
                  const int32_t* skin_count);
int32_t or_model_size(const or_state* s);
void or_get_model(const or_state* s, double* ref_pos, double* ref_nrm, double* ref_radius,
                  double* ref_conf, int32_t* ref_t_init, int32_t* ref_t_obs,
                  double* live_pos, double* live_nrm, double* live_radius,
                  double* live_conf, int32_t* live_t_init, int32_t* live_t_obs,
                  int32_t* skin_idx, double* skin_w, int32_t* skin_count);
void or_set_nodes(or_state* s, int32_t n, const double* pos, const double* sigma,
                  const double* dq, const int32_t* nbr, const int32_t* nbr_count);
int32_t or_num_nodes(const or_state* s);
void or_get_nodes(const or_state* s, double* pos, double* sigma, double* dq, int32_t* nbr,
                  int32_t* nbr_count);

/* frame maps (depth_processing.cpp:103-138) */
int32_t or_build_frame(or_state* s, const uint16_t* depth, int32_t w, int32_t h,
                       int32_t frame_index);
void or_get_frame(const or_state* s, double* vert, double* nrm, double* conf, double* radius,
                  uint8_t* vertex_valid, uint8_t* valid, int32_t* valid_count);
void or_set_frame(or_state* s, int32_t w, int32_t h, int32_t frame_index, const double* vert,
                  const double* nrm, const double* conf, const double* radius,
                  const uint8_t* vertex_valid, const uint8_t* valid);
int32_t or_backproject(const uint16_t* depth, int32_t w, int32_t h, const or_config* cfg,
                       double* vert, uint8_t* vvalid);
void or_estimate_normals(const double* vert, const uint8_t* vvalid, int32_t w, int32_t h,
                         double* nrm, uint8_t* nvalid);
double or_compute_confidence(double px, double py, const or_config* cfg);
double or_compute_radius(double depth_m, double focal_px, double n_z);
void or_bilateral_filter(const uint16_t* depth, int32_t w, int32_t h, double sigma_space,
                         double sigma_depth, uint16_t* out);

/* warp field (warp_field.cpp) */
int32_t or_init_warp_field(or_state* s);
void or_compute_node_edges(or_state* s, int32_t k);
int32_t or_forward_warp(or_state* s);
int32_t or_inverse_warp_surfel(const or_state* s, int32_t i, double* pos, double* nrm);
int32_t or_extend_warp_field(or_state* s, int32_t n, const double* positions);
void or_update_skinning_incremental(or_state* s, int32_t first_new_node);
int32_t or_voxel_knn(const double* points, int32_t n, double cell, const double* q, int32_t k,
                     int32_t* out_idx);
int32_t or_voxel_has_point_within(const double* points, int32_t n, double cell,
                                  const double* q, double radius);

/* raster (raster.cpp) */
void or_render_index_map(const or_state* s, const double* pose, int32_t factor, int32_t* idx,
                         double* depth);
void or_render_model_maps(const or_state* s, const double* pose, int32_t t_now,
                          int32_t t_last_reinit, int32_t* idx, double* vert, double* nrm,
                          double* depth, uint8_t* valid);

/* solver (solver.cpp) */
int32_t or_find_correspondences(const or_state* s, const int32_t* mm_idx,
                                const double* mm_vert, const double* mm_nrm,
                                const uint8_t* mm_valid, int32_t mw, int32_t mh,
                                const double* pose, int32_t cap, int32_t* surfel, int32_t* px,
                                int32_t* py, double* v_model, double* v_depth,
                                double* n_depth);
int32_t or_normal_equations(or_state* s, const double* pose, int32_t t_now,
                            int32_t t_last_reinit, double* h, double* g, uint8_t* touched,
                            double* e_pre, int32_t* n_pairs);
int32_t or_solve_nonrigid(or_state* s, const double* pose, int32_t t_now,
                          int32_t t_last_reinit, or_solver_report* out);
int32_t or_rigid_align(or_state* s, const double* render_pose, const double* init_pose,
                       int32_t t_now, int32_t t_last_reinit, or_rigid_result* out);
double or_data_energy(const or_state* s, int32_t n_pairs, const int32_t* surfel,
                      const double* v_depth, const double* n_depth);
double or_reg_energy(const or_state* s);
int32_t or_blend_jacobian(const or_state* s, int32_t i, double* y3, double* dy_db24,
                          double* node_jac /* count x 3x6 */);
void or_reg_terms(const double* dq_j, const double* dq_i, const double* p_j, double* r3,
                  double* jj18, double* ji18);
int32_t or_ldlt_solve(int32_t n, const double* a, const double* b, double* x);
/* Dense LM step x = A^-1 b (A: n x n row-major, symmetric). Returns 0 on success. */
typedef int32_t (*or_dense_solver_fn)(int32_t n, const double* a, const double* b, double* x);
/* Replaces the restated Eigen LDLT of solve_nonrigid's LM step (NULL restores it). */
void or_set_dense_solver(or_dense_solver_fn fn);
/* Number of LM-step dense solves performed so far (process-wide). */
int64_t or_dense_solve_count(void);
int32_t or_assert_normal_equations(int32_t dim, const double* h);

/* fusion (fusion.cpp) */
int32_t or_fuse_depth(or_state* s, const int32_t* index_map, int32_t factor, const double* pose,
                      int32_t t_now, int32_t cap, int32_t* n_candidates, double* cand_pos,
                      double* cand_nrm, double* cand_radius, double* cand_conf,
                      int32_t* cand_px, int32_t* cand_py);
int32_t or_skin_appended(const or_state* s, const double* live_pos, const double* node_live,
                         int32_t* idx8, double* w8, int32_t* count);
int32_t or_inverse_warp_strain(const or_state* s, const double* x, const int32_t* idx,
                               const double* w, int32_t count, const double* node_live,
                               double* strain9);
int32_t or_check_compressive(const or_state* s, const double* x, const int32_t* idx,
                             const double* w, int32_t count, const double* node_live);
double or_sigma_max3(const double* m9);
void or_remove_surfels(const or_state* s, const int32_t* index_map, int32_t factor,
                       const double* pose, int32_t t_now, uint8_t* mask);
int32_t or_apply_fusion(or_state* s, const double* pose, int32_t t_now, or_fusion_outcome* out);

/* reinit (reinit.cpp) */
int32_t or_should_reinitialize(int32_t n, const double* mean_residuals, const int32_t* appended,
                               int32_t t_now, int32_t t_last_reinit, const or_config* cfg);
int32_t or_clean_and_reset(or_state* s, const double* pose, int32_t* removed,
                           int32_t* survivors);

/* geometry (geometry.cpp) */
void or_dq_from_se3(const double* pose, double* dq);
void or_dq_to_se3(const double* dq, double* pose);
void or_dq_mul(const double* a, const double* b, double* out);
void or_dq_normalized(const double* dq, double* out);
int32_t or_blend(int32_t n, const double* dqs, const double* w, double* out);
double or_skinning_weight(const double* x, const double* p, double sigma);
void or_se3_increment(const double* omega, const double* dt, const double* pose, double* out);
void or_dq_increment(const double* omega, const double* dt, double* out);
void or_quat_from_rotvec(const double* omega, double* q);
void or_quat_from_matrix(const double* r9, double* q);
void or_matrix_from_quat(const double* q, double* r9);

/* pipeline (pipeline.cpp:37-142) */
or_pipeline* or_pipeline_new(const or_config* cfg, int32_t mirror_fp32);
void or_pipeline_free(or_pipeline* p);
int32_t or_pipeline_process_frame(or_pipeline* p, const uint16_t* depth, int32_t w, int32_t h,
                                  int32_t frame_index, or_frame_stats* out);
or_state* or_pipeline_state(or_pipeline* p);
void or_pipeline_pose(const or_pipeline* p, double* pose);
int32_t or_pipeline_last_reinit(const or_pipeline* p);

#ifdef __cplusplus
}
#endif
#endif
