// ds_context.cuh — device-resident state of one sequence and the host-side
// stage entry points (implemented across the k_*.cu translation units).
//
// HBM layout (per context, one sequence, one stream):
//   surfels   SoA, double-buffered for stable compaction (fusion.cpp:264-284)
//             ref_pr/live_pr float4 (x,y,z,radius), ref_nc/live_nc float4
//             (nx,ny,nz,confidence), t int2 (t_init,t_observed), knn int4 +
//             w float4 (K=4 skinning, -1 = empty slot)            104 B/surfel
//   nodes     pos double4 (x,y,z,sigma), dq 2 x double4 (real, dual), nbr int[8],
//             se3 cache double[12] (per GN iteration)
//   frame     depth u16, vert/nrm double4 (x,y,z,radius)/(n,confidence), flags u8
//   maps      model-map point/splat keys (fp64 depth bits) + index, index map
//             (supersampled W*f x H*f) keys + index
//   solver    per-pixel pair slot (surfel, 4x6 fp32 Jacobian rows, fp64 residual),
//             per-surfel pair lists, term->block records sorted per frame,
//             BSR 6x6 fp32 blocks, PCG vectors fp64
#pragma once
#include <cuda_runtime.h>
#include <stdint.h>

#include <deque>
#include <utility>
#include <string>
#include <vector>

#include "../../include/dynsurf_b200.h"
#include "ds_math.cuh"

namespace ds {

struct Error {
  ds_status code;
  std::string msg;
};
[[noreturn]] void fail(ds_status code, const std::string& msg);
void cuda_check(cudaError_t e, const char* what);
#define DS_CUDA(call) ::ds::cuda_check((call), #call)

enum KernelKind {
  KK_FRAME_MAPS = 0,
  KK_FORWARD_WARP,
  KK_COMPACT_INVERSE_WARP,
  KK_MODEL_MAP_SPLAT,
  KK_ASSOCIATE,
  KK_INDEX_MAP,
  KK_PAIR_TERMS,
  KK_PAIR_LISTS,
  KK_PATTERN,
  KK_BLOCK_ASSEMBLY,
  KK_PCG,
  KK_NODE_UPDATE,
  KK_ENERGY,
  KK_REDUCE,
  KK_RIGID,
  KK_FUSE,
  KK_SKIN_APPEND,
  KK_REMOVE,
  KK_GREEDY_NODES,
  KK_NODE_EDGES,
  KK_SKIN_KNN,
  KK_SKIN_INCREMENTAL,
  KK_SCAN,
  KK_MISC,
  KK_COUNT
};
extern const char* kKernelNames[KK_COUNT];

struct ModelBuf {
  float4* rp = nullptr;  // reference (x,y,z,radius)
  float4* rn = nullptr;  // reference (nx,ny,nz,confidence)
  float4* lp = nullptr;  // live
  float4* ln = nullptr;
  int2* t = nullptr;     // (t_init, t_observed), shared by both arrays
  int4* ki = nullptr;    // skinning node indices (-1 empty)
  float4* kw = nullptr;  // skinning weights
};

// Small device-side scalars read back once per sync point.
struct DevScalars {
  int valid_count, degenerate, any_stable, n_pairs;
  int n_pairs_ok, fused, n_cand, n_accept;
  int low_support, comp_rejected, removed, n_keep;
  int n_nodes, n_new_nodes, err, finite;
  int up_blocks, full_blocks, pcg_iters, mean_cnt;
  int rigid_pairs, rigid_low, n_records, survivors;
  int rmax_bits, pair_list_n;
  double e_data, e_reg, ginf, htrace;
  double e_data_pre, e_reg_pre, g_sq, mu, mu_floor;
  double pcg_rr, pcg_rr0, mean_abs_r, rigid_abs;
  // device-resident LM loop (solver.cpp:296-406 state, k_lm_decide)
  int lm_iter, lm_attempt, lm_relin, lm_done;
  int lm_accepted, lm_attempts_total, pcg_iter_total, lm_rounds;
  int lm_relins, lm_pairs, any_stable_pat, _pad_lm1;  // any_stable_pat: build_pattern's copy
  double lm_e_pre, lm_gnorm, lm_initial, lm_final;
  double rigid_pose[12];
  // JtJ pattern counts, published by its last kernel (read with the frame's
  // next scalar fetch instead of host syncs inside the pattern build)
  int pat_n_up, pat_n_full, pat_n_chunks, pat_n_multi, pat_err, ne_err;
  int surv_old, fuse_err;  // apply_fusion: appended survivors' offset, append error (device-side)
  unsigned ne_scale_bits, _pad_ne;  // assert_normal_equations: max|H| (fp32 bits)
};

enum DevErr { DERR_NODE_CAP = 1, DERR_HASH_CELL = 2, DERR_HASH_FULL = 4, DERR_BLOCK_CAP = 8 };
// assert_normal_equations (solver.cpp:157-167) failures, DevScalars::ne_err
enum NeErr { NE_ASYMMETRIC = 1, NE_NOT_PSD = 2 };

struct GraphSlot {
  cudaGraphExec_t exec = nullptr;
  int64_t kernels = 0;  // kernel launches per replay (accounting)
  int64_t kernels_lin = 0;  // device LM loop: kernels per linearisation round
  int64_t kernels_tail = 0;  // device LM loop: kernels after the loop (the report)
};

struct ProfRec {
  int kind;
  cudaEvent_t a, b;
};

// Uniform-grid index over a node set (ds_knn.cuh / k_knn.cu).
constexpr int kKnnMaxPoints = 1 << 20;  // grid index capacity (points)
struct KnnGrid {
  long long* key = nullptr;
  int2* range = nullptr;
  int* ids = nullptr;
  double4* cpos = nullptr;  // the points' positions in cell order (copy of pos[ids[k]])
  double* prm = nullptr;
  int* pslot = nullptr;  // build scratch: slot of every point
  int* fill = nullptr;   // build scratch: per-slot scatter counters
  int mask = 0;      // slots - 1 of the current build (<= cap_mask)
  int cap_mask = 0;  // allocated slots - 1
  bool valid = false;
};

struct Ctx {
  ds_config cfg{};
  int device = 0;
  cudaStream_t stream = nullptr;
  bool own_stream = false;
  cudaStream_t side = nullptr;  // fork/join branch inside the GN step (parallel graph branch)
  cudaEvent_t ev_fork = nullptr, ev_mid = nullptr, ev_join = nullptr, ev_live = nullptr;
  bool live_pending = false, live_grid = false;  // prepare_live_nodes_async in flight
  cudaEvent_t ev_nodes = nullptr;  // new-node seeds / edges on the side stream
  bool nodes_pending = false;
  bool warp_in_index_map = false;  // next apply_fusion: forward warp fused into index pass 1
  int num_sms = 148;
  int W = 0, H = 0, P = 0;
  int S_cap = 0, N_cap = 0, R_cap = 0, UB_cap = 0, B_cap = 0, HT = 0;

  // model
  ModelBuf mb[2];
  int cur = 0;
  int capacity_growths = 0;
  // geometric re-allocations so far (grow_capacity)
  int n_surfels = 0;
  // nodes
  int n_nodes = 0;
  double4* node_pos = nullptr;
  double4* node_dq = nullptr;
  double4* node_dq_cand = nullptr;
  int* node_nbr = nullptr;
  double* node_se3 = nullptr;
  double* node_se3_cand = nullptr;
  double4* node_live = nullptr;
  float4* node_live_f = nullptr;  // fp32 copy for K-NN pre-tests
  // frame
  uint16_t* depth = nullptr;
  uint16_t* depth_f = nullptr;
  double4* f_vert = nullptr;
  double4* f_nrm = nullptr;
  uint8_t* f_flag = nullptr;  // bit0 vertex_valid, bit1 valid
  int frame_index = 0;
  int valid_count = 0;
  bool frame_ready = false;
  // model maps
  unsigned long long* mm_pkey = nullptr;
  unsigned long long* mm_skey = nullptr;
  int* mm_pidx = nullptr;
  int* mm_sidx = nullptr;
  int* mm_idx = nullptr;
  double mm_pose[12];
  bool mm_ready = false;
  bool mm_clean = false;  // model-map z-buffers hold the cleared state (in stream order)
  int* any_stable_pre = nullptr;  // "some surfel is stable", computed by the fusion's compaction
  bool any_stable_ready = false;  // ... and valid for the current model
  // supersampled index map
  unsigned long long* im_key = nullptr;
  int* im_idx = nullptr;
  int im_factor = 0;
  double im_pose[12];
  bool im_ready = false;
  // pairs / surfel lists
  int* pair_s = nullptr;     // per pixel: surfel or -1
  uint8_t* pair_ok = nullptr;
  float* pair_rows = nullptr;  // per pixel 4 x 6
  double* pair_r = nullptr;
  int* s_cnt = nullptr;
  int* s_head = nullptr;  // lowest pixel of the surfel's pairs
  int* s_base = nullptr;  // segment base in p_list (surfels with > 1 pair)
  int* s_fill = nullptr;  // segment fill counter
  int* p_list = nullptr;  // per pixel: pixels of multi-pair surfels, segmented
  int* p_next = nullptr;  // per pixel: next pixel of the same surfel (pixel order)
  // term -> block records and BSR
  int* rec_key = nullptr;
  int* rec_val = nullptr;
  int* rec_key2 = nullptr;
  int* rec_val2 = nullptr;
  int* rec_flag = nullptr;
  int* up_key = nullptr;
  int* up_start = nullptr;
  int* up_pos = nullptr;
  int* up_mpos = nullptr;
  int* row_ptr = nullptr;
  int* row_cnt = nullptr;
  int* bsr_col = nullptr;
  int* bsr_tag = nullptr;  // upper block id << 1 | mirrored
  float* bsr_val = nullptr;
  uint8_t* bsr_touch = nullptr;
  int* diag_pos = nullptr;
  int* chunk_first = nullptr;  // per upper block: first assembly chunk (n_up + 1)
  int* chunk_ub = nullptr;     // per chunk: upper block
  int4* chunk_d0 = nullptr;    // per chunk: assembly descriptor (k_chunk_fill)
  int4* chunk_d1 = nullptr;
  float* part_h = nullptr;     // per chunk: 6x6 partial
  double* part_g = nullptr;    // per chunk: g partial
  int* part_t = nullptr;       // per chunk: touched
  // regulariser terms, assembled apart from the surfel records (per frame:
  // the reg records' sorted positions grouped by upper block; per GN
  // iteration: their 6x6 sums on the side branch, added by the assembly)
  int* reg_rec = nullptr;        // reg record words (edge, type) in sorted order
  int* reg_ub = nullptr;         // their upper blocks
  int* reg_bf = nullptr;         // block-start flags -> exclusive scan (reg_bscan)
  int* reg_bscan = nullptr;
  int* reg_blk_start = nullptr;  // per reg block: first reg record (+ end)
  int* ub_reg = nullptr;         // per upper block: reg block or -1
  double* reg_h = nullptr;       // per reg block: 6x6 sum
  double* reg_g = nullptr;       // per reg block: g sum (diagonal blocks)
  int REG_cap = 0, RB_cap = 0, reg_cap_now = 0;
  int* elig = nullptr;  // render-eligible surfels of the current frame's solve
  int n_elig = 0;
  int n_records = 0, n_up = 0, n_full = 0, n_chunks = 0, n_multi = 0, CH_cap = 0;
  int* multi_flag = nullptr;
  int* multi_scan = nullptr;
  int* multi_list = nullptr;
  double n_pairs_ok_est = 0;
  bool pattern_ready = false;
  bool pattern_pending = false;  // enqueued, counts not adopted yet (pattern_adopt)
  void* cub_tmp = nullptr;
  size_t cub_tmp_bytes = 0;
  // PCG
  double* g = nullptr;
  double* pcg_x = nullptr;
  unsigned* pcgc_idx = nullptr;  // cluster PCG index scratch (k_pcg_cluster.cu)
  int rigid_grid_cap = 0;  // DS_RIGID_GRID: rigid-ICP term kernel grid cap (0: 2 CTAs per SM)
  int spmv_tma = 0;  // DS_SPMV_TMA: stand-alone SpMV 0 rows kernel, 1 TMA-staged, 2 persistent TMA
  bool check_ne = false;          // DS_CHECK_NE: assert_normal_equations every GN iteration
  int pcg_cluster = 0;            // DS_PCG_CLUSTER: 0 off (default), 2..16 cluster size
  int pcgc_smem_cap = 1 << 30;    // DS_PCGC_SMEM: cluster PCG carve bytes (tests shrink it)
  double* pcg_p0 = nullptr;
  double* pcg_p1 = nullptr;
  double* pcg_p2 = nullptr;
  double* pcg_q = nullptr;
  double* pcg_minv = nullptr;
  double* pcg_items = nullptr;
  double* pcg_vec = nullptr;
  double* gst_part = nullptr;
  int* pcg_slices = nullptr;  // per PCG CTA (r0, r1, bb0, bb1)
  unsigned long long* pcg_trace = nullptr;  // DS_PCG_TRACE diagnostics
  double* reg_ab = nullptr;
  double* pcg_part = nullptr;
  int pcg_grid = 0;
  // fusion
  int* cand_flag = nullptr;
  int* cand_scan = nullptr;
  int* cand_pix = nullptr;
  float4* cand_p = nullptr;
  float4* cand_n = nullptr;
  int4* cand_ki = nullptr;
  float4* cand_kw = nullptr;
  int* cand_ok = nullptr;
  int* cand_ok_scan = nullptr;
  int* keep = nullptr;
  int* keep_scan = nullptr;
  float4* ext_pos = nullptr;  // uncovered extension candidates (ordered)
  // greedy node hash
  KnnGrid grid_ref, grid_live;  // reference / live node positions
  KnnGrid grid_new;             // the nodes added this frame (incremental reskinning)
  double* new_bbox = nullptr;   // their bounding box (6 doubles, side-stream scratch)
  bool use_pdl = true;
  bool no_defer = false;        // DS_NO_DEFER=1: join the side stream at the end of each fusion          // programmatic dependent launch in the GN chain (DS_NO_PDL=1 disables)
  int incr_grid_min = 16;       // new nodes above which grid_new is used (DS_INCR_GRID_MIN)
  double incr_cell = 4.0;       // grid_new cell size in node_sigma (DS_INCR_CELL)
  double live_cell = 2.0;       // grid_live (screening) cell size in node_sigma (DS_LIVE_CELL)
  double ref_cell = 2.0;        // grid_ref (edges, seeds, skinning) cell size (DS_REF_CELL)
  long long* ht_key = nullptr;
  int* ht_cnt = nullptr;
  int* ht_ids = nullptr;
  // scratch
  int* scan_tmp = nullptr;
  unsigned long long* scan_status = nullptr;  // look-back scan tile status words
  int scan_tmp_n = 0;
  double* red_part = nullptr;
  int red_part_n = 0;
  double* d_pose = nullptr;  // 12 doubles
  unsigned* tickets = nullptr;  // last-block tickets of fused grid reductions
  DevScalars* dsc = nullptr;
  DevScalars* hsc = nullptr;  // pinned mirror
  uint16_t* h_depth_pinned = nullptr;

  // host pipeline state (Pipeline, pipeline.hpp:52-59)
  double pose[12];
  bool initialized = false;
  int t_last_reinit = 0;
  std::deque<double> win_residual;
  std::deque<int> win_appended;

  // accounting
  int64_t launches[KK_COUNT] = {0};
  double prof_ms[KK_COUNT] = {0};
  double prof_bytes[KK_COUNT] = {0};
  int64_t prof_launches[KK_COUNT] = {0};
  int64_t total_launches = 0;
  std::vector<ProfRec> prof_pending;
  std::vector<cudaEvent_t> event_pool;
  std::vector<void*> allocations;
  // per-frame extras
  int lm_attempts = 0, pcg_iterations = 0;
  // CUDA graphs of the GN step / LM attempt (re-captured per frame, updated in place)
  bool use_graphs = true;
  int knn_edges_grid = 8192;
  bool screen_grid = true;  // DS_SCREEN_GRID=0: brute-force two-pass screening K-NN
  int pcg_smem_cap = 200 * 1024;  // DS_PCG_SMEM: slice bytes allowed in shared memory (tests: 0)  // node count above which edges / seeds use the grid
  bool trace_host = false;  // DS_TRACE_HOST: host-side timing prints
  bool device_lm = true;
  int pattern_frame = -1;  // frame whose JtJ pattern was built ahead (overlapping the rigid ICP)  // LM loop as a device-side WHILE graph (DS_HOST_LM=1: host loop)
  GraphSlot g_step, g_attempt, g_solve;
  double* h_mu = nullptr;  // pinned staging for mu
  int* h_int = nullptr;    // pinned staging for small ints

  ModelBuf& M() { return mb[cur]; }
  ModelBuf& Malt() { return mb[cur ^ 1]; }
};

// ---- launch accounting (every kernel of the library goes through these)
void launch_begin(Ctx& c, int kind);
void launch_end(Ctx& c, int kind, double bytes);
void prof_flush(Ctx& c);
// Programmatic dependent launch (PDL): the kernel may be scheduled while its
// stream predecessor drains; it must call pdl_wait() before touching anything
// the predecessor produces (every kernel launched with DS_LAUNCH_PDL does so
// first thing; without the attribute the wait is a no-op).
// (no early launch_dependents trigger: measured slower -- the dependents'
// waiting CTAs then take slots from the draining predecessor)
__device__ __forceinline__ void pdl_wait() { asm volatile("griddepcontrol.wait;" ::: "memory"); }

template <typename... KArgs, typename... Args>
inline cudaError_t launch_pdl(Ctx& c, dim3 grid, dim3 block, size_t smem, void (*k)(KArgs...),
                              Args&&... args) {
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = grid;
  cfg.blockDim = block;
  cfg.dynamicSmemBytes = smem;
  cfg.stream = c.stream;
  cudaLaunchAttribute at[1];
  at[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  at[0].val.programmaticStreamSerializationAllowed = 1;
  cfg.attrs = at;
  cfg.numAttrs = c.use_pdl ? 1 : 0;
  return cudaLaunchKernelEx(&cfg, k, std::forward<Args>(args)...);
}
#define DS_LAUNCH_PDL(ctx, kind, bytes, grid, block, smem, kernel, ...)                    \
  do {                                                                                     \
    ::ds::launch_begin((ctx), (kind));                                                     \
    DS_CUDA(::ds::launch_pdl((ctx), dim3(grid), dim3(block), (smem), kernel, __VA_ARGS__)); \
    ::ds::launch_end((ctx), (kind), (double)(bytes));                                      \
  } while (0)

#define DS_LAUNCH(ctx, kind, bytes, grid, block, smem, kernel, ...)        \
  do {                                                                     \
    ::ds::launch_begin((ctx), (kind));                                     \
    kernel<<<(grid), (block), (smem), (ctx).stream>>>(__VA_ARGS__);        \
    ::ds::launch_end((ctx), (kind), (double)(bytes));                      \
  } while (0)

inline int cdiv(long long a, long long b) { return int((a + b - 1) / b); }
void sync(Ctx& c);                   // stream sync + profile flush
void fetch_scalars(Ctx& c);          // D2H of DevScalars (syncs)
void clear_scalars(Ctx& c);

// ---- utilities (k_scan.cu)
// exclusive scan of n ints: out[0..n] (out[n] = total). in may alias out only if n+1 storage.
void scan_exclusive(Ctx& c, const int* in, int* out, int n);
void sort_pairs(Ctx& c, int* keys, int* vals, int* keys_alt, int* vals_alt, int n, int end_bit,
                int** keys_out, int** vals_out, int kind = KK_PATTERN);

// ---- frame (k_frame.cu)
void frame_maps(Ctx& c, const uint16_t* depth_dev, int frame_index);
void init_surfels_from_frame(Ctx& c);  // initialize_from_frame (pipeline.cpp:42-72) surfels

// ---- warp field (k_warp.cu, k_skin.cu)
int forward_warp(Ctx& c, bool count_degenerate);
void node_se3(Ctx& c, const double4* dq, double* se3);
void node_live_positions(Ctx& c);
void apply_increments(Ctx& c, const double* delta, double4* out, double* se3 = nullptr);  // solver.cpp:277-286
void init_warp_field(Ctx& c);
void compute_node_edges(Ctx& c, bool build_grid = true);
bool build_knn_grid(Ctx& c, KnnGrid& g, const double4* pos, int n, double h, int load_inv = 2);
int extend_warp_field(Ctx& c, const float4* positions, int n);  // returns appended
// the same over positions base[*off_dev .. *end_dev) with the count on the
// device (<= bound); its greedy pass ends with a full scalar fetch
int extend_warp_field_dev(Ctx& c, const float4* base, const int* off_dev, const int* end_dev,
                          int bound);
void update_skinning_incremental(Ctx& c, int first_new);

// ---- raster (k_raster.cu)
void render_model_maps(Ctx& c, const double* pose, int t_now, int t_last, bool associate,
                       const double* assoc_pose, bool consume_reset = false);
void render_index_map(Ctx& c, const double* pose, int factor, const double4* warp_dq = nullptr);
// model maps + association over a precomputed render-eligible surfel list
void render_model_maps_list(Ctx& c, const double* pose, int t_now, int t_last,
                            const double* assoc_pose, const int* list, int n,
                            const double4* warp_dq = nullptr, bool resolve = true, bool clear = true);
// resets the model-map z-buffers (the GN iteration kernel resets what it consumed)
void clear_model_maps(Ctx& c);

// ---- solver (k_solver.cu, k_rigid.cu)
void solve_nonrigid(Ctx& c, const double* pose, int t_now, int t_last, ds_solver_report* out);
void gn_linearize(Ctx& c, const double* pose, int t_now, int t_last, double* e_pre, int* n_pairs);
void pcg_solve(Ctx& c, double mu, int max_iters, double tol, int* iters, double* rel_res);
// assert_normal_equations (solver.cpp:157-167) on the assembled BSR system:
// enqueue the device check (flags in dsc->ne_err) / run it and fail with
// DS_ERR_NUMERICAL like the reference's dynsurf::Error
void check_normal_equations_async(Ctx& c);
void check_normal_equations(Ctx& c);
// cluster-resident PCG (k_pcg_cluster.cu); false when it does not apply
bool pcg_cluster_launch(Ctx& c, int max_iters, double tol);
void rigid_align(Ctx& c, const double* render_pose, const double* init_pose, int t_now,
                 int t_last, ds_rigid_result* out);
// rigid_align split: enqueue the device work / wait and assemble the result
void rigid_align_enqueue(Ctx& c, const double* render_pose, const double* init_pose, int t_now,
                         int t_last);
void rigid_align_finish(Ctx& c, const double* init_pose, ds_rigid_result* out);
void prepare_live_nodes_async(Ctx& c);
// main stream waits for side-stream node updates (seeds / edges), if any
inline void join_node_updates(Ctx& c) {
  if (!c.nodes_pending) return;
  DS_CUDA(cudaStreamWaitEvent(c.stream, c.ev_nodes, 0));
  c.nodes_pending = false;
}

// ---- fusion (k_fusion.cu)
void apply_fusion(Ctx& c, const double* pose, int t_now, ds_fusion_outcome* out);
void fuse_depth(Ctx& c, const double* pose, int t_now, int* fused, int* n_cand);
void screen_candidates(Ctx& c, int n_cand, int* low_support, int* comp_rejected, int* accepted);
void removal_mask(Ctx& c, const double* pose, int t_now, int n);
int clean_and_reset(Ctx& c, const double* pose, int* survivors);

// capacity guards
void ensure_surfel_capacity(Ctx& c, long long n);
void ensure_node_capacity(Ctx& c, long long n);

}  // namespace ds
