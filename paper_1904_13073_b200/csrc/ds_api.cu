// ds_api.cu — context lifetime, state transfer, the per-frame process call and
// the C ABI (include/dynsurf_b200.h). Host orchestration mirrors
// Pipeline::process_frame (pipeline.cpp:74-142) and initialize_from_frame
// (pipeline.cpp:42-72); all stage work is on the device.
#include <cub/cub.cuh>

#include <cstdio>
#include <cstdlib>

#include <algorithm>
#include <chrono>
#include <cmath>
#include <cstring>
#include <string>
#include <vector>

#include "ds_blend.cuh"
#include "ds_context.cuh"

namespace ds {

const char* kKernelNames[KK_COUNT] = {
    "frame_maps",   "forward_warp", "compact_inverse_warp", "model_map_splat", "associate",
    "index_map",    "pair_terms",   "pair_lists",           "pattern",         "block_assembly",
    "pcg",          "node_update",  "energy",               "reduce",          "rigid_icp",
    "fuse",         "skin_append",  "remove",               "greedy_nodes",    "node_edges",
    "skin_knn",     "skin_incremental", "scan",             "misc"};

size_t sort_temp_bytes(int n);
int pcg_max_grid(int num_sms);
void build_pattern(Ctx& c, int t_now, int t_last);
void build_pattern_enqueue(Ctx& c, int t_now, int t_last);
void pattern_adopt(Ctx& c, bool have_scalars);
double bsr_spmv(Ctx& c, const double* x_dev, double* y_dev, double mu, int reps);
void gn_linearize_async(Ctx& c, const double* pose, int t_now, int t_last, bool lm_floor,
                        bool maps_clean = false);
void fuse_depth_async(Ctx& c, const double* pose, int t_now);

thread_local std::string g_last_error;

void fail(ds_status code, const std::string& msg) { throw Error{code, msg}; }
void cuda_check(cudaError_t e, const char* what) {
  if (e != cudaSuccess) {
    cudaGetLastError();
    throw Error{DS_ERR_CUDA, std::string(what) + ": " + cudaGetErrorString(e)};
  }
}

void launch_begin(Ctx& c, int kind) {
  if (!c.cfg.profile) return;
  ProfRec r;
  r.kind = kind;
  if (c.event_pool.size() >= 2) {
    r.b = c.event_pool.back();
    c.event_pool.pop_back();
    r.a = c.event_pool.back();
    c.event_pool.pop_back();
  } else {
    DS_CUDA(cudaEventCreate(&r.a));
    DS_CUDA(cudaEventCreate(&r.b));
  }
  DS_CUDA(cudaEventRecord(r.a, c.stream));
  c.prof_pending.push_back(r);
}
void launch_end(Ctx& c, int kind, double bytes) {
  const cudaError_t e = cudaGetLastError();
  if (e != cudaSuccess)
    throw Error{DS_ERR_CUDA, std::string("kernel ") + kKernelNames[kind] + ": " + cudaGetErrorString(e)};
  c.launches[kind] += 1;
  c.total_launches += 1;
  if (c.cfg.profile && !c.prof_pending.empty()) {
    // launches/bytes of the profiled launches only, so bytes / ms is a rate
    DS_CUDA(cudaEventRecord(c.prof_pending.back().b, c.stream));
    c.prof_launches[kind] += 1;
    c.prof_bytes[kind] += bytes;
  }
}
void prof_flush(Ctx& c) {
  // launches on another stream (the side branch) may still be running after
  // this stream's sync: keep those records for a later flush
  std::vector<ProfRec> keep;
  for (auto& r : c.prof_pending) {
    if (cudaEventQuery(r.b) != cudaSuccess) {
      cudaGetLastError();
      keep.push_back(r);
      continue;
    }
    float ms = 0;
    DS_CUDA(cudaEventElapsedTime(&ms, r.a, r.b));
    c.prof_ms[r.kind] += ms;
    c.event_pool.push_back(r.a);
    c.event_pool.push_back(r.b);
  }
  c.prof_pending.swap(keep);
}
void sync(Ctx& c) {
  DS_CUDA(cudaStreamSynchronize(c.stream));
  prof_flush(c);
}
void fetch_scalars(Ctx& c) {
  DS_CUDA(cudaMemcpyAsync(c.hsc, c.dsc, sizeof(DevScalars), cudaMemcpyDeviceToHost, c.stream));
  sync(c);
}
void clear_scalars(Ctx& c) { DS_CUDA(cudaMemsetAsync(c.dsc, 0, sizeof(DevScalars), c.stream)); }

void ensure_surfel_capacity(Ctx& c, long long n) {
  if (n > c.S_cap) fail(DS_ERR_CAPACITY, "surfel capacity exceeded (" + std::to_string(n) + " > " +
                                             std::to_string(c.S_cap) + ")");
}
void ensure_node_capacity(Ctx& c, long long n) {
  if (n > c.N_cap) fail(DS_ERR_CAPACITY, "node capacity exceeded");
}

namespace {

template <typename T>
T* dalloc(Ctx& c, size_t count) {
  void* p = nullptr;
  DS_CUDA(cudaMalloc(&p, std::max<size_t>(count, 1) * sizeof(T)));
  c.allocations.push_back(p);
  return static_cast<T*>(p);
}

void validate(const ds_config& k) {  // PipelineConfig::validate (config.cpp:121-144)
  auto req = [](bool ok, const char* what) {
    if (!ok) fail(DS_ERR_CONFIG, std::string("config: ") + what);
  };
  req(k.node_sigma > 0, "node_sigma must be positive");
  req(k.knn_k >= 1 && k.knn_k <= 8, "knn_k out of range");
  req(k.node_neighbor_k >= 1, "node_neighbor_k must be positive");
  req(k.lambda >= 0, "lambda must be nonnegative");
  req(k.max_gn_iters >= 1, "max_gn_iters must be positive");
  req(k.delta_distance > 0, "delta_distance must be positive");
  req(k.delta_normal > 0 && k.delta_normal <= 1, "delta_normal must be in (0,1]");
  req(k.epsilon > 0 && k.epsilon < 1, "epsilon must be in (0,1)");
  req(k.delta_stable > 0, "delta_stable must be positive");
  req(k.t_low_confid > 0, "t_low_confid must be positive");
  req(k.delta_recent >= 0, "delta_recent must be nonnegative");
  req(k.delta_nn > 0, "delta_nn must be positive");
  req(k.supersample_factor >= 1, "supersample_factor must be >= 1");
  req(k.depth_min > 0 && k.depth_max > k.depth_min, "depth range invalid");
  req(k.reinit_energy_threshold > 0, "reinit_energy_threshold must be positive");
  req(k.reinit_append_threshold > 0, "reinit_append_threshold must be positive");
  req(k.reinit_window >= 1, "reinit_window must be positive");
  req(k.periodic_reinit_interval >= 0, "periodic_reinit_interval must be >= 0");
  req(k.delta_distance_reinit > 0, "delta_distance_reinit must be positive");
  // Pipeline::Pipeline (pipeline.cpp:37-40)
  req(k.fx > 0 && k.fy > 0 && k.width > 0 && k.height > 0, "pipeline: invalid intrinsics");
  // device layout limits
  req(k.knn_k <= 4, "device path keeps at most knn_k = 4 skinning nodes");
  req(k.node_neighbor_k <= 8, "device path keeps at most node_neighbor_k = 8 edges");
  req(k.supersample_factor <= 8, "supersample_factor > 8 not supported on device");
}

void allocate(Ctx& c) {
  const ds_config& k = c.cfg;
  c.W = k.width;
  c.H = k.height;
  c.P = c.W * c.H;
  c.S_cap = k.max_surfels > 0 ? k.max_surfels : std::max(8 * c.P, 4096);
  c.N_cap = k.max_nodes > 0 ? k.max_nodes : 8192;
  c.R_cap = c.S_cap * 10 + c.N_cap * 24;
  c.UB_cap = std::min(c.R_cap, std::max(48 * c.N_cap, 65536));
  c.B_cap = 2 * c.UB_cap;
  c.HT = 1;
  while (c.HT < 2 * c.N_cap) c.HT <<= 1;
  const size_t P = c.P, S = c.S_cap, N = c.N_cap;
  const int f = k.supersample_factor;
  for (int b = 0; b < 2; ++b) {
    ModelBuf& m = c.mb[b];
    m.rp = dalloc<float4>(c, S);
    m.rn = dalloc<float4>(c, S);
    m.lp = dalloc<float4>(c, S);
    m.ln = dalloc<float4>(c, S);
    m.t = dalloc<int2>(c, S);
    m.ki = dalloc<int4>(c, S);
    m.kw = dalloc<float4>(c, S);
  }
  c.node_pos = dalloc<double4>(c, N);
  c.node_dq = dalloc<double4>(c, 2 * N);
  c.node_dq_cand = dalloc<double4>(c, 2 * N);
  c.node_nbr = dalloc<int>(c, 8 * N);
  c.node_se3 = dalloc<double>(c, 12 * N);
  c.node_se3_cand = dalloc<double>(c, 12 * N);
  c.node_live = dalloc<double4>(c, N);
  c.node_live_f = dalloc<float4>(c, N);
  c.depth = dalloc<uint16_t>(c, P);
  c.depth_f = dalloc<uint16_t>(c, P);
  c.f_vert = dalloc<double4>(c, P);
  c.f_nrm = dalloc<double4>(c, P);
  c.f_flag = dalloc<uint8_t>(c, P);
  c.mm_pkey = dalloc<unsigned long long>(c, P);
  c.mm_skey = dalloc<unsigned long long>(c, P);
  c.mm_pidx = dalloc<int>(c, P);
  c.mm_sidx = dalloc<int>(c, P);
  c.mm_idx = dalloc<int>(c, P);
  c.im_key = dalloc<unsigned long long>(c, P * f * f);
  c.im_idx = dalloc<int>(c, P * f * f);
  c.pair_s = dalloc<int>(c, P);
  c.pair_ok = dalloc<uint8_t>(c, P);
  c.pair_rows = dalloc<float>(c, P * 24);
  c.pair_r = dalloc<double>(c, P);
  c.s_cnt = dalloc<int>(c, S + 1);
  c.s_head = dalloc<int>(c, S + 1);
  c.s_base = dalloc<int>(c, S + 1);
  c.s_fill = dalloc<int>(c, S + 1);
  c.p_list = dalloc<int>(c, P);
  c.p_next = dalloc<int>(c, P);
  c.rec_key = dalloc<int>(c, c.R_cap);
  c.rec_val = dalloc<int>(c, c.R_cap);
  c.rec_key2 = dalloc<int>(c, c.R_cap);
  c.rec_val2 = dalloc<int>(c, c.R_cap + 1);
  c.rec_flag = dalloc<int>(c, c.R_cap + 1);
  c.up_key = dalloc<int>(c, c.UB_cap);
  c.up_start = dalloc<int>(c, c.UB_cap + 1);
  c.up_pos = dalloc<int>(c, c.UB_cap);
  c.up_mpos = dalloc<int>(c, c.UB_cap);
  c.row_ptr = dalloc<int>(c, N + 1);
  c.row_cnt = dalloc<int>(c, N + 1);
  c.bsr_col = dalloc<int>(c, c.B_cap + 4);  // + the TMA SpMV's 16 B-aligned column copies
  c.bsr_tag = dalloc<int>(c, c.B_cap);
  c.bsr_val = dalloc<float>(c, (size_t)c.B_cap * 36);
  c.bsr_touch = dalloc<uint8_t>(c, c.B_cap);
  c.diag_pos = dalloc<int>(c, N);
  c.CH_cap = c.R_cap / 64 + c.UB_cap + 1;
  c.chunk_first = dalloc<int>(c, c.UB_cap + 1);
  c.multi_flag = dalloc<int>(c, c.UB_cap + 1);
  c.multi_scan = dalloc<int>(c, c.UB_cap + 1);
  c.multi_list = dalloc<int>(c, c.UB_cap + 1);
  c.chunk_ub = dalloc<int>(c, c.CH_cap);
  c.chunk_d0 = dalloc<int4>(c, c.CH_cap);
  c.chunk_d1 = dalloc<int4>(c, c.CH_cap);
  c.part_h = dalloc<float>(c, (size_t)c.CH_cap * 36);
  c.part_g = dalloc<double>(c, (size_t)c.CH_cap * 6);
  c.part_t = dalloc<int>(c, c.CH_cap);
  c.REG_cap = 24 * N;  // 3 records per directed edge, 8 edges per node
  c.RB_cap = 9 * N;    // distinct upper blocks of the graph: N diagonal + <= 8 N edges
  c.reg_rec = dalloc<int>(c, c.REG_cap + 1);
  c.reg_ub = dalloc<int>(c, c.REG_cap + 1);
  c.reg_bf = dalloc<int>(c, c.REG_cap + 1);
  c.reg_bscan = dalloc<int>(c, c.REG_cap + 2);
  c.reg_blk_start = dalloc<int>(c, c.RB_cap + 2);
  c.ub_reg = dalloc<int>(c, c.UB_cap + 1);
  c.reg_h = dalloc<double>(c, (size_t)c.RB_cap * 36);
  c.reg_g = dalloc<double>(c, (size_t)c.RB_cap * 6);
  c.elig = dalloc<int>(c, S);
  c.cub_tmp_bytes = std::max(sort_temp_bytes(c.R_cap), sort_temp_bytes(P));
  c.cub_tmp = dalloc<char>(c, c.cub_tmp_bytes);
  c.g = dalloc<double>(c, 6 * N);
  c.pcg_x = dalloc<double>(c, 6 * N);
  c.pcg_p0 = dalloc<double>(c, 6 * N);
  c.pcg_p1 = dalloc<double>(c, 6 * N);
  c.pcg_p2 = dalloc<double>(c, 6 * N);
  c.pcg_q = dalloc<double>(c, 6 * N);
  c.pcg_minv = dalloc<double>(c, 36 * N);
  c.pcg_items = dalloc<double>(c, 6 * (size_t)c.B_cap);
  // cluster PCG: block source codes + halo lists when they do not fit on chip
  c.pcgc_idx = dalloc<unsigned>(c, (size_t)c.B_cap + 16 * (size_t)N + 16);
  c.pcg_vec = dalloc<double>(c, 60 * (size_t)N);
  c.gst_part = dalloc<double>(c, 3 * (size_t)cdiv(N, 256) + 8);
  c.reg_ab = dalloc<double>(c, 48 * (size_t)N);
  c.pcg_grid = pcg_max_grid(c.num_sms);
  if (const char* e = std::getenv("DS_PCG_GRID")) {  // tuning knob (capped at co-residency)
    const int g = std::atoi(e);
    if (g > 0) c.pcg_grid = std::min(c.pcg_grid, g);
  }
  c.pcg_part = dalloc<double>(c, 8 * (size_t)c.pcg_grid);
  c.pcg_slices = dalloc<int>(c, 4 * (size_t)c.pcg_grid + 4);
  if (std::getenv("DS_PCG_TRACE")) c.pcg_trace = dalloc<unsigned long long>(c, 64);
  c.cand_flag = dalloc<int>(c, P + 1);
  c.cand_scan = dalloc<int>(c, P + 1);
  c.cand_pix = dalloc<int>(c, P);
  c.cand_p = dalloc<float4>(c, P);
  c.cand_n = dalloc<float4>(c, P);
  c.cand_ki = dalloc<int4>(c, P);
  c.cand_kw = dalloc<float4>(c, P);
  c.cand_ok = dalloc<int>(c, P + 1);
  c.cand_ok_scan = dalloc<int>(c, P + 1);
  c.keep = dalloc<int>(c, S + P + 1);
  c.keep_scan = dalloc<int>(c, S + P + 1);
  c.ext_pos = dalloc<float4>(c, P);
  for (KnnGrid* g : {&c.grid_ref, &c.grid_live, &c.grid_new}) {
    int slots = 1;
    while (slots < 2 * std::min(c.N_cap, kKnnMaxPoints)) slots <<= 1;
    g->key = dalloc<long long>(c, slots);
    g->range = dalloc<int2>(c, slots);
    g->ids = dalloc<int>(c, std::min(c.N_cap, kKnnMaxPoints));
    g->cpos = dalloc<double4>(c, std::min(c.N_cap, kKnnMaxPoints));
    g->prm = dalloc<double>(c, 8);
    g->pslot = dalloc<int>(c, std::min(c.N_cap, kKnnMaxPoints));
    g->fill = dalloc<int>(c, slots);
    g->mask = g->cap_mask = slots - 1;
  }
  c.new_bbox = dalloc<double>(c, 8);
  c.any_stable_pre = dalloc<int>(c, 1);
  c.ht_key = dalloc<long long>(c, c.HT);
  c.ht_cnt = dalloc<int>(c, c.HT);
  c.ht_ids = dalloc<int>(c, 8 * (size_t)c.HT);
  const size_t scan_max = std::max({(size_t)c.R_cap, S + P, P * f * f, N + 1});
  c.scan_tmp_n = cdiv((long long)scan_max, 4096) + 16;
  c.scan_tmp = dalloc<int>(c, c.scan_tmp_n);
  c.scan_status = dalloc<unsigned long long>(c, c.scan_tmp_n);
  c.red_part_n = cdiv(c.P, 256) * 29 + cdiv(8 * (long long)N, 256) + cdiv(c.P, 256) + 64;
  c.red_part = dalloc<double>(c, c.red_part_n);
  c.d_pose = dalloc<double>(c, 12);
  c.tickets = dalloc<unsigned>(c, 16);
  DS_CUDA(cudaMemsetAsync(c.tickets, 0, 16 * sizeof(unsigned), c.stream));
  c.dsc = dalloc<DevScalars>(c, 1);
  DS_CUDA(cudaMallocHost(&c.hsc, sizeof(DevScalars)));
  DS_CUDA(cudaMallocHost(&c.h_depth_pinned, sizeof(uint16_t) * P));
  DS_CUDA(cudaMallocHost(&c.h_mu, sizeof(double)));
  DS_CUDA(cudaMallocHost(&c.h_int, 4 * sizeof(int)));
  if (const char* e = std::getenv("DS_NO_GRAPHS")) c.use_graphs = e[0] == '0';
  if (const char* e = std::getenv("DS_HOST_LM")) c.device_lm = e[0] == '0';
  c.trace_host = std::getenv("DS_TRACE_HOST") != nullptr;
  if (const char* e = std::getenv("DS_KNN_EDGES_GRID")) c.knn_edges_grid = std::atoi(e);
  if (const char* e = std::getenv("DS_SCREEN_GRID")) c.screen_grid = e[0] != '0';
  if (const char* e = std::getenv("DS_INCR_GRID_MIN")) c.incr_grid_min = std::atoi(e);
  if (const char* e = std::getenv("DS_NO_PDL")) c.use_pdl = e[0] == '0';
  if (const char* e = std::getenv("DS_NO_DEFER")) c.no_defer = e[0] != '0';
  if (const char* e = std::getenv("DS_INCR_CELL")) c.incr_cell = std::atof(e);
  if (const char* e = std::getenv("DS_LIVE_CELL")) c.live_cell = std::atof(e);
  if (const char* e = std::getenv("DS_REF_CELL")) c.ref_cell = std::atof(e);
  if (const char* e = std::getenv("DS_PCG_SMEM")) c.pcg_smem_cap = std::min(std::atoi(e), c.pcg_smem_cap);
  if (const char* e = std::getenv("DS_PCG_CLUSTER")) c.pcg_cluster = std::atoi(e);
  if (const char* e = std::getenv("DS_CHECK_NE")) c.check_ne = e[0] != '0';
  if (const char* e = std::getenv("DS_SPMV_TMA")) c.spmv_tma = std::atoi(e);
  if (const char* e = std::getenv("DS_RIGID_GRID")) c.rigid_grid_cap = std::max(1, std::atoi(e));
  if (const char* e = std::getenv("DS_PCGC_SMEM")) c.pcgc_smem_cap = std::atoi(e);
  DS_CUDA(cudaMemsetAsync(c.dsc, 0, sizeof(DevScalars), c.stream));
  DS_CUDA(cudaMemsetAsync(c.node_nbr, 0xff, sizeof(int) * 8 * N, c.stream));
}

void release(Ctx& c) {
  for (auto& r : c.prof_pending) {
    cudaEventDestroy(r.a);
    cudaEventDestroy(r.b);
  }
  for (auto e : c.event_pool) cudaEventDestroy(e);
  for (void* p : c.allocations) cudaFree(p);
  if (c.hsc) cudaFreeHost(c.hsc);
  if (c.h_depth_pinned) cudaFreeHost(c.h_depth_pinned);
  if (c.h_mu) cudaFreeHost(c.h_mu);
  if (c.h_int) cudaFreeHost(c.h_int);
  if (c.g_step.exec) cudaGraphExecDestroy(c.g_step.exec);
  if (c.g_attempt.exec) cudaGraphExecDestroy(c.g_attempt.exec);
  if (c.g_solve.exec) cudaGraphExecDestroy(c.g_solve.exec);
  if (c.own_stream && c.stream) cudaStreamDestroy(c.stream);
  if (c.side) cudaStreamDestroy(c.side);
  if (c.ev_fork) cudaEventDestroy(c.ev_fork);
  if (c.ev_join) cudaEventDestroy(c.ev_join);
  if (c.ev_mid) cudaEventDestroy(c.ev_mid);
  if (c.ev_live) cudaEventDestroy(c.ev_live);
  if (c.ev_nodes) cudaEventDestroy(c.ev_nodes);
}

void set_identity(double* p) {
  for (int i = 0; i < 12; ++i) p[i] = (i == 0 || i == 4 || i == 8) ? 1.0 : 0.0;
}

// Geometric capacity growth at a frame boundary (the reference's containers
// are unbounded std::vectors: types.hpp:66-80, warp_field.cpp:142-184). Every
// device buffer is sized from the surfel / node capacities, so growing
// re-allocates the context's device state: the persistent state (the current
// model SoA, node positions / transforms / edges, the device scalars) is
// parked in temporary buffers, the context is re-allocated at the new
// capacities and the state copied back; everything else is per frame.
void grow_capacity(Ctx& c, long long need_surfels, long long need_nodes) {
  join_node_updates(c);
  DS_CUDA(cudaStreamSynchronize(c.side));
  sync(c);
  const int n = c.n_surfels, N = c.n_nodes;
  const long long S_new = std::max<long long>(c.S_cap, need_surfels);
  const long long N_new = std::max<long long>(c.N_cap, need_nodes);
  if (S_new * 10 + N_new * 24 >= 0x7fffffffLL)
    fail(DS_ERR_CAPACITY, "capacity growth beyond 32-bit record indices");
  const ModelBuf old = c.M();
  struct Park {
    void* p;
    size_t bytes;
    const void* src;
  };
  std::vector<Park> park = {
      {nullptr, sizeof(float4) * n, old.rp}, {nullptr, sizeof(float4) * n, old.rn},
      {nullptr, sizeof(float4) * n, old.lp}, {nullptr, sizeof(float4) * n, old.ln},
      {nullptr, sizeof(int2) * n, old.t},    {nullptr, sizeof(int4) * n, old.ki},
      {nullptr, sizeof(float4) * n, old.kw}, {nullptr, sizeof(double4) * N, c.node_pos},
      {nullptr, sizeof(double4) * 2 * N, c.node_dq}, {nullptr, sizeof(int) * 8 * N, c.node_nbr},
      {nullptr, sizeof(DevScalars), c.dsc}, {nullptr, sizeof(uint16_t) * c.P, c.depth}};
  for (auto& q : park) {
    DS_CUDA(cudaMalloc(&q.p, std::max<size_t>(q.bytes, 1)));
    if (q.bytes) DS_CUDA(cudaMemcpyAsync(q.p, q.src, q.bytes, cudaMemcpyDeviceToDevice, c.stream));
  }
  sync(c);
  // device and pinned allocations only (streams and events stay)
  for (void* p : c.allocations) cudaFree(p);
  c.allocations.clear();
  for (void** h : {(void**)&c.hsc, (void**)&c.h_depth_pinned, (void**)&c.h_mu, (void**)&c.h_int})
    if (*h) {
      cudaFreeHost(*h);
      *h = nullptr;
    }
  for (GraphSlot* g : {&c.g_step, &c.g_attempt, &c.g_solve})
    if (g->exec) {
      cudaGraphExecDestroy(g->exec);
      g->exec = nullptr;
    }
  c.cfg.max_surfels = (int)S_new;
  c.cfg.max_nodes = (int)N_new;
  allocate(c);
  c.cur = 0;
  const ModelBuf& m = c.M();
  void* dst[] = {m.rp,       m.rn,      m.lp,       m.ln,  m.t,    m.ki,
                 m.kw,       c.node_pos, c.node_dq, c.node_nbr, c.dsc, c.depth};
  for (size_t k = 0; k < park.size(); ++k) {
    if (park[k].bytes)
      DS_CUDA(cudaMemcpyAsync(dst[k], park[k].p, park[k].bytes, cudaMemcpyDeviceToDevice, c.stream));
  }
  sync(c);
  for (auto& q : park) cudaFree(q.p);
  c.pattern_ready = false;
  c.pattern_frame = -1;
  c.mm_ready = c.im_ready = c.frame_ready = false;
  c.mm_clean = false;
  c.any_stable_ready = false;
  c.live_pending = false;
  c.nodes_pending = false;
  for (KnnGrid* g : {&c.grid_ref, &c.grid_live, &c.grid_new}) g->valid = false;
  ++c.capacity_growths;
}

// Frame-boundary headroom: a frame appends at most one surfel per valid pixel
// (fusion.cpp:235-257); the node set is kept below half the node capacity.
void ensure_frame_headroom(Ctx& c) {
  const long long need_s = (long long)c.n_surfels + c.P;
  const bool grow_s = need_s > c.S_cap;
  const bool grow_n = (long long)c.n_nodes * 2 > (long long)c.N_cap;
  if (!grow_s && !grow_n)
    return;
  grow_capacity(c, grow_s ? std::max(2LL * c.S_cap, need_s + c.P) : c.S_cap,
                grow_n ? 2LL * c.N_cap : c.N_cap);
}

// initialize_from_frame (pipeline.cpp:42-72)
void initialize_from_frame(Ctx& c) {
  init_surfels_from_frame(c);
  init_warp_field(c);
  c.t_last_reinit = c.frame_index;
  c.win_residual.clear();
  c.win_appended.clear();
  c.initialized = true;
  c.pattern_ready = false;
}

// should_reinitialize (reinit.cpp:9-26)
bool should_reinitialize(Ctx& c, int t_now) {
  const ds_config& k = c.cfg;
  if (k.periodic_reinit_interval > 0 && t_now - c.t_last_reinit >= k.periodic_reinit_interval)
    return true;
  if ((int)c.win_residual.size() < k.reinit_window) return false;
  const size_t n = c.win_residual.size();
  for (int i = 0; i < k.reinit_window; ++i) {
    if (c.win_residual[n - 1 - i] <= k.reinit_energy_threshold) return false;
    if (c.win_appended[n - 1 - i] <= k.reinit_append_threshold) return false;
  }
  return true;
}

struct PhaseEvents {
  cudaEvent_t e[6];
  PhaseEvents() {
    for (auto& x : e) DS_CUDA(cudaEventCreate(&x));
  }
  ~PhaseEvents() {
    for (auto& x : e) cudaEventDestroy(x);
  }
};

float elapsed(cudaEvent_t a, cudaEvent_t b) {
  float ms = 0;
  DS_CUDA(cudaEventElapsedTime(&ms, a, b));
  return ms;
}

// Pipeline::process_frame (pipeline.cpp:74-142)
void process_frame_impl(Ctx& c, const uint16_t* depth_dev, int fi, ds_frame_stats* st);
void process_frame(Ctx& c, const uint16_t* depth_dev, int fi, ds_frame_stats* st) {
  const auto t0 = std::chrono::steady_clock::now();
  process_frame_impl(c, depth_dev, fi, st);
  if (c.trace_host)
    std::fprintf(stderr, "frame %d host %.1f us gpu %.1f us\n", fi,
                 std::chrono::duration<double, std::micro>(std::chrono::steady_clock::now() - t0)
                     .count(),
                 st->total_ms * 1e3);
}
void process_frame_impl(Ctx& c, const uint16_t* depth_dev, int fi, ds_frame_stats* st) {
  std::memset(st, 0, sizeof *st);
  st->frame = fi;
  const int64_t launches0 = c.total_launches;
  if (c.initialized) {  // geometric growth happens between frames
    const bool own = depth_dev == c.depth;
    ensure_frame_headroom(c);
    if (own) depth_dev = c.depth;
  }
  PhaseEvents ev;
  DS_CUDA(cudaEventRecord(ev.e[0], c.stream));
  frame_maps(c, depth_dev, fi);
  DS_CUDA(cudaEventRecord(ev.e[1], c.stream));
  if (!c.initialized) {
    join_node_updates(c);  // deferred side-stream work must not race the new warp field
    c.any_stable_ready = false;
    set_identity(c.pose);
    for (int attempt = 0;; ++attempt) {  // the node count is known only after sampling
      try {
        initialize_from_frame(c);
        break;
      } catch (const Error& e) {
        if (e.code != DS_ERR_CAPACITY || attempt >= 16) throw;
        const bool own = depth_dev == c.depth;  // ds_process_frame's upload buffer
        c.n_surfels = 0;
        c.n_nodes = 0;
        grow_capacity(c, c.S_cap, 2LL * c.N_cap);
        if (own) depth_dev = c.depth;  // re-allocated, content kept
        frame_maps(c, depth_dev, fi);  // per-frame buffers were re-allocated
      }
    }
    DS_CUDA(cudaEventRecord(ev.e[5], c.stream));
    fetch_scalars(c);
    st->valid_pixels = c.hsc->valid_count;
    st->surfel_count = c.n_surfels;
    st->node_count = c.n_nodes;
    std::copy(c.pose, c.pose + 12, st->pose);
    st->depth_ms = elapsed(ev.e[0], ev.e[1]);
    st->total_ms = elapsed(ev.e[0], ev.e[5]);
    st->kernel_launches = (int)(c.total_launches - launches0);
    return;
  }
  const int t_now = fi;
  // the rigid ICP (main stream) and the frame's JtJ pattern build (side stream,
  // independent of the pose) overlap; the pattern's host syncs wait only on it
  rigid_align_enqueue(c, c.pose, c.pose, t_now, c.t_last_reinit);
  join_node_updates(c);  // last frame's deferred node / skinning updates (side stream)
  if (c.n_nodes > 0 && c.n_surfels > 0) {
    cudaStream_t main_stream = c.stream;
    c.stream = c.side;
    const auto tp0 = std::chrono::steady_clock::now();
    try {
      build_pattern_enqueue(c, t_now, c.t_last_reinit);
      if (c.trace_host)
        std::fprintf(stderr, "build_pattern (side, host) %.1f us\n",
                     std::chrono::duration<double, std::micro>(std::chrono::steady_clock::now() - tp0)
                         .count());
    } catch (...) {
      c.stream = main_stream;
      throw;
    }
    c.stream = main_stream;
    c.pattern_frame = t_now;
    DS_CUDA(cudaEventRecord(c.ev_join, c.side));  // work enqueued after its last sync
    DS_CUDA(cudaStreamWaitEvent(c.stream, c.ev_join, 0));
  }
  const auto tr0 = std::chrono::steady_clock::now();
  rigid_align_finish(c, c.pose, &st->rigid);
  pattern_adopt(c, true);  // counts came with the rigid ICP's scalar fetch
  if (c.trace_host)
    std::fprintf(stderr, "pattern (side) built; rigid wait %.1f us\n",
                 std::chrono::duration<double, std::micro>(std::chrono::steady_clock::now() - tr0)
                     .count());
  std::copy(st->rigid.pose, st->rigid.pose + 12, c.pose);
  DS_CUDA(cudaEventRecord(ev.e[2], c.stream));
  solve_nonrigid(c, c.pose, t_now, c.t_last_reinit, &st->solver);
  DS_CUDA(cudaEventRecord(ev.e[3], c.stream));
  if (c.n_nodes > 0) prepare_live_nodes_async(c);  // overlaps the warp / index map / fusion
  c.warp_in_index_map = true;  // forward_warp (pipeline.cpp:108) fused into the index map pass
  apply_fusion(c, c.pose, t_now, &st->fusion);
  DS_CUDA(cudaEventRecord(ev.e[4], c.stream));
  if (c.live_pending) {  // not consumed (no fusion): keep the stream order
    DS_CUDA(cudaStreamWaitEvent(c.stream, c.ev_live, 0));
    c.live_pending = false;
  }
  c.win_residual.push_back(st->solver.mean_residual);
  c.win_appended.push_back(st->fusion.appended);
  while ((int)c.win_residual.size() > c.cfg.reinit_window) c.win_residual.pop_front();
  while ((int)c.win_appended.size() > c.cfg.reinit_window) c.win_appended.pop_front();
  if (should_reinitialize(c, t_now)) {
    join_node_updates(c);  // the reset rebuilds nodes and skinning
    c.any_stable_ready = false;
    st->reinit = 1;
    try {
      st->reinit_removed = clean_and_reset(c, c.pose, nullptr);
    } catch (const Error& e) {
      if (e.code != DS_ERR_EMPTY_GEOMETRY) throw;
      st->reinit_removed = c.n_surfels;
      initialize_from_frame(c);
    }
    c.t_last_reinit = t_now;
    c.win_residual.clear();
    c.win_appended.clear();
  }
  DS_CUDA(cudaEventRecord(ev.e[5], c.stream));
  fetch_scalars(c);
  st->valid_pixels = c.hsc->valid_count;
  st->surfel_count = c.n_surfels;
  st->node_count = c.n_nodes;
  std::copy(c.pose, c.pose + 12, st->pose);
  st->depth_ms = elapsed(ev.e[0], ev.e[1]);
  st->rigid_ms = elapsed(ev.e[1], ev.e[2]);
  st->solve_ms = elapsed(ev.e[2], ev.e[3]);
  st->fusion_ms = elapsed(ev.e[3], ev.e[4]);
  st->reinit_ms = elapsed(ev.e[4], ev.e[5]);
  st->total_ms = elapsed(ev.e[0], ev.e[5]);
  st->lm_attempts = c.lm_attempts;
  st->pcg_iterations = c.pcg_iterations;
  st->gn_blocks = c.n_full;
  st->kernel_launches = (int)(c.total_launches - launches0);
}

// -------------------------------------------------------------- small kernels
__global__ void k_pair_flags(const int* __restrict__ pair_s, int P, int* __restrict__ f) {
  const int c = blockIdx.x * blockDim.x + threadIdx.x;
  if (c < P) f[c] = pair_s[c] >= 0 ? 1 : 0;
}
__global__ void k_pair_export(const int* __restrict__ pair_s, const int* __restrict__ scan, int P,
                              int W, ModelBuf m, const double4* __restrict__ fvert,
                              const double4* __restrict__ fnrm, Rig pose, int cap, int* surfel,
                              int* px, int* py, double* vm, double* vd, double* nd) {
  const int c = blockIdx.x * blockDim.x + threadIdx.x;
  if (c >= P) return;
  const int s = pair_s[c];
  if (s < 0) return;
  const int k = scan[c];
  if (k >= cap) return;
  surfel[k] = s;
  px[k] = c % W;
  py[k] = c / W;
  const float4 lp = m.lp[s];
  const double4 fv = fvert[c], fn = fnrm[c];
  const V3 v = rig_apply(pose, v3(fv.x, fv.y, fv.z));
  const V3 n = rig_rotate(pose, v3(fn.x, fn.y, fn.z));
  vm[3 * k] = lp.x;
  vm[3 * k + 1] = lp.y;
  vm[3 * k + 2] = lp.z;
  vd[3 * k] = v.x;
  vd[3 * k + 1] = v.y;
  vd[3 * k + 2] = v.z;
  nd[3 * k] = n.x;
  nd[3 * k + 1] = n.y;
  nd[3 * k + 2] = n.z;
}
__global__ void k_associate_only(const int* __restrict__ mm_idx, ModelBuf m,
                                 const double4* __restrict__ fvert, const double4* __restrict__ fnrm,
                                 const uint8_t* __restrict__ fflag, Rig pose, int P,
                                 int* __restrict__ pair_s) {
  const int c = blockIdx.x * blockDim.x + threadIdx.x;
  if (c >= P) return;
  const int win = mm_idx[c];
  int ps = -1;
  if (win >= 0 && (fflag[c] & 2)) {
    const double4 fv = fvert[c], fn = fnrm[c];
    const V3 vd = rig_apply(pose, v3(fv.x, fv.y, fv.z));
    const V3 nd = rig_rotate(pose, v3(fn.x, fn.y, fn.z));
    const float4 lp = m.lp[win], ln = m.ln[win];
    if (nrm(sub(v3(lp.x, lp.y, lp.z), vd)) < 0.03 && dot(v3(ln.x, ln.y, ln.z), nd) > 0.7) ps = win;
  }
  pair_s[c] = ps;
}

}  // namespace
}  // namespace ds

// ================================================================== C ABI
using ds::Ctx;

struct ds_context {
  Ctx c;
};

#define API_BEGIN try {
#define API_END                                      \
  }                                                  \
  catch (const ds::Error& e) {                       \
    ds::g_last_error = e.msg;                        \
    return e.code;                                   \
  }                                                  \
  catch (const std::exception& e) {                  \
    ds::g_last_error = e.what();                     \
    return DS_ERR_CUDA;                              \
  }                                                  \
  return DS_OK;
#define REQUIRE(cond, msg)                                      \
  do {                                                          \
    if (!(cond)) ds::fail(DS_ERR_INVALID_ARGUMENT, (msg));      \
  } while (0)

// every API call sees the side stream's deferred node / skinning updates
// (process_frame joins them itself, after launching the rigid ICP)
static void bind_nojoin(Ctx& c) { DS_CUDA(cudaSetDevice(c.device)); }
static void bind(Ctx& c) {
  bind_nojoin(c);
  ds::join_node_updates(c);
  c.any_stable_ready = false;  // the call may change the model
}

extern "C" {

void ds_default_config(ds_config* k) {
  std::memset(k, 0, sizeof *k);
  k->node_sigma = 0.025;
  k->knn_k = 4;
  k->node_neighbor_k = 8;
  k->lambda = 5.0;
  k->max_gn_iters = 10;
  k->delta_distance = 0.001;
  k->delta_normal = 0.85;
  k->epsilon = 0.2;
  k->delta_stable = 10.0;
  k->t_low_confid = 30;
  k->delta_recent = 2;
  k->delta_nn = 0.03;
  k->supersample_factor = 4;
  k->compressive_check = 1;
  k->depth_min = 0.1;
  k->depth_max = 5.0;
  k->bilateral_sigma_space = 4.5;
  k->bilateral_sigma_depth = 30.0;
  k->reinit_energy_threshold = 0.005;
  k->reinit_append_threshold = 3000;
  k->reinit_window = 3;
  k->periodic_reinit_interval = 0;
  k->delta_distance_reinit = 0.010;
  k->pcg_max_iters = 10;
  k->pcg_tol = 0.0;
}

const char* ds_last_error(void) { return ds::g_last_error.c_str(); }
int32_t ds_version(void) { return 1; }

ds_status ds_validate_config(const ds_config* cfg) {
  API_BEGIN
  REQUIRE(cfg, "null config");
  ds::validate(*cfg);
  API_END
}

ds_status ds_create(const ds_config* cfg, int32_t device, void* stream, ds_context** out) {
  ds_context* ctx = nullptr;
  try {
    REQUIRE(cfg && out, "null argument");
    ds::validate(*cfg);
    int count = 0;
    const cudaError_t e = cudaGetDeviceCount(&count);
    if (e != cudaSuccess || count == 0)
      ds::fail(DS_ERR_CUDA, "no CUDA device available (the B200 path has no CPU fallback)");
    if (device < 0 || device >= count) ds::fail(DS_ERR_INVALID_ARGUMENT, "bad device index");
    ctx = new ds_context();
    Ctx& c = ctx->c;
    c.cfg = *cfg;
    c.device = device;
    DS_CUDA(cudaSetDevice(device));
    DS_CUDA(cudaDeviceGetAttribute(&c.num_sms, cudaDevAttrMultiProcessorCount, device));
    if (stream) {
      c.stream = static_cast<cudaStream_t>(stream);
    } else {
      DS_CUDA(cudaStreamCreateWithFlags(&c.stream, cudaStreamNonBlocking));
      c.own_stream = true;
    }
    DS_CUDA(cudaStreamCreateWithFlags(&c.side, cudaStreamNonBlocking));
    DS_CUDA(cudaEventCreateWithFlags(&c.ev_fork, cudaEventDisableTiming));
    DS_CUDA(cudaEventCreateWithFlags(&c.ev_join, cudaEventDisableTiming));
    DS_CUDA(cudaEventCreateWithFlags(&c.ev_mid, cudaEventDisableTiming));
    DS_CUDA(cudaEventCreateWithFlags(&c.ev_live, cudaEventDisableTiming));
    DS_CUDA(cudaEventCreateWithFlags(&c.ev_nodes, cudaEventDisableTiming));
    ds::set_identity(c.pose);
    ds::allocate(c);
    ds::sync(c);
    *out = ctx;
    return DS_OK;
  } catch (const ds::Error& e) {
    ds::g_last_error = e.msg;
    if (ctx) {
      ds::release(ctx->c);
      delete ctx;
    }
    return e.code;
  }
}

ds_status ds_destroy(ds_context* ctx) {
  if (!ctx) return DS_OK;
  cudaSetDevice(ctx->c.device);
  cudaStreamSynchronize(ctx->c.stream);
  ds::release(ctx->c);
  delete ctx;
  return DS_OK;
}

ds_status ds_synchronize(ds_context* ctx) {
  API_BEGIN
  REQUIRE(ctx, "null context");
  bind(ctx->c);
  ds::sync(ctx->c);
  API_END
}

ds_status ds_capacity(const ds_context* ctx, int32_t* surfel_capacity, int32_t* node_capacity,
                      int32_t* growths) {
  API_BEGIN
  REQUIRE(ctx, "null context");
  if (surfel_capacity) *surfel_capacity = ctx->c.S_cap;
  if (node_capacity) *node_capacity = ctx->c.N_cap;
  if (growths) *growths = ctx->c.capacity_growths;
  API_END
}

ds_status ds_join_deferred(ds_context* ctx) {
  API_BEGIN
  REQUIRE(ctx, "null context");
  bind(ctx->c);
  API_END
}

static void check_dims(Ctx& c, int w, int h) {
  if (w != c.W || h != c.H)
    ds::fail(DS_ERR_DIMENSION_MISMATCH, "depth image size does not match intrinsics");
}

ds_status ds_process_frame(ds_context* ctx, const uint16_t* depth, int32_t w, int32_t h,
                           int32_t fi, ds_frame_stats* out) {
  API_BEGIN
  REQUIRE(ctx && depth && out, "null argument");
  Ctx& c = ctx->c;
  bind_nojoin(c);
  check_dims(c, w, h);
  std::memcpy(c.h_depth_pinned, depth, sizeof(uint16_t) * c.P);
  DS_CUDA(cudaMemcpyAsync(c.depth, c.h_depth_pinned, sizeof(uint16_t) * c.P,
                          cudaMemcpyHostToDevice, c.stream));
  ds::process_frame(c, c.depth, fi, out);
  API_END
}

ds_status ds_process_frame_device(ds_context* ctx, const uint16_t* depth_dev, int32_t w, int32_t h,
                                  int32_t fi, ds_frame_stats* out) {
  API_BEGIN
  REQUIRE(ctx && depth_dev && out, "null argument");
  Ctx& c = ctx->c;
  bind_nojoin(c);
  check_dims(c, w, h);
  ds::process_frame(c, depth_dev, fi, out);
  API_END
}

ds_status ds_is_initialized(const ds_context* ctx, int32_t* init, int32_t* last) {
  API_BEGIN
  REQUIRE(ctx, "null context");
  if (init) *init = ctx->c.initialized ? 1 : 0;
  if (last) *last = ctx->c.t_last_reinit;
  API_END
}

ds_status ds_reset(ds_context* ctx) {
  API_BEGIN
  REQUIRE(ctx, "null context");
  Ctx& c = ctx->c;
  bind(c);  // the deferred side-stream node / skinning work writes the buffers the reset frees
  c.initialized = false;
  c.n_surfels = 0;
  c.n_nodes = 0;
  c.t_last_reinit = 0;
  c.win_residual.clear();
  c.win_appended.clear();
  c.pattern_ready = false;
  c.mm_ready = c.im_ready = c.frame_ready = false;
  ds::set_identity(c.pose);
  API_END
}

ds_status ds_upload_model(ds_context* ctx, int32_t n, const double* rp, const double* rn,
                          const double* lp, const double* ln, const double* radius,
                          const double* conf, const int32_t* ti, const int32_t* to,
                          const int32_t* sidx, const double* sw, const int32_t* scount) {
  API_BEGIN
  REQUIRE(ctx && n >= 0, "bad argument");
  Ctx& c = ctx->c;
  bind(c);
  ds::ensure_surfel_capacity(c, n);
  std::vector<float4> a(n), b(n), d(n), e(n), w(n);
  std::vector<int2> t(n);
  std::vector<int4> k(n);
  for (int i = 0; i < n; ++i) {
    a[i] = make_float4((float)rp[3 * i], (float)rp[3 * i + 1], (float)rp[3 * i + 2], (float)radius[i]);
    b[i] = make_float4((float)rn[3 * i], (float)rn[3 * i + 1], (float)rn[3 * i + 2], (float)conf[i]);
    d[i] = make_float4((float)lp[3 * i], (float)lp[3 * i + 1], (float)lp[3 * i + 2], (float)radius[i]);
    e[i] = make_float4((float)ln[3 * i], (float)ln[3 * i + 1], (float)ln[3 * i + 2], (float)conf[i]);
    t[i] = make_int2(ti[i], to[i]);
    const int cnt = scount[i];
    if (cnt < 0 || cnt > 4) ds::fail(DS_ERR_INVALID_ARGUMENT, "device keeps at most 4 skinning slots");
    int id[4] = {-1, -1, -1, -1};
    float ww[4] = {0, 0, 0, 0};
    for (int m = 0; m < cnt; ++m) {
      id[m] = sidx[8 * i + m];
      ww[m] = (float)sw[8 * i + m];
    }
    k[i] = make_int4(id[0], id[1], id[2], id[3]);
    w[i] = make_float4(ww[0], ww[1], ww[2], ww[3]);
  }
  ds::ModelBuf& m = c.M();
  DS_CUDA(cudaMemcpyAsync(m.rp, a.data(), sizeof(float4) * n, cudaMemcpyHostToDevice, c.stream));
  DS_CUDA(cudaMemcpyAsync(m.rn, b.data(), sizeof(float4) * n, cudaMemcpyHostToDevice, c.stream));
  DS_CUDA(cudaMemcpyAsync(m.lp, d.data(), sizeof(float4) * n, cudaMemcpyHostToDevice, c.stream));
  DS_CUDA(cudaMemcpyAsync(m.ln, e.data(), sizeof(float4) * n, cudaMemcpyHostToDevice, c.stream));
  DS_CUDA(cudaMemcpyAsync(m.t, t.data(), sizeof(int2) * n, cudaMemcpyHostToDevice, c.stream));
  DS_CUDA(cudaMemcpyAsync(m.ki, k.data(), sizeof(int4) * n, cudaMemcpyHostToDevice, c.stream));
  DS_CUDA(cudaMemcpyAsync(m.kw, w.data(), sizeof(float4) * n, cudaMemcpyHostToDevice, c.stream));
  ds::sync(c);
  c.n_surfels = n;
  c.pattern_ready = false;
  API_END
}

ds_status ds_model_size(const ds_context* ctx, int32_t* n) {
  API_BEGIN
  REQUIRE(ctx && n, "null argument");
  *n = ctx->c.n_surfels;
  API_END
}

ds_status ds_download_model(ds_context* ctx, double* rp, double* rn, double* lp, double* ln,
                            double* radius, double* conf, int32_t* ti, int32_t* to, int32_t* sidx,
                            double* sw, int32_t* scount) {
  API_BEGIN
  REQUIRE(ctx, "null context");
  Ctx& c = ctx->c;
  bind(c);
  const int n = c.n_surfels;
  std::vector<float4> a(n), b(n), d(n), e(n), w(n);
  std::vector<int2> t(n);
  std::vector<int4> k(n);
  ds::ModelBuf& m = c.M();
  DS_CUDA(cudaMemcpyAsync(a.data(), m.rp, sizeof(float4) * n, cudaMemcpyDeviceToHost, c.stream));
  DS_CUDA(cudaMemcpyAsync(b.data(), m.rn, sizeof(float4) * n, cudaMemcpyDeviceToHost, c.stream));
  DS_CUDA(cudaMemcpyAsync(d.data(), m.lp, sizeof(float4) * n, cudaMemcpyDeviceToHost, c.stream));
  DS_CUDA(cudaMemcpyAsync(e.data(), m.ln, sizeof(float4) * n, cudaMemcpyDeviceToHost, c.stream));
  DS_CUDA(cudaMemcpyAsync(t.data(), m.t, sizeof(int2) * n, cudaMemcpyDeviceToHost, c.stream));
  DS_CUDA(cudaMemcpyAsync(k.data(), m.ki, sizeof(int4) * n, cudaMemcpyDeviceToHost, c.stream));
  DS_CUDA(cudaMemcpyAsync(w.data(), m.kw, sizeof(float4) * n, cudaMemcpyDeviceToHost, c.stream));
  ds::sync(c);
  for (int i = 0; i < n; ++i) {
    if (rp) { rp[3 * i] = a[i].x; rp[3 * i + 1] = a[i].y; rp[3 * i + 2] = a[i].z; }
    if (rn) { rn[3 * i] = b[i].x; rn[3 * i + 1] = b[i].y; rn[3 * i + 2] = b[i].z; }
    if (lp) { lp[3 * i] = d[i].x; lp[3 * i + 1] = d[i].y; lp[3 * i + 2] = d[i].z; }
    if (ln) { ln[3 * i] = e[i].x; ln[3 * i + 1] = e[i].y; ln[3 * i + 2] = e[i].z; }
    if (radius) radius[i] = d[i].w;
    if (conf) conf[i] = e[i].w;
    if (ti) ti[i] = t[i].x;
    if (to) to[i] = t[i].y;
    const int ids[4] = {k[i].x, k[i].y, k[i].z, k[i].w};
    const float ws[4] = {w[i].x, w[i].y, w[i].z, w[i].w};
    int cnt = 0;
    while (cnt < 4 && ids[cnt] >= 0) ++cnt;
    if (scount) scount[i] = cnt;
    for (int m2 = 0; m2 < 8; ++m2) {
      if (sidx) sidx[8 * i + m2] = m2 < cnt ? ids[m2] : -1;
      if (sw) sw[8 * i + m2] = m2 < cnt ? (double)ws[m2] : 0.0;
    }
  }
  API_END
}

ds_status ds_upload_nodes(ds_context* ctx, int32_t n, const double* pos, const double* sigma,
                          const double* dq, const int32_t* nbr, const int32_t* nbr_count) {
  API_BEGIN
  REQUIRE(ctx && n >= 0, "bad argument");
  Ctx& c = ctx->c;
  bind(c);
  ds::ensure_node_capacity(c, n);
  std::vector<double4> p(n), q(2 * (size_t)n);
  std::vector<int> nb(8 * (size_t)n, -1);
  for (int j = 0; j < n; ++j) {
    p[j] = make_double4(pos[3 * j], pos[3 * j + 1], pos[3 * j + 2], sigma[j]);
    q[2 * j] = make_double4(dq[8 * j], dq[8 * j + 1], dq[8 * j + 2], dq[8 * j + 3]);
    q[2 * j + 1] = make_double4(dq[8 * j + 4], dq[8 * j + 5], dq[8 * j + 6], dq[8 * j + 7]);
    const int cnt = nbr_count ? nbr_count[j] : 0;
    if (cnt < 0 || cnt > 8) ds::fail(DS_ERR_INVALID_ARGUMENT, "device keeps at most 8 node edges");
    for (int k = 0; k < cnt; ++k) nb[8 * j + k] = nbr[8 * j + k];
  }
  DS_CUDA(cudaMemcpyAsync(c.node_pos, p.data(), sizeof(double4) * n, cudaMemcpyHostToDevice, c.stream));
  DS_CUDA(cudaMemcpyAsync(c.node_dq, q.data(), sizeof(double4) * 2 * n, cudaMemcpyHostToDevice, c.stream));
  DS_CUDA(cudaMemcpyAsync(c.node_nbr, nb.data(), sizeof(int) * 8 * n, cudaMemcpyHostToDevice, c.stream));
  ds::sync(c);
  c.n_nodes = n;
  c.pattern_ready = false;
  API_END
}

ds_status ds_num_nodes(const ds_context* ctx, int32_t* n) {
  API_BEGIN
  REQUIRE(ctx && n, "null argument");
  *n = ctx->c.n_nodes;
  API_END
}

ds_status ds_download_nodes(ds_context* ctx, double* pos, double* sigma, double* dq, int32_t* nbr,
                            int32_t* nbr_count) {
  API_BEGIN
  REQUIRE(ctx, "null context");
  Ctx& c = ctx->c;
  bind(c);
  const int n = c.n_nodes;
  std::vector<double4> p(n), q(2 * (size_t)n);
  std::vector<int> nb(8 * (size_t)n);
  DS_CUDA(cudaMemcpyAsync(p.data(), c.node_pos, sizeof(double4) * n, cudaMemcpyDeviceToHost, c.stream));
  DS_CUDA(cudaMemcpyAsync(q.data(), c.node_dq, sizeof(double4) * 2 * n, cudaMemcpyDeviceToHost, c.stream));
  DS_CUDA(cudaMemcpyAsync(nb.data(), c.node_nbr, sizeof(int) * 8 * n, cudaMemcpyDeviceToHost, c.stream));
  ds::sync(c);
  for (int j = 0; j < n; ++j) {
    if (pos) { pos[3 * j] = p[j].x; pos[3 * j + 1] = p[j].y; pos[3 * j + 2] = p[j].z; }
    if (sigma) sigma[j] = p[j].w;
    if (dq) {
      const double v[8] = {q[2 * j].x, q[2 * j].y, q[2 * j].z, q[2 * j].w,
                           q[2 * j + 1].x, q[2 * j + 1].y, q[2 * j + 1].z, q[2 * j + 1].w};
      std::memcpy(dq + 8 * j, v, sizeof v);
    }
    int cnt = 0;
    while (cnt < 8 && nb[8 * j + cnt] >= 0) ++cnt;
    if (nbr_count) nbr_count[j] = cnt;
    if (nbr)
      for (int k = 0; k < 8; ++k) nbr[8 * j + k] = k < cnt ? nb[8 * j + k] : -1;
  }
  API_END
}

ds_status ds_set_pose(ds_context* ctx, const double* pose) {
  API_BEGIN
  REQUIRE(ctx && pose, "null argument");
  std::copy(pose, pose + 12, ctx->c.pose);
  API_END
}
ds_status ds_get_pose(ds_context* ctx, double* pose) {
  API_BEGIN
  REQUIRE(ctx && pose, "null argument");
  std::copy(ctx->c.pose, ctx->c.pose + 12, pose);
  API_END
}

ds_status ds_frame_maps(ds_context* ctx, const uint16_t* depth, int32_t w, int32_t h, int32_t fi,
                        int32_t* valid_count) {
  API_BEGIN
  REQUIRE(ctx && depth, "null argument");
  Ctx& c = ctx->c;
  bind(c);
  check_dims(c, w, h);
  DS_CUDA(cudaMemcpyAsync(c.depth, depth, sizeof(uint16_t) * c.P, cudaMemcpyHostToDevice, c.stream));
  ds::frame_maps(c, c.depth, fi);
  ds::fetch_scalars(c);
  if (valid_count) *valid_count = c.hsc->valid_count;
  API_END
}

ds_status ds_download_frame(ds_context* ctx, double* vert, double* nrm, double* conf,
                            double* radius, uint8_t* vvalid, uint8_t* valid) {
  API_BEGIN
  REQUIRE(ctx, "null context");
  Ctx& c = ctx->c;
  bind(c);
  std::vector<double4> v(c.P), n(c.P);
  std::vector<uint8_t> f(c.P);
  DS_CUDA(cudaMemcpyAsync(v.data(), c.f_vert, sizeof(double4) * c.P, cudaMemcpyDeviceToHost, c.stream));
  DS_CUDA(cudaMemcpyAsync(n.data(), c.f_nrm, sizeof(double4) * c.P, cudaMemcpyDeviceToHost, c.stream));
  DS_CUDA(cudaMemcpyAsync(f.data(), c.f_flag, c.P, cudaMemcpyDeviceToHost, c.stream));
  ds::sync(c);
  for (int i = 0; i < c.P; ++i) {
    if (vert) { vert[3 * i] = v[i].x; vert[3 * i + 1] = v[i].y; vert[3 * i + 2] = v[i].z; }
    if (nrm) { nrm[3 * i] = n[i].x; nrm[3 * i + 1] = n[i].y; nrm[3 * i + 2] = n[i].z; }
    if (radius) radius[i] = v[i].w;
    if (conf) conf[i] = n[i].w;
    if (vvalid) vvalid[i] = f[i] & 1;
    if (valid) valid[i] = (f[i] >> 1) & 1;
  }
  API_END
}

ds_status ds_upload_frame(ds_context* ctx, int32_t w, int32_t h, int32_t fi, const double* vert,
                          const double* nrm, const double* conf, const double* radius,
                          const uint8_t* vvalid, const uint8_t* valid) {
  API_BEGIN
  REQUIRE(ctx && vert && nrm && conf && radius && vvalid && valid, "null argument");
  Ctx& c = ctx->c;
  bind(c);
  check_dims(c, w, h);
  std::vector<double4> v(c.P), n(c.P);
  std::vector<uint8_t> f(c.P);
  int vc = 0;
  for (int i = 0; i < c.P; ++i) {
    v[i] = make_double4(vert[3 * i], vert[3 * i + 1], vert[3 * i + 2], radius[i]);
    n[i] = make_double4(nrm[3 * i], nrm[3 * i + 1], nrm[3 * i + 2], conf[i]);
    f[i] = (vvalid[i] ? 1 : 0) | (valid[i] ? 2 : 0);
    vc += valid[i] ? 1 : 0;
  }
  DS_CUDA(cudaMemcpyAsync(c.f_vert, v.data(), sizeof(double4) * c.P, cudaMemcpyHostToDevice, c.stream));
  DS_CUDA(cudaMemcpyAsync(c.f_nrm, n.data(), sizeof(double4) * c.P, cudaMemcpyHostToDevice, c.stream));
  DS_CUDA(cudaMemcpyAsync(c.f_flag, f.data(), c.P, cudaMemcpyHostToDevice, c.stream));
  DS_CUDA(cudaMemcpyAsync(&c.dsc->valid_count, &vc, sizeof(int), cudaMemcpyHostToDevice, c.stream));
  ds::sync(c);
  c.frame_index = fi;
  c.frame_ready = true;
  API_END
}

ds_status ds_init_warp_field(ds_context* ctx) {
  API_BEGIN
  REQUIRE(ctx, "null context");
  bind(ctx->c);
  ds::init_warp_field(ctx->c);
  ctx->c.pattern_ready = false;
  ds::sync(ctx->c);
  API_END
}

ds_status ds_compute_node_edges(ds_context* ctx) {
  API_BEGIN
  REQUIRE(ctx, "null context");
  bind(ctx->c);
  ds::compute_node_edges(ctx->c);
  ctx->c.pattern_ready = false;
  ds::sync(ctx->c);
  API_END
}

ds_status ds_forward_warp(ds_context* ctx, int32_t* degenerate) {
  API_BEGIN
  REQUIRE(ctx, "null context");
  bind(ctx->c);
  const int d = ds::forward_warp(ctx->c, true);
  if (degenerate) *degenerate = d;
  API_END
}

ds_status ds_render_index_map(ds_context* ctx, const double* pose, int32_t factor, int32_t* idx) {
  API_BEGIN
  REQUIRE(ctx && pose && factor >= 1, "bad argument");
  Ctx& c = ctx->c;
  bind(c);
  ds::render_index_map(c, pose, factor);
  if (idx) {
    const size_t cells = (size_t)c.P * factor * factor;
    DS_CUDA(cudaMemcpyAsync(idx, c.im_idx, sizeof(int) * cells, cudaMemcpyDeviceToHost, c.stream));
    ds::sync(c);
    for (size_t i = 0; i < cells; ++i)
      if (idx[i] == 0x7f7f7f7f) idx[i] = -1;
  } else {
    ds::sync(c);
  }
  API_END
}

ds_status ds_render_model_maps(ds_context* ctx, const double* pose, int32_t t_now, int32_t t_last,
                               int32_t* idx, double* vert, double* nrm, double* depth,
                               uint8_t* valid) {
  API_BEGIN
  REQUIRE(ctx && pose, "bad argument");
  Ctx& c = ctx->c;
  bind(c);
  ds::render_model_maps(c, pose, t_now, t_last, false, nullptr);
  std::vector<int> mi(c.P), pi(c.P);
  std::vector<unsigned long long> pk(c.P), sk(c.P);
  DS_CUDA(cudaMemcpyAsync(mi.data(), c.mm_idx, sizeof(int) * c.P, cudaMemcpyDeviceToHost, c.stream));
  DS_CUDA(cudaMemcpyAsync(pi.data(), c.mm_pidx, sizeof(int) * c.P, cudaMemcpyDeviceToHost, c.stream));
  DS_CUDA(cudaMemcpyAsync(pk.data(), c.mm_pkey, 8 * (size_t)c.P, cudaMemcpyDeviceToHost, c.stream));
  DS_CUDA(cudaMemcpyAsync(sk.data(), c.mm_skey, 8 * (size_t)c.P, cudaMemcpyDeviceToHost, c.stream));
  std::vector<float4> lp(c.n_surfels), ln(c.n_surfels);
  DS_CUDA(cudaMemcpyAsync(lp.data(), c.M().lp, sizeof(float4) * c.n_surfels, cudaMemcpyDeviceToHost, c.stream));
  DS_CUDA(cudaMemcpyAsync(ln.data(), c.M().ln, sizeof(float4) * c.n_surfels, cudaMemcpyDeviceToHost, c.stream));
  ds::sync(c);
  for (int i = 0; i < c.P; ++i) {
    const int w = mi[i];
    if (idx) idx[i] = w;
    if (valid) valid[i] = w >= 0 ? 1 : 0;
    double d = INFINITY;
    if (w >= 0) {
      const unsigned long long k = (pi[i] != 0x7f7f7f7f) ? pk[i] : sk[i];
      std::memcpy(&d, &k, sizeof d);
    }
    if (depth) depth[i] = d;
    for (int a = 0; a < 3; ++a) {
      if (vert) vert[3 * i + a] = w >= 0 ? (&lp[w].x)[a] : 0.0;
      if (nrm) nrm[3 * i + a] = w >= 0 ? (&ln[w].x)[a] : 0.0;
    }
  }
  API_END
}

ds_status ds_associate(ds_context* ctx, const double* pose, int32_t cap, int32_t* n_pairs,
                       int32_t* surfel, int32_t* px, int32_t* py, double* vm, double* vd,
                       double* nd) {
  API_BEGIN
  REQUIRE(ctx && pose && n_pairs, "bad argument");
  Ctx& c = ctx->c;
  bind(c);
  REQUIRE(c.mm_ready && c.frame_ready, "associate: no model maps / frame");
  DS_LAUNCH(c, ds::KK_ASSOCIATE, 113.0 * c.P, ds::cdiv(c.P, 256), 256, 0, ds::k_associate_only,
            c.mm_idx, c.M(), c.f_vert, c.f_nrm, c.f_flag, ds::rig_load(pose), c.P, c.pair_s);
  DS_LAUNCH(c, ds::KK_MISC, 8.0 * c.P, ds::cdiv(c.P, 256), 256, 0, ds::k_pair_flags, c.pair_s, c.P,
            c.cand_flag);
  ds::scan_exclusive(c, c.cand_flag, c.cand_scan, c.P);
  int total = 0;
  DS_CUDA(cudaMemcpyAsync(&total, c.cand_scan + c.P, sizeof(int), cudaMemcpyDeviceToHost, c.stream));
  ds::sync(c);
  *n_pairs = total;
  const int m = std::min(total, cap);
  if (m > 0 && surfel && px && py && vm && vd && nd) {
    int *d_s = nullptr, *d_x = nullptr, *d_y = nullptr;
    double *d_vm = nullptr, *d_vd = nullptr, *d_nd = nullptr;
    DS_CUDA(cudaMalloc(&d_s, sizeof(int) * m * 3));
    DS_CUDA(cudaMalloc(&d_vm, sizeof(double) * m * 9));
    d_x = d_s + m;
    d_y = d_s + 2 * m;
    d_vd = d_vm + 3 * m;
    d_nd = d_vm + 6 * m;
    DS_LAUNCH(c, ds::KK_MISC, 80.0 * m, ds::cdiv(c.P, 256), 256, 0, ds::k_pair_export, c.pair_s,
              c.cand_scan, c.P, c.W, c.M(), c.f_vert, c.f_nrm, ds::rig_load(pose), m, d_s, d_x, d_y,
              d_vm, d_vd, d_nd);
    DS_CUDA(cudaMemcpyAsync(surfel, d_s, sizeof(int) * m, cudaMemcpyDeviceToHost, c.stream));
    DS_CUDA(cudaMemcpyAsync(px, d_x, sizeof(int) * m, cudaMemcpyDeviceToHost, c.stream));
    DS_CUDA(cudaMemcpyAsync(py, d_y, sizeof(int) * m, cudaMemcpyDeviceToHost, c.stream));
    DS_CUDA(cudaMemcpyAsync(vm, d_vm, sizeof(double) * 3 * m, cudaMemcpyDeviceToHost, c.stream));
    DS_CUDA(cudaMemcpyAsync(vd, d_vd, sizeof(double) * 3 * m, cudaMemcpyDeviceToHost, c.stream));
    DS_CUDA(cudaMemcpyAsync(nd, d_nd, sizeof(double) * 3 * m, cudaMemcpyDeviceToHost, c.stream));
    ds::sync(c);
    cudaFree(d_s);
    cudaFree(d_vm);
  }
  API_END
}

ds_status ds_build_normal_equations(ds_context* ctx, const double* pose, int32_t t_now,
                                    int32_t t_last, int32_t* n_blocks, int32_t* n_pairs,
                                    double* e_pre) {
  API_BEGIN
  REQUIRE(ctx && pose, "bad argument");
  Ctx& c = ctx->c;
  bind(c);
  REQUIRE(c.frame_ready, "no frame maps");
  ds::build_pattern(c, t_now, t_last);
  ds::gn_linearize(c, pose, t_now, t_last, e_pre, n_pairs);
  if (n_blocks) *n_blocks = c.n_full;
  API_END
}

ds_status ds_download_normal_equations(ds_context* ctx, int32_t* row_ptr, int32_t* col,
                                       double* values, uint8_t* touched, double* g) {
  API_BEGIN
  REQUIRE(ctx, "null context");
  Ctx& c = ctx->c;
  bind(c);
  const int N = c.n_nodes, B = c.n_full;
  std::vector<float> v((size_t)B * 36);
  if (row_ptr) DS_CUDA(cudaMemcpyAsync(row_ptr, c.row_ptr, sizeof(int) * (N + 1), cudaMemcpyDeviceToHost, c.stream));
  if (col) DS_CUDA(cudaMemcpyAsync(col, c.bsr_col, sizeof(int) * B, cudaMemcpyDeviceToHost, c.stream));
  DS_CUDA(cudaMemcpyAsync(v.data(), c.bsr_val, sizeof(float) * 36 * B, cudaMemcpyDeviceToHost, c.stream));
  if (touched) DS_CUDA(cudaMemcpyAsync(touched, c.bsr_touch, B, cudaMemcpyDeviceToHost, c.stream));
  if (g) DS_CUDA(cudaMemcpyAsync(g, c.g, sizeof(double) * 6 * N, cudaMemcpyDeviceToHost, c.stream));
  ds::sync(c);
  if (values)
    for (size_t i = 0; i < v.size(); ++i) values[i] = v[i];
  API_END
}

ds_status ds_check_normal_equations(ds_context* ctx) {
  API_BEGIN
  REQUIRE(ctx, "null context");
  Ctx& c = ctx->c;
  bind(c);
  REQUIRE(c.pattern_ready, "no assembled system");
  ds::check_normal_equations(c);
  API_END
}

ds_status ds_set_normal_equation_values(ds_context* ctx, const double* values, const double* g) {
  API_BEGIN
  REQUIRE(ctx && values, "null argument");
  Ctx& c = ctx->c;
  bind(c);
  REQUIRE(c.pattern_ready, "no assembled system");
  const int B = c.n_full;
  std::vector<float> v((size_t)B * 36);
  for (size_t i = 0; i < v.size(); ++i) v[i] = (float)values[i];
  DS_CUDA(cudaMemcpyAsync(c.bsr_val, v.data(), sizeof(float) * v.size(), cudaMemcpyHostToDevice,
                          c.stream));
  if (g)
    DS_CUDA(cudaMemcpyAsync(c.g, g, sizeof(double) * 6 * c.n_nodes, cudaMemcpyHostToDevice, c.stream));
  ds::sync(c);
  API_END
}

ds_status ds_pcg_solve(ds_context* ctx, double mu, int32_t max_iters, double tol, double* delta,
                       int32_t* iters, double* rel) {
  API_BEGIN
  REQUIRE(ctx, "null context");
  Ctx& c = ctx->c;
  bind(c);
  REQUIRE(c.pattern_ready, "no assembled system");
  int it = 0;
  double rr = 0;
  ds::pcg_solve(c, mu, max_iters, tol, &it, &rr);
  if (iters) *iters = it;
  if (rel) *rel = rr;
  if (delta) {
    DS_CUDA(cudaMemcpyAsync(delta, c.pcg_x, sizeof(double) * 6 * c.n_nodes, cudaMemcpyDeviceToHost,
                            c.stream));
    ds::sync(c);
  }
  if (c.pcg_trace) {  // DS_PCG_TRACE: phase timestamps of CTA 0, us from kernel start
    unsigned long long tr[64];
    DS_CUDA(cudaMemcpy(tr, c.pcg_trace, sizeof tr, cudaMemcpyDeviceToHost));
    std::fprintf(stderr, "pcg_trace");
    for (int k = 1; k < 64; ++k)
      if (tr[k] >= tr[0] && tr[k] - tr[0] < 100000000ull)
        std::fprintf(stderr, " %d:%.2f", k, (tr[k] - tr[0]) * 1e-3);
    std::fprintf(stderr, "\n");
    DS_CUDA(cudaMemset(c.pcg_trace, 0, sizeof tr));
  }
  API_END
}

ds_status ds_bsr_spmv(ds_context* ctx, const double* x, double* y, double mu, int32_t reps,
                      double* mean_ms) {
  API_BEGIN
  REQUIRE(ctx && x && y && reps >= 0, "bad argument");
  Ctx& c = ctx->c;
  bind(c);
  REQUIRE(c.pattern_ready, "no assembled system");
  const size_t n6 = 6 * (size_t)c.n_nodes;
  DS_CUDA(cudaMemcpyAsync(c.pcg_p0, x, sizeof(double) * n6, cudaMemcpyHostToDevice, c.stream));
  const double ms = ds::bsr_spmv(c, c.pcg_p0, c.pcg_q, mu, std::max(1, (int)reps));
  DS_CUDA(cudaMemcpyAsync(y, c.pcg_q, sizeof(double) * n6, cudaMemcpyDeviceToHost, c.stream));
  ds::sync(c);
  if (mean_ms) *mean_ms = ms;
  API_END
}

ds_status ds_solve_nonrigid(ds_context* ctx, const double* pose, int32_t t_now, int32_t t_last,
                            ds_solver_report* out) {
  API_BEGIN
  REQUIRE(ctx && pose && out, "bad argument");
  Ctx& c = ctx->c;
  bind(c);
  REQUIRE(c.frame_ready, "no frame maps");
  ds::solve_nonrigid(c, pose, t_now, t_last, out);
  API_END
}

ds_status ds_rigid_align(ds_context* ctx, const double* render_pose, const double* init_pose,
                         int32_t t_now, int32_t t_last, ds_rigid_result* out) {
  API_BEGIN
  REQUIRE(ctx && render_pose && init_pose && out, "bad argument");
  Ctx& c = ctx->c;
  bind(c);
  REQUIRE(c.frame_ready, "no frame maps");
  ds::rigid_align(c, render_pose, init_pose, t_now, t_last, out);
  API_END
}

ds_status ds_apply_fusion(ds_context* ctx, const double* pose, int32_t t_now, ds_fusion_outcome* out) {
  API_BEGIN
  REQUIRE(ctx && pose && out, "bad argument");
  Ctx& c = ctx->c;
  bind(c);
  REQUIRE(c.frame_ready, "no frame maps");
  ds::apply_fusion(c, pose, t_now, out);
  API_END
}

ds_status ds_fuse_depth(ds_context* ctx, const double* pose, int32_t t_now, int32_t* fused,
                        int32_t* n_cand) {
  API_BEGIN
  REQUIRE(ctx && pose, "bad argument");
  Ctx& c = ctx->c;
  bind(c);
  int f = 0, nc = 0;
  ds::fuse_depth(c, pose, t_now, &f, &nc);
  if (fused) *fused = f;
  if (n_cand) *n_cand = nc;
  API_END
}

ds_status ds_download_candidates(ds_context* ctx, double* pos, double* nrm, double* radius,
                                 double* conf, int32_t* px, int32_t* py) {
  API_BEGIN
  REQUIRE(ctx, "null context");
  Ctx& c = ctx->c;
  bind(c);
  ds::fetch_scalars(c);
  const int n = c.hsc->n_cand;
  std::vector<float4> p(n), q(n);
  std::vector<int> pix(n);
  DS_CUDA(cudaMemcpyAsync(p.data(), c.cand_p, sizeof(float4) * n, cudaMemcpyDeviceToHost, c.stream));
  DS_CUDA(cudaMemcpyAsync(q.data(), c.cand_n, sizeof(float4) * n, cudaMemcpyDeviceToHost, c.stream));
  DS_CUDA(cudaMemcpyAsync(pix.data(), c.cand_pix, sizeof(int) * n, cudaMemcpyDeviceToHost, c.stream));
  ds::sync(c);
  for (int i = 0; i < n; ++i) {
    if (pos) { pos[3 * i] = p[i].x; pos[3 * i + 1] = p[i].y; pos[3 * i + 2] = p[i].z; }
    if (nrm) { nrm[3 * i] = q[i].x; nrm[3 * i + 1] = q[i].y; nrm[3 * i + 2] = q[i].z; }
    if (radius) radius[i] = p[i].w;
    if (conf) conf[i] = q[i].w;
    if (px) px[i] = pix[i] % c.W;
    if (py) py[i] = pix[i] / c.W;
  }
  API_END
}

ds_status ds_skin_appended(ds_context* ctx, int32_t n, const double* positions,
                           const double* node_live, int32_t* sidx, double* sw, int32_t* scount,
                           uint8_t* supported, uint8_t* comp_ok) {
  API_BEGIN
  REQUIRE(ctx && positions && n >= 0 && n <= ctx->c.P, "bad argument");
  Ctx& c = ctx->c;
  bind(c);
  std::vector<float4> p(n);
  for (int i = 0; i < n; ++i)
    p[i] = make_float4((float)positions[3 * i], (float)positions[3 * i + 1],
                       (float)positions[3 * i + 2], 0.f);
  DS_CUDA(cudaMemcpyAsync(c.cand_p, p.data(), sizeof(float4) * n, cudaMemcpyHostToDevice, c.stream));
  (void)node_live;  // node live positions are derived on the device from the node transforms
  int low = 0, comp = 0, acc = 0;
  ds::screen_candidates(c, n, &low, &comp, &acc);
  std::vector<int4> ki(n);
  std::vector<float4> kw(n);
  std::vector<int> res(n);
  DS_CUDA(cudaMemcpyAsync(ki.data(), c.cand_ki, sizeof(int4) * n, cudaMemcpyDeviceToHost, c.stream));
  DS_CUDA(cudaMemcpyAsync(kw.data(), c.cand_kw, sizeof(float4) * n, cudaMemcpyDeviceToHost, c.stream));
  DS_CUDA(cudaMemcpyAsync(res.data(), c.cand_flag, sizeof(int) * n, cudaMemcpyDeviceToHost, c.stream));
  ds::sync(c);
  for (int i = 0; i < n; ++i) {
    const int ids[4] = {ki[i].x, ki[i].y, ki[i].z, ki[i].w};
    const float ws[4] = {kw[i].x, kw[i].y, kw[i].z, kw[i].w};
    int cnt = 0;
    while (cnt < 4 && ids[cnt] >= 0) ++cnt;
    if (scount) scount[i] = cnt;
    for (int m = 0; m < 8; ++m) {
      if (sidx) sidx[8 * i + m] = m < cnt ? ids[m] : -1;
      if (sw) sw[8 * i + m] = m < cnt ? (double)ws[m] : 0.0;
    }
    if (supported) supported[i] = res[i] >= 1 ? 1 : 0;  // skin_appended returned an entry
    if (comp_ok) comp_ok[i] = res[i] == 2 ? 1 : 0;      // and check_compressive kept it
  }
  API_END
}

ds_status ds_remove_mask(ds_context* ctx, const double* pose, int32_t t_now, uint8_t* mask) {
  API_BEGIN
  REQUIRE(ctx && pose, "bad argument");
  Ctx& c = ctx->c;
  bind(c);
  REQUIRE(c.im_ready, "remove_mask: no index map rendered");
  const int n = c.n_surfels;
  ds::removal_mask(c, pose, t_now, n);
  std::vector<int> keep(n);
  DS_CUDA(cudaMemcpyAsync(keep.data(), c.keep, sizeof(int) * n, cudaMemcpyDeviceToHost, c.stream));
  ds::sync(c);
  if (mask)
    for (int i = 0; i < n; ++i) mask[i] = keep[i] ? 0 : 1;
  API_END
}

ds_status ds_extend_warp_field(ds_context* ctx, int32_t n, const double* positions,
                               int32_t* appended) {
  API_BEGIN
  REQUIRE(ctx && (n == 0 || positions) && n <= ctx->c.P, "bad argument");
  Ctx& c = ctx->c;
  bind(c);
  std::vector<float4> p(n);
  for (int i = 0; i < n; ++i)
    p[i] = make_float4((float)positions[3 * i], (float)positions[3 * i + 1],
                       (float)positions[3 * i + 2], 0.f);
  DS_CUDA(cudaMemcpyAsync(c.cand_p, p.data(), sizeof(float4) * n, cudaMemcpyHostToDevice, c.stream));
  const int a = ds::extend_warp_field(c, c.cand_p, n);
  ds::join_node_updates(c);
  ds::sync(c);
  c.pattern_ready = false;
  if (appended) *appended = a;
  API_END
}

ds_status ds_update_skinning_incremental(ds_context* ctx, int32_t first_new) {
  API_BEGIN
  REQUIRE(ctx, "null context");
  bind(ctx->c);
  ds::update_skinning_incremental(ctx->c, first_new);
  ctx->c.pattern_ready = false;
  ds::sync(ctx->c);
  API_END
}

ds_status ds_clean_and_reset(ds_context* ctx, const double* pose, int32_t* removed,
                             int32_t* survivors) {
  API_BEGIN
  REQUIRE(ctx && pose, "bad argument");
  Ctx& c = ctx->c;
  bind(c);
  REQUIRE(c.frame_ready, "no frame maps");
  int s = 0;
  const int r = ds::clean_and_reset(c, pose, &s);
  ds::sync(c);
  if (removed) *removed = r;
  if (survivors) *survivors = s;
  API_END
}

int32_t ds_num_kernel_kinds(void) { return ds::KK_COUNT; }
const char* ds_kernel_name(int32_t kind) {
  return (kind >= 0 && kind < ds::KK_COUNT) ? ds::kKernelNames[kind] : "unknown";
}
ds_status ds_kernel_stats(ds_context* ctx, int32_t kind, int64_t* launches, double* total_ms,
                          double* bytes) {
  API_BEGIN
  REQUIRE(ctx && kind >= 0 && kind < ds::KK_COUNT, "bad argument");
  Ctx& c = ctx->c;
  bind(c);
  ds::sync(c);
  if (launches) *launches = c.cfg.profile || c.prof_launches[kind] ? c.prof_launches[kind]
                                                                  : c.launches[kind];
  if (total_ms) *total_ms = c.prof_ms[kind];
  if (bytes) *bytes = c.prof_bytes[kind];
  API_END
}
ds_status ds_reset_kernel_stats(ds_context* ctx) {
  API_BEGIN
  REQUIRE(ctx, "null context");
  Ctx& c = ctx->c;
  bind(c);
  ds::sync(c);
  for (int k = 0; k < ds::KK_COUNT; ++k) {
    c.launches[k] = 0;
    c.prof_launches[k] = 0;
    c.prof_ms[k] = 0;
    c.prof_bytes[k] = 0;
  }
  c.total_launches = 0;
  API_END
}
ds_status ds_set_profiling(ds_context* ctx, int32_t enable) {
  API_BEGIN
  REQUIRE(ctx, "null context");
  Ctx& c = ctx->c;
  bind(c);
  ds::sync(c);
  c.cfg.profile = enable ? 1 : 0;
  API_END
}
// PNG spec 9.2 row filters (None, Sub, Up, Average, Paeth), host code
ds_status ds_png_unfilter(const uint8_t* data, int64_t size, int32_t width, int32_t height,
                          int32_t bpp, uint8_t* out) {
  if (!data || !out || width < 0 || height < 0 || bpp < 1) return DS_ERR_INVALID_ARGUMENT;
  const int64_t stride = int64_t(width) * bpp;
  if (size != int64_t(height) * (stride + 1)) return DS_ERR_DIMENSION_MISMATCH;
  for (int64_t y = 0; y < height; ++y) {
    const uint8_t ft = data[y * (stride + 1)];
    const uint8_t* in = data + y * (stride + 1) + 1;
    uint8_t* cur = out + y * stride;
    const uint8_t* prior = y ? cur - stride : nullptr;
    if (ft > 4) return DS_ERR_INVALID_ARGUMENT;
    for (int64_t i = 0; i < stride; ++i) {
      const int a = i >= bpp ? cur[i - bpp] : 0;
      const int b = prior ? prior[i] : 0;
      const int c = (prior && i >= bpp) ? prior[i - bpp] : 0;
      int v = in[i];
      if (ft == 1) {
        v += a;
      } else if (ft == 2) {
        v += b;
      } else if (ft == 3) {
        v += (a + b) >> 1;
      } else if (ft == 4) {
        const int p = a + b - c, pa = std::abs(p - a), pb = std::abs(p - b), pc = std::abs(p - c);
        v += (pa <= pb && pa <= pc) ? a : (pb <= pc ? b : c);
      }
      cur[i] = uint8_t(v);
    }
  }
  return DS_OK;
}

ds_status ds_total_launches(const ds_context* ctx, int64_t* launches) {
  API_BEGIN
  REQUIRE(ctx && launches, "bad argument");
  *launches = ctx->c.total_launches;
  API_END
}

}  // extern "C"
