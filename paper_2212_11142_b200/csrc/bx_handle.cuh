// bx_handle.cuh — the library's private state behind the C ABI (include/bx_sm100.h): the handle
// with every device buffer and switch, and the helpers the bx_*.cu translation units share
// (status / error text, uploads, device views of the handle, the posterior launcher).
// No exception crosses the boundary; every failure becomes a status code + bx_last_error().
#pragma once
#include <algorithm>
#include <cmath>
#include <cstdarg>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <string>
#include <vector>
#include <unordered_map>
#include <mutex>

#include "bx_common.cuh"

namespace bx {
int score_max_partials(int sm_count);
size_t lml_scratch_doubles(int n, int c);
}  // namespace bx

using namespace bx;

namespace {

struct DevBuf {
  void* p = nullptr;
  size_t bytes = 0;
  cudaError_t ensure(size_t need) {
    if (need <= bytes) return cudaSuccess;
    if (p) cudaFree(p);
    p = nullptr;
    bytes = 0;
    cudaError_t e = cudaMalloc(&p, need < 256 ? 256 : need);
    if (e == cudaSuccess) bytes = need < 256 ? 256 : need;
    return e;
  }
  void release() {
    if (p) cudaFree(p);
    p = nullptr;
    bytes = 0;
  }
  template <typename T>
  T* as() const { return reinterpret_cast<T*>(p); }
};

}  // namespace

struct bx_handle {
  int device = 0;
  int sm_count = 148;
  std::string err;
  // space
  bool has_space = false;
  int n_params = 0, row_words = 0, n_features = 0, n_slots = 0;
  std::vector<bx_param_desc> params;
  std::vector<int32_t> rank_host;
  DevBuf d_params, d_coord, d_rank, d_feat_param, d_feat_sub, d_slot_param, d_slot_move;
  // gp
  bool has_gp = false;
  int gp_n = 0, gp_ncols = 0, gp_rows = 0, gp_lda = 0;
  double outputscale = 1, y_mean = 0, y_std = 1;
  DevBuf d_A, d_L, d_planes, d_kmask, d_inv_l, d_inv_l2, d_disc_tab, d_disc_off, d_train;
  // forest
  bool has_forest = false;
  ForestDev forest{};
  DevBuf d_nodes, d_roots, d_cnodes, d_leaf_val, d_leaf_idx, d_real_thr, d_code_param, d_code_sub;
  DevBuf d_qmask, d_qvid, d_quval, d_qsoff, d_qcode_param, d_qcode_sub, d_qrthr, d_qiidx, d_qimask,
      d_qcode_param2, d_qcode_sub2, d_qcode_mul;
  bool no_coded_forest = false;  // BX_FOREST_GENERIC debug switch (env)
  std::vector<int32_t> feat_param_host, feat_sub_host;
  std::vector<double> coord_host;
  // evaluated
  int ev_count = 0, ev_mask = 0;
  DevBuf d_ev_rows, d_ev_table;
  // cot
  bool has_cot = false;
  CotDev cot{};
  DevBuf d_g_kind, d_g_pbeg, d_g_params, d_g_root, d_child_begin, d_child_count, d_child_value;
  // constraints
  bool has_constraints = false;
  ConstraintDev cons{};
  DevBuf d_prog_begin, d_code, d_consts, d_vtag, d_vint, d_vflt, d_voff, d_str_id, d_fault;
  // scratch
  DevBuf d_probs, d_partials, d_summary, d_lml_scratch;
  cudaStream_t copy_stream = nullptr;
  cudaEvent_t ev_copy = nullptr, ev_done = nullptr;
  cudaEvent_t ev_t[5] = {nullptr, nullptr, nullptr, nullptr, nullptr};  // rf / gp / merge timing
  float t_ms[3] = {0, 0, 0};
  // register-resident fused GP path (gp_fused.cu)
  bool use_fused = false;
  bool no_fused = false;  // BX_GP_GENERIC debug switch (env)
  // tensor-core posterior (gp_tc.cu): digit-sliced [L^-1; alpha^T] + row scales
  bool use_tc = false;
  bool no_tc = false;     // BX_GP_DMMA=1 forces the FP64 DMMA kernel
  bool no_qs_forest = false;        // BX_FOREST_WALK=1: node walks instead of QuickScorer tables
  bool rf_after_gp = false;         // last score_impl ran the forest + summary kernel after the posterior
  int tc_debug = 0;                 // BX_TC_DEBUG (timing experiments)
  // streaming host pools (bx_score_host on the tensor-core path): the pool in device memory, one
  // ready flag per copied chunk, pinned ones to write the flags with the copy engine
  DevBuf d_pool, d_ready;
  uint32_t* h_ones = nullptr;
  int64_t h_ones_len = 0;
  const uint32_t* stream_ready = nullptr;  // set while a streaming posterior launch is enqueued
  const uint32_t* stream_packed = nullptr; // ... whose pool arrives packed (unpacked into d_pool)
  int stream_shift = 0;
  // distances on the FP64 tensor cores over the embedding of W (bx_set_gp decides): tc_ks k-steps,
  // 0 -> FMA distances
  int tc_ks = 0;
  bool tc_aug = false;
  std::vector<EmbDim> tc_emb;
  std::vector<double> tc_tab;
  DevBuf d_emb, d_emb_tab, d_emb_planes, d_emb_yy;
  bool tc_no_dmma = false;                 // BX_TC_NO_DMMA=1: FMA distances
  bool tc_trace = false;                   // BX_TC_TRACE set (role timeline dump)
  bool lml_narrow = false;                 // BX_LML_NARROW=1: _lml_core always one CTA per setting
  int lml_small_max = 40;                  // _lml_core in one CTA's shared memory up to this n (BX_LML_SMALL_MAX)
  int tc_nsl = 0, tc_nch = 0;
  double tc_kscale = 0;
  DevBuf d_mdig, d_rowscale, d_tc_part;
  DevBuf d_factor;  // bx_gp_factor: distances, z, hyperparameters, one setting's factorisation scratch
  bool matern_precise = false;  // BX_MATERN_PRECISE debug switch (env)
  int mt = 0, rows8 = 0, n_kendall = 0;
  int32_t kendall_param[BX_MAX_PARAMS] = {0};
  PackSpec pack{};                  // packed wire format of the space (bx_set_space)
  const uint8_t* pw_rows = nullptr;  // per-row forest summation order for the next score_impl (bx_climb)
  DevBuf d_climb;                    // bx_climb scratch
  int32_t* h_climb_flag = nullptr;   // pinned: bx_climb's per-step active count (an async 4-byte read)
  void* h_lml_stage = nullptr;       // pinned staging of bx_lml_core_host (parameters in, results out)
  size_t h_lml_stage_bytes = 0;
  DevBuf d_lml_stage;
  DevBuf d_fit;                      // bx_rf_fit buffers
  DevBuf d_packed;                  // streamed packed pool
  DevBuf d_panels, d_ei, d_grad_scratch, d_leaf_count, d_gen_rows;
  bool has_leaf_count = false;
  cudaStream_t rf_stream = nullptr;
  cudaEvent_t ev_fork = nullptr, ev_rf = nullptr;
};


namespace {

// 2^(j/64) and 2^(j/256), correctly rounded (long double), computed once per process
struct Exp2Tables {
  double t64[64], t256[256];
  Exp2Tables() {
    for (int j = 0; j < 64; ++j) t64[j] = (double)exp2l((long double)j / 64.0L);
    for (int j = 0; j < 256; ++j) t256[j] = (double)exp2l((long double)j / 256.0L);
  }
};
const Exp2Tables& exp2_tables() {
  static const Exp2Tables t;
  return t;
}

int fail(bx_handle* h, int code, const char* fmt, ...) {
  char buf[512];
  va_list ap;
  va_start(ap, fmt);
  vsnprintf(buf, sizeof buf, fmt, ap);
  va_end(ap);
  if (h) h->err = buf;
  return code;
}

#define BX_CUDA(h, call)                                                                       \
  do {                                                                                         \
    cudaError_t e_ = (call);                                                                   \
    if (e_ != cudaSuccess)                                                                     \
      return fail(h, BX_ERR_CUDA, "%s failed: %s", #call, cudaGetErrorString(e_));             \
  } while (0)

template <typename T>
cudaError_t upload(DevBuf& b, const T* host, size_t count) {
  cudaError_t e = b.ensure(count * sizeof(T) + 16);
  if (e != cudaSuccess) return e;
  if (count == 0) return cudaSuccess;
  return cudaMemcpy(b.p, host, count * sizeof(T), cudaMemcpyHostToDevice);
}

SpaceDev space_dev(const bx_handle* h) {
  SpaceDev s;
  s.params = h->d_params.as<bx_param_desc>();
  s.coord_lut = h->d_coord.as<double>();
  s.rank_lut = h->d_rank.as<int32_t>();
  s.feat_param = h->d_feat_param.as<int32_t>();
  s.feat_sub = h->d_feat_sub.as<int32_t>();
  s.slot_param = h->d_slot_param.as<int32_t>();
  s.slot_move = h->d_slot_move.as<int32_t>();
  s.n_params = h->n_params;
  s.row_words = h->row_words;
  s.n_features = h->n_features;
  s.n_slots = h->n_slots;
  return s;
}

GpDev gp_dev(const bx_handle* h) {
  GpDev g;
  g.n = h->gp_n;
  g.ncols_pad = h->gp_ncols;
  g.rows_pad = h->gp_rows;
  g.lda = h->gp_lda;
  g.A = h->d_A.as<double>();
  g.planes = h->d_planes.as<uint64_t>();
  g.kmask = h->d_kmask.as<uint64_t>();
  g.inv_l = h->d_inv_l.as<double>();
  g.inv_l2 = h->d_inv_l2.as<double>();
  g.disc_tab = h->d_disc_tab.as<double>();
  g.disc_off = h->d_disc_off.as<int32_t>();
  g.outputscale = h->outputscale;
  g.y_mean = h->y_mean;
  g.y_std = h->y_std;
  return g;
}

EvalSetDev eval_dev(const bx_handle* h) {
  EvalSetDev e;
  e.rows = h->d_ev_rows.as<uint32_t>();
  e.table = h->d_ev_table.as<int32_t>();
  e.count = h->ev_count;
  e.table_mask = h->ev_mask;
  return e;
}

uint64_t host_row_hash(const uint32_t* row, int words) {
  uint64_t hsh = 1469598103934665603ull;
  for (int w = 0; w < words; ++w) {
    hsh ^= row[w];
    hsh *= 1099511628211ull;
    hsh ^= hsh >> 29;
  }
  return hsh;
}

int check_space(bx_handle* h) {
  if (!h) return BX_ERR_ARG;
  if (!h->has_space) return fail(h, BX_ERR_STATE, "bx_set_space has not been called");
  return BX_OK;
}

int max_partials(int sm_count) {
  const int a = score_max_partials(sm_count), b = summary_max_partials(sm_count);
  return a > b ? a : b;
}

FusedArgs fused_args(const bx_handle* h, const uint32_t* rows, int64_t q, double f_model) {
  FusedArgs f{};
  f.space = space_dev(h);
  f.gp = gp_dev(h);
  f.panels = h->d_panels.as<double>();
  f.rows = rows;
  f.q = q;
  f.f_model = f_model;
  f.mt = h->mt;
  f.n_kendall = h->n_kendall;
  for (int i = 0; i < h->n_kendall; ++i) f.kendall_param[i] = h->kendall_param[i];
  f.n_num = f.n_cat = f.n_perm = 0;
  for (int k = 0; k < h->n_params; ++k) {
    const int kind = h->params[k].kind;
    if (kind == BX_CATEGORICAL) f.cat_param[f.n_cat++] = k;
    else if (kind == BX_PERMUTATION) f.perm_param[f.n_perm++] = k;
    else f.num_param[f.n_num++] = k;
  }
  std::memcpy(f.exp2tab, exp2_tables().t64, sizeof(f.exp2tab));
  f.precise = h->matern_precise ? 1 : 0;
  return f;
}

// the posterior kernels that take FusedArgs (tensor-core or register-resident DMMA)
bool fused_path(const bx_handle* h) { return h->use_tc || h->use_fused; }

cudaError_t launch_posterior(const bx_handle* h, const FusedArgs& f, cudaStream_t s) {
  if (h->use_tc) {
    TcArgs t{};
    t.f = f;
    t.mdig = h->d_mdig.as<unsigned char>();
    t.rowscale = h->d_rowscale.as<double>();
    t.n_slices = h->tc_nsl;
    t.n_chunks = h->tc_nch;
    t.kscale = h->tc_kscale;
    t.ready = h->stream_ready;
    t.ready_shift = h->stream_shift;
    t.packed = h->stream_packed;
    t.pack = h->pack;
    t.ks = h->tc_ks;
    t.n_emb = (int32_t)h->tc_emb.size();
    t.aug = h->tc_aug ? 1 : 0;
    t.emb = h->d_emb.as<EmbDim>();
    t.emb_tab = h->d_emb_tab.as<double>();
    t.emb_tab_len = (int32_t)h->tc_tab.size();
    t.emb_planes = h->d_emb_planes.as<double>();
    t.emb_yy = h->d_emb_yy.as<double>();
    t.part = h->tc_nsl > 8 ? h->d_tc_part.as<double>() : nullptr;
    t.n_coord = (int32_t)h->coord_host.size();
    std::memcpy(t.exp2tab256, exp2_tables().t256, sizeof(t.exp2tab256));
    t.debug = h->tc_debug;
    const char* trace = h->tc_trace ? getenv("BX_TC_TRACE") : nullptr;  // profiling aid: CTA 0's timeline
    if (!trace || !trace[0]) return launch_gp_tc(t, h->sm_count, s);
    const size_t bytes = 4 * 4096 * 2 * sizeof(long long);
    std::vector<long long> host(bytes / sizeof(long long));
    long long* dev = nullptr;
    cudaError_t e = cudaMalloc(&dev, bytes);
    if (e == cudaSuccess) e = cudaMemsetAsync(dev, 0, bytes, s);
    t.trace = dev;
    if (e == cudaSuccess) e = launch_gp_tc(t, h->sm_count, s);
    if (e == cudaSuccess) e = cudaMemcpyAsync(host.data(), dev, bytes, cudaMemcpyDeviceToHost, s);
    if (e == cudaSuccess) e = cudaStreamSynchronize(s);
    cudaFree(dev);
    if (FILE* f = fopen(trace, "wb")) {
      fwrite(host.data(), 1, bytes, f);
      fclose(f);
    }
    return e;
  }
  return launch_gp_fused(f, h->sm_count, s);
}

int check_gp(bx_handle* h) {
  int r = check_space(h);
  if (r) return r;
  if (!h->has_gp) return fail(h, BX_ERR_STATE, "bx_set_gp has not been called");
  return BX_OK;
}

}  // namespace


// shared across the translation units (defined in bx_score.cu / bx_model.cu)
int score_impl(bx_handle* h, const uint32_t* rows, int64_t q, int64_t index_base, double f_model, double eps_f,
               int32_t k, int32_t flags, double* values, double* probs_out, Partial* partials, int* n_partials,
               cudaStream_t s, int timing, bool track_prob = false, cudaEvent_t rows_ready = nullptr);
