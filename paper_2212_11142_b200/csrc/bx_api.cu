// bx_api.cu — the C ABI (include/bx_sm100.h): handle, model-state uploads, launches.
// No exception crosses the boundary; every failure becomes a status code + bx_last_error().
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
  DevBuf d_qmask, d_qvid, d_quval, d_qsoff, d_qcode_param, d_qcode_sub, d_qrthr, d_qiidx, d_qimask;
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
  int tc_nsl = 0, tc_nch = 0;
  double tc_kscale = 0;
  DevBuf d_mdig, d_rowscale, d_tc_part;
  bool matern_precise = false;  // BX_MATERN_PRECISE debug switch (env)
  int mt = 0, rows8 = 0, n_kendall = 0;
  int32_t kendall_param[BX_MAX_PARAMS] = {0};
  PackSpec pack{};                  // packed wire format of the space (bx_set_space)
  const uint8_t* pw_rows = nullptr;  // per-row forest summation order for the next score_impl (bx_climb)
  DevBuf d_climb;                    // bx_climb scratch
  DevBuf d_packed;                  // streamed packed pool
  DevBuf d_panels, d_ei, d_grad_scratch, d_leaf_count, d_gen_rows;
  bool has_leaf_count = false;
  cudaStream_t rf_stream = nullptr;
  cudaEvent_t ev_fork = nullptr, ev_rf = nullptr;
};

cudaError_t bx::set_smem_once(const void* fn, int bytes) {
  static std::mutex mu;
  static std::unordered_map<const void*, int> done;
  std::lock_guard<std::mutex> lock(mu);
  int& have = done[fn];
  if (bytes <= have) return cudaSuccess;
  const cudaError_t e = cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize, bytes);
  if (e == cudaSuccess) have = bytes;
  return e;
}

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

static int build_coded_forest(bx_handle* h, const std::vector<RfNode>& nodes,
                              const std::vector<int32_t>& roots, int max_depth);


// Helmert basis: (L - 1) x L orthonormal rows spanning the sum-zero subspace of R^L
static std::vector<double> helmert(int L) {
  std::vector<double> Q((size_t)(L - 1) * L, 0.0);
  for (int j = 1; j < L; ++j) {
    const double nrm = std::sqrt((double)j * (j + 1));
    for (int i = 0; i < j; ++i) Q[(size_t)(j - 1) * L + i] = 1.0 / nrm;
    Q[(size_t)(j - 1) * L + j] = -(double)j / nrm;
  }
  return Q;
}

// The Euclidean embedding of W = sum_k sq_k / l_k^2 (surrogate.py:173-223; EmbDim in bx_common.cuh),
// centred on the training mean; planes = the DMMA B operand [4 ks][npad] (-2 y', then |y'|^2 and 1
// when they fit the padding: *aug), yy[npad] = |y'|^2.  False when a metric does not embed (naive
// permutation indicator) or the centred coordinates are too large for the |x|^2 + |y|^2 - 2 x.y
// form (bound 256: the cancellation error stays near the 2^-40 fixed point of K*).
static bool build_embedding(const bx_handle* h, const uint32_t* train_rows, int n, const double* inv_l,
                            const double* inv_l2, int npad, std::vector<EmbDim>& emb, std::vector<double>& tab,
                            std::vector<double>& planes, std::vector<double>& yy, bool* aug) {
  std::vector<int> seg;  // table entries per coordinate that carry the centring
  for (int k = 0; k < h->n_params; ++k) {
    const bx_param_desc& p = h->params[k];
    if (p.kind == BX_INTEGER || p.kind == BX_ORDINAL) {
      emb.push_back(EmbDim{BX_EMB_CODE, p.word, 0, 0, 0, (int)tab.size()});
      for (int i = 0; i < p.size; ++i) tab.push_back(h->coord_host[p.coord + i] * inv_l[k]);
      seg.push_back(p.size);
    } else if (p.kind == BX_REAL) {
      emb.push_back(EmbDim{BX_EMB_REAL, p.word, 0, 0, 0, (int)tab.size()});
      tab.push_back(inv_l[k]);
      tab.push_back(0.0);
      seg.push_back(0);
    } else if (p.kind == BX_CATEGORICAL) {
      const int L = p.size;
      const std::vector<double> Q = helmert(L);
      const double sw = std::sqrt(inv_l2[k] / 2.0);  // unit-edge simplex: |V_a - V_b|^2 = 1
      for (int j = 0; j + 1 < L; ++j) {
        emb.push_back(EmbDim{BX_EMB_CODE, p.word, 0, 0, 0, (int)tab.size()});
        for (int a = 0; a < L; ++a) tab.push_back(Q[(size_t)j * L + a] * sw);
        seg.push_back(L);
      }
    } else {  // permutation
      const int m = p.size;
      const double wm = inv_l2[k] / p.raw_mx;
      if (p.metric == BX_SPEARMAN) {
        const std::vector<double> Q = helmert(m);
        for (int j = 0; j + 1 < m; ++j) {
          emb.push_back(EmbDim{BX_EMB_PERM_LIN, p.word, 0, 0, m, (int)tab.size()});
          for (int i = 0; i < m; ++i) tab.push_back(Q[(size_t)j * m + i] * std::sqrt(wm));
          tab.push_back(0.0);
          seg.push_back(-1);
        }
      } else if (p.metric == BX_KENDALL) {
        for (int a = 0; a < m; ++a)
          for (int b = a + 1; b < m; ++b) {
            emb.push_back(EmbDim{BX_EMB_KENDALL, p.word, a, b, m, (int)tab.size()});
            tab.push_back(0.0);
            tab.push_back(std::sqrt(wm));
            seg.push_back(2);
          }
      } else if (p.metric == BX_HAMMING) {
        const std::vector<double> Q = helmert(m);
        for (int pos = 0; pos < m; ++pos)
          for (int j = 0; j + 1 < m; ++j) {
            emb.push_back(EmbDim{BX_EMB_PERM_HOT, p.word, pos, 0, m, (int)tab.size()});
            for (int v = 0; v < m; ++v) tab.push_back(Q[(size_t)j * m + v] * std::sqrt(wm / 2.0));
            seg.push_back(m);
          }
      } else {
        return false;  // the naive indicator 1{a != b} over m! permutations does not embed cheaply
      }
    }
    if (emb.size() > 32) return false;
  }
  const int E = (int)emb.size();
  if (E == 0) return false;
  // centre on the training mean (translation leaves every distance unchanged)
  for (int e = 0; e < E; ++e) {
    double mu = 0.0;
    for (int j = 0; j < n; ++j) mu += emb_value(emb[e], train_rows + (size_t)j * h->row_words, tab.data());
    mu /= n;
    const EmbDim& d = emb[e];
    if (seg[e] > 0) {
      for (int i = 0; i < seg[e]; ++i) tab[d.off + i] -= mu;
    } else if (d.kind == BX_EMB_REAL) {
      tab[d.off + 1] = -mu;
    } else {
      tab[d.off + d.m] = -mu;
    }
  }
  // magnitude bound over the whole domain
  double bound = 0.0;
  for (int e = 0; e < E; ++e) {
    const EmbDim& d = emb[e];
    double mx = 0.0;
    if (seg[e] > 0) {
      for (int i = 0; i < seg[e]; ++i) mx = std::max(mx, std::fabs(tab[d.off + i]));
    } else if (d.kind == BX_EMB_REAL) {
      int kp = 0;
      while (kp + 1 < h->n_params && h->params[kp].word != d.word) ++kp;
      const bx_param_desc& p = h->params[kp];
      for (int i : {0, p.size - 1}) mx = std::max(mx, std::fabs(h->coord_host[p.coord + i] * tab[d.off] + tab[d.off + 1]));
    } else {
      mx = std::fabs(tab[d.off + d.m]);
      for (int i = 0; i < d.m; ++i) mx += std::fabs(tab[d.off + i]) * (d.m - 1);
    }
    bound += mx * mx;
  }
  if (!(bound <= 256.0)) return false;
  const int ks = (E + 3) / 4;
  *aug = E + 2 <= 4 * ks;
  planes.assign((size_t)4 * ks * npad, 0.0);
  yy.assign((size_t)npad, 0.0);
  for (int j = 0; j < n; ++j) {
    const uint32_t* row = train_rows + (size_t)j * h->row_words;
    double s2 = 0.0;
    for (int e = 0; e < E; ++e) {
      const double y = emb_value(emb[e], row, tab.data());
      planes[(size_t)e * npad + j] = -2.0 * y;
      s2 = std::fma(y, y, s2);
    }
    yy[j] = s2;
    if (*aug) {
      planes[(size_t)E * npad + j] = s2;
      planes[(size_t)(E + 1) * npad + j] = 1.0;
    }
  }
  return true;
}


namespace bx {
__global__ void unpack_kernel(PackSpec spec, const uint32_t* packed, int64_t q, int words, uint32_t* rows) {
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < q; i += (int64_t)gridDim.x * blockDim.x)
    unpack_row(spec, packed + (size_t)i * spec.pw, rows + (size_t)i * words, words);
}
cudaError_t launch_unpack(const PackSpec& spec, const uint32_t* packed, int64_t q, int words, uint32_t* rows,
                          cudaStream_t s) {
  int64_t blocks = (q + 255) / 256;
  if (blocks > 148 * 16) blocks = 148 * 16;
  unpack_kernel<<<(int)blocks, 256, 0, s>>>(spec, packed, q, words, rows);
  return cudaGetLastError();
}
}  // namespace bx


namespace bx {
// bx_climb state on the device: per start the current row, value and an active flag; the tracker
struct ClimbState {
  int32_t n_active;
  int32_t pad;
  TopRec best;                       // index >= 0 once set
  uint32_t best_row[BX_MAX_ROW_WORDS];
};

// per-row forest order: a start whose CoT-filtered list has exactly one neighbour is scored like
// the reference's _scores on one configuration (q == 1: numpy's pairwise tree sum)
__global__ void climb_flags_kernel(int A, int S, const int32_t* active, const uint8_t* valid, uint8_t* pw) {
  for (int a = threadIdx.x; a < A; a += blockDim.x) {
    int cnt = 0;
    for (int s = 0; s < S; ++s) cnt += valid[a * S + s] ? 1 : 0;
    for (int s = 0; s < S; ++s) pw[a * S + s] = (active[a] && cnt == 1) ? 1 : 0;
  }
}

// one step's bookkeeping (acquisition.py:193-201): per active start the argbest neighbour under
// (value desc, configuration asc) (_argbest, :87-94), moved to iff strictly better; every scored
// neighbour folded into the tracker (_Tracker.update, :105-111).  Warp a = start a: its lanes scan
// the slots, then a shuffle reduction under the same total orders; thread 0 folds the starts'
// tracker candidates.
__device__ __forceinline__ bool climb_better(const SpaceDev& sp, const uint32_t* nb, int W, double v1, int r1, double v2,
                                             int r2) {
  if (r1 < 0) return false;
  if (r2 < 0) return true;
  if (v1 != v2) return v1 > v2;
  return key_cmp(sp.params, sp.n_params, sp.rank_lut, nb + (size_t)r1 * W, nb + (size_t)r2 * W) < 0;
}

__global__ void climb_update_kernel(SpaceDev sp, EvalSetDev ev, int A, int S, int32_t* active, uint32_t* cur,
                                    double* curv, const uint32_t* nb, const uint8_t* valid, const double* vals,
                                    ClimbState* st) {
  __shared__ int s_trk[BX_MAX_K];
  __shared__ int s_moved[BX_MAX_K];
  const int W = sp.row_words;
  const int a = threadIdx.x >> 5, lane = threadIdx.x & 31;
  if (a < A) {
    int br = -1, tr = -1;  // argbest row and tracker-candidate row of this lane
    double bv = -INFINITY, tv = -INFINITY;
    if (active[a])
      for (int s2 = lane; s2 < S; s2 += 32) {
        const int r = a * S + s2;
        if (!valid[r]) continue;
        const double v = vals[r];
        if (climb_better(sp, nb, W, v, r, bv, br)) {
          bv = v;
          br = r;
        }
        if (v != -INFINITY && !(ev.count > 0 && is_evaluated(ev, nb + (size_t)r * W, W)) &&
            climb_better(sp, nb, W, v, r, tv, tr)) {
          tv = v;
          tr = r;
        }
      }
#pragma unroll
    for (int o = 16; o; o >>= 1) {
      const double ov = __shfl_xor_sync(0xffffffffu, bv, o), otv = __shfl_xor_sync(0xffffffffu, tv, o);
      const int orow = __shfl_xor_sync(0xffffffffu, br, o), otr = __shfl_xor_sync(0xffffffffu, tr, o);
      if (climb_better(sp, nb, W, ov, orow, bv, br)) {
        bv = ov;
        br = orow;
      }
      if (climb_better(sp, nb, W, otv, otr, tv, tr)) {
        tv = otv;
        tr = otr;
      }
    }
    if (lane == 0) {
      s_trk[a] = tr;
      int moved = 0;
      if (active[a]) {
        if (br >= 0 && bv > curv[a]) {  // acquisition.py:200
          curv[a] = bv;
          moved = 1;
        } else {
          active[a] = 0;  // no neighbours, or no improvement: this start stops
        }
      }
      s_moved[a] = moved ? br : -1;
    }
    __syncwarp();
    const int mr = __shfl_sync(0xffffffffu, lane == 0 ? s_moved[a] : 0, 0);
    if (mr >= 0)
      for (int w = lane; w < W; w += 32) cur[(size_t)a * W + w] = nb[(size_t)mr * W + w];
  }
  __syncthreads();
  if (threadIdx.x == 0) {
    int n_active = 0;
    for (int i = 0; i < A; ++i) {
      n_active += s_moved[i] >= 0 ? 1 : 0;
      const int r = s_trk[i];
      if (r < 0) continue;
      const double v = vals[r];
      const uint32_t* row = nb + (size_t)r * W;
      bool take = st->best.index < 0 || v > st->best.value;
      if (!take && v == st->best.value) take = key_cmp(sp.params, sp.n_params, sp.rank_lut, row, st->best_row) < 0;
      if (take) {
        st->best = TopRec{v, 0.0, 0};
        for (int w = 0; w < W; ++w) st->best_row[w] = row[w];
      }
    }
    st->n_active = n_active;
  }
}
}  // namespace bx

extern "C" {

int bx_abi_version(void) { return BX_ABI_VERSION; }

bx_handle* bx_create(int device) {
  if (cudaSetDevice(device) != cudaSuccess) return nullptr;
  bx_handle* h = new (std::nothrow) bx_handle();
  if (!h) return nullptr;
  h->device = device;
  const char* generic = getenv("BX_FOREST_GENERIC");
  h->no_coded_forest = generic && generic[0] == '1';
  cudaDeviceGetAttribute(&h->sm_count, cudaDevAttrMultiProcessorCount, device);
  cudaStreamCreateWithFlags(&h->copy_stream, cudaStreamNonBlocking);
  cudaEventCreateWithFlags(&h->ev_copy, cudaEventDisableTiming);
  cudaEventCreateWithFlags(&h->ev_done, cudaEventDisableTiming);
  for (int i = 0; i < 5; ++i) cudaEventCreate(&h->ev_t[i]);
  const char* gpg = getenv("BX_GP_GENERIC");
  h->no_fused = gpg && gpg[0] == '1';
  if (const char* dbg = getenv("BX_TC_DEBUG")) h->tc_debug = atoi(dbg);
  h->tc_trace = getenv("BX_TC_TRACE") != nullptr;
  if (const char* ln = getenv("BX_LML_NARROW")) h->lml_narrow = ln[0] == '1';
  if (const char* nd = getenv("BX_TC_NO_DMMA")) h->tc_no_dmma = nd[0] == '1';
  const char* fw = getenv("BX_FOREST_WALK");
  h->no_qs_forest = fw && fw[0] == '1';
  const char* dm = getenv("BX_GP_DMMA");
  h->no_tc = h->no_fused || (dm && dm[0] == '1');
  const char* mp = getenv("BX_MATERN_PRECISE");
  h->matern_precise = mp && mp[0] == '1';
  cudaStreamCreateWithFlags(&h->rf_stream, cudaStreamNonBlocking);
  cudaEventCreateWithFlags(&h->ev_fork, cudaEventDisableTiming);
  cudaEventCreateWithFlags(&h->ev_rf, cudaEventDisableTiming);
  return h;
}

void bx_destroy(bx_handle* h) {
  if (!h) return;
  cudaSetDevice(h->device);
  DevBuf* bufs[] = {&h->d_params, &h->d_coord, &h->d_rank, &h->d_feat_param, &h->d_feat_sub,
                    &h->d_slot_param, &h->d_slot_move, &h->d_A, &h->d_L, &h->d_planes,
                    &h->d_kmask, &h->d_inv_l, &h->d_inv_l2, &h->d_disc_tab, &h->d_disc_off,
                    &h->d_train, &h->d_nodes, &h->d_roots, &h->d_ev_rows, &h->d_ev_table,
                    &h->d_g_kind, &h->d_g_pbeg, &h->d_g_params, &h->d_g_root,
                    &h->d_child_begin, &h->d_child_count, &h->d_child_value, &h->d_prog_begin, &h->d_code,
                    &h->d_consts, &h->d_vtag, &h->d_vint, &h->d_vflt, &h->d_voff, &h->d_str_id,
                    &h->d_fault, &h->d_probs, &h->d_partials, &h->d_summary, &h->d_lml_scratch,
                    &h->d_cnodes, &h->d_leaf_val,
                    &h->d_real_thr, &h->d_code_param, &h->d_code_sub, &h->d_leaf_idx,
                    &h->d_qmask, &h->d_qvid, &h->d_quval, &h->d_qsoff, &h->d_qcode_param,
                    &h->d_qcode_sub, &h->d_qrthr, &h->d_qiidx, &h->d_qimask};
  for (DevBuf* b : bufs) b->release();
  if (h->copy_stream) cudaStreamDestroy(h->copy_stream);
  if (h->ev_copy) cudaEventDestroy(h->ev_copy);
  if (h->ev_done) cudaEventDestroy(h->ev_done);
  for (int i = 0; i < 5; ++i)
    if (h->ev_t[i]) cudaEventDestroy(h->ev_t[i]);
  h->d_panels.release();
  h->d_pool.release();
  h->d_ready.release();
  h->d_emb.release();
  h->d_packed.release();
  h->d_climb.release();
  h->d_emb_tab.release();
  h->d_emb_planes.release();
  h->d_emb_yy.release();
  if (h->h_ones) cudaFreeHost(h->h_ones);
  h->d_mdig.release();
  h->d_rowscale.release();
  h->d_tc_part.release();
  h->d_ei.release();
  h->d_grad_scratch.release();
  h->d_leaf_count.release();
  h->d_gen_rows.release();
  if (h->rf_stream) cudaStreamDestroy(h->rf_stream);
  if (h->ev_fork) cudaEventDestroy(h->ev_fork);
  if (h->ev_rf) cudaEventDestroy(h->ev_rf);
  delete h;
}

const char* bx_last_error(bx_handle* h) { return h ? h->err.c_str() : "null handle"; }

int bx_device_sm_count(bx_handle* h) { return h ? h->sm_count : 0; }

int bx_gp_kernel(bx_handle* h) {
  if (!h) return BX_GP_GENERIC;
  return h->use_tc ? BX_GP_TENSOR : h->use_fused ? BX_GP_DMMA : BX_GP_GENERIC;
}

int bx_gp_distance_ksteps(bx_handle* h) { return h && h->use_tc ? h->tc_ks : 0; }

int bx_set_option(bx_handle* h, int32_t option, int32_t value) {
  if (!h) return BX_ERR_ARG;
  if (option == BX_OPT_LML_NARROW) {
    h->lml_narrow = value != 0;
    return BX_OK;
  }
  return fail(h, BX_ERR_ARG, "unknown option %d", option);
}

int bx_packed_row_words(bx_handle* h) { return h && h->has_space ? h->pack.pw : 0; }

int bx_pack_rows(bx_handle* h, const uint32_t* rows, int64_t q, uint32_t* packed) {
  int r = check_space(h);
  if (r) return r;
  if (q < 0 || (q > 0 && (!rows || !packed))) return fail(h, BX_ERR_ARG, "bad buffers");
  for (int64_t i = 0; i < q; ++i) pack_row(h->pack, rows + (size_t)i * h->row_words, packed + (size_t)i * h->pack.pw);
  return BX_OK;
}

int bx_unpack_rows(bx_handle* h, const uint32_t* packed, int64_t q, uint32_t* rows) {
  int r = check_space(h);
  if (r) return r;
  if (q < 0 || (q > 0 && (!rows || !packed))) return fail(h, BX_ERR_ARG, "bad buffers");
  for (int64_t i = 0; i < q; ++i)
    unpack_row(h->pack, packed + (size_t)i * h->pack.pw, rows + (size_t)i * h->row_words, h->row_words);
  return BX_OK;
}

int bx_set_space(bx_handle* h, const bx_param_desc* params, int32_t n_params, int32_t row_words,
                 const double* coord_lut, int32_t coord_len, const int32_t* rank_lut,
                 int32_t rank_len, int32_t n_features) {
  if (!h) return BX_ERR_ARG;
  if (n_params < 1 || n_params > BX_MAX_PARAMS)
    return fail(h, BX_ERR_UNSUPPORTED, "n_params=%d outside [1, %d]", n_params, BX_MAX_PARAMS);
  if (row_words < 1 || row_words > BX_MAX_ROW_WORDS)
    return fail(h, BX_ERR_UNSUPPORTED, "row_words=%d outside [1, %d]", row_words, BX_MAX_ROW_WORDS);
  cudaSetDevice(h->device);
  std::vector<int32_t> fparam, fsub, sparam, smove;
  for (int k = 0; k < n_params; ++k) {
    const bx_param_desc& p = params[k];
    int nw = p.kind == BX_REAL ? 4 : (p.kind == BX_PERMUTATION ? 2 : 1);
    if (p.word < 0 || p.word + nw > row_words)
      return fail(h, BX_ERR_ARG, "parameter %d overflows the row (%d words)", k, row_words);
    if (p.kind == BX_PERMUTATION) {
      if (p.size < 2 || p.size > BX_MAX_PERM)
        return fail(h, BX_ERR_UNSUPPORTED, "permutation size %d outside [2, 16]", p.size);
      if ((p.word & 1) != 0) return fail(h, BX_ERR_ARG, "permutation %d not 8-byte aligned", k);
      for (int e = 0; e < p.size; ++e) { fparam.push_back(k); fsub.push_back(e); }
      for (int m = 0; m < p.size * (p.size - 1) / 2; ++m) { sparam.push_back(k); smove.push_back(m); }
    } else if (p.kind == BX_CATEGORICAL) {
      for (int e = 0; e < p.size; ++e) { fparam.push_back(k); fsub.push_back(e); }
      for (int m = 0; m < p.size - 1; ++m) { sparam.push_back(k); smove.push_back(m); }
    } else {
      if (p.kind == BX_REAL && (p.word & 1) != 0)
        return fail(h, BX_ERR_ARG, "real parameter %d not 8-byte aligned", k);
      fparam.push_back(k);
      fsub.push_back(0);
      sparam.push_back(k); smove.push_back(0);
      sparam.push_back(k); smove.push_back(1);
    }
  }
  if ((int)fparam.size() != n_features)
    return fail(h, BX_ERR_ARG, "n_features=%d but the parameters imply %d", n_features,
                (int)fparam.size());
  BX_CUDA(h, upload(h->d_params, params, n_params));
  BX_CUDA(h, upload(h->d_coord, coord_lut, (size_t)coord_len));
  BX_CUDA(h, upload(h->d_rank, rank_lut, (size_t)rank_len));
  BX_CUDA(h, upload(h->d_feat_param, fparam.data(), fparam.size()));
  BX_CUDA(h, upload(h->d_feat_sub, fsub.data(), fsub.size()));
  BX_CUDA(h, upload(h->d_slot_param, sparam.data(), sparam.size()));
  BX_CUDA(h, upload(h->d_slot_move, smove.data(), smove.size()));
  h->params.assign(params, params + n_params);
  h->feat_param_host = fparam;
  h->feat_sub_host = fsub;
  h->coord_host.assign(coord_lut, coord_lut + coord_len);
  h->rank_host.assign(rank_lut, rank_lut + rank_len);
  h->n_params = n_params;
  h->row_words = row_words;
  h->n_features = n_features;
  h->n_slots = (int)sparam.size();
  // packed wire format: parameters in order at their bit widths
  {
    PackSpec& ps = h->pack;
    ps = PackSpec{};
    ps.n = n_params;
    int bit = 0;
    for (int k = 0; k < n_params; ++k) {
      const bx_param_desc& p = params[k];
      PackParam& q = ps.p[k];
      q.kind = p.kind;
      q.word = p.word;
      q.bit = bit;
      q.lo = p.lo;
      q.hi = p.hi;
      if (p.kind == BX_REAL) {
        q.carry_coord = p.is_log ? 1 : 0;
        q.bits = q.carry_coord ? 128 : 64;
      } else if (p.kind == BX_PERMUTATION) {
        q.bits = 4 * p.size;
      } else {
        int b = 1;
        while ((1 << b) < p.size) ++b;
        q.bits = b;
      }
      bit += q.bits;
    }
    ps.pw = (bit + 31) / 32;
  }
  h->has_space = true;
  // every other piece of model state is expressed in the old space's rows / features / domain
  // indices: drop it, so a caller that forgets to re-set it gets BX_ERR_STATE, not stale reads
  h->has_gp = false;
  h->has_forest = false;
  h->has_cot = false;
  h->has_leaf_count = false;
  h->has_constraints = false;
  h->ev_count = 0;
  return BX_OK;
}

int bx_set_gp(bx_handle* h, const uint32_t* train_rows, int32_t n, const double* L,
              const double* alpha, double outputscale, const double* lengthscales, double y_mean,
              double y_std, void* stream) {
  int r = check_space(h);
  if (r) return r;
  if (n < 1) return fail(h, BX_ERR_ARG, "need at least one training point");
  if (!(outputscale > 0)) return fail(h, BX_ERR_ARG, "outputscale must be positive");
  cudaSetDevice(h->device);
  cudaStream_t s = (cudaStream_t)stream;
  const int D = h->n_params;
  std::vector<double> inv_l(D), inv_l2(D);
  std::vector<int32_t> disc_off(D, 0);
  std::vector<double> disc;
  for (int k = 0; k < D; ++k) {
    const double l = lengthscales[k];
    if (!(l > 0)) return fail(h, BX_ERR_ARG, "lengthscale %d must be positive", k);
    inv_l[k] = 1.0 / l;
    inv_l2[k] = 1.0 / (l * l);  // surrogate.py:222 1.0 / l ** 2
    const bx_param_desc& p = h->params[k];
    disc_off[k] = (int)disc.size();
    if (p.kind == BX_PERMUTATION) {
      const int m = p.size;
      int raw_max = m * m * m;  // >= every semimetric maximum
      for (int raw = 0; raw <= raw_max; ++raw) disc.push_back(((double)raw / p.raw_mx) * inv_l2[k]);
    } else if (p.kind == BX_CATEGORICAL) {
      disc.push_back(0.0);
      disc.push_back(inv_l2[k]);
    }
  }
  disc.push_back(0.0);
  h->gp_n = n;
  h->gp_ncols = ((n + 15) / 16) * 16;
  h->gp_rows = ((n + 1 + 15) / 16) * 16;
  h->gp_lda = h->gp_ncols;
  const size_t a_elems = (size_t)h->gp_rows * h->gp_lda;
  BX_CUDA(h, h->d_A.ensure(a_elems * 8));
  BX_CUDA(h, cudaMemsetAsync(h->d_A.p, 0, a_elems * 8, s));
  BX_CUDA(h, h->d_L.ensure((size_t)n * n * 8));
  BX_CUDA(h, cudaMemcpyAsync(h->d_L.p, L, (size_t)n * n * 8, cudaMemcpyHostToDevice, s));
  BX_CUDA(h, cudaMemcpyAsync(h->d_A.as<double>() + (size_t)n * h->gp_lda, alpha, (size_t)n * 8,
                             cudaMemcpyHostToDevice, s));
  BX_CUDA(h, h->d_train.ensure((size_t)n * h->row_words * 4));
  BX_CUDA(h, cudaMemcpyAsync(h->d_train.p, train_rows, (size_t)n * h->row_words * 4,
                             cudaMemcpyHostToDevice, s));
  BX_CUDA(h, h->d_inv_l.ensure(D * 8));
  BX_CUDA(h, cudaMemcpyAsync(h->d_inv_l.p, inv_l.data(), D * 8, cudaMemcpyHostToDevice, s));
  BX_CUDA(h, h->d_inv_l2.ensure(D * 8));
  BX_CUDA(h, cudaMemcpyAsync(h->d_inv_l2.p, inv_l2.data(), D * 8, cudaMemcpyHostToDevice, s));
  BX_CUDA(h, h->d_disc_tab.ensure(disc.size() * 8));
  BX_CUDA(h, cudaMemcpyAsync(h->d_disc_tab.p, disc.data(), disc.size() * 8, cudaMemcpyHostToDevice, s));
  BX_CUDA(h, h->d_disc_off.ensure(D * 4));
  BX_CUDA(h, cudaMemcpyAsync(h->d_disc_off.p, disc_off.data(), D * 4, cudaMemcpyHostToDevice, s));
  BX_CUDA(h, h->d_planes.ensure((size_t)D * n * 8));
  BX_CUDA(h, h->d_kmask.ensure((size_t)D * n * 16));
  BX_CUDA(h, launch_tri_inverse(h->d_L.as<double>(), n, h->d_A.as<double>(), h->gp_lda, s));
  BX_CUDA(h, launch_gp_planes(space_dev(h), h->d_train.as<uint32_t>(), n, h->d_inv_l.as<double>(),
                              h->d_planes.as<uint64_t>(), h->d_kmask.as<uint64_t>(), s));
  // register-resident path: n + 1 rows must fit 8 * 32 register rows and the smem budget
  h->use_fused = false;
  h->n_kendall = 0;
  for (int k = 0; k < D; ++k)
    if (h->params[k].kind == BX_PERMUTATION && h->params[k].metric == BX_KENDALL)
      h->kendall_param[h->n_kendall++] = k;
  const int mt = ((n + 1 + 15) / 16) * 2;  // m-tiles of 8 rows covering rows 0..n, even count
  if (!h->no_fused && 8 * mt <= fused_max_rows()) {
    const size_t smem = fused_smem_bytes(n, D, h->n_kendall, 8 * mt);
    if (smem <= 200 * 1024) {
      h->mt = mt;
      h->rows8 = 8 * mt;
      BX_CUDA(h, h->d_panels.ensure(panels_doubles(h->gp_ncols, h->rows8) * 8));
      BX_CUDA(h, launch_build_panels(h->d_A.as<double>(), h->gp_lda, h->gp_rows, h->gp_ncols,
                                     h->rows8, h->d_panels.as<double>(), s));
      h->use_fused = true;
    }
  }
  // tensor-core path: n <= 511 (32 row chunks; n > 255 runs two column passes per tile) and the
  // shared-memory budget.  Distances on the FP64 tensor cores over the Euclidean embedding of W
  // (EmbDim) when every metric embeds and the centred coordinates stay small, else FMA distances.
  h->use_tc = false;
  h->tc_ks = 0;
  if (!h->no_tc && n <= 511) {
    h->tc_emb.clear();
    h->tc_tab.clear();
    std::vector<double> planes, yy;
    const int nsl = (n + 31) / 32;
    bool dmma = !h->tc_no_dmma && !h->matern_precise &&
                build_embedding(h, train_rows, n, inv_l.data(), inv_l2.data(), 32 * nsl, h->tc_emb, h->tc_tab,
                                planes, yy, &h->tc_aug);
    const int E = (int)h->tc_emb.size();
    const int ks = dmma ? (E + 3) / 4 : 0;
    dmma = dmma && ks >= 1 && ks <= 8 &&
           tc_smem_bytes(n, D, h->n_kendall, h->row_words, ks, E, (int)h->tc_tab.size(), h->tc_aug, false) <= 227 * 1024;
    if (dmma || tc_smem_bytes(n, D, h->n_kendall, h->row_words, 0, 0, 0, false, false) <= 227 * 1024) {
      int Ex = 0;
      const double m = frexp(outputscale, &Ex);  // sigma < 2^Ex = sc
      if (m > 1.0 - ldexp(1.0, -20)) ++Ex;        // headroom: K* * 2^40 / sc < 2^40 - 2^20
      h->tc_nsl = nsl;
      h->tc_nch = n / 16 + 1;
      h->tc_kscale = ldexp(1.0, 40 - Ex);
      BX_CUDA(h, h->d_mdig.ensure(tc_mdig_bytes(n)));
      BX_CUDA(h, h->d_rowscale.ensure(2 * 512 * 8));
      if (h->tc_nsl > 8)  // pass-0 partial sums of rows >= 256: [CTA][256 rows][128 candidates]
        BX_CUDA(h, h->d_tc_part.ensure((size_t)h->sm_count * 256 * 128 * 8));
      if (dmma) {
        h->tc_ks = ks;
        BX_CUDA(h, upload(h->d_emb, h->tc_emb.data(), h->tc_emb.size()));
        BX_CUDA(h, upload(h->d_emb_tab, h->tc_tab.data(), h->tc_tab.size()));
        planes.resize((size_t)4 * ks * 32 * nsl, 0.0);  // k-rows beyond E (+2) are zero
        BX_CUDA(h, upload(h->d_emb_planes, planes.data(), planes.size()));
        BX_CUDA(h, upload(h->d_emb_yy, yy.data(), yy.size()));
      }
      h->use_tc = true;
      BX_CUDA(h, launch_build_mdig(h->d_A.as<double>(), h->gp_lda, n, ldexp(1.0, Ex),
                                   h->d_mdig.as<unsigned char>(), h->d_rowscale.as<double>(), dmma ? 1 : 0, s));
    }
  }
  BX_CUDA(h, cudaStreamSynchronize(s));  // host vectors above go out of scope
  h->outputscale = outputscale;
  h->y_mean = y_mean;
  h->y_std = y_std;
  h->has_gp = true;
  return BX_OK;
}

int bx_set_forest(bx_handle* h, const int32_t* feature, const double* threshold, const int32_t* left,
                  const int32_t* right, const double* value, int32_t n_nodes, const int32_t* roots,
                  int32_t n_trees, int32_t max_depth, double constant) {
  int r = check_space(h);
  if (r) return r;
  cudaSetDevice(h->device);
  h->forest = ForestDev{};
  if (!std::isnan(constant)) {
    h->forest.has_trees = 0;
    h->forest.constant = constant;
    h->forest.n_trees = 0;
    h->has_forest = true;
    return BX_OK;
  }
  if (n_trees < 1 || !roots)
    return fail(h, BX_ERR_NO_TREES, "feasibility model has no trees");
  // Re-pack breadth-first per tree so that children are adjacent; keep values of every node.
  std::vector<RfNode> nodes;
  nodes.reserve(n_nodes);
  std::vector<int32_t> new_roots(n_trees);
  std::vector<int32_t> queue;
  for (int t = 0; t < n_trees; ++t) {
    const int root = roots[t];
    if (root < 0 || root >= n_nodes) return fail(h, BX_ERR_ARG, "root %d out of range", root);
    new_roots[t] = (int)nodes.size();
    nodes.push_back(RfNode{threshold[root], value[root], feature[root], -1});
    queue.assign(1, root);
    std::vector<int32_t> slot(1, new_roots[t]);
    for (size_t qi = 0; qi < queue.size(); ++qi) {
      const int old = queue[qi];
      const int me = slot[qi];
      if (feature[old] < 0) continue;
      if (feature[old] >= h->n_features)
        return fail(h, BX_ERR_ARG, "node %d splits on feature %d >= %d", old, feature[old], h->n_features);
      const int l = left[old], rr = right[old];
      if (l < 0 || l >= n_nodes || rr < 0 || rr >= n_nodes)
        return fail(h, BX_ERR_ARG, "node %d has a child out of range", old);
      nodes[me].child = (int)nodes.size();
      nodes.push_back(RfNode{threshold[l], value[l], feature[l], -1});
      nodes.push_back(RfNode{threshold[rr], value[rr], feature[rr], -1});
      queue.push_back(l);
      slot.push_back(nodes[me].child);
      queue.push_back(rr);
      slot.push_back(nodes[me].child + 1);
    }
  }
  BX_CUDA(h, upload(h->d_nodes, nodes.data(), nodes.size()));
  BX_CUDA(h, upload(h->d_roots, new_roots.data(), new_roots.size()));
  h->forest.nodes = h->d_nodes.as<RfNode>();
  h->forest.roots = h->d_roots.as<int32_t>();
  h->forest.n_trees = n_trees;
  h->forest.max_depth = max_depth;
  h->forest.has_trees = 1;
  h->forest.constant = 0.0;
  h->forest.coded = 0;
  h->has_forest = true;
  if (!h->no_coded_forest) {
    r = build_coded_forest(h, nodes, new_roots, max_depth);
    if (r) return r;
  }
  return BX_OK;
}

// Integer-coded node table for rf_coded_kernel (see CodedForestDev).  Falls back to the generic
// kernel (coded = 0) whenever an assumption does not hold: a leaf deeper than max_depth, a
// non-monotone coordinate table, or a field overflow.
}  // extern "C"

static int build_coded_forest(bx_handle* h, const std::vector<RfNode>& nodes,
                              const std::vector<int32_t>& roots, int max_depth) {
  const int D = h->n_params;
  std::vector<int32_t> slot_base(D), code_param, code_sub;
  for (int k = 0; k < D; ++k) {
    const bx_param_desc& p = h->params[k];
    slot_base[k] = (int)code_param.size();
    // one code per encode_configs column: a one-hot label and a permutation position each get
    // their own slot, so every non-real split is `code < cut`
    const int cnt = (p.kind == BX_PERMUTATION || p.kind == BX_CATEGORICAL) ? p.size : 1;
    for (int e = 0; e < cnt; ++e) {
      code_param.push_back(k);
      code_sub.push_back(e);
    }
    if (p.kind == BX_INTEGER || p.kind == BX_ORDINAL)
      for (int i = 1; i < p.size; ++i)
        if (!(h->coord_host[p.coord + i - 1] <= h->coord_host[p.coord + i])) return BX_OK;
  }
  if ((int)code_param.size() > 64) return BX_OK;
  // depth of every node (breadth-first layout: children after parents)
  std::vector<int> depth(nodes.size(), -1);
  for (int32_t r : roots) depth[r] = 0;
  for (size_t u = 0; u < nodes.size(); ++u) {
    if (depth[u] < 0) return BX_OK;
    if (nodes[u].feat >= 0) {
      if (depth[u] + 1 > max_depth) return BX_OK;  // traversal would stop on an internal node
      depth[nodes[u].child] = depth[nodes[u].child + 1] = depth[u] + 1;
    }
  }
  std::vector<uint64_t> coded(nodes.size());
  std::vector<uint32_t> leaf_idx(nodes.size(), 0);
  std::vector<double> leaf_val, real_thr;
  bool has_real = false;
  for (size_t u = 0; u < nodes.size(); ++u) {
    const RfNode& nd = nodes[u];
    uint64_t type, slot = 0, arg, child;
    if (nd.feat < 0) {
      // leaf: `code[0] >= 0xFFFFFF` never holds and the left child is the leaf itself, so a walk
      // that reached it stays; its value index lives in leaf_idx
      type = 2;
      arg = 0xFFFFFF;
      leaf_idx[u] = (uint32_t)leaf_val.size();
      leaf_val.push_back(nd.val);
      child = (uint64_t)u;
      coded[u] = arg | (type << 30) | (child << 32);
      continue;
    } else {
      const int k = h->feat_param_host[nd.feat], sub = h->feat_sub_host[nd.feat];
      const bx_param_desc& p = h->params[k];
      const double t = nd.thr;
      child = (uint64_t)(uint32_t)nd.child;
      if (p.kind == BX_REAL) {
        type = 1;
        slot = slot_base[k];
        arg = real_thr.size();
        real_thr.push_back(t);
        has_real = true;
      } else {
        type = 0;
        int cut1 = 0;  // number of code values whose feature value is <= t
        slot = slot_base[k] + ((p.kind == BX_PERMUTATION || p.kind == BX_CATEGORICAL) ? sub : 0);
        if (p.kind == BX_PERMUTATION) {
          for (int i = 0; i < p.size; ++i) cut1 += ((double)i <= t) ? 1 : 0;
        } else if (p.kind == BX_CATEGORICAL) {
          cut1 = (0.0 <= t ? 1 : 0) + (1.0 <= t ? 1 : 0);  // one-hot code in {0, 1}
        } else {
          for (int i = 0; i < p.size; ++i) cut1 += (h->coord_host[p.coord + i] <= t) ? 1 : 0;
        }
        arg = (uint64_t)cut1;
      }
    }
    if (arg >= (1u << 24) || slot >= 64) return BX_OK;
    coded[u] = arg | (slot << 24) | (type << 30) | (child << 32);
  }
  h->forest.cf.has_real = has_real ? 1 : 0;
  if (leaf_val.empty()) leaf_val.push_back(0.0);
  if (real_thr.empty()) real_thr.push_back(0.0);
  BX_CUDA(h, upload(h->d_cnodes, coded.data(), coded.size()));
  BX_CUDA(h, upload(h->d_leaf_val, leaf_val.data(), leaf_val.size()));
  BX_CUDA(h, upload(h->d_leaf_idx, leaf_idx.data(), leaf_idx.size()));
  h->forest.cf.leaf_idx = h->d_leaf_idx.as<uint32_t>();
  BX_CUDA(h, upload(h->d_real_thr, real_thr.data(), real_thr.size()));
  BX_CUDA(h, upload(h->d_code_param, code_param.data(), code_param.size()));
  BX_CUDA(h, upload(h->d_code_sub, code_sub.data(), code_sub.size()));
  CodedForestDev& cf = h->forest.cf;
  cf.nodes = h->d_cnodes.as<uint64_t>();
  cf.leaf_val = h->d_leaf_val.as<double>();
  cf.real_thr = h->d_real_thr.as<double>();
  cf.roots = h->forest.roots;
  cf.code_param = h->d_code_param.as<int32_t>();
  cf.code_sub = h->d_code_sub.as<int32_t>();
  cf.n_nodes = (int)coded.size();
  cf.n_codes = (int)code_param.size();
  cf.n_trees = h->forest.n_trees;
  cf.max_depth = max_depth;
  cf.n_leaves = (int)leaf_val.size();
  cf.nodes_in_smem = 0;  // decided at launch from the smem budget
  h->forest.coded = 1;

  // QuickScorer tables (QsForestDev): integer splits only, <= 64 leaves per tree
  QsForestDev& qs = h->forest.qs;
  qs = QsForestDev{};
  // real features: the code of a real parameter is the number of its distinct split thresholds
  // below the candidate's coordinate, so `x <= thr_j` (go left) is `code < j + 1` like every other
  // split (thresholds sorted per parameter; the device finds the code by binary search)
  std::vector<std::vector<double>> rthr(D);
  std::vector<int32_t> qcut(nodes.size(), 0);
  bool rthr_ok = true;
  if (has_real) {
    for (size_t u = 0; u < nodes.size(); ++u)
      if (nodes[u].feat >= 0 && h->params[h->feat_param_host[nodes[u].feat]].kind == BX_REAL)
        rthr[h->feat_param_host[nodes[u].feat]].push_back(nodes[u].thr);
    for (int k = 0; k < D; ++k) {
      std::sort(rthr[k].begin(), rthr[k].end());
      rthr[k].erase(std::unique(rthr[k].begin(), rthr[k].end()), rthr[k].end());
      if (rthr[k].size() >= 32768) rthr_ok = false;
    }
    for (size_t u = 0; u < nodes.size(); ++u)
      if (nodes[u].feat >= 0 && h->params[h->feat_param_host[nodes[u].feat]].kind == BX_REAL) {
        const std::vector<double>& tv = rthr[h->feat_param_host[nodes[u].feat]];
        qcut[u] = (int32_t)(std::lower_bound(tv.begin(), tv.end(), nodes[u].thr) - tv.begin()) + 1;
      }
  }
  std::vector<int32_t> roff(D, 0);
  std::vector<double> rflat;
  for (int k = 0; k < D; ++k) {
    roff[k] = (int32_t)rflat.size();
    rflat.insert(rflat.end(), rthr[k].begin(), rthr[k].end());
  }
  if (rflat.size() >= 65536) rthr_ok = false;
  if (rflat.empty()) rflat.push_back(0.0);
  if (rthr_ok) {
    const int S = (int)code_param.size();
    std::vector<int32_t> soff(S), range(S);
    int stride = 0;
    for (int c = 0; c < S; ++c) {
      const bx_param_desc& p = h->params[code_param[c]];
      range[c] = p.kind == BX_CATEGORICAL ? 2 : (p.kind == BX_REAL ? (int)rthr[code_param[c]].size() + 1 : p.size);
      soff[c] = stride;
      stride += range[c];
    }
    const int T = h->forest.n_trees;
    std::vector<uint64_t> mask((size_t)T * stride, ~0ull);
    std::vector<uint16_t> vid((size_t)T * 64, 0);
    std::vector<double> uval;
    bool ok = (size_t)T * stride <= ((size_t)1 << 24);  // host tables; the shared-memory budget is checked below
    std::vector<int32_t> lo(nodes.size()), mid(nodes.size()), hi(nodes.size());
    for (int t = 0; ok && t < T; ++t) {
      // left-to-right leaf numbering and subtree leaf ranges by an explicit post-order walk
      int leaves = 0;
      std::vector<std::pair<int, int>> stack{{roots[t], 0}};  // (node, phase)
      while (!stack.empty() && ok) {
        const int u = stack.back().first;
        const int phase = stack.back().second;
        const RfNode& nd = nodes[u];
        if (nd.feat < 0) {
          if (leaves >= 64) { ok = false; break; }
          const double v = nd.val;
          size_t id = 0;
          while (id < uval.size() && std::memcmp(&uval[id], &v, 8) != 0) ++id;
          if (id == uval.size()) uval.push_back(v);
          if (id > 65535) { ok = false; break; }
          vid[(size_t)t * 64 + leaves] = (uint16_t)id;
          lo[u] = leaves;
          hi[u] = ++leaves;
          stack.pop_back();
        } else if (phase == 0) {
          stack.back().second = 1;
          lo[u] = leaves;
          stack.push_back({nd.child, 0});
        } else if (phase == 1) {
          stack.back().second = 2;
          mid[u] = leaves;
          stack.push_back({nd.child + 1, 0});
        } else {
          hi[u] = leaves;
          // going right (code >= cut) rules out the left subtree's leaves [lo, mid)
          const uint32_t lo32 = (uint32_t)coded[u];
          const bool real_split = ((coded[u] >> 30) & 3u) == 1u;
          const int slot = (int)((lo32 >> 24) & 63u), cut = real_split ? qcut[u] : (int)(lo32 & 0xFFFFFFu);
          const uint64_t left = ((mid[u] - lo[u]) >= 64 ? ~0ull : ((1ull << (mid[u] - lo[u])) - 1)) << lo[u];
          for (int v = cut; v < range[slot]; ++v) mask[(size_t)t * stride + soff[slot] + v] &= ~left;
          stack.pop_back();
        }
      }
    }
    // one code per categorical parameter instead of one per one-hot feature: the mask of label L
    // is the AND over the parameter's one-hot codes of their masks at [L == sub] (fewer table
    // loads per candidate: one per parameter and tree)
    std::vector<int32_t> qparam, qsub, qsoff, qrange;
    if (ok) {
      std::vector<int> merged(h->n_params, -1), newidx(S, -1);
      for (int c = 0; c < S; ++c) {
        const bx_param_desc& p = h->params[code_param[c]];
        if (p.kind == BX_CATEGORICAL) {
          if (merged[code_param[c]] >= 0) continue;
          merged[code_param[c]] = (int)qparam.size();
          qparam.push_back(code_param[c]);
          qsub.push_back(-1);
          qrange.push_back(p.size);
        } else {
          newidx[c] = (int)qparam.size();
          qparam.push_back(code_param[c]);
          // a real code carries its threshold run: offset | count << 16 into qs.rthr
          qsub.push_back(p.kind == BX_REAL ? (int32_t)(roff[code_param[c]] | (rthr[code_param[c]].size() << 16))
                                           : code_sub[c]);
          qrange.push_back(range[c]);
        }
      }
      int stride2 = 0;
      for (size_t c = 0; c < qparam.size(); ++c) {
        qsoff.push_back(stride2);
        stride2 += qrange[c];
      }
      {
        std::vector<uint64_t> m2((size_t)T * stride2, ~0ull);
        for (int t = 0; t < T; ++t) {
          for (int c = 0; c < S; ++c) {
            const bx_param_desc& p = h->params[code_param[c]];
            if (p.kind == BX_CATEGORICAL) {
              const int mc = merged[code_param[c]];
              for (int L = 0; L < p.size; ++L)
                m2[(size_t)t * stride2 + qsoff[mc] + L] &=
                    mask[(size_t)t * stride + soff[c] + (L == code_sub[c] ? 1 : 0)];
            } else {
              const int c2 = newidx[c];
              for (int v = 0; v < range[c]; ++v)
                m2[(size_t)t * stride2 + qsoff[c2] + v] = mask[(size_t)t * stride + soff[c] + v];
            }
          }
        }
        mask.swap(m2);
        stride = stride2;
      }
    }
    // indirect slots: real parameters whose codes span many thresholds keep, per tree, only the few
    // distinct masks its own splits produce (runs of equal masks along the code) and a [code][tree]
    // u16 index into them
    // indirect slots (QsForestDev): a real parameter whose codes span many thresholds, and a
    // permutation of <= 5 elements as ONE slot coded by its rank (m! codes, the AND of its element
    // positions' masks) instead of m position slots
    struct Ind {
      int param, sub, range;
      std::vector<int> slots;  // the q-slots it replaces
    };
    std::vector<Ind> ind;
    std::vector<char> taken(qparam.size(), 0);
    std::vector<int32_t> dparam, dsub, dsoff;
    int dstride = 0;
    if (ok) {
      for (size_t c = 0; c < qparam.size() && ind.size() < 4; ++c)
        if (h->params[qparam[c]].kind == BX_REAL && qrange[c] > 32) {
          ind.push_back(Ind{qparam[c], qsub[c], qrange[c], {(int)c}});
          taken[c] = 1;
        }
      for (int k = 0; k < h->n_params && ind.size() < 4; ++k) {
        const bx_param_desc& p = h->params[k];
        if (p.kind != BX_PERMUTATION || p.size > 5) continue;
        Ind d{k, -1, 1, std::vector<int>(p.size, -1)};
        for (int i = 2; i <= p.size; ++i) d.range *= i;
        for (size_t c = 0; c < qparam.size(); ++c)
          if (qparam[c] == k) d.slots[qsub[c]] = (int)c;  // slot of element e (code = its position)
        if (std::find(d.slots.begin(), d.slots.end(), -1) != d.slots.end()) continue;
        for (int c : d.slots) taken[c] = 1;
        ind.push_back(d);
      }
      for (size_t c = 0; c < qparam.size(); ++c) {
        if (taken[c]) continue;
        dparam.push_back(qparam[c]);
        dsub.push_back(qsub[c]);
        dsoff.push_back(dstride);
        dstride += qrange[c];
      }
      ok = (size_t)T * dstride * 8 <= 160 * 1024;
    }
    if (ok) {
      if (uval.empty()) uval.push_back(0.0);
      // direct slots transposed to [slot value][tree] so a group of 8 trees is one 64-byte run per
      // slot; odd row length (in 8-byte words): the <= 16 distinct code-value rows a half-warp reads
      // with 8-byte loads fall in 16 distinct bank pairs (groups of 8 trees read t .. t+7)
      int tpad = (T + 7) / 8 * 8 + 1;
      std::vector<uint64_t> mt((size_t)std::max(dstride, 1) * tpad, ~0ull);
      for (size_t c = 0, d = 0; c < qparam.size(); ++c) {
        if (taken[c]) continue;
        for (int v = 0; v < qrange[c]; ++v)
          for (int t = 0; t < T; ++t) mt[(size_t)(dsoff[d] + v) * tpad + t] = mask[(size_t)t * stride + qsoff[c] + v];
        ++d;
      }
      // indirect tables: rows (slot, code) x itpad u16 indices (itpad = 8 * odd: 16-byte rows)
      int itpad = (T + 7) / 8 * 8;
      if ((itpad / 8) % 2 == 0) itpad += 8;
      int irows = 0;
      for (const Ind& d : ind) irows += d.range;
      ok = (size_t)irows * itpad * 2 <= 96 * 1024;
      std::vector<uint16_t> iidx((size_t)std::max(irows, 1) * itpad, 0);
      std::vector<uint64_t> imask;
      qs.n_ind = (int)ind.size();
      int ioff = 0;
      for (size_t i = 0; i < ind.size() && ok; ++i) {
        const Ind& d = ind[i];
        qs.ind_param[i] = d.param;
        qs.ind_sub[i] = d.sub;
        qs.ind_off[i] = ioff;
        const bx_param_desc& p = h->params[d.param];
        for (int t = 0; t < T && ok; ++t) {
          int cur = -1;
          for (int v = 0; v < d.range; ++v) {
            uint64_t mv;
            if (p.kind == BX_REAL) {
              mv = mask[(size_t)t * stride + qsoff[d.slots[0]] + v];
            } else {  // permutation of rank v (Lehmer code): AND of the element-position masks
              int a[16], used = 0, r = v;
              for (int i = 0; i < p.size; ++i) {
                int f = 1;
                for (int j = 2; j <= p.size - 1 - i; ++j) f *= j;
                int c = r / f;
                r %= f;
                for (int e = 0; e < p.size; ++e)
                  if (!((used >> e) & 1) && c-- == 0) {
                    a[i] = e;
                    used |= 1 << e;
                    break;
                  }
              }
              mv = ~0ull;
              for (int i = 0; i < p.size; ++i) mv &= mask[(size_t)t * stride + qsoff[d.slots[a[i]]] + i];
            }
            if (cur < 0 || imask[cur] != mv) {
              cur = -1;
              for (size_t u = imask.size() > 64 ? imask.size() - 64 : 0; u < imask.size(); ++u)
                if (imask[u] == mv) cur = (int)u;  // reuse a recent equal mask (same tree)
              if (cur < 0) {
                cur = (int)imask.size();
                imask.push_back(mv);
              }
            }
            if (cur > 65535) { ok = false; break; }
            iidx[(size_t)(ioff + v) * itpad + t] = (uint16_t)cur;
          }
        }
        ioff += d.range;
      }
      if (imask.empty()) imask.push_back(~0ull);
      if (ok) {
        qs.tpad = tpad;
        BX_CUDA(h, upload(h->d_qmask, mt.data(), mt.size()));
        BX_CUDA(h, upload(h->d_qvid, vid.data(), vid.size()));
        BX_CUDA(h, upload(h->d_quval, uval.data(), uval.size()));
        if (dsoff.empty()) { dsoff.push_back(0); dparam.push_back(0); dsub.push_back(0); }
        BX_CUDA(h, upload(h->d_qsoff, dsoff.data(), dsoff.size()));
        BX_CUDA(h, upload(h->d_qcode_param, dparam.data(), dparam.size()));
        BX_CUDA(h, upload(h->d_qcode_sub, dsub.data(), dsub.size()));
        BX_CUDA(h, upload(h->d_qrthr, rflat.data(), rflat.size()));
        BX_CUDA(h, upload(h->d_qiidx, iidx.data(), iidx.size()));
        BX_CUDA(h, upload(h->d_qimask, imask.data(), imask.size()));
        qs.rthr = h->d_qrthr.as<double>();
        qs.has_real = has_real ? 1 : 0;
        qs.mask = h->d_qmask.as<uint64_t>();
        qs.vid = h->d_qvid.as<uint16_t>();
        qs.uval = h->d_quval.as<double>();
        qs.soff = h->d_qsoff.as<int32_t>();
        qs.code_param = h->d_qcode_param.as<int32_t>();
        qs.code_sub = h->d_qcode_sub.as<int32_t>();
        qs.iidx = h->d_qiidx.as<uint16_t>();
        qs.imask = h->d_qimask.as<uint64_t>();
        qs.itpad = itpad;
        qs.n_iidx_rows = irows;
        qs.n_imask = (int)imask.size();
        qs.n_trees = T;
        qs.n_codes = dstride > 0 ? (int)dparam.size() : 0;
        qs.stride = dstride;
        qs.n_uvals = (int)uval.size();
        qs.enabled = h->no_qs_forest ? 0 : 1;
        if (getenv("BX_QS_INFO"))  // development aid: table geometry
          fprintf(stderr, "qs: trees %d codes %d (+%d indirect: %d rows, %d masks) stride %d tpad %d uvals %d masks %zu B summary smem %zu B\n",
                  T, qs.n_codes, qs.n_ind, irows, qs.n_imask, dstride, tpad, qs.n_uvals, (size_t)dstride * tpad * 8,
                  (size_t)qs_summary_smem_bytes(qs));
      }
    }
  }
  return BX_OK;
}

extern "C" {

int bx_clear_forest(bx_handle* h) {
  if (!h) return BX_ERR_ARG;
  h->has_forest = false;
  return BX_OK;
}

int bx_set_evaluated(bx_handle* h, const uint32_t* rows, int32_t count) {
  int r = check_space(h);
  if (r) return r;
  cudaSetDevice(h->device);
  const int W = h->row_words;
  h->ev_count = count > 0 ? count : 0;
  if (h->ev_count == 0) return BX_OK;
  int size = 16;
  while (size < 2 * count) size <<= 1;
  std::vector<int32_t> table(size, -1);
  for (int i = 0; i < count; ++i) {
    const uint32_t* row = rows + (size_t)i * W;
    int slot = (int)(host_row_hash(row, W) & (uint64_t)(size - 1));
    while (table[slot] >= 0) {
      if (std::memcmp(rows + (size_t)table[slot] * W, row, W * 4) == 0) break;  // duplicate
      slot = (slot + 1) & (size - 1);
    }
    if (table[slot] < 0) table[slot] = i;
  }
  BX_CUDA(h, upload(h->d_ev_rows, rows, (size_t)count * W));
  BX_CUDA(h, upload(h->d_ev_table, table.data(), table.size()));
  h->ev_mask = size - 1;
  return BX_OK;
}

int bx_set_cot(bx_handle* h, int32_t n_groups, const int32_t* group_kind,
               const int32_t* group_param_begin, const int32_t* group_params,
               const int32_t* group_root, int32_t n_nodes, const int32_t* child_begin,
               const int32_t* child_count, const int32_t* node_value,
               const int64_t* node_leaf_count) {
  int r = check_space(h);
  if (r) return r;
  if (n_groups < 0 || n_nodes < 0) return fail(h, BX_ERR_ARG, "bad chain-of-trees sizes");
  cudaSetDevice(h->device);
  const int np = group_param_begin[n_groups];
  for (int g = 0; g < n_groups; ++g) {
    if (group_kind[g] == 0 && (group_root[g] < 0 || group_root[g] >= n_nodes))
      return fail(h, BX_ERR_ARG, "group %d root out of range", g);
  }
  for (int u = 0; u < n_nodes; ++u)
    if (child_count[u] < 0 || child_begin[u] < 0 || child_begin[u] + child_count[u] > n_nodes)
      return fail(h, BX_ERR_ARG, "node %d children out of range", u);
  BX_CUDA(h, upload(h->d_g_kind, group_kind, n_groups));
  BX_CUDA(h, upload(h->d_g_pbeg, group_param_begin, n_groups + 1));
  BX_CUDA(h, upload(h->d_g_params, group_params, np));
  BX_CUDA(h, upload(h->d_g_root, group_root, n_groups));
  BX_CUDA(h, upload(h->d_child_begin, child_begin, n_nodes));
  BX_CUDA(h, upload(h->d_child_count, child_count, n_nodes));
  BX_CUDA(h, upload(h->d_child_value, node_value, n_nodes));
  h->cot.n_groups = n_groups;
  h->cot.group_kind = h->d_g_kind.as<int32_t>();
  h->cot.group_param_begin = h->d_g_pbeg.as<int32_t>();
  h->cot.group_params = h->d_g_params.as<int32_t>();
  h->cot.group_root = h->d_g_root.as<int32_t>();
  h->cot.child_begin = h->d_child_begin.as<int32_t>();
  h->cot.child_count = h->d_child_count.as<int32_t>();
  h->cot.node_value = h->d_child_value.as<int32_t>();
  h->has_leaf_count = node_leaf_count != nullptr;
  if (node_leaf_count) BX_CUDA(h, upload(h->d_leaf_count, node_leaf_count, n_nodes));
  h->has_cot = true;
  return BX_OK;
}

int bx_clear_cot(bx_handle* h) {
  if (!h) return BX_ERR_ARG;
  h->has_cot = false;
  return BX_OK;
}

int bx_set_constraints(bx_handle* h, int32_t n_constraints, const int32_t* prog_begin,
                       const int32_t* code, int32_t code_len, const double* consts,
                       int32_t n_consts, const int32_t* value_tag, const int64_t* value_int,
                       const double* value_float, const int32_t* value_str, int32_t n_values) {
  int r = check_space(h);
  if (r) return r;
  if (n_constraints < 0 || code_len < 0 || n_consts < 0)
    return fail(h, BX_ERR_ARG, "bad constraint program sizes");
  cudaSetDevice(h->device);
  const int D = h->n_params;
  std::vector<int32_t> voff(D);
  int total = 0;
  for (int k = 0; k < D; ++k) {
    voff[k] = total;
    const bx_param_desc& p = h->params[k];
    total += (p.kind == BX_REAL || p.kind == BX_PERMUTATION) ? 0 : p.size;
  }
  if (total != n_values)
    return fail(h, BX_ERR_ARG, "constraint value tables: expected %d entries, got %d", total, n_values);
  if (n_constraints > 0 && prog_begin[n_constraints] != code_len)
    return fail(h, BX_ERR_ARG, "prog_begin[n] != code_len");
  const int lit = n_consts;
  std::vector<int32_t> vtag(value_tag, value_tag + total), sid(value_str, value_str + total);
  std::vector<int64_t> vint(value_int, value_int + total);
  std::vector<double> vflt(value_float, value_float + total);
  vtag.push_back(0); sid.push_back(0); vint.push_back(0); vflt.push_back(0.0);
  BX_CUDA(h, upload(h->d_prog_begin, prog_begin, n_constraints + 1));
  BX_CUDA(h, upload(h->d_code, code, code_len));
  BX_CUDA(h, upload(h->d_consts, consts, lit));
  BX_CUDA(h, upload(h->d_vtag, vtag.data(), vtag.size()));
  BX_CUDA(h, upload(h->d_vint, vint.data(), vint.size()));
  BX_CUDA(h, upload(h->d_vflt, vflt.data(), vflt.size()));
  BX_CUDA(h, upload(h->d_voff, voff.data(), voff.size()));
  BX_CUDA(h, upload(h->d_str_id, sid.data(), sid.size()));
  BX_CUDA(h, h->d_fault.ensure(16));
  BX_CUDA(h, cudaMemset(h->d_fault.p, 0, 16));
  h->cons.n_constraints = n_constraints;
  h->cons.prog_begin = h->d_prog_begin.as<int32_t>();
  h->cons.code = h->d_code.as<int32_t>();
  h->cons.consts = h->d_consts.as<double>();
  h->cons.vtag = h->d_vtag.as<int32_t>();
  h->cons.vint = h->d_vint.as<int64_t>();
  h->cons.vflt = h->d_vflt.as<double>();
  h->cons.voff = h->d_voff.as<int32_t>();
  h->cons.str_id = h->d_str_id.as<int32_t>();
  h->cons.fault = h->d_fault.as<int32_t>();
  h->has_constraints = true;
  return BX_OK;
}

// ---- scoring --------------------------------------------------------------------------------

// Summary pass over the EI / probability buffers of the last fused scoring launch.
static SummaryArgs last_summary_args(bx_handle* h, const uint32_t* rows, int64_t q,
                                     int64_t index_base, double eps_f, int32_t k, double* values,
                                     double* probs_out, Partial* partials) {
  const bool forest = h->has_forest && h->forest.has_trees;
  SummaryArgs m{};
  m.space = space_dev(h);
  m.evald = eval_dev(h);
  m.rows = rows;
  m.q = q;
  m.index_base = index_base;
  m.ei = h->d_ei.as<double>();
  m.probs_in = forest ? h->d_probs.as<double>() : nullptr;
  m.use_forest = h->has_forest ? 1 : 0;
  m.has_trees = forest ? 1 : 0;
  m.constant = h->forest.constant;
  m.eps_f = eps_f;
  m.k = k;
  m.values_out = values;
  m.probs_out = probs_out;
  m.partials = partials;
  return m;
}

static int score_impl(bx_handle* h, const uint32_t* rows, int64_t q, int64_t index_base,
                      double f_model, double eps_f, int32_t k, int32_t flags, double* values,
                      double* probs_out, Partial* partials, int* n_partials, cudaStream_t s,
                      int timing, bool track_prob = false, cudaEvent_t rows_ready = nullptr) {
  ScoreArgs a{};
  a.space = space_dev(h);
  a.gp = gp_dev(h);
  a.evald = eval_dev(h);
  a.rows = rows;
  a.q = q;
  a.index_base = index_base;
  a.f_model = f_model;
  a.eps_f = eps_f;
  a.k = k;
  a.flags = flags;
  a.use_forest = h->has_forest ? 1 : 0;
  a.forest = h->forest;
  a.values_out = values;
  a.probs_out = probs_out;
  a.partials = partials;
  const bool forest = h->has_forest && h->forest.has_trees;
  if (forest) BX_CUDA(h, h->d_probs.ensure((size_t)q * 8));
  if (fused_path(h)) {
    // posterior (mean / var) -> forest -> summary.  With a summary wanted and QuickScorer tables
    // that fit, the forest and the summary are one kernel after the posterior (it evaluates the EI
    // only for the candidates whose probability passes eps_f); otherwise the stand-alone forest
    // kernel runs before the posterior and the summary kernel after it.  The forest and posterior
    // kernels each fill every SM's shared memory, so they run back to back on the caller's stream
    // (which also makes the per-kernel CUDA-event timing exact).
    const bool rf_summ = forest && !(flags & BX_SCORE_RF_PAIRWISE) && !h->pw_rows && partials != nullptr &&
                         qs_summary_available(h->forest);
    h->rf_after_gp = rf_summ;
    // a stand-alone forest kernel before the posterior reads the rows: a streaming pool must be in
    if (rows_ready && forest && !rf_summ) BX_CUDA(h, cudaStreamWaitEvent(s, rows_ready, 0));
    if (timing == 1 && !rf_summ) BX_CUDA(h, cudaEventRecord(h->ev_t[0], s));
    if (forest && !rf_summ)
      BX_CUDA(h, launch_rf(a.space, h->forest, rows, q, (flags & BX_SCORE_RF_PAIRWISE) ? 1 : 0,
                           h->d_probs.as<double>(), s, h->pw_rows));
    if (timing == 1 && !rf_summ) BX_CUDA(h, cudaEventRecord(h->ev_t[1], s));
    BX_CUDA(h, h->d_ei.ensure((size_t)q * 16));
    FusedArgs f = fused_args(h, rows, q, f_model);
    f.mean_out = h->d_ei.as<double>();
    f.var_out = h->d_ei.as<double>() + q;
    if (timing) BX_CUDA(h, cudaEventRecord(h->ev_t[2], s));
    BX_CUDA(h, launch_posterior(h, f, s));
    if (timing) BX_CUDA(h, cudaEventRecord(h->ev_t[3], s));
    SummaryArgs m = last_summary_args(h, rows, q, index_base, eps_f, k, values, probs_out, partials);
    m.track_prob = track_prob ? 1 : 0;
    m.mean = h->d_ei.as<double>();
    m.var = h->d_ei.as<double>() + q;
    m.f_model = f_model;
    if (rows_ready) BX_CUDA(h, cudaStreamWaitEvent(s, rows_ready, 0));  // streaming pool fully copied
    if (rf_summ) {
      if (timing == 1) BX_CUDA(h, cudaEventRecord(h->ev_t[0], s));
      BX_CUDA(h, launch_rf_summary(a.space, h->forest, m, h->sm_count, s, n_partials));
      if (timing == 1) BX_CUDA(h, cudaEventRecord(h->ev_t[1], s));
      return BX_OK;
    }
    BX_CUDA(h, launch_summary(m, h->sm_count, s, n_partials));
    return BX_OK;
  }
  if (timing == 1) BX_CUDA(h, cudaEventRecord(h->ev_t[0], s));
  if (forest) {
    BX_CUDA(h, launch_rf(a.space, h->forest, rows, q, (flags & BX_SCORE_RF_PAIRWISE) ? 1 : 0,
                         h->d_probs.as<double>(), s, h->pw_rows));
    a.probs_in = h->d_probs.as<double>();
  }
  if (timing == 1) BX_CUDA(h, cudaEventRecord(h->ev_t[1], s));
  if (timing) BX_CUDA(h, cudaEventRecord(h->ev_t[2], s));
  BX_CUDA(h, launch_score(a, h->sm_count, s, n_partials));
  if (timing) BX_CUDA(h, cudaEventRecord(h->ev_t[3], s));
  return BX_OK;
}

int bx_score(bx_handle* h, const uint32_t* rows, int64_t q, int64_t index_base, double f_model,
             double eps_f, int32_t k, int32_t flags, double* values, double* probs,
             bx_score_summary* summary, void* stream) {
  int r = check_gp(h);
  if (r) return r;
  if (q < 1) return fail(h, BX_ERR_ARG, "empty candidate pool");
  if (k < 0 || k > BX_MAX_K) return fail(h, BX_ERR_ARG, "k=%d outside [0, %d]", k, BX_MAX_K);
  cudaSetDevice(h->device);
  cudaStream_t s = (cudaStream_t)stream;
  const bool want = !(flags & BX_SCORE_NO_SUMMARY) && summary != nullptr;
  const int timing = (flags & BX_SCORE_TIMING) ? 1 : ((flags & BX_SCORE_TIMING_POSTERIOR) ? 2 : 0);
  Partial* partials = nullptr;
  if (want) {
    BX_CUDA(h, h->d_partials.ensure(sizeof(Partial) * (size_t)max_partials(h->sm_count)));
    BX_CUDA(h, h->d_summary.ensure(sizeof(bx_score_summary)));
    partials = h->d_partials.as<Partial>();
  }
  int np = 0;
  r = score_impl(h, rows, q, index_base, f_model, eps_f, k, flags, values, probs, partials, &np, s,
                 timing);
  if (r) return r;
  if (want) {
    BX_CUDA(h, launch_summary_merge(partials, np, space_dev(h), k, rows, index_base,
                                    h->d_summary.as<bx_score_summary>(), s));
    if (timing == 1) BX_CUDA(h, cudaEventRecord(h->ev_t[4], s));
    BX_CUDA(h, cudaMemcpyAsync(summary, h->d_summary.p, sizeof(bx_score_summary),
                               cudaMemcpyDeviceToHost, s));
  } else if (timing == 1) {
    BX_CUDA(h, cudaEventRecord(h->ev_t[4], s));
  }
  if (want || timing) BX_CUDA(h, cudaStreamSynchronize(s));
  if (want && summary->n_finite == 0 && fused_path(h)) {
    // every value is -inf: only now is the probability tracker needed (acquisition.py:179-184)
    // rerun the step with the tracker on (it is the only rare path, so no state is kept for it)
    r = score_impl(h, rows, q, index_base, f_model, eps_f, k, flags & ~(BX_SCORE_TIMING | BX_SCORE_TIMING_POSTERIOR),
                   values, probs, partials, &np, s, 0, true);
    if (r) return r;
    BX_CUDA(h, launch_summary_merge(partials, np, space_dev(h), k, rows, index_base,
                                    h->d_summary.as<bx_score_summary>(), s));
    BX_CUDA(h, cudaMemcpyAsync(summary, h->d_summary.p, sizeof(bx_score_summary),
                               cudaMemcpyDeviceToHost, s));
    BX_CUDA(h, cudaStreamSynchronize(s));
  }
  if (timing == 1) {
    cudaEventElapsedTime(&h->t_ms[0], h->ev_t[0], h->ev_t[1]);
    cudaEventElapsedTime(&h->t_ms[1], h->ev_t[2], h->ev_t[3]);
    cudaEventElapsedTime(&h->t_ms[2], h->rf_after_gp ? h->ev_t[1] : h->ev_t[3], h->ev_t[4]);
  } else if (timing == 2) {  // the posterior only: the other kernels run back to back, unobserved
    cudaEventElapsedTime(&h->t_ms[1], h->ev_t[2], h->ev_t[3]);
    h->t_ms[0] = h->t_ms[2] = -1.0f;
  }
  return BX_OK;
}

int bx_last_timing(bx_handle* h, float* rf_ms, float* score_ms, float* merge_ms) {
  if (!h) return BX_ERR_ARG;
  if (rf_ms) *rf_ms = h->t_ms[0];
  if (score_ms) *score_ms = h->t_ms[1];
  if (merge_ms) *merge_ms = h->t_ms[2];
  return BX_OK;
}

int bx_score_host(bx_handle* h, const uint32_t* host_rows, int64_t q, int64_t index_base,
                  double f_model, double eps_f, int32_t k, int32_t flags,
                  bx_score_summary* summary, void* stream) {
  int r = check_gp(h);
  if (r) return r;
  if (q < 1) return fail(h, BX_ERR_ARG, "empty candidate pool");
  if (!summary) return fail(h, BX_ERR_ARG, "bx_score_host needs a summary");
  if (k < 0 || k > BX_MAX_K) return fail(h, BX_ERR_ARG, "k=%d outside [0, %d]", k, BX_MAX_K);
  cudaSetDevice(h->device);
  cudaStream_t s = (cudaStream_t)stream;
  const int W = h->row_words;
  const bool packed = (flags & BX_SCORE_PACKED) != 0;
  const int HW = packed ? h->pack.pw : W;  // words per host row
  flags &= ~(BX_SCORE_PACKED | BX_SCORE_NO_SUMMARY);
  BX_CUDA(h, h->d_pool.ensure((size_t)q * W * 4));
  if (packed) BX_CUDA(h, h->d_packed.ensure((size_t)q * HW * 4));
  BX_CUDA(h, h->d_partials.ensure(sizeof(Partial) * (size_t)max_partials(h->sm_count)));
  BX_CUDA(h, h->d_summary.ensure(sizeof(bx_score_summary)));
  uint32_t* pool = h->d_pool.as<uint32_t>();
  uint32_t* dst = packed ? h->d_packed.as<uint32_t>() : pool;  // where the host rows land
  Partial* parts = h->d_partials.as<Partial>();
  const bool forest = h->has_forest && h->forest.has_trees;
  if (h->use_tc && (!forest || qs_summary_available(h->forest)) && !(flags & BX_SCORE_RF_PAIRWISE) &&
      (!packed || h->pack.pw <= 16)) {
    // Streaming: the whole pool is copied in 2^16-row chunks on the copy stream, each followed by a
    // 4-byte ready flag written by the copy engine; one posterior launch consumes tiles as their
    // chunk lands (the row prefetcher waits on the flag; packed rows are unpacked by its decoders,
    // which write the full rows for the kernels after it), so only the first chunk's copy is
    // exposed and there is no per-chunk launch cost.  The forest + summary kernel runs after the
    // last copy.
    const int shift = 16;
    const int64_t n_chunks = (q + (1 << shift) - 1) >> shift;
    BX_CUDA(h, h->d_ready.ensure((size_t)n_chunks * 4));
    if (h->h_ones_len < n_chunks) {
      if (h->h_ones) cudaFreeHost(h->h_ones);
      h->h_ones = nullptr;
      BX_CUDA(h, cudaMallocHost(&h->h_ones, (size_t)n_chunks * 4));
      for (int64_t i = 0; i < n_chunks; ++i) h->h_ones[i] = 1u;
      h->h_ones_len = n_chunks;
    }
    uint32_t* ready = h->d_ready.as<uint32_t>();
    BX_CUDA(h, cudaMemsetAsync(ready, 0, (size_t)n_chunks * 4, s));
    BX_CUDA(h, cudaEventRecord(h->ev_done, s));
    BX_CUDA(h, cudaStreamWaitEvent(h->copy_stream, h->ev_done, 0));
    for (int64_t c = 0; c < n_chunks; ++c) {
      const int64_t off = c << shift, len = std::min<int64_t>((int64_t)1 << shift, q - off);
      BX_CUDA(h, cudaMemcpyAsync(dst + (size_t)off * HW, host_rows + (size_t)off * HW, (size_t)len * HW * 4,
                                 cudaMemcpyHostToDevice, h->copy_stream));
      BX_CUDA(h, cudaMemcpyAsync(ready + c, h->h_ones + c, 4, cudaMemcpyHostToDevice, h->copy_stream));
    }
    BX_CUDA(h, cudaEventRecord(h->ev_copy, h->copy_stream));
    for (int pass = 0; pass < 2; ++pass) {  // pass 2 (probability tracker) only if every value is -inf
      int np = 0;
      h->stream_ready = pass == 0 ? ready : nullptr;
      h->stream_shift = shift;
      h->stream_packed = (pass == 0 && packed) ? dst : nullptr;  // pass 2 reads the unpacked pool
      r = score_impl(h, pool, q, index_base, f_model, eps_f, k, flags, nullptr, nullptr, parts, &np, s, false,
                     pass == 1, pass == 0 ? h->ev_copy : nullptr);
      h->stream_ready = nullptr;
      h->stream_packed = nullptr;
      if (r) return r;
      BX_CUDA(h, launch_summary_merge(parts, np, space_dev(h), k, nullptr, 0,
                                      h->d_summary.as<bx_score_summary>(), s));
      BX_CUDA(h, cudaMemcpyAsync(summary, h->d_summary.p, sizeof(bx_score_summary), cudaMemcpyDeviceToHost, s));
      BX_CUDA(h, cudaStreamSynchronize(s));
      if (summary->n_finite != 0) break;
    }
  } else {
    // the other kernel paths: one copy (and a device unpack), then the device-resident path
    BX_CUDA(h, cudaMemcpyAsync(dst, host_rows, (size_t)q * HW * 4, cudaMemcpyHostToDevice, s));
    if (packed) BX_CUDA(h, launch_unpack(h->pack, dst, q, W, pool, s));
    r = bx_score(h, pool, q, index_base, f_model, eps_f, k, flags, nullptr, nullptr, summary, stream);
    if (r) return r;
  }
  // the pool is host-resident: the top-k rows come straight from the caller's buffer
  for (int i = 0; i < summary->n_top; ++i) {
    const uint32_t* src = host_rows + (size_t)(summary->top[i].index - index_base) * HW;
    if (packed) unpack_row(h->pack, src, summary->top[i].row, W);
    else std::memcpy(summary->top[i].row, src, (size_t)W * 4);
  }
  return BX_OK;
}

int bx_gp_predict(bx_handle* h, const uint32_t* rows, int64_t q, double* mean, double* var,
                  void* stream) {
  int r = check_gp(h);
  if (r) return r;
  if (q < 1) return BX_OK;
  cudaSetDevice(h->device);
  ScoreArgs a{};
  a.space = space_dev(h);
  a.gp = gp_dev(h);
  a.evald = EvalSetDev{};
  a.rows = rows;
  a.q = q;
  a.f_model = 0.0;
  a.mean_out = mean;
  a.var_out = var;
  int np = 0;
  if (fused_path(h)) {
    FusedArgs f = fused_args(h, rows, q, 0.0);
    f.mean_out = mean;
    f.var_out = var;
    BX_CUDA(h, launch_posterior(h, f, (cudaStream_t)stream));
    return BX_OK;
  }
  BX_CUDA(h, launch_score(a, h->sm_count, (cudaStream_t)stream, &np));
  return BX_OK;
}

int bx_rf_predict(bx_handle* h, const uint32_t* rows, int64_t q, int32_t flags, double* probs,
                  void* stream) {
  int r = check_space(h);
  if (r) return r;
  if (!h->has_forest) return fail(h, BX_ERR_STATE, "bx_set_forest has not been called");
  if (q < 1) return BX_OK;
  cudaSetDevice(h->device);
  cudaStream_t s = (cudaStream_t)stream;
  if (!h->forest.has_trees) {
    std::vector<double> c((size_t)q, h->forest.constant);
    BX_CUDA(h, cudaMemcpyAsync(probs, c.data(), (size_t)q * 8, cudaMemcpyHostToDevice, s));
    BX_CUDA(h, cudaStreamSynchronize(s));
    return BX_OK;
  }
  BX_CUDA(h, launch_rf(space_dev(h), h->forest, rows, q, (flags & BX_SCORE_RF_PAIRWISE) ? 1 : 0,
                       probs, s));
  return BX_OK;
}

int bx_neighbor_slots(bx_handle* h) { return (h && h->has_space) ? h->n_slots : -1; }

int bx_climb(bx_handle* h, const uint32_t* dev_pool_rows, const int64_t* host_start_index,
             const double* host_start_values, int32_t n_starts, int32_t use_cot, double f_model, double eps_f,
             int32_t max_steps, bx_cand* host_best, int32_t* host_steps, void* stream) {
  int r = check_gp(h);
  if (r) return r;
  if (n_starts < 0 || n_starts > BX_MAX_K || !host_best) return fail(h, BX_ERR_ARG, "bad climb arguments");
  if (use_cot && !h->has_cot) return fail(h, BX_ERR_STATE, "bx_set_cot has not been called");
  if (host_steps) *host_steps = 0;
  if (n_starts == 0) return BX_OK;
  cudaSetDevice(h->device);
  cudaStream_t s = (cudaStream_t)stream;
  const int A = n_starts, S = h->n_slots, W = h->row_words;
  // scratch: cur rows, values, active flags, neighbour rows, valid, pairwise flags, values, state
  size_t off = 0;
  auto take = [&](size_t bytes) { const size_t o = off; off += (bytes + 255) & ~(size_t)255; return o; };
  const size_t o_cur = take((size_t)A * W * 4), o_curv = take((size_t)A * 8), o_act = take((size_t)A * 4),
               o_nb = take((size_t)A * S * W * 4), o_val = take((size_t)A * S), o_pw = take((size_t)A * S),
               o_vals = take((size_t)A * S * 8), o_probs = take((size_t)A * S * 8), o_st = take(sizeof(ClimbState));
  BX_CUDA(h, h->d_climb.ensure(off));
  unsigned char* base = h->d_climb.as<unsigned char>();
  uint32_t* cur = reinterpret_cast<uint32_t*>(base + o_cur);
  double* curv = reinterpret_cast<double*>(base + o_curv);
  int32_t* act = reinterpret_cast<int32_t*>(base + o_act);
  uint32_t* nb = reinterpret_cast<uint32_t*>(base + o_nb);
  uint8_t* valid = base + o_val;
  uint8_t* pw = base + o_pw;
  double* vals = reinterpret_cast<double*>(base + o_vals);
  double* probs = reinterpret_cast<double*>(base + o_probs);
  ClimbState* st = reinterpret_cast<ClimbState*>(base + o_st);
  ClimbState hs{};
  hs.n_active = A;
  hs.best = TopRec{host_best->value, host_best->prob, host_best->index};
  std::memcpy(hs.best_row, host_best->row, sizeof(hs.best_row));
  std::vector<int32_t> ones(A, 1);
  for (int a = 0; a < A; ++a)  // the start rows, gathered from the pool
    BX_CUDA(h, cudaMemcpyAsync(cur + (size_t)a * W, dev_pool_rows + (size_t)host_start_index[a] * W, (size_t)W * 4,
                               cudaMemcpyDeviceToDevice, s));
  BX_CUDA(h, cudaMemcpyAsync(curv, host_start_values, (size_t)A * 8, cudaMemcpyHostToDevice, s));
  BX_CUDA(h, cudaMemcpyAsync(act, ones.data(), (size_t)A * 4, cudaMemcpyHostToDevice, s));
  BX_CUDA(h, cudaMemcpyAsync(st, &hs, sizeof(ClimbState), cudaMemcpyHostToDevice, s));
  int steps = 0;
  for (int step = 0; step < max_steps && hs.n_active > 0; ++step) {
    BX_CUDA(h, launch_neighbors(space_dev(h), use_cot ? &h->cot : nullptr, cur, A, nb, valid, s));
    climb_flags_kernel<<<1, 32, 0, s>>>(A, S, act, valid, pw);
    BX_CUDA(h, cudaGetLastError());
    h->pw_rows = pw;
    int np = 0;
    r = score_impl(h, nb, (int64_t)A * S, 0, f_model, eps_f, 0, 0, vals, probs, nullptr, &np, s, 0);
    h->pw_rows = nullptr;
    if (r) return r;
    climb_update_kernel<<<1, 32 * A, 0, s>>>(space_dev(h), eval_dev(h), A, S, act, cur, curv, nb, valid, vals, st);
    BX_CUDA(h, cudaGetLastError());
    BX_CUDA(h, cudaMemcpyAsync(&hs.n_active, &st->n_active, 4, cudaMemcpyDeviceToHost, s));
    BX_CUDA(h, cudaStreamSynchronize(s));  // the one device -> host read per step
    ++steps;
  }
  BX_CUDA(h, cudaMemcpyAsync(&hs, st, sizeof(ClimbState), cudaMemcpyDeviceToHost, s));
  BX_CUDA(h, cudaStreamSynchronize(s));
  host_best->value = hs.best.value;
  host_best->prob = hs.best.prob;
  host_best->index = hs.best.index;
  std::memcpy(host_best->row, hs.best_row, sizeof(hs.best_row));
  if (host_steps) *host_steps = steps;
  return BX_OK;
}

int bx_neighbors(bx_handle* h, const uint32_t* rows, int32_t count, int32_t use_cot,
                 uint32_t* out_rows, uint8_t* out_valid, void* stream) {
  int r = check_space(h);
  if (r) return r;
  if (use_cot && !h->has_cot) return fail(h, BX_ERR_STATE, "bx_set_cot has not been called");
  cudaSetDevice(h->device);
  BX_CUDA(h, launch_neighbors(space_dev(h), use_cot ? &h->cot : nullptr, rows, count, out_rows,
                              out_valid, (cudaStream_t)stream));
  return BX_OK;
}

int bx_cot_contains(bx_handle* h, const uint32_t* rows, int64_t q, uint8_t* mask, void* stream) {
  int r = check_space(h);
  if (r) return r;
  if (!h->has_cot) return fail(h, BX_ERR_STATE, "bx_set_cot has not been called");
  cudaSetDevice(h->device);
  BX_CUDA(h, launch_cot_contains(space_dev(h), h->cot, rows, q, mask, (cudaStream_t)stream));
  return BX_OK;
}

int bx_constraints_eval(bx_handle* h, const uint32_t* rows, int64_t q, uint8_t* mask, void* stream) {
  int r = check_space(h);
  if (r) return r;
  if (!h->has_constraints) return fail(h, BX_ERR_STATE, "bx_set_constraints has not been called");
  cudaSetDevice(h->device);
  cudaStream_t s = (cudaStream_t)stream;
  BX_CUDA(h, cudaMemsetAsync(h->d_fault.p, 0, 4, s));
  BX_CUDA(h, launch_constraints(space_dev(h), h->cons, rows, q, mask, s));
  int fault = 0;
  BX_CUDA(h, cudaMemcpyAsync(&fault, h->d_fault.p, 4, cudaMemcpyDeviceToHost, s));
  BX_CUDA(h, cudaStreamSynchronize(s));
  if (fault)
    return fail(h, BX_ERR_UNSUPPORTED,
                "constraint arithmetic left the exact int64/2^53 envelope of the device evaluator");
  return BX_OK;
}

int bx_lml_batched(bx_handle* h, const double* sq, int32_t n, int32_t D, const double* z,
                   const double* thetas, int32_t c, double* out, void* stream) {
  if (!h) return BX_ERR_ARG;
  if (n < 1 || D < 1 || D > BX_MAX_PARAMS || c < 0)
    return fail(h, BX_ERR_ARG, "bad lml shape n=%d D=%d c=%d", n, D, c);
  cudaSetDevice(h->device);
  if (lml_wide_supported(n) && !h->lml_narrow) {
    // blocked Cholesky batched over the settings, in groups that keep the factors under 1 GiB
    const int np = (n + 31) / 32 * 32;
    const int group = (int)std::max<size_t>(1, std::min<size_t>((size_t)c, (1ull << 30) / ((size_t)np * np * 8)));
    BX_CUDA(h, h->d_lml_scratch.ensure(lml_coarse_wide_scratch_doubles(n, group) * sizeof(double)));
    for (int c0 = 0; c0 < c; c0 += group)
      BX_CUDA(h, launch_lml_coarse_wide(sq, n, D, z, thetas + (size_t)c0 * (2 + D), std::min(group, c - c0),
                                        out + c0, h->d_lml_scratch.as<double>(), (cudaStream_t)stream));
    return BX_OK;
  }
  const size_t bytes = ((size_t)n * (n + 1) / 2 + n) * sizeof(double);
  double* scratch = nullptr;
  if (bytes > 200 * 1024) {
    BX_CUDA(h, h->d_lml_scratch.ensure(lml_scratch_doubles(n, c) * sizeof(double)));
    scratch = h->d_lml_scratch.as<double>();
  }
  BX_CUDA(h, launch_lml(sq, n, D, z, thetas, c, out, scratch, (cudaStream_t)stream));
  return BX_OK;
}

static int check_generate(bx_handle* h, int32_t mode) {
  int r = check_space(h);
  if (r) return r;
  if (mode < 0 || mode > 2) return fail(h, BX_ERR_ARG, "generation mode %d not in {0, 1, 2}", mode);
  if (mode == 1 && !(h->has_cot && h->has_leaf_count))
    return fail(h, BX_ERR_STATE, "mode 1 needs bx_set_cot with node leaf counts");
  if (mode == 2 && !h->has_cot) return fail(h, BX_ERR_STATE, "mode 2 needs bx_set_cot");
  return BX_OK;
}

int bx_generate(bx_handle* h, uint64_t seed, int64_t index_base, int64_t q, int32_t mode,
                uint32_t* rows, void* stream) {
  int r = check_generate(h, mode);
  if (r) return r;
  cudaSetDevice(h->device);
  CotDev cot = h->has_cot ? h->cot : CotDev{};
  BX_CUDA(h, launch_generate(space_dev(h), cot, h->d_leaf_count.as<int64_t>(), mode, seed, index_base,
                             q, rows, (cudaStream_t)stream));
  return BX_OK;
}

int bx_score_generated(bx_handle* h, uint64_t seed, int64_t index_base, int64_t q, int32_t mode,
                       double f_model, double eps_f, int32_t k, bx_score_summary* summary,
                       void* stream) {
  int r = check_gp(h);
  if (r) return r;
  r = check_generate(h, mode);
  if (r) return r;
  if (q < 1) return fail(h, BX_ERR_ARG, "empty candidate pool");
  if (!summary) return fail(h, BX_ERR_ARG, "bx_score_generated needs a summary");
  if (k < 0 || k > BX_MAX_K) return fail(h, BX_ERR_ARG, "k=%d outside [0, %d]", k, BX_MAX_K);
  cudaSetDevice(h->device);
  cudaStream_t s = (cudaStream_t)stream;
  const int W = h->row_words;
  const int64_t chunk = 1 << 22;
  const int64_t n_chunks = (q + chunk - 1) / chunk;
  const size_t per_chunk = (size_t)max_partials(h->sm_count);
  BX_CUDA(h, h->d_partials.ensure(sizeof(Partial) * per_chunk * (size_t)n_chunks));
  BX_CUDA(h, h->d_summary.ensure(sizeof(bx_score_summary)));
  BX_CUDA(h, h->d_gen_rows.ensure((size_t)chunk * W * 4));
  CotDev cot = h->has_cot ? h->cot : CotDev{};
  Partial* base = h->d_partials.as<Partial>();
  // Partials per chunk: one per SM (forest + summary kernel) or two (summary kernel).  They are
  // merged once at the end when all of them fit the fast merge, else folded into a running
  // partial after every chunk.
  const bool rf_summ = h->use_tc && h->has_forest && h->forest.has_trees && qs_summary_available(h->forest);
  const int64_t np_max = fused_path(h) ? (rf_summ ? 1 : 2) * (int64_t)h->sm_count : (int64_t)per_chunk;
  const bool fits_once = np_max * n_chunks <= 1024 &&
                         np_max * n_chunks * (k > 0 ? k : 1) * (int64_t)sizeof(TopRec) <= 200 * 1024;
  const bool running = !fits_once && np_max + 1 <= 1024 &&
                       (np_max + 1) * (k > 0 ? k : 1) * (int64_t)sizeof(TopRec) <= 200 * 1024;
  for (int pass = 0; pass < 2; ++pass) {
    int total = 0;
    for (int64_t c = 0; c < n_chunks; ++c) {
      const int64_t off = c * chunk;
      const int64_t len = (q - off) < chunk ? (q - off) : chunk;
      BX_CUDA(h, launch_generate(space_dev(h), cot, h->d_leaf_count.as<int64_t>(), mode, seed,
                                 index_base + off, len, h->d_gen_rows.as<uint32_t>(), s));
      int np = 0;
      Partial* dst = running ? base + 1 : base + total;
      r = score_impl(h, h->d_gen_rows.as<uint32_t>(), len, index_base + off, f_model, eps_f, k, 0,
                     nullptr, nullptr, dst, &np, s, false, pass == 1);
      if (r) return r;
      if (running)
        BX_CUDA(h, c == 0 ? launch_partial_merge(base + 1, np, space_dev(h), k, base, s)
                          : launch_partial_merge(base, np + 1, space_dev(h), k, base, s));
      total = running ? 1 : total + np;
    }
    BX_CUDA(h, launch_summary_merge(base, total, space_dev(h), k, nullptr, 0,
                                    h->d_summary.as<bx_score_summary>(), s));
    BX_CUDA(h, cudaMemcpyAsync(summary, h->d_summary.p, sizeof(bx_score_summary),
                               cudaMemcpyDeviceToHost, s));
    BX_CUDA(h, cudaStreamSynchronize(s));
    if (summary->n_finite != 0 || !fused_path(h)) break;
  }
  // regenerate the top-k rows from their global indices
  int64_t idx[BX_MAX_K];
  for (int i = 0; i < summary->n_top; ++i) idx[i] = summary->top[i].index;
  if (summary->n_top > 0) {
    BX_CUDA(h, launch_generate_indexed(space_dev(h), cot, h->d_leaf_count.as<int64_t>(), mode, seed,
                                       idx, summary->n_top, h->d_gen_rows.as<uint32_t>(), s));
    std::vector<uint32_t> rows((size_t)summary->n_top * W);
    BX_CUDA(h, cudaMemcpyAsync(rows.data(), h->d_gen_rows.p, rows.size() * 4, cudaMemcpyDeviceToHost, s));
    BX_CUDA(h, cudaStreamSynchronize(s));
    for (int i = 0; i < summary->n_top; ++i)
      std::memcpy(summary->top[i].row, rows.data() + (size_t)i * W, (size_t)W * 4);
  }
  return BX_OK;
}

int bx_lml_core(bx_handle* h, const double* sq, int32_t n, int32_t D, const double* z,
                const double* params, int32_t c, double prior_shape, double prior_rate,
                int32_t use_prior, int32_t want_grad, double* value, double* grad, int32_t* ok,
                void* stream) {
  if (!h) return BX_ERR_ARG;
  if (n < 1 || D < 1 || D > BX_MAX_PARAMS || c < 0)
    return fail(h, BX_ERR_ARG, "bad lml shape n=%d D=%d c=%d", n, D, c);
  if (want_grad && !grad) return fail(h, BX_ERR_ARG, "want_grad needs a gradient buffer");
  cudaSetDevice(h->device);
  // the whole-GPU pipeline, settings side by side on grid.y (a setting's arithmetic does not depend
  // on the batch: the batched L-BFGS-B restarts get the values a single call gives), in groups that
  // keep the scratch under 1 GiB; BX_OPT_LML_NARROW: one CTA per setting
  if (lml_wide_supported(n) && !h->lml_narrow) {
    const size_t per = lml_wide_scratch_doubles(n, D, 1) * sizeof(double);
    const int group = (int)std::max<size_t>(1, std::min<size_t>((size_t)std::max(c, 1), (1ull << 30) / per));
    BX_CUDA(h, h->d_grad_scratch.ensure(lml_wide_scratch_doubles(n, D, group) * sizeof(double)));
    for (int c0 = 0; c0 < c; c0 += group) {
      const int g = std::min(group, c - c0);
      BX_CUDA(h, launch_lml_wide(sq, n, D, z, params + (size_t)c0 * (2 + D), g, prior_shape, prior_rate, use_prior,
                                 want_grad, value + c0, want_grad ? grad + (size_t)c0 * (2 + D) : nullptr, ok + c0,
                                 h->d_grad_scratch.as<double>(), (cudaStream_t)stream));
    }
    return BX_OK;
  }
  BX_CUDA(h, h->d_grad_scratch.ensure(lml_grad_scratch_doubles(n, c) * sizeof(double)));
  BX_CUDA(h, launch_lml_grad(sq, n, D, z, params, c, prior_shape, prior_rate, use_prior, want_grad,
                             value, grad, ok, h->d_grad_scratch.as<double>(), (cudaStream_t)stream));
  return BX_OK;
}

int bx_pairwise_sq(bx_handle* h, const uint32_t* a, int32_t qa, const uint32_t* b, int32_t qb,
                   double* out, void* stream) {
  int r = check_space(h);
  if (r) return r;
  cudaSetDevice(h->device);
  BX_CUDA(h, launch_pairwise_sq(space_dev(h), a, qa, b, qb, out, (cudaStream_t)stream));
  return BX_OK;
}

}  // extern "C"
