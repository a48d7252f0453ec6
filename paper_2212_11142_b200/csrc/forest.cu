// forest.cu — random-forest feasibility probability (FeasibilityModel.predict_proba_batch,
// feasibility.py:72-89) over encoded rows, bit-exact.
//
// One thread per candidate walks the trees in tree order.  Feature values are produced on the fly
// from the row exactly as encode_configs builds them (feasibility.py:33-51): the host-made
// coordinate of a numeric parameter, 0/1 one-hot for a categorical label, and the position of an
// element inside a permutation.  The comparison is the reference's `x <= threshold` on doubles and
// no arithmetic touches x, so the leaf reached is identical.  The mean over trees reproduces
// numpy's summation order: sequential over trees when q >= 2 (the (T, q) reduction over axis 0)
// and numpy's pairwise_sum (8 accumulators, 128-element blocks) when q == 1.
#include "bx_common.cuh"

namespace bx {

namespace {

__device__ __forceinline__ double feature_value(const SpaceDev& sp, const bx_param_desc* params,
                                                const uint32_t* row, int f) {
  const int k = sp.feat_param[f];
  const int sub = sp.feat_sub[f];
  const bx_param_desc& p = params[k];
  if (p.kind == BX_CATEGORICAL) return (int)row[p.word] == sub ? 1.0 : 0.0;
  if (p.kind == BX_PERMUTATION) return (double)perm_pos(row_u64(row, p.word), p.size, sub);
  return row_coord(p, sp.coord_lut, row);
}

__device__ __forceinline__ double leaf_value(const SpaceDev& sp, const bx_param_desc* params,
                                             const ForestDev& f, const uint32_t* row, int tree) {
  int cur = f.roots[tree];
  // feasibility.py:80-88: at most max_depth + 1 descents
  for (int it = 0; it <= f.max_depth; ++it) {
    const RfNode nd = f.nodes[cur];
    if (nd.feat < 0) break;
    const double x = feature_value(sp, params, row, nd.feat);
    cur = (x <= nd.thr) ? nd.child : nd.child + 1;
  }
  return f.nodes[cur].val;
}

// numpy pairwise_sum (numpy/_core/src/umath/loops_utils.h.src) over the leaf values of trees
// [t0, t0 + cnt), evaluated with the same association.
__device__ double pairwise_leaf_sum(const SpaceDev& sp, const bx_param_desc* params,
                                    const ForestDev& f, const uint32_t* row, int t0, int cnt) {
  if (cnt < 8) {
    double res = 0.0;
    for (int i = 0; i < cnt; ++i) res = __dadd_rn(res, leaf_value(sp, params, f, row, t0 + i));
    return res;
  }
  if (cnt <= 128) {
    double r[8];
    for (int i = 0; i < 8; ++i) r[i] = leaf_value(sp, params, f, row, t0 + i);
    int i = 8;
    for (; i < cnt - (cnt % 8); i += 8)
      for (int j = 0; j < 8; ++j) r[j] = __dadd_rn(r[j], leaf_value(sp, params, f, row, t0 + i + j));
    double res = __dadd_rn(__dadd_rn(__dadd_rn(r[0], r[1]), __dadd_rn(r[2], r[3])),
                           __dadd_rn(__dadd_rn(r[4], r[5]), __dadd_rn(r[6], r[7])));
    for (; i < cnt; ++i) res = __dadd_rn(res, leaf_value(sp, params, f, row, t0 + i));
    return res;
  }
  int n2 = cnt / 2;
  n2 -= n2 % 8;
  return __dadd_rn(pairwise_leaf_sum(sp, params, f, row, t0, n2),
                   pairwise_leaf_sum(sp, params, f, row, t0 + n2, cnt - n2));
}

__global__ void __launch_bounds__(256) rf_kernel(SpaceDev sp, ForestDev f, const uint32_t* rows,
                                                 int64_t q, int pairwise, double* probs) {
  __shared__ bx_param_desc params[BX_MAX_PARAMS];
  for (int i = threadIdx.x; i < sp.n_params * (int)sizeof(bx_param_desc) / 4; i += blockDim.x)
    reinterpret_cast<int32_t*>(params)[i] = reinterpret_cast<const int32_t*>(sp.params)[i];
  __syncthreads();
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < q;
       i += (int64_t)gridDim.x * blockDim.x) {
    const uint32_t* row = rows + (size_t)i * sp.row_words;
    double sum;
    if (pairwise) {
      sum = pairwise_leaf_sum(sp, params, f, row, 0, f.n_trees);
    } else {
      sum = leaf_value(sp, params, f, row, 0);
      for (int t = 1; t < f.n_trees; ++t) sum = __dadd_rn(sum, leaf_value(sp, params, f, row, t));
    }
    probs[i] = __ddiv_rn(sum, (double)f.n_trees);  // np.mean: sum / count
  }
}

// ---- integer-coded fast path -------------------------------------------------------------------
constexpr int kRfThreads = 256;

struct CodeView {
  const int32_t* code;  // smem [n_codes][kRfThreads]
  const double* real;   // smem [n_codes][kRfThreads] (only real slots used)
  int t;
};

__device__ __forceinline__ double coded_leaf(const CodedForestDev& cf, const uint64_t* nodes,
                                             const CodeView& cv, int tree) {
  int cur = cf.roots[tree];
  for (int it = 0; it <= cf.max_depth; ++it) {
    const uint64_t nd = nodes[cur];
    const int type = (int)(nd & 3u);
    if (type == 0) break;
    const int slot = (int)((nd >> 2) & 63u);
    const uint32_t arg = (uint32_t)(nd >> 8) & 0xFFFFFFu;
    bool left;
    if (type == 1) {
      left = cv.code[slot * kRfThreads + cv.t] < (int)arg;  // arg = cut + 1
    } else if (type == 2) {
      const bool eq = cv.code[slot * kRfThreads + cv.t] == (int)(arg & 0x3FFFFFu);
      left = eq ? ((arg >> 22) & 1u) : ((arg >> 23) & 1u);
    } else {
      left = cv.real[slot * kRfThreads + cv.t] <= cf.real_thr[arg];
    }
    cur = (int)(nd >> 32) + (left ? 0 : 1);
  }
  return cf.leaf_val[(uint32_t)(nodes[cur] >> 8) & 0xFFFFFFu];
}

// G trees walked in lockstep (independent dependency chains: G node loads in flight per thread);
// the leaf values are still added strictly in tree order.
template <int G>
__device__ __forceinline__ void coded_leaves(const CodedForestDev& cf, const uint64_t* nodes,
                                             const CodeView& cv, int t0, double* out) {
  int cur[G];
  bool live[G];
#pragma unroll
  for (int s = 0; s < G; ++s) {
    cur[s] = cf.roots[t0 + s];
    live[s] = true;
  }
  for (int it = 0; it <= cf.max_depth; ++it) {
    bool any = false;
#pragma unroll
    for (int s = 0; s < G; ++s) {
      if (!live[s]) continue;
      const uint64_t nd = nodes[cur[s]];
      const int type = (int)(nd & 3u);
      if (type == 0) {
        live[s] = false;
        continue;
      }
      any = true;
      const int slot = (int)((nd >> 2) & 63u);
      const uint32_t arg = (uint32_t)(nd >> 8) & 0xFFFFFFu;
      bool left;
      if (type == 1) {
        left = cv.code[slot * kRfThreads + cv.t] < (int)arg;
      } else if (type == 2) {
        const bool eq = cv.code[slot * kRfThreads + cv.t] == (int)(arg & 0x3FFFFFu);
        left = eq ? ((arg >> 22) & 1u) : ((arg >> 23) & 1u);
      } else {
        left = cv.real[slot * kRfThreads + cv.t] <= cf.real_thr[arg];
      }
      cur[s] = (int)(nd >> 32) + (left ? 0 : 1);
    }
    if (!any) break;
  }
#pragma unroll
  for (int s = 0; s < G; ++s) out[s] = cf.leaf_val[(uint32_t)(nodes[cur[s]] >> 8) & 0xFFFFFFu];
}

__device__ double coded_pairwise(const CodedForestDev& cf, const uint64_t* nodes, const CodeView& cv,
                                 int t0, int cnt) {
  if (cnt < 8) {
    double res = 0.0;
    for (int i = 0; i < cnt; ++i) res = __dadd_rn(res, coded_leaf(cf, nodes, cv, t0 + i));
    return res;
  }
  if (cnt <= 128) {
    double r[8];
    for (int i = 0; i < 8; ++i) r[i] = coded_leaf(cf, nodes, cv, t0 + i);
    int i = 8;
    for (; i < cnt - (cnt % 8); i += 8)
      for (int j = 0; j < 8; ++j) r[j] = __dadd_rn(r[j], coded_leaf(cf, nodes, cv, t0 + i + j));
    double res = __dadd_rn(__dadd_rn(__dadd_rn(r[0], r[1]), __dadd_rn(r[2], r[3])),
                           __dadd_rn(__dadd_rn(r[4], r[5]), __dadd_rn(r[6], r[7])));
    for (; i < cnt; ++i) res = __dadd_rn(res, coded_leaf(cf, nodes, cv, t0 + i));
    return res;
  }
  int n2 = cnt / 2;
  n2 -= n2 % 8;
  return __dadd_rn(coded_pairwise(cf, nodes, cv, t0, n2),
                   coded_pairwise(cf, nodes, cv, t0 + n2, cnt - n2));
}

__global__ void __launch_bounds__(kRfThreads) rf_coded_kernel(SpaceDev sp, CodedForestDev cf,
                                                              const uint32_t* rows, int64_t q,
                                                              int pairwise, double* probs) {
  extern __shared__ __align__(16) unsigned char smem[];
  __shared__ bx_param_desc params[BX_MAX_PARAMS];
  uint64_t* snodes = reinterpret_cast<uint64_t*>(smem);
  const size_t node_bytes = cf.nodes_in_smem ? (size_t)cf.n_nodes * 8 : 0;
  int32_t* code = reinterpret_cast<int32_t*>(smem + node_bytes);
  double* real = reinterpret_cast<double*>(smem + node_bytes + (size_t)cf.n_codes * kRfThreads * 4 +
                                           ((cf.n_codes & 1) ? kRfThreads * 4 : 0));
  for (int i = threadIdx.x; i < sp.n_params * (int)sizeof(bx_param_desc) / 4; i += blockDim.x)
    reinterpret_cast<int32_t*>(params)[i] = reinterpret_cast<const int32_t*>(sp.params)[i];
  if (cf.nodes_in_smem)
    for (int i = threadIdx.x; i < cf.n_nodes; i += blockDim.x) snodes[i] = cf.nodes[i];
  __syncthreads();
  const uint64_t* nodes = cf.nodes_in_smem ? snodes : cf.nodes;
  CodeView cv{code, real, (int)threadIdx.x};
  const int64_t stride = (int64_t)gridDim.x * blockDim.x;
  const int64_t n_iter = (q + stride - 1) / stride;
  for (int64_t it = 0; it < n_iter; ++it) {
    const int64_t i = it * stride + (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= q) break;
    const uint32_t* row = rows + (size_t)i * sp.row_words;
    for (int c = 0; c < cf.n_codes; ++c) {
      const bx_param_desc& p = params[cf.code_param[c]];
      int v = 0;
      if (p.kind == BX_PERMUTATION) {
        v = perm_pos(row_u64(row, p.word), p.size, cf.code_sub[c]);
      } else if (p.kind == BX_REAL) {
        real[c * kRfThreads + threadIdx.x] = row_f64(row, p.word + 2);
      } else {
        v = (int)row[p.word];
      }
      code[c * kRfThreads + threadIdx.x] = v;
    }
    double sum;
    if (pairwise) {
      sum = coded_pairwise(cf, nodes, cv, 0, cf.n_trees);
    } else {
      sum = coded_leaf(cf, nodes, cv, 0);
      for (int t = 1; t < cf.n_trees; ++t) sum = __dadd_rn(sum, coded_leaf(cf, nodes, cv, t));
    }
    probs[i] = __ddiv_rn(sum, (double)cf.n_trees);
  }
}

}  // namespace

size_t rf_coded_smem(const CodedForestDev& cf) {
  return (cf.nodes_in_smem ? (size_t)cf.n_nodes * 8 : 0) + (size_t)cf.n_codes * kRfThreads * 4 +
         ((cf.n_codes & 1) ? kRfThreads * 4 : 0) + (size_t)cf.n_codes * kRfThreads * 8;
}

cudaError_t launch_rf(const SpaceDev& space, const ForestDev& f, const uint32_t* rows, int64_t q,
                      int pairwise, double* probs, cudaStream_t s) {
  if (q <= 0) return cudaSuccess;
  if (f.coded) {
    const size_t bytes = rf_coded_smem(f.cf);
    cudaError_t e = cudaFuncSetAttribute(rf_coded_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                         (int)bytes);
    if (e != cudaSuccess) return e;
    int per_sm = 0, dev = 0, sms = 148;
    e = cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, rf_coded_kernel, kRfThreads, bytes);
    if (e != cudaSuccess) return e;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    int64_t blocks = (q + kRfThreads - 1) / kRfThreads;
    const int64_t cap = (int64_t)sms * (per_sm > 0 ? per_sm : 1);
    if (blocks > cap) blocks = cap;
    rf_coded_kernel<<<(int)blocks, kRfThreads, bytes, s>>>(space, f.cf, rows, q, pairwise, probs);
    return cudaGetLastError();
  }
  int64_t blocks = (q + 255) / 256;
  if (blocks > 148 * 16) blocks = 148 * 16;
  rf_kernel<<<(int)blocks, 256, 0, s>>>(space, f, rows, q, pairwise, probs);
  return cudaGetLastError();
}

}  // namespace bx
