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

}  // namespace

cudaError_t launch_rf(const SpaceDev& space, const ForestDev& f, const uint32_t* rows, int64_t q,
                      int pairwise, double* probs, cudaStream_t s) {
  if (q <= 0) return cudaSuccess;
  int64_t blocks = (q + 255) / 256;
  if (blocks > 148 * 16) blocks = 148 * 16;
  rf_kernel<<<(int)blocks, 256, 0, s>>>(space, f, rows, q, pairwise, probs);
  return cudaGetLastError();
}

}  // namespace bx
