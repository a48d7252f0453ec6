// merge.cu — reduce per-block partial summaries into the bx_score_summary of a call.
//
// 128 threads: each folds a strided subset of the partials into its own top-k list in shared
// memory, then a log2(128)-level tree merges pairs of sorted lists (two-pointer merge, keep k)
// and the two tracker bests (value / probability desc, ties -> smaller configuration via
// key_cmp on the partials' stored rows).  Orders: acquisition.py:188 (top-k), :97-111 (trackers).
#include "summary.cuh"

namespace bx {

namespace {

constexpr int kMergeThreads = 128;

__device__ bool better_by_key(const Partial* parts, int a, int b, bool by_prob,
                              const bx_param_desc* params, int n_params, const int32_t* rank_lut) {
  if (a < 0) return false;
  if (b < 0) return true;
  const TopRec& ra = by_prob ? parts[a].best_prob : parts[a].best;
  const TopRec& rb = by_prob ? parts[b].best_prob : parts[b].best;
  const double x = by_prob ? ra.prob : ra.value, y = by_prob ? rb.prob : rb.value;
  if (x != y) return x > y;
  return key_cmp(params, n_params, rank_lut, by_prob ? parts[a].best_prob_row : parts[a].best_row,
                 by_prob ? parts[b].best_prob_row : parts[b].best_row) < 0;
}

// merge sorted list b (nb) into sorted list a (na), keeping k entries
__device__ void merge_lists(TopRec* a, int& na, const TopRec* b, int nb, int k) {
  TopRec tmp[BX_MAX_K];
  int i = 0, j = 0, o = 0;
  while (o < k && (i < na || j < nb)) {
    if (j >= nb || (i < na && !top_before(b[j].value, b[j].index, a[i])))
      tmp[o++] = a[i++];
    else
      tmp[o++] = b[j++];
  }
  for (int t = 0; t < o; ++t) a[t] = tmp[t];
  na = o;
}

__global__ void __launch_bounds__(kMergeThreads) merge_kernel(const Partial* parts, int n_parts,
                                                              SpaceDev space, int k,
                                                              const uint32_t* pool_rows,
                                                              int64_t index_base,
                                                              bx_score_summary* out) {
  extern __shared__ __align__(16) unsigned char smem[];
  TopRec* lists = reinterpret_cast<TopRec*>(smem);  // [kMergeThreads][k]
  __shared__ bx_param_desc params[BX_MAX_PARAMS];
  __shared__ int cnt[kMergeThreads], bi[kMergeThreads], pi[kMergeThreads];
  __shared__ long long sc[kMergeThreads], fi[kMergeThreads];
  const int t = threadIdx.x;
  for (int i = t; i < space.n_params * (int)sizeof(bx_param_desc) / 4; i += blockDim.x)
    reinterpret_cast<int32_t*>(params)[i] = reinterpret_cast<const int32_t*>(space.params)[i];
  __syncthreads();
  TopRec* mine = lists + (size_t)t * (k > 0 ? k : 1);
  int n = 0, b = -1, p = -1;
  long long s = 0, f = 0;
  for (int q = t; q < n_parts; q += blockDim.x) {
    const Partial& P = parts[q];
    s += P.n_scored;
    f += P.n_finite;
    if (k > 0) merge_lists(mine, n, P.top, P.n_top, k);
    if (P.best.index >= 0 && better_by_key(parts, q, b, false, params, space.n_params, space.rank_lut))
      b = q;
    if (P.best_prob.index >= 0 &&
        better_by_key(parts, q, p, true, params, space.n_params, space.rank_lut))
      p = q;
  }
  cnt[t] = n;
  bi[t] = b;
  pi[t] = p;
  sc[t] = s;
  fi[t] = f;
  __syncthreads();
  for (int stride = kMergeThreads / 2; stride > 0; stride >>= 1) {
    if (t < stride) {
      const int o = t + stride;
      int na = cnt[t];
      if (k > 0) merge_lists(mine, na, lists + (size_t)o * k, cnt[o], k);
      cnt[t] = na;
      if (better_by_key(parts, bi[o], bi[t], false, params, space.n_params, space.rank_lut)) bi[t] = bi[o];
      if (better_by_key(parts, pi[o], pi[t], true, params, space.n_params, space.rank_lut)) pi[t] = pi[o];
      sc[t] += sc[o];
      fi[t] += fi[o];
    }
    __syncthreads();
  }
  const int W = space.row_words;
  if (t == 0) {
    out->n_scored = sc[0];
    out->n_finite = fi[0];
    out->k = k;
    out->n_top = cnt[0];
    for (int i = 0; i < cnt[0]; ++i) {
      out->top[i].value = lists[i].value;
      out->top[i].prob = lists[i].prob;
      out->top[i].index = lists[i].index;
    }
    out->best.index = -1;
    out->best.value = out->best.prob = -INFINITY;
    if (bi[0] >= 0) {
      const Partial& P = parts[bi[0]];
      out->best.value = P.best.value;
      out->best.prob = P.best.prob;
      out->best.index = P.best.index;
      for (int w = 0; w < W; ++w) out->best.row[w] = P.best_row[w];
    }
    out->best_prob.index = -1;
    out->best_prob.value = out->best_prob.prob = -INFINITY;
    if (pi[0] >= 0) {
      const Partial& P = parts[pi[0]];
      out->best_prob.value = P.best_prob.value;
      out->best_prob.prob = P.best_prob.prob;
      out->best_prob.index = P.best_prob.index;
      for (int w = 0; w < W; ++w) out->best_prob.row[w] = P.best_prob_row[w];
    }
  }
  __syncthreads();
  if (pool_rows) {  // gather the rows of the top-k entries from the device pool
    for (int i = t; i < cnt[0] * W; i += blockDim.x) {
      const int e = i / W, w = i % W;
      out->top[e].row[w] = pool_rows[(size_t)(lists[e].index - index_base) * W + w];
    }
  }
}

}  // namespace

cudaError_t launch_summary_merge(const Partial* partials, int n_partials, const SpaceDev& space,
                                 int k, const uint32_t* pool_rows, int64_t index_base,
                                 bx_score_summary* out, cudaStream_t s) {
  const size_t bytes = (size_t)kMergeThreads * (k > 0 ? k : 1) * sizeof(TopRec);
  cudaError_t e = cudaFuncSetAttribute(merge_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                       (int)bytes);
  if (e != cudaSuccess) return e;
  merge_kernel<<<1, kMergeThreads, bytes, s>>>(partials, n_partials, space, k, pool_rows,
                                                index_base, out);
  return cudaGetLastError();
}

}  // namespace bx
