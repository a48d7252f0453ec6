// score_summary.cu — acquisition value, eps_f filter and per-warp summaries over precomputed EI.
//
// value = ei                                  without a forest             (acquisition.py:75-76)
//       = -inf if p < eps_f else ei * p       with a forest                 (acquisition.py:77-79)
// Each lane owns one candidate; a ballot against the warp's current thresholds (which only
// tighten) selects the few candidates that can still enter the stable top-k or either tracker, and
// lane 0 folds them in sequentially.  The evaluated-set check (acquisition.py:107) is an exact row
// match through the handle's hash table.
#include "summary.cuh"

namespace bx {

namespace {

constexpr int kSumThreads = 256;
constexpr int kSumWarps = kSumThreads / 32;

__global__ void __launch_bounds__(kSumThreads) summary_kernel(SummaryArgs a) {
  __shared__ bx_param_desc params[BX_MAX_PARAMS];
  __shared__ Partial parts[kSumWarps];
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  for (int i = tid; i < a.space.n_params * (int)sizeof(bx_param_desc) / 4; i += blockDim.x)
    reinterpret_cast<int32_t*>(params)[i] = reinterpret_cast<const int32_t*>(a.space.params)[i];
  Partial* summ = &parts[warp];
  const bool want = a.partials != nullptr;
  if (want && lane == 0) partial_init(summ);
  __syncthreads();
  const int words = a.space.row_words;
  const int64_t stride = (int64_t)gridDim.x * kSumThreads;
  for (int64_t base = (int64_t)blockIdx.x * kSumThreads + warp * 32; base < a.q; base += stride) {
    const int64_t gi = base + lane;
    const bool valid = gi < a.q;
    double value = -INFINITY, prob = -INFINITY;
    if (valid) {
      const double ei = a.mean ? ei_value(a.mean[gi], a.var[gi], a.f_model) : a.ei[gi];
      if (a.use_forest) {
        prob = a.has_trees ? a.probs_in[gi] : a.constant;
        value = (prob < a.eps_f) ? -INFINITY : ei * prob;
      } else {
        prob = 1.0;
        value = ei;
      }
      if (a.values_out) a.values_out[gi] = value;
      if (a.probs_out) a.probs_out[gi] = prob;
    }
    if (!want) continue;
    const bool fin = valid && value != -INFINITY;
    // thresholds snapshot (warp-uniform reads of lane 0's partial)
    const bool top_open = a.k > 0 && summ->n_top < a.k;
    const double kth = (a.k > 0 && !top_open) ? summ->top[a.k - 1].value : -INFINITY;
    const bool prob_ok = a.track_prob && prob >= summ->best_prob.prob;
    const bool maybe = valid && ((fin && a.k > 0 && (top_open || value >= kth)) ||
                                 (fin && value >= summ->best.value) || prob_ok);
    bool evaluated = false;
    if (maybe && a.evald.count > 0) evaluated = is_evaluated(a.evald, a.rows + (size_t)gi * words, words);
    const bool pass = maybe && ((fin && a.k > 0 && (top_open || value >= kth)) ||
                                (!evaluated && ((fin && value >= summ->best.value) || prob_ok)));
    const unsigned vmask = __ballot_sync(0xffffffffu, valid);
    const unsigned fmask = __ballot_sync(0xffffffffu, fin);
    unsigned pmask = __ballot_sync(0xffffffffu, pass);
    const unsigned emask = __ballot_sync(0xffffffffu, evaluated);
    if (lane == 0) {
      summ->n_scored += __popc(vmask);
      summ->n_finite += __popc(fmask);
    }
    while (pmask) {
      const int c = __ffs(pmask) - 1;
      pmask &= pmask - 1;
      const double vc = __shfl_sync(0xffffffffu, value, c);
      const double pc = __shfl_sync(0xffffffffu, prob, c);
      if (lane == 0)
        partial_add(summ, a.k, params, a.space.n_params, a.space.rank_lut, words, vc, pc,
                    a.index_base + base + c, (emask >> c) & 1u, a.rows + (size_t)(base + c) * words,
                    a.track_prob != 0);
      __syncwarp();
    }
  }
  if (want) {
    __syncthreads();  // fold the block's warp partials into one
    if (tid == 0)
      for (int w = 1; w < kSumWarps; ++w)
        partial_merge(&parts[0], &parts[w], a.k, params, a.space.n_params, a.space.rank_lut, words);
    __syncthreads();
    const int32_t* src = reinterpret_cast<const int32_t*>(&parts[0]);
    int32_t* dst = reinterpret_cast<int32_t*>(a.partials + blockIdx.x);
    for (int i = tid; i < (int)(sizeof(Partial) / 4); i += kSumThreads) dst[i] = src[i];
  }
}

}  // namespace

int summary_max_partials(int sm_count) { return sm_count * 2 * kSumWarps; }

cudaError_t launch_summary(const SummaryArgs& a, int sm_count, cudaStream_t s, int* n_partials) {
  int64_t blocks = (a.q + kSumThreads - 1) / kSumThreads;
  if (blocks > (int64_t)sm_count * 2) blocks = (int64_t)sm_count * 2;
  if (blocks < 1) blocks = 1;
  *n_partials = (int)blocks;
  summary_kernel<<<(int)blocks, kSumThreads, 0, s>>>(a);
  return cudaGetLastError();
}

}  // namespace bx
