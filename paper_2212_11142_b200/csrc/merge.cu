// merge.cu — reduce per-block partial summaries into the bx_score_summary of a call.
//
// Fast path (n_partials <= 1024, lists <= 200 KB): a two-level warp tournament (merge_fast_kernel).
// Otherwise
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

// ---- fast path: a two-level warp tournament over the partials' sorted top-k lists -------------
// Every partial's list is copied to shared memory; warp w merges the lists of partials
// [w G, (w+1) G) by k rounds of a warp argmax over the list heads (order: value desc, index asc),
// then warp 0 merges the 32 warp lists the same way.  Trackers: warp argmax by (value desc, key).
constexpr int kFastThreads = 1024;
constexpr int kFastBytes = 200 * 1024;  // n_parts * k * sizeof(TopRec) must fit

__device__ __forceinline__ bool rec_before(const TopRec& a, const TopRec& b) {
  return a.value > b.value || (a.value == b.value && a.index < b.index);
}

__device__ __forceinline__ TopRec shfl_rec(const TopRec& r, int src) {
  TopRec o;
  o.value = __shfl_sync(0xffffffffu, r.value, src);
  o.prob = __shfl_sync(0xffffffffu, r.prob, src);
  o.index = __shfl_sync(0xffffffffu, r.index, src);
  return o;
}

// k rounds of a warp argmax over up to 32 sorted lists (lane l owns list l: base + l * stride,
// length len); writes the merged top-k to dst (lane 0) and returns its length
__device__ int warp_tournament(const TopRec* base, int stride, int len, int k, TopRec* dst) {
  const int lane = threadIdx.x & 31;
  int pos = 0, o = 0;
  for (; o < k; ++o) {
    TopRec head = pos < len ? base[lane * stride + pos] : TopRec{-INFINITY, -INFINITY, INT64_MAX};
    int win = lane;
    for (int off = 16; off; off >>= 1) {
      const TopRec other = shfl_rec(head, lane ^ off);
      const int ow = __shfl_xor_sync(0xffffffffu, win, off);
      if (rec_before(other, head)) {
        head = other;
        win = ow;
      }
    }
    if (head.index == INT64_MAX) break;  // every list exhausted (warp-uniform)
    if (lane == 0) dst[o] = head;
    if (lane == win) ++pos;
  }
  return o;
}

// tracker argmax over lanes: candidate partial index q (or -1) per lane; the value is held in a
// register and the configuration key is only read on an exact value tie (then the earlier partial
// wins an exact key tie too, as the reference's first-seen rule does)
__device__ int warp_best(const Partial* parts, int q, bool by_prob, const bx_param_desc* params, int n_params,
                         const int32_t* rank_lut) {
  double v = -INFINITY;
  if (q >= 0) v = by_prob ? parts[q].best_prob.prob : parts[q].best.value;
  for (int off = 16; off; off >>= 1) {
    const int o = __shfl_xor_sync(0xffffffffu, q, off);
    const double ov = __shfl_xor_sync(0xffffffffu, v, off);
    bool take = false;
    if (o >= 0) {
      if (q < 0 || ov > v) {
        take = true;
      } else if (ov == v) {
        const int c = key_cmp(params, n_params, rank_lut, by_prob ? parts[o].best_prob_row : parts[o].best_row,
                              by_prob ? parts[q].best_prob_row : parts[q].best_row);
        take = c < 0 || (c == 0 && o < q);
      }
    }
    if (take) {
      q = o;
      v = ov;
    }
  }
  return q;
}

// acc_out != nullptr: write the merged Partial (running summary of a chunked pool); otherwise the
// final bx_score_summary (+ top-k rows gathered from pool_rows when given).
__global__ void __launch_bounds__(kFastThreads) merge_fast_kernel(const Partial* parts, int n_parts, SpaceDev space,
                                                                  int k, const uint32_t* pool_rows,
                                                                  int64_t index_base, bx_score_summary* out,
                                                                  Partial* acc_out) {
  extern __shared__ __align__(16) unsigned char smem[];
  TopRec* lists = reinterpret_cast<TopRec*>(smem);  // [n_parts][k]
  __shared__ bx_param_desc params[BX_MAX_PARAMS];
  __shared__ TopRec wl[32][BX_MAX_K];
  __shared__ int wn[32], wb[32], wp[32];
  __shared__ long long wsc[32], wfi[32];
  const int t = threadIdx.x, lane = t & 31, warp = t >> 5;
  for (int i = t; i < space.n_params * (int)sizeof(bx_param_desc) / 4; i += blockDim.x)
    reinterpret_cast<int32_t*>(params)[i] = reinterpret_cast<const int32_t*>(space.params)[i];
  const int kk = k > 0 ? k : 1;
  for (int i = t; i < n_parts * kk; i += blockDim.x) lists[i] = parts[i / kk].top[i % kk];
  const int G = (n_parts + 31) / 32;  // partials per warp (n_parts <= 1024)
  const int p = warp * G + lane;
  const bool mine = lane < G && p < n_parts;
  long long sc = mine ? parts[p].n_scored : 0, fi = mine ? parts[p].n_finite : 0;
  for (int off = 16; off; off >>= 1) {
    sc += __shfl_xor_sync(0xffffffffu, sc, off);
    fi += __shfl_xor_sync(0xffffffffu, fi, off);
  }
  int qb = (mine && parts[p].best.index >= 0) ? p : -1;
  int qp = (mine && parts[p].best_prob.index >= 0) ? p : -1;
  qb = warp_best(parts, qb, false, params, space.n_params, space.rank_lut);
  qp = warp_best(parts, qp, true, params, space.n_params, space.rank_lut);
  __syncthreads();  // lists staged
  const int n_w = k > 0 ? warp_tournament(lists + (size_t)warp * G * kk, kk, mine ? parts[p].n_top : 0, k, wl[warp]) : 0;
  if (lane == 0) {
    wn[warp] = n_w;
    wb[warp] = qb;
    wp[warp] = qp;
    wsc[warp] = sc;
    wfi[warp] = fi;
  }
  __syncthreads();
  __shared__ TopRec fin[BX_MAX_K];
  __shared__ int n_top_s, best_s, bestp_s;
  __shared__ long long sc_s, fi_s;
  if (warp == 0) {
    const int nw = (int)(blockDim.x >> 5);
    const int n_top = k > 0 ? warp_tournament(&wl[0][0], BX_MAX_K, lane < nw ? wn[lane] : 0, k, fin) : 0;
    long long a1 = lane < nw ? wsc[lane] : 0, a2 = lane < nw ? wfi[lane] : 0;
    for (int off = 16; off; off >>= 1) {
      a1 += __shfl_xor_sync(0xffffffffu, a1, off);
      a2 += __shfl_xor_sync(0xffffffffu, a2, off);
    }
    const int b1 = warp_best(parts, lane < nw ? wb[lane] : -1, false, params, space.n_params, space.rank_lut);
    const int b2 = warp_best(parts, lane < nw ? wp[lane] : -1, true, params, space.n_params, space.rank_lut);
    if (lane == 0) {
      n_top_s = n_top;
      best_s = b1;
      bestp_s = b2;
      sc_s = a1;
      fi_s = a2;
    }
  }
  __syncthreads();
  const int n_top = n_top_s, best = best_s, bestp = bestp_s;
  const int W = space.row_words;
  if (acc_out) {  // parts may alias acc_out: read everything into registers, then write
    const TopRec tb = best >= 0 ? parts[best].best : TopRec{-INFINITY, -INFINITY, -1};
    const TopRec tp = bestp >= 0 ? parts[bestp].best_prob : TopRec{-INFINITY, -INFINITY, -1};
    const uint32_t rb = (t < W && best >= 0) ? parts[best].best_row[t] : 0u;
    const uint32_t rp = (t < W && bestp >= 0) ? parts[bestp].best_prob_row[t] : 0u;
    __syncthreads();
    if (t == 0) {
      acc_out->n_scored = sc_s;
      acc_out->n_finite = fi_s;
      acc_out->n_top = n_top;
      acc_out->best = tb;
      acc_out->best_prob = tp;
    }
    if (t < n_top) acc_out->top[t] = fin[t];
    if (t < W) {
      acc_out->best_row[t] = rb;
      acc_out->best_prob_row[t] = rp;
    }
    return;
  }
  if (t == 0) {
    out->n_scored = sc_s;
    out->n_finite = fi_s;
    out->k = k;
    out->n_top = n_top;
    out->best.index = -1;
    out->best.value = out->best.prob = -INFINITY;
    if (best >= 0) {
      out->best.value = parts[best].best.value;
      out->best.prob = parts[best].best.prob;
      out->best.index = parts[best].best.index;
    }
    out->best_prob.index = -1;
    out->best_prob.value = out->best_prob.prob = -INFINITY;
    if (bestp >= 0) {
      out->best_prob.value = parts[bestp].best_prob.value;
      out->best_prob.prob = parts[bestp].best_prob.prob;
      out->best_prob.index = parts[bestp].best_prob.index;
    }
  }
  if (t < n_top) {
    out->top[t].value = fin[t].value;
    out->top[t].prob = fin[t].prob;
    out->top[t].index = fin[t].index;
  }
  if (t < W) {
    if (best >= 0) out->best.row[t] = parts[best].best_row[t];
    if (bestp >= 0) out->best_prob.row[t] = parts[bestp].best_prob_row[t];
  }
  if (pool_rows)
    for (int i = t; i < n_top * W; i += blockDim.x) {
      const int e = i / W, w = i % W;
      out->top[e].row[w] = pool_rows[(size_t)(fin[e].index - index_base) * W + w];
    }
}

}  // namespace

cudaError_t launch_partial_merge(const Partial* partials, int n_partials, const SpaceDev& space, int k,
                                 Partial* acc_out, cudaStream_t s) {
  const size_t bytes = (size_t)n_partials * (k > 0 ? k : 1) * sizeof(TopRec);
  if (n_partials > 1024 || bytes > (size_t)kFastBytes) return cudaErrorInvalidValue;
  cudaError_t e = set_smem(merge_fast_kernel, (int)bytes);
  if (e != cudaSuccess) return e;
  merge_fast_kernel<<<1, kFastThreads, bytes, s>>>(partials, n_partials, space, k, nullptr, 0, nullptr, acc_out);
  return cudaGetLastError();
}

cudaError_t launch_summary_merge(const Partial* partials, int n_partials, const SpaceDev& space,
                                 int k, const uint32_t* pool_rows, int64_t index_base,
                                 bx_score_summary* out, cudaStream_t s) {
  const size_t fb = (size_t)n_partials * (k > 0 ? k : 1) * sizeof(TopRec);
  if (n_partials <= 1024 && fb <= (size_t)kFastBytes) {
    cudaError_t e = set_smem(merge_fast_kernel, (int)fb);
    if (e != cudaSuccess) return e;
    merge_fast_kernel<<<1, kFastThreads, fb, s>>>(partials, n_partials, space, k, pool_rows, index_base, out,
                                                   nullptr);
    return cudaGetLastError();
  }
  const size_t bytes = (size_t)kMergeThreads * (k > 0 ? k : 1) * sizeof(TopRec);
  cudaError_t e = set_smem(merge_kernel, (int)bytes);
  if (e != cudaSuccess) return e;
  merge_kernel<<<1, kMergeThreads, bytes, s>>>(partials, n_partials, space, k, pool_rows,
                                                index_base, out);
  return cudaGetLastError();
}

}  // namespace bx
