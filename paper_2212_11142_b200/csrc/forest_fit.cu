// forest_fit.cu — rf_fit's tree building (feasibility.py:95-197, _TreeBuilder.build) on the device,
// bit-exact: one CTA per tree walks the tree depth first exactly as the reference's recursion does,
// so node ids come out in the reference's creation (preorder) order and the i-th node that draws a
// feature subset gets the i-th subset of the tree's generator (drawn on the host, in order: the
// RNG stream is numpy's own).  Per node the 256 threads evaluate every drawn feature:
//   * the node's rows in their current order (bootstrap order, then stable partitions);
//   * a stable sort by the feature value (bitonic over (value, position) pairs = np.argsort kind
//     "stable");
//   * positives by prefix counts (the reference's cumsum of 0/1 values: exact integers);
//   * the weighted Gini of every cut between distinct values with the reference's operation order
//     (IEEE operations, no contraction), the first minimum (np.argmin), strict improvement across
//     features in drawing order;
//   * threshold = 0.5 (x_i + x_i+1), left = x <= threshold, stable partition of the rows.
// A tree that needs more subsets than were drawn reports it (status 1) and the host draws more from
// the same generator and builds it again.
#include <cfloat>

#include "bx_common.cuh"

namespace bx {

namespace {

constexpr int kFitThreads = 256;

struct FitStack {
  int s, e, depth, parent;  // row segment [s, e), depth, parent node (its right child)
};

__device__ __forceinline__ bool key_less(double va, int ia, double vb, int ib) {
  return va < vb || (va == vb && ia < ib);
}

// bitonic sort of (key, idx) over np elements (a power of two) in shared memory, ascending
__device__ void bitonic(double* key, int* idx, int np) {
  for (int size = 2; size <= np; size <<= 1) {
    for (int stride = size >> 1; stride > 0; stride >>= 1) {
      __syncthreads();
      for (int t = threadIdx.x; t < np / 2; t += blockDim.x) {
        const int lo = 2 * t - (t & (stride - 1));
        const int hi = lo + stride;
        const bool up = ((lo & size) == 0);
        const bool swap = up ? key_less(key[hi], idx[hi], key[lo], idx[lo]) : key_less(key[lo], idx[lo], key[hi], idx[hi]);
        if (swap) {
          const double k = key[lo];
          key[lo] = key[hi];
          key[hi] = k;
          const int i = idx[lo];
          idx[lo] = idx[hi];
          idx[hi] = i;
        }
      }
    }
  }
  __syncthreads();
}

// block-wide inclusive prefix sum of cnt[0..n) (ints), in place
__device__ void block_scan(int* cnt, int n, int* warp_tot) {
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  int carry = 0;
  for (int base = 0; base < n; base += blockDim.x) {
    const int i = base + threadIdx.x;
    int v = i < n ? cnt[i] : 0;
    for (int o = 1; o < 32; o <<= 1) {
      const int u = __shfl_up_sync(0xffffffffu, v, o);
      if (lane >= o) v += u;
    }
    if (lane == 31) warp_tot[warp] = v;
    __syncthreads();
    if (warp == 0) {
      int w = lane < (int)(blockDim.x >> 5) ? warp_tot[lane] : 0;
      for (int o = 1; o < 32; o <<= 1) {
        const int u = __shfl_up_sync(0xffffffffu, w, o);
        if (lane >= o) w += u;
      }
      if (lane < (int)(blockDim.x >> 5)) warp_tot[lane] = w;
    }
    __syncthreads();
    const int add = carry + (warp > 0 ? warp_tot[warp - 1] : 0);
    if (i < n) cnt[i] = v + add;
    carry += warp_tot[(blockDim.x >> 5) - 1];
    __syncthreads();
  }
}

__global__ void __launch_bounds__(kFitThreads) rf_fit_kernel(const double* X, const double* y, int n, int F,
                                                               const int32_t* boot, const int32_t* feats,
                                                               const int32_t* n_drawn, int max_draws, int k,
                                                               int max_depth, int max_nodes, int32_t* o_feature,
                                                               double* o_threshold, int32_t* o_left, int32_t* o_right,
                                                               double* o_value, int32_t* o_n_nodes,
                                                               int32_t* o_status, FitStack* stack_g) {
  extern __shared__ __align__(16) unsigned char smem[];
  const int np2 = [&] { int p = 1; while (p < n) p <<= 1; return p; }();
  double* key = reinterpret_cast<double*>(smem);          // [np2]
  int* idx = reinterpret_cast<int*>(key + np2);            // [np2]
  int* rows = idx + np2;                                   // [n]
  int* tmp = rows + n;                                     // [n]
  int* cnt = tmp + n;                                      // [n]
  __shared__ int warp_tot[kFitThreads / 32];
  __shared__ double red_s[kFitThreads / 32];
  __shared__ int red_i[kFitThreads / 32];
  __shared__ int s_n_nodes, s_draw, s_sp, s_status, s_best_f, s_best_cut_i;
  __shared__ double s_best_score, s_best_thr;
  const int t = blockIdx.x, tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int base = t * max_nodes;
  FitStack* stack = stack_g + (size_t)t * max_nodes;
  for (int i = tid; i < n; i += blockDim.x) rows[i] = boot[(size_t)t * n + i];
  if (tid == 0) {
    s_n_nodes = 0;
    s_draw = 0;
    s_status = 0;
    s_sp = 1;
    stack[0] = FitStack{0, n, 0, -1};
  }
  __syncthreads();
  while (true) {
    __syncthreads();
    if (s_sp == 0 || s_status != 0) break;
    const FitStack cur = stack[s_sp - 1];
    __syncthreads();
    if (tid == 0) --s_sp;
    const int s = cur.s, e = cur.e, m = e - s;
    // new_node(): preorder id; the parent of a right child learns it now
    const int node = s_n_nodes;
    __syncthreads();
    if (tid == 0) {
      s_n_nodes = node + 1;
      if (node >= max_nodes) s_status = 2;
      if (cur.parent >= 0) o_right[base + cur.parent] = node;
    }
    __syncthreads();
    if (s_status) break;
    // value = mean of y over the node's rows (0/1 values: an exact count)
    int pc = 0;
    for (int i = tid; i < m; i += blockDim.x) pc += y[rows[s + i]] > 0.5 ? 1 : 0;
    for (int o = 16; o; o >>= 1) pc += __shfl_xor_sync(0xffffffffu, pc, o);
    if (lane == 0) warp_tot[warp] = pc;
    __syncthreads();
    int npos = 0;
    for (int w = 0; w < kFitThreads / 32; ++w) npos += warp_tot[w];
    const double mean = (double)npos / (double)m;
    if (tid == 0) {
      o_feature[base + node] = -1;
      o_threshold[base + node] = 0.0;
      o_left[base + node] = -1;
      o_right[base + node] = -1;
      o_value[base + node] = mean;
    }
    if (cur.depth >= max_depth || m < 2 || mean == 0.0 || mean == 1.0) continue;  // leaf
    const int d = s_draw;
    __syncthreads();
    if (tid == 0) {
      s_draw = d + 1;
      if (d >= n_drawn[t] || d >= max_draws) s_status = 1;  // more feature subsets needed
      s_best_f = -1;
      s_best_score = INFINITY;
    }
    __syncthreads();
    if (s_status) break;
    int np = 1;
    while (np < m) np <<= 1;
    for (int j = 0; j < k; ++j) {
      const int f = feats[((size_t)t * max_draws + d) * k + j];
      for (int i = tid; i < np; i += blockDim.x) {
        key[i] = i < m ? X[(size_t)rows[s + i] * F + f] : INFINITY;
        idx[i] = i < m ? i : (1 << 30) + i;
      }
      bitonic(key, idx, np);
      // positives among sorted[0..i]
      for (int i = tid; i < m; i += blockDim.x) cnt[i] = y[rows[s + idx[i]]] > 0.5 ? 1 : 0;
      __syncthreads();
      block_scan(cnt, m, warp_tot);
      const double total = (double)cnt[m - 1];
      // weighted Gini of every cut between distinct values; first minimum
      double bs = INFINITY;
      int bi = 1 << 30;
      for (int i = tid; i < m - 1; i += blockDim.x) {
        if (!(key[i] != key[i + 1])) continue;
        const double nl = (double)(i + 1), nr = (double)(m - 1 - i);
        const double pl = (double)cnt[i], pr = __dsub_rn(total, pl);
        const double a = __ddiv_rn(pl, nl), b = __ddiv_rn(__dsub_rn(nl, pl), nl);
        const double gl = __dsub_rn(__dsub_rn(1.0, __dmul_rn(a, a)), __dmul_rn(b, b));
        const double c = __ddiv_rn(pr, nr), dd = __ddiv_rn(__dsub_rn(nr, pr), nr);
        const double gr = __dsub_rn(__dsub_rn(1.0, __dmul_rn(c, c)), __dmul_rn(dd, dd));
        const double sc = __ddiv_rn(__dadd_rn(__dmul_rn(nl, gl), __dmul_rn(nr, gr)), (double)m);
        if (sc < bs || (sc == bs && i < bi)) {
          bs = sc;
          bi = i;
        }
      }
      for (int o = 16; o; o >>= 1) {
        const double os = __shfl_xor_sync(0xffffffffu, bs, o);
        const int oi = __shfl_xor_sync(0xffffffffu, bi, o);
        if (os < bs || (os == bs && oi < bi)) {
          bs = os;
          bi = oi;
        }
      }
      if (lane == 0) {
        red_s[warp] = bs;
        red_i[warp] = bi;
      }
      __syncthreads();
      if (tid == 0) {
        for (int w = 1; w < kFitThreads / 32; ++w)
          if (red_s[w] < bs || (red_s[w] == bs && red_i[w] < bi)) {
            bs = red_s[w];
            bi = red_i[w];
          }
        if (bi < (1 << 30) && (s_best_f < 0 || bs < s_best_score)) {  // feasibility.py:143
          s_best_score = bs;
          s_best_f = f;
          s_best_thr = __dmul_rn(0.5, __dadd_rn(key[bi], key[bi + 1]));
          s_best_cut_i = bi;
        }
      }
      __syncthreads();
    }
    if (s_best_f < 0) continue;  // no cut in any drawn feature: a leaf (the subset was still drawn)
    const int bf = s_best_f;
    const double thr = s_best_thr;
    // stable partition of the node's rows: x <= thr first (rows[left_mask], then rows[~left_mask])
    for (int i = tid; i < m; i += blockDim.x) cnt[i] = X[(size_t)rows[s + i] * F + bf] <= thr ? 1 : 0;
    __syncthreads();
    block_scan(cnt, m, warp_tot);
    const int nleft = cnt[m - 1];
    for (int i = tid; i < m; i += blockDim.x) {
      const bool lft = X[(size_t)rows[s + i] * F + bf] <= thr;
      const int before = i > 0 ? cnt[i - 1] : 0;
      tmp[lft ? before : nleft + (i - before)] = rows[s + i];
    }
    __syncthreads();
    for (int i = tid; i < m; i += blockDim.x) rows[s + i] = tmp[i];
    if (tid == 0) {
      o_feature[base + node] = bf;
      o_threshold[base + node] = thr;
      o_left[base + node] = node + 1;  // the left child is created next (preorder)
      stack[s_sp] = FitStack{s + nleft, e, cur.depth + 1, node};  // right, after the left subtree
      stack[s_sp + 1] = FitStack{s, s + nleft, cur.depth + 1, -1};
      s_sp += 2;
      if (s_sp + 2 > max_nodes) s_status = 2;
    }
  }
  __syncthreads();
  if (tid == 0) {
    o_n_nodes[t] = s_n_nodes;
    o_status[t] = s_status;
  }
}

}  // namespace

size_t rf_fit_smem_bytes(int n) {
  int p = 1;
  while (p < n) p <<= 1;
  return (size_t)p * 12 + (size_t)n * 12 + 16;
}

cudaError_t launch_rf_fit(const double* X, const double* y, int n, int F, int T, const int32_t* boot,
                          const int32_t* feats, const int32_t* n_drawn, int max_draws, int k, int max_depth,
                          int max_nodes, int32_t* feature, double* threshold, int32_t* left, int32_t* right,
                          double* value, int32_t* n_nodes, int32_t* status, void* stack, cudaStream_t s) {
  const size_t bytes = rf_fit_smem_bytes(n);
  cudaError_t e = set_smem(rf_fit_kernel, (int)bytes);
  if (e != cudaSuccess) return e;
  rf_fit_kernel<<<T, kFitThreads, bytes, s>>>(X, y, n, F, boot, feats, n_drawn, max_draws, k, max_depth, max_nodes,
                                                feature, threshold, left, right, value, n_nodes, status,
                                                reinterpret_cast<FitStack*>(stack));
  return cudaGetLastError();
}

size_t rf_fit_stack_bytes(int T, int max_nodes) { return (size_t)T * max_nodes * sizeof(FitStack); }

}  // namespace bx
