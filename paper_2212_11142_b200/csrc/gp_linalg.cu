// gp_linalg.cu — once-per-iteration GP state and the batched coarse marginal likelihood.
//
//   gp_planes_kernel     training planes for the cross-covariance (surrogate.py:163-218)
//   tri_inverse_kernel   L^-1 by column forward substitution (the TRSM of surrogate.py:323 done once)
//   pairwise_sq_kernel   pairwise_sq_distances (surrogate.py:173-198), bit-exact
//   lml_kernel           _batched_coarse_lml (surrogate.py:420-456): one CTA per hyperparameter
//                        candidate, Gram build + right-looking Cholesky in shared memory (packed
//                        lower triangle) or in an L2-resident global scratch when n is large,
//                        -inf when a pivot is not positive (LAPACK potrf info > 0).
#include "bx_common.cuh"

namespace bx {

namespace {

__global__ void gp_planes_kernel(SpaceDev sp, const uint32_t* train, int n, const double* inv_l,
                                 uint64_t* planes, uint64_t* kmask) {
  const int64_t total = (int64_t)sp.n_params * n;
  for (int64_t t = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; t < total;
       t += (int64_t)gridDim.x * blockDim.x) {
    const int k = (int)(t / n), j = (int)(t % n);
    const bx_param_desc& p = sp.params[k];
    const uint32_t* row = train + (size_t)j * sp.row_words;
    uint64_t v;
    if (p.kind == BX_PERMUTATION) {
      v = row_u64(row, p.word);
      uint64_t lo = 0, hi = 0;
      if (p.metric == BX_KENDALL) kendall_mask(v, p.size, lo, hi);
      kmask[((size_t)k * n + j) * 2] = lo;
      kmask[((size_t)k * n + j) * 2 + 1] = hi;
    } else if (p.kind == BX_CATEGORICAL) {
      v = row[p.word];
    } else {
      v = (uint64_t)__double_as_longlong(row_coord(p, sp.coord_lut, row) * inv_l[k]);
    }
    planes[(size_t)k * n + j] = v;
  }
}

// One warp per column j of L^-1: x_i = -(sum_{k=j}^{i-1} L_ik x_k) / L_ii, the dot product split
// across the lanes and reduced with shuffles; the column lives in shared memory.
constexpr int kInvWarps = 8;
__global__ void __launch_bounds__(kInvWarps * 32) tri_inverse_kernel(const double* L, int n, double* A, int lda) {
  extern __shared__ double xcol[];  // [warps][n]
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int j = blockIdx.x * (blockDim.x >> 5) + warp;
  if (j >= n) return;
  double* x = xcol + (size_t)warp * n;
  if (lane == 0) x[j] = 1.0 / L[(size_t)j * n + j];
  __syncwarp();
  for (int i = j + 1; i < n; ++i) {
    const double* Li = L + (size_t)i * n;
    double s = 0.0;
    for (int k = j + lane; k < i; k += 32) s = fma(Li[k], x[k], s);
#pragma unroll
    for (int off = 16; off; off >>= 1) s += __shfl_xor_sync(0xffffffffu, s, off);
    if (lane == 0) x[i] = -s / Li[i];
    __syncwarp();
  }
  for (int i = j + lane; i < n; i += 32) A[(size_t)i * lda + j] = x[i];
}

__global__ void pairwise_sq_kernel(SpaceDev sp, const uint32_t* a, int qa, const uint32_t* b, int qb,
                                   double* out) {
  const int64_t total = (int64_t)qa * qb;
  for (int64_t t = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; t < total;
       t += (int64_t)gridDim.x * blockDim.x) {
    const int ia = (int)(t / qb), ib = (int)(t % qb);
    const uint32_t* ra = a + (size_t)ia * sp.row_words;
    const uint32_t* rb = b + (size_t)ib * sp.row_words;
    for (int k = 0; k < sp.n_params; ++k) {
      const bx_param_desc& p = sp.params[k];
      double v;
      if (p.kind == BX_CATEGORICAL) {
        v = ra[p.word] != rb[p.word] ? 1.0 : 0.0;  // surrogate.py:193
      } else if (p.kind == BX_PERMUTATION) {
        const uint64_t x = row_u64(ra, p.word), y = row_u64(rb, p.word);
        uint64_t xl = 0, xh = 0, yl = 0, yh = 0;
        if (p.metric == BX_KENDALL) {
          kendall_mask(x, p.size, xl, xh);
          kendall_mask(y, p.size, yl, yh);
        }
        const int raw = perm_raw(p.metric, p.size, x, y, xl, xh, yl, yh);
        v = __ddiv_rn((double)raw, p.raw_mx);  // surrogate.py:218
      } else {
        const double d = __dsub_rn(row_coord(p, sp.coord_lut, ra), row_coord(p, sp.coord_lut, rb));
        v = __dmul_rn(d, d);  // surrogate.py:187-188
      }
      out[((size_t)k * qa + ia) * qb + ib] = v;
    }
  }
}

__device__ __forceinline__ size_t tri_idx(int i, int k) { return (size_t)i * (i + 1) / 2 + k; }

constexpr int kLmlThreads = 256;

// One CTA per hyperparameter candidate.
__global__ void __launch_bounds__(kLmlThreads) lml_kernel(const double* sq, int n, int D,
                                                          const double* z, const double* thetas,
                                                          double* out, double* scratch,
                                                          int use_smem) {
  extern __shared__ __align__(16) unsigned char smem_raw[];
  const int c = blockIdx.x;
  const int tid = threadIdx.x;
  const size_t tri = (size_t)n * (n + 1) / 2;
  double* K = use_smem ? reinterpret_cast<double*>(smem_raw) : scratch + (size_t)c * (tri + n);
  double* u = use_smem ? K + tri : scratch + (size_t)c * (tri + n) + tri;
  __shared__ double inv_sq[BX_MAX_PARAMS];
  __shared__ double red[kLmlThreads / 32];
  __shared__ int failed;
  const double* th = thetas + (size_t)c * (2 + D);
  const double sigma = exp(th[0]);
  const double noise = fmax(exp(th[1]), 1e-6);  // NOISE_FLOOR
  for (int k = tid; k < D; k += blockDim.x) inv_sq[k] = exp(-2.0 * th[2 + k]);
  if (tid == 0) failed = 0;
  __syncthreads();

  // Gram (lower triangle): sigma * (1 + sqrt5 d + 5/3 W) * exp(-sqrt5 d)   (surrogate.py:430-434)
  for (size_t t = tid; t < tri; t += blockDim.x) {
    int i = (int)((sqrt(8.0 * (double)t + 1.0) - 1.0) * 0.5);
    while (tri_idx(i + 1, 0) <= t) ++i;
    while (tri_idx(i, 0) > t) --i;
    const int k2 = (int)(t - tri_idx(i, 0));
    double W = 0.0;
    for (int k = 0; k < D; ++k) W = fma(sq[((size_t)k * n + i) * n + k2], inv_sq[k], W);
    const double d = sqrt(fmax(W, 0.0));
    double v = sigma * (1.0 + kSqrt5 * d + (5.0 / 3.0) * W) * exp(-kSqrt5 * d);
    if (i == k2) v += noise + 1e-9;  // JITTER
    K[t] = v;
  }
  for (int i = tid; i < n; i += blockDim.x) u[i] = z[i];
  __syncthreads();

  // right-looking Cholesky, lower
  for (int j = 0; j < n; ++j) {
    const double piv = K[tri_idx(j, j)];
    if (!(piv > 0.0)) {  // potrf: ajj <= 0 or NaN -> info > 0
      if (tid == 0) failed = 1;
      break;
    }
    const double ljj = sqrt(piv);
    __syncthreads();
    if (tid == 0) K[tri_idx(j, j)] = ljj;
    for (int i = j + 1 + tid; i < n; i += blockDim.x) K[tri_idx(i, j)] /= ljj;
    __syncthreads();
    const int m = n - j - 1;  // trailing size
    const size_t work = (size_t)m * (m + 1) / 2;
    for (size_t t = tid; t < work; t += blockDim.x) {
      int r = (int)((sqrt(8.0 * (double)t + 1.0) - 1.0) * 0.5);
      while (tri_idx(r + 1, 0) <= t) ++r;
      while (tri_idx(r, 0) > t) --r;
      const int cc = (int)(t - tri_idx(r, 0));
      const int i = j + 1 + r, k = j + 1 + cc;
      K[tri_idx(i, k)] -= K[tri_idx(i, j)] * K[tri_idx(k, j)];
    }
    __syncthreads();
  }
  __syncthreads();
  if (failed) {
    if (tid == 0) out[c] = -INFINITY;
    return;
  }
  // u = L^-1 z (column sweep)
  for (int j = 0; j < n; ++j) {
    __syncthreads();
    const double uj = u[j] / K[tri_idx(j, j)];
    __syncthreads();
    if (tid == 0) u[j] = uj;
    for (int i = j + 1 + tid; i < n; i += blockDim.x) u[i] -= K[tri_idx(i, j)] * uj;
  }
  __syncthreads();
  double quad = 0.0, logdet = 0.0;
  for (int i = tid; i < n; i += blockDim.x) {
    quad = fma(u[i], u[i], quad);
    logdet += log(K[tri_idx(i, i)]);
  }
  for (int off = 16; off; off >>= 1) {
    quad += __shfl_xor_sync(0xffffffffu, quad, off);
    logdet += __shfl_xor_sync(0xffffffffu, logdet, off);
  }
  __shared__ double red2[kLmlThreads / 32];
  if ((tid & 31) == 0) { red[tid >> 5] = quad; red2[tid >> 5] = logdet; }
  __syncthreads();
  if (tid == 0) {
    double q = 0.0, l = 0.0;
    for (int w = 0; w < kLmlThreads / 32; ++w) { q += red[w]; l += red2[w]; }
    // surrogate.py:453-455
    out[c] = -0.5 * q - 0.5 * (2.0 * l) - 0.5 * n * log(2.0 * 3.14159265358979323846);
  }
}

// ---- _lml_core with gradient (surrogate.py:356-400), one CTA per hyperparameter setting ------
// params row: (sigma, noise, l_1 .. l_D) in natural units, as _lml_core receives them.
// Scratch per CTA: K (n x n), L (n x n), X = L^-1 (n x n), u, alpha (n).
constexpr int kGradThreads = 256;

__device__ __forceinline__ double block_sum(double v, double* red) {
  for (int off = 16; off; off >>= 1) v += __shfl_xor_sync(0xffffffffu, v, off);
  __syncthreads();
  if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = v;
  __syncthreads();
  double s = 0.0;
  for (int w = 0; w < (int)(blockDim.x >> 5); ++w) s += red[w];
  return s;
}

__global__ void __launch_bounds__(kGradThreads) lml_grad_kernel(const double* sq, int n, int D,
                                                                const double* z, const double* prm,
                                                                double prior_k, double prior_rate,
                                                                int use_prior, int want_grad,
                                                                double* out_value, double* out_grad,
                                                                int* out_ok, double* scratch) {
  const int c = blockIdx.x, tid = threadIdx.x;
  const size_t nn = (size_t)n * n;
  double* K = scratch + (size_t)c * (3 * nn + 2 * n);
  double* L = K + nn;
  double* X = L + nn;
  double* u = X + nn;
  double* al = u + n;
  __shared__ double inv_l2[BX_MAX_PARAMS];
  __shared__ double red[kGradThreads / 32];
  __shared__ int failed;
  const double* p = prm + (size_t)c * (2 + D);
  const double sigma = p[0];
  const double noise = fmax(p[1], 1e-6);  // NOISE_FLOOR
  for (int k = tid; k < D; k += blockDim.x) inv_l2[k] = 1.0 / (p[2 + k] * p[2 + k]);
  if (tid == 0) failed = 0;
  __syncthreads();
  // K and Ky = K + (noise + jitter) I  (surrogate.py:365-371)
  for (size_t t = tid; t < nn; t += blockDim.x) {
    const int i = (int)(t / n), j = (int)(t % n);
    double W = 0.0;
    for (int k = 0; k < D; ++k) W = fma(sq[(size_t)k * nn + t], inv_l2[k], W);
    const double d = sqrt(fmax(W, 0.0));
    const double E = exp(-kSqrt5 * d);
    const double kv = sigma * ((1.0 + kSqrt5 * d + (5.0 / 3.0) * W) * E);
    K[t] = kv;
    L[t] = (i == j) ? kv + noise + 1e-9 : kv;
  }
  __syncthreads();
  // right-looking Cholesky on the lower triangle of L
  for (int j = 0; j < n; ++j) {
    const double piv = L[(size_t)j * n + j];
    if (!(piv > 0.0)) {
      if (tid == 0) failed = 1;
      break;
    }
    const double ljj = sqrt(piv);
    __syncthreads();
    if (tid == 0) L[(size_t)j * n + j] = ljj;
    for (int i = j + 1 + tid; i < n; i += blockDim.x) L[(size_t)i * n + j] /= ljj;
    __syncthreads();
    const int m = n - j - 1;
    for (int t = tid; t < m * m; t += blockDim.x) {
      const int i = j + 1 + t / m, k = j + 1 + t % m;
      if (k <= i) L[(size_t)i * n + k] -= L[(size_t)i * n + j] * L[(size_t)k * n + j];
    }
    __syncthreads();
  }
  __syncthreads();
  if (failed) {
    if (tid == 0) {
      out_ok[c] = 0;
      out_value[c] = -INFINITY;
    }
    if (want_grad)
      for (int k = tid; k < 2 + D; k += blockDim.x) out_grad[(size_t)c * (2 + D) + k] = 0.0;
    return;
  }
  // u = L^-1 z, alpha = L^-T u (the two TRTRS calls, surrogate.py:373-374)
  for (int i = tid; i < n; i += blockDim.x) u[i] = z[i];
  for (int j = 0; j < n; ++j) {
    __syncthreads();
    const double uj = u[j] / L[(size_t)j * n + j];
    __syncthreads();
    if (tid == 0) u[j] = uj;
    for (int i = j + 1 + tid; i < n; i += blockDim.x) u[i] -= L[(size_t)i * n + j] * uj;
  }
  __syncthreads();
  for (int i = tid; i < n; i += blockDim.x) al[i] = u[i];
  for (int j = n - 1; j >= 0; --j) {
    __syncthreads();
    const double aj = al[j] / L[(size_t)j * n + j];
    __syncthreads();
    if (tid == 0) al[j] = aj;
    for (int i = tid; i < j; i += blockDim.x) al[i] -= L[(size_t)j * n + i] * aj;
  }
  __syncthreads();
  double za = 0.0, ld = 0.0;
  for (int i = tid; i < n; i += blockDim.x) {
    za = fma(z[i], al[i], za);
    ld += log(L[(size_t)i * n + i]);
  }
  za = block_sum(za, red);
  ld = block_sum(ld, red);
  double value = -0.5 * za - ld - 0.5 * n * log(2.0 * 3.14159265358979323846);
  if (use_prior) {  // Gamma(k, rate) log density per lengthscale (surrogate.py:380-383)
    double sl = 0.0, sll = 0.0;
    for (int k = 0; k < D; ++k) {
      sl += p[2 + k];
      sll += log(p[2 + k]);
    }
    value += D * (prior_k * log(prior_rate) - lgamma(prior_k)) + (prior_k - 1.0) * sll - prior_rate * sl;
  }
  if (tid == 0) {
    out_ok[c] = 1;
    out_value[c] = value;
  }
  if (!want_grad) return;
  // X = L^-1, one column per thread (forward substitution)
  for (int j = tid; j < n; j += blockDim.x) {
    for (int i = 0; i < j; ++i) X[(size_t)i * n + j] = 0.0;
    X[(size_t)j * n + j] = 1.0 / L[(size_t)j * n + j];
    for (int i = j + 1; i < n; ++i) {
      double s = 0.0;
      for (int k = j; k < i; ++k) s = fma(L[(size_t)i * n + k], X[(size_t)k * n + j], s);
      X[(size_t)i * n + j] = -s / L[(size_t)i * n + i];
    }
  }
  __syncthreads();
  // M = alpha alpha^T - X^T X; gradient sums (surrogate.py:386-399)
  double g0 = 0.0, g1 = 0.0;
  double gl[BX_MAX_PARAMS];
  for (int k = 0; k < D; ++k) gl[k] = 0.0;
  for (size_t t = tid; t < nn; t += blockDim.x) {
    const int a = (int)(t / n), b = (int)(t % n);
    const int k0 = a > b ? a : b;
    double kinv = 0.0;
    for (int k = k0; k < n; ++k) kinv = fma(X[(size_t)k * n + a], X[(size_t)k * n + b], kinv);
    const double M = al[a] * al[b] - kinv;
    g0 = fma(M, K[t], g0);
    if (a == b) g1 += M;
    double W = 0.0;
    for (int k = 0; k < D; ++k) W = fma(sq[(size_t)k * nn + t], inv_l2[k], W);
    const double d = sqrt(fmax(W, 0.0));
    const double MG = M * ((1.0 + kSqrt5 * d) * exp(-kSqrt5 * d));
    for (int k = 0; k < D; ++k) gl[k] = fma(MG, sq[(size_t)k * nn + t], gl[k]);
  }
  g0 = block_sum(g0, red);
  g1 = block_sum(g1, red);
  double* g = out_grad + (size_t)c * (2 + D);
  if (tid == 0) {
    g[0] = 0.5 * g0;
    g[1] = 0.5 * noise * g1;
  }
  const double scale = (5.0 / 6.0) * sigma;
  for (int k = 0; k < D; ++k) {
    const double s = block_sum(gl[k], red);
    if (tid == 0) {
      const double l = p[2 + k];
      double gk = (scale / (l * l)) * s;
      if (use_prior) gk += (prior_k - 1.0) - prior_rate * l;
      g[2 + k] = gk;
    }
  }
}

// ---- _lml_core for small n: one CTA per setting, everything in shared memory ---------------------
// The lower triangle of Ky (packed, row-major: (i, k) at i (i + 1) / 2 + k) is factored in place
// (right-looking, a warp per row of the trailing update), u = L^-1 z and alpha = L^-T u are one
// warp's forward / backward sweeps, L is inverted in place (X = L^-1, columns from the last: X_ij =
// -(sum_{k=j+1..i} X_ik L_kj) / L_jj with column j of L saved first), and the gradient sums take
// K^-1_ab = sum_{k >= a} X_ka X_kb per lower entry (a thread per entry).  Same formulas and
// operation order within each entry as lml_grad_kernel (surrogate.py:356-400); a setting's
// arithmetic does not depend on the batch.  n <= kSmallLmlMaxN (the triangle plus three vectors fit
// in 227 KB); launch latency and block-wide steps instead of global-memory round trips.
constexpr int kSmallThreads = 512;
constexpr int kSmallLmlMaxN = 232;

// u = L^-1 z and alpha = L^-T u (the two TRTRS calls, surrogate.py:373-374) by one warp as column
// sweeps: lane l keeps the running sums of rows l, l + 32, ... (R register slots) in registers;
// each step the owner of row i finishes it and broadcasts the solved entry, every lane folds it
// into its rows (one division, one shuffle and one FMA per step instead of a five-level reduction
// per row).  R is the smallest power of two >= ceil(n / 32): the per-step bookkeeping is R wide.
template <int R>
__device__ __forceinline__ void small_sweeps(int n, const double* z, const double* Lp, double* u, double* al,
                                             int lane) {
  double acc[R], zr[R];
#pragma unroll
  for (int m = 0; m < R; ++m) {
    acc[m] = 0.0;
    zr[m] = lane + 32 * m < n ? z[lane + 32 * m] : 0.0;  // z out of the step chain (global memory)
  }
  for (int i = 0; i < n; ++i) {
    double ui = 0.0;
#pragma unroll
    for (int m = 0; m < R; ++m)
      if (lane + 32 * m == i) ui = (zr[m] - acc[m]) / Lp[tri_idx(i, i)];
    ui = __shfl_sync(0xffffffffu, ui, i & 31);
    if (lane == (i & 31)) u[i] = ui;
#pragma unroll
    for (int m = 0; m < R; ++m) {
      const int k = lane + 32 * m;
      if (k > i && k < n) acc[m] = fma(Lp[tri_idx(k, i)], ui, acc[m]);
    }
  }
#pragma unroll
  for (int m = 0; m < R; ++m) acc[m] = 0.0;
  __syncwarp();
  for (int i = n - 1; i >= 0; --i) {
    double ai = 0.0;
#pragma unroll
    for (int m = 0; m < R; ++m)
      if (lane + 32 * m == i) ai = (u[i] - acc[m]) / Lp[tri_idx(i, i)];
    ai = __shfl_sync(0xffffffffu, ai, i & 31);
    if (lane == (i & 31)) al[i] = ai;
    const size_t r0 = tri_idx(i, 0);
#pragma unroll
    for (int m = 0; m < R; ++m) {
      const int j = lane + 32 * m;
      if (j < i) acc[m] = fma(Lp[r0 + j], ai, acc[m]);
    }
  }
}

__global__ void __launch_bounds__(kSmallThreads) lml_small_kernel(const double* sq, int n, int D, const double* z,
                                                                  const double* prm, double prior_k, double prior_rate,
                                                                  int use_prior, int want_grad, double* out_value,
                                                                  double* out_grad, int* out_ok, int sep_x) {
  extern __shared__ __align__(16) double sm[];
  const int c = blockIdx.x, tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  constexpr int kWarps = kSmallThreads / 32;
  const size_t tri = (size_t)n * (n + 1) / 2, nn = (size_t)n * n;
  double* Lp = sm;            // [tri]
  double* u = Lp + tri;       // [n]
  double* al = u + n;         // [n]
  double* col = al + n;       // [n] column j of L while it is inverted in place
  double* Xs = col + n;       // [tri] X = L^-1 beside L when sep_x (launch_lml_small)
  __shared__ double inv_l2[BX_MAX_PARAMS];
  __shared__ double red[kWarps];
  __shared__ int failed;
  const double* p = prm + (size_t)c * (2 + D);
  const double sigma = p[0];
  const double noise = fmax(p[1], 1e-6);  // NOISE_FLOOR
  for (int k = tid; k < D; k += blockDim.x) inv_l2[k] = 1.0 / (p[2 + k] * p[2 + k]);
  if (tid == 0) failed = 0;
  __syncthreads();
  // Ky lower triangle (surrogate.py:365-371); a warp per row: contiguous packed entries
  for (int i = warp; i < n; i += kWarps) {
    const size_t r0 = tri_idx(i, 0);
    for (int k2 = lane; k2 <= i; k2 += 32) {
      const size_t t = (size_t)i * n + k2;
      double W = 0.0;
      for (int k = 0; k < D; ++k) W = fma(sq[(size_t)k * nn + t], inv_l2[k], W);
      const double d = sqrt(fmax(W, 0.0));
      const double E = exp(-kSqrt5 * d);
      const double kv = sigma * ((1.0 + kSqrt5 * d + (5.0 / 3.0) * W) * E);
      Lp[r0 + k2] = (i == k2) ? kv + noise + 1e-9 : kv;
    }
  }
  __syncthreads();
  // right-looking Cholesky
  for (int j = 0; j < n; ++j) {
    const double piv = Lp[tri_idx(j, j)];
    if (!(piv > 0.0)) {  // potrf: a_jj <= 0 or NaN (uniform: every thread reads the same value)
      if (tid == 0) failed = 1;
      break;
    }
    const double ljj = sqrt(piv);
    for (int i = j + 1 + tid; i < n; i += blockDim.x) col[i] = Lp[tri_idx(i, j)] / ljj;
    __syncthreads();
    if (tid == 0) Lp[tri_idx(j, j)] = ljj;
    for (int i = j + 1 + warp; i < n; i += kWarps) {
      const size_t r0 = tri_idx(i, 0);
      const double ci = col[i];
      if (lane == 0) Lp[r0 + j] = ci;
      for (int k = j + 1 + lane; k <= i; k += 32) Lp[r0 + k] -= ci * col[k];
    }
    __syncthreads();
  }
  __syncthreads();
  if (failed) {
    if (tid == 0) {
      out_ok[c] = 0;
      out_value[c] = -INFINITY;
    }
    if (want_grad)
      for (int k = tid; k < 2 + D; k += blockDim.x) out_grad[(size_t)c * (2 + D) + k] = 0.0;
    return;
  }
  // u = L^-1 z and alpha = L^-T u: warp 0 (small_sweeps)
  if (warp == 0) {
    const int rpl = (n + 31) >> 5;  // rows per lane: the fewest register slots that cover n
    if (rpl <= 1) small_sweeps<1>(n, z, Lp, u, al, lane);
    else if (rpl <= 2) small_sweeps<2>(n, z, Lp, u, al, lane);
    else if (rpl <= 4) small_sweeps<4>(n, z, Lp, u, al, lane);
    else small_sweeps<8>(n, z, Lp, u, al, lane);
  }
  __syncthreads();
  double za = 0.0, ld = 0.0;
  for (int i = tid; i < n; i += blockDim.x) {
    za = fma(z[i], al[i], za);
    ld += log(Lp[tri_idx(i, i)]);
  }
  za = block_sum(za, red);
  ld = block_sum(ld, red);
  double value = -0.5 * za - ld - 0.5 * n * log(2.0 * 3.14159265358979323846);
  if (use_prior) {  // Gamma(k, rate) log density per lengthscale (surrogate.py:380-383)
    double sl = 0.0, sll = 0.0;
    for (int k = 0; k < D; ++k) {
      sl += p[2 + k];
      sll += log(p[2 + k]);
    }
    value += D * (prior_k * log(prior_rate) - lgamma(prior_k)) + (prior_k - 1.0) * sll - prior_rate * sl;
  }
  if (tid == 0) {
    out_ok[c] = 1;
    out_value[c] = value;
  }
  if (!want_grad) return;
  // X = L^-1: X_ii = 1 / L_ii, X_ij = -(sum_{k=j+1..i} X_ik L_kj) / L_jj for j < i
  const double* X = Lp;
  if (sep_x) {
    // beside L (which stays intact): a row needs only its own entries and L, so each warp runs its
    // rows from the diagonal leftwards with no block-wide step - the same sums in the same order
    // as the in-place sweep below, hence the same bits
    for (int i = warp; i < n; i += kWarps) {
      const size_t r0 = tri_idx(i, 0);
      if (lane == 0) Xs[r0 + i] = 1.0 / Lp[r0 + i];
      __syncwarp();
      for (int j = i - 1; j >= 0; --j) {
        const double xjj = 1.0 / Lp[tri_idx(j, j)];
        double s = 0.0;
        for (int k = j + 1 + lane; k <= i; k += 32) s = fma(Xs[r0 + k], Lp[tri_idx(k, j)], s);
        for (int off = 16; off; off >>= 1) s += __shfl_xor_sync(0xffffffffu, s, off);
        if (lane == 0) Xs[r0 + j] = -s * xjj;
        __syncwarp();
      }
    }
    X = Xs;
  } else {
    // in place, last column first (column j of L saved before its rows are overwritten)
    for (int j = n - 1; j >= 0; --j) {
      for (int i = j + 1 + tid; i < n; i += blockDim.x) col[i] = Lp[tri_idx(i, j)];
      __syncthreads();
      const double xjj = 1.0 / Lp[tri_idx(j, j)];
      for (int i = j + 1 + warp; i < n; i += kWarps) {
        const size_t r0 = tri_idx(i, 0);
        double s = 0.0;
        for (int k = j + 1 + lane; k <= i; k += 32) s = fma(Lp[r0 + k], col[k], s);
        for (int off = 16; off; off >>= 1) s += __shfl_xor_sync(0xffffffffu, s, off);
        if (lane == 0) Lp[r0 + j] = -s * xjj;
      }
      __syncthreads();
      if (tid == 0) Lp[tri_idx(j, j)] = xjj;
    }
  }
  __syncthreads();
  // M = alpha alpha^T - X^T X; gradient sums over the full matrix (symmetric: off-diagonal lower
  // entries counted twice) (surrogate.py:386-399)
  double g0 = 0.0, g1 = 0.0;
  double gl[BX_MAX_PARAMS];
  for (int k = 0; k < D; ++k) gl[k] = 0.0;
  for (size_t t = tid; t < tri; t += blockDim.x) {
    int a = (int)((sqrt(8.0 * (double)t + 1.0) - 1.0) * 0.5);
    while (tri_idx(a + 1, 0) <= t) ++a;
    while (tri_idx(a, 0) > t) --a;
    const int b = (int)(t - tri_idx(a, 0));  // a >= b
    double kinv = 0.0;
    for (int k = a; k < n; ++k) kinv = fma(X[tri_idx(k, a)], X[tri_idx(k, b)], kinv);
    const double M = al[a] * al[b] - kinv;
    const double w = a == b ? 1.0 : 2.0;
    const size_t e = (size_t)a * n + b;
    double W = 0.0;
    for (int k = 0; k < D; ++k) W = fma(sq[(size_t)k * nn + e], inv_l2[k], W);
    const double d = sqrt(fmax(W, 0.0));
    const double E = exp(-kSqrt5 * d);
    const double kv = sigma * ((1.0 + kSqrt5 * d + (5.0 / 3.0) * W) * E);
    g0 = fma(w * M, kv, g0);
    if (a == b) g1 += M;
    const double MG = w * M * ((1.0 + kSqrt5 * d) * E);
    for (int k = 0; k < D; ++k) gl[k] = fma(MG, sq[(size_t)k * nn + e], gl[k]);
  }
  // the 2 + D block sums in one pass: each warp's xor-reduced partial per quantity, then thread 0
  // adds the warps in order (block_sum's arithmetic, one barrier instead of 2 (2 + D))
  __shared__ double red_all[BX_MAX_PARAMS + 2][kWarps];
  for (int q = 0; q < 2 + D; ++q) {
    double v = q == 0 ? g0 : (q == 1 ? g1 : gl[q - 2]);
    for (int off = 16; off; off >>= 1) v += __shfl_xor_sync(0xffffffffu, v, off);
    if (lane == 0) red_all[q][warp] = v;
  }
  __syncthreads();
  if (tid == 0) {
    double tot[BX_MAX_PARAMS + 2];
    for (int q = 0; q < 2 + D; ++q) {
      double s = 0.0;
      for (int w = 0; w < kWarps; ++w) s += red_all[q][w];
      tot[q] = s;
    }
    double* g = out_grad + (size_t)c * (2 + D);
    g[0] = 0.5 * tot[0];
    g[1] = 0.5 * noise * tot[1];
    const double scale = (5.0 / 6.0) * sigma;
    for (int k = 0; k < D; ++k) {
      const double l = p[2 + k];
      double gk = (scale / (l * l)) * tot[2 + k];
      if (use_prior) gk += (prior_k - 1.0) - prior_rate * l;
      g[2 + k] = gk;
    }
  }
}

int grid_for(int64_t work, int threads) {
  int64_t b = (work + threads - 1) / threads;
  if (b > 148 * 16) b = 148 * 16;
  if (b < 1) b = 1;
  return (int)b;
}

}  // namespace

size_t lml_scratch_doubles(int n, int c) { return (size_t)c * ((size_t)n * (n + 1) / 2 + n); }

size_t lml_grad_scratch_doubles(int n, int c) { return (size_t)c * (3 * (size_t)n * n + 2 * (size_t)n); }

cudaError_t launch_lml_grad(const double* sq, int n, int D, const double* z, const double* prm,
                            int c, double prior_k, double prior_rate, int use_prior, int want_grad,
                            double* out_value, double* out_grad, int* out_ok, double* scratch,
                            cudaStream_t s) {
  if (c <= 0) return cudaSuccess;
  lml_grad_kernel<<<c, kGradThreads, 0, s>>>(sq, n, D, z, prm, prior_k, prior_rate, use_prior,
                                              want_grad, out_value, out_grad, out_ok, scratch);
  return cudaGetLastError();
}

bool lml_small_supported(int n) { return n >= 1 && n <= kSmallLmlMaxN; }

cudaError_t launch_lml_small(const double* sq, int n, int D, const double* z, const double* prm, int c,
                             double prior_k, double prior_rate, int use_prior, int want_grad, double* out_value,
                             double* out_grad, int* out_ok, cudaStream_t s) {
  if (c <= 0) return cudaSuccess;
  if (!lml_small_supported(n)) return cudaErrorInvalidValue;
  const size_t tri = (size_t)n * (n + 1) / 2;
  // X = L^-1 beside L (warp-per-row inverse, no block barriers) when both triangles fit
  const int sep_x = want_grad && (2 * tri + 3 * (size_t)n) * sizeof(double) <= 200 * 1024 ? 1 : 0;
  const size_t bytes = ((sep_x ? 2 : 1) * tri + 3 * (size_t)n) * sizeof(double);
  cudaError_t e = set_smem(lml_small_kernel, (int)bytes);
  if (e != cudaSuccess) return e;
  lml_small_kernel<<<c, kSmallThreads, bytes, s>>>(sq, n, D, z, prm, prior_k, prior_rate, use_prior, want_grad,
                                                   out_value, out_grad, out_ok, sep_x);
  return cudaGetLastError();
}

cudaError_t launch_lml(const double* sq, int n, int D, const double* z, const double* thetas, int c,
                       double* out, double* scratch, cudaStream_t s) {
  if (c <= 0) return cudaSuccess;
  const size_t bytes = ((size_t)n * (n + 1) / 2 + n) * sizeof(double);
  const int use_smem = bytes <= 200 * 1024;
  if (use_smem) {
    cudaError_t e = set_smem(lml_kernel, (int)bytes);
    if (e != cudaSuccess) return e;
  }
  lml_kernel<<<c, kLmlThreads, use_smem ? bytes : 0, s>>>(sq, n, D, z, thetas, out, scratch, use_smem);
  return cudaGetLastError();
}

cudaError_t launch_pairwise_sq(const SpaceDev& space, const uint32_t* a, int qa, const uint32_t* b,
                               int qb, double* out, cudaStream_t s) {
  if ((int64_t)qa * qb <= 0) return cudaSuccess;
  pairwise_sq_kernel<<<grid_for((int64_t)qa * qb, 256), 256, 0, s>>>(space, a, qa, b, qb, out);
  return cudaGetLastError();
}

cudaError_t launch_gp_planes(const SpaceDev& space, const uint32_t* train_rows, int n,
                             const double* inv_l, uint64_t* planes, uint64_t* kmask,
                             cudaStream_t s) {
  gp_planes_kernel<<<grid_for((int64_t)space.n_params * n, 256), 256, 0, s>>>(
      space, train_rows, n, inv_l, planes, kmask);
  return cudaGetLastError();
}

cudaError_t launch_tri_inverse(const double* L, int n, double* A, int lda, cudaStream_t s) {
  int warps = kInvWarps;
  while (warps > 1 && (size_t)warps * n * 8 > 200 * 1024) warps >>= 1;
  const size_t smem = (size_t)warps * n * 8;
  if (smem > 200 * 1024) return cudaErrorInvalidValue;  // n > 25600
  if (smem > 48 * 1024) {
    cudaError_t e = set_smem(tri_inverse_kernel, (int)smem);
    if (e != cudaSuccess) return e;
  }
  tri_inverse_kernel<<<(n + warps - 1) / warps, warps * 32, smem, s>>>(L, n, A, lda);
  return cudaGetLastError();
}

}  // namespace bx
