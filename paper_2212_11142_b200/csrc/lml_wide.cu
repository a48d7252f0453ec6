// lml_wide.cu — _lml_core (surrogate.py:356-400) for ONE hyperparameter setting spread over the
// whole GPU.  The L-BFGS-B refinement calls the objective with a single setting (~200 times per BO
// iteration), so the one-CTA-per-setting kernel of gp_linalg.cu leaves 147 SMs idle; here every
// stage is tiled across CTAs:
//
//   lw_gram_kernel     K and Ky = K + (noise + 1e-9) I  (surrogate.py:365-371), padded to 32-multiples
//                      with an identity block so the tiles need no bounds
//   lw_chol_kernel     blocked right-looking Cholesky, one launch per 32-column block: every CTA owns
//                      one 32-row block of the panel, applies the updates from the previous block
//                      columns, factors the diagonal block (redundantly, in shared memory) and solves
//                      its rows — LAPACK potrf's failure rule (a pivot that is not > 0) sets a flag
//   lw_inverse_kernel  X = L^-1, one warp per column (forward substitution)
//   lw_value_kernel    u = X z, alpha = X^T u (the two TRTRS of :373-374), value (+ Gamma prior :380-383)
//   lw_grad_kernel     K^-1 = X^T X by 32 x 32 tiles (lower tile triangle, symmetric weight 2) fused
//                      with the gradient sums of M = alpha alpha^T - K^-1 (:386-399) into per-tile
//                      partials
//   lw_final_kernel    reduces the partials: d/dlog sigma, d/dlog noise, d/dlog l_k (+ prior)
#include <algorithm>

#include "bx_common.cuh"

namespace bx {

namespace {

constexpr int kT = 32;  // tile edge

// logspace: prm rows are thetas (log sigma, log noise, log l_k) as _batched_coarse_lml takes them
// (surrogate.py:428-434: exp, exp(-2 theta)); else natural units as _lml_core takes them.  Setting
// blockIdx.y writes its own K / A (K may be null: the coarse LML needs only A).
__global__ void __launch_bounds__(256) lw_gram_kernel(const double* sq, int n, int np, int D, const double* prm0,
                                                      int logspace, double* K0, double* A0) {
  __shared__ double il2[BX_MAX_PARAMS];
  const double* prm = prm0 + (size_t)blockIdx.y * (2 + D);
  double* K = K0 ? K0 + (size_t)blockIdx.y * np * np : nullptr;
  double* A = A0 + (size_t)blockIdx.y * np * np;
  for (int k = threadIdx.x; k < D; k += blockDim.x)
    il2[k] = logspace ? exp(-2.0 * prm[2 + k]) : 1.0 / (prm[2 + k] * prm[2 + k]);
  __syncthreads();
  const double sigma = logspace ? exp(prm[0]) : prm[0];
  const double noise = fmax(logspace ? exp(prm[1]) : prm[1], 1e-6);  // NOISE_FLOOR
  const size_t nn = (size_t)n * n, total = (size_t)np * np;
  for (size_t t = (size_t)blockIdx.x * blockDim.x + threadIdx.x; t < total; t += (size_t)gridDim.x * blockDim.x) {
    const int i = (int)(t / np), j = (int)(t % np);
    if (i < n && j < n) {
      const size_t s = (size_t)i * n + j;
      double W = 0.0;
      for (int k = 0; k < D; ++k) W = fma(sq[(size_t)k * nn + s], il2[k], W);
      const double d = sqrt(fmax(W, 0.0));
      const double E = exp(-kSqrt5 * d);
      const double kv = sigma * ((1.0 + kSqrt5 * d + (5.0 / 3.0) * W) * E);
      if (K) K[t] = kv;
      A[t] = (i == j) ? kv + noise + 1e-9 : kv;  // JITTER
    } else {
      if (K) K[t] = 0.0;
      A[t] = (i == j) ? 1.0 : 0.0;
    }
  }
}

// Block column J of the Cholesky factor (A holds L in the finished block columns).  CTA b owns row
// block I = J + b; 256 threads = 8 warps, thread (ty, tx) covers rows ty + 8 s of column tx.
__global__ void __launch_bounds__(256) lw_chol_kernel(double* A0, int np, int J, int* fail0) {
  __shared__ double Dg[kT][kT + 1], T[kT][kT + 1], P[kT][kT + 1], Q[kT][kT + 1];
  double* A = A0 + (size_t)blockIdx.y * np * np;  // setting blockIdx.y
  int* fail = fail0 + blockIdx.y;
  const int I = J + blockIdx.x;
  const int tid = threadIdx.x, tx = tid & 31, ty = tid >> 5;
  const bool diag = I == J;
  const double* Ab = A;
  for (int s = 0; s < 4; ++s) {
    const int r = ty + 8 * s;
    Dg[r][tx] = Ab[(size_t)(J * kT + r) * np + J * kT + tx];
    if (!diag) T[r][tx] = Ab[(size_t)(I * kT + r) * np + J * kT + tx];
  }
  for (int kb = 0; kb < J; ++kb) {
    __syncthreads();
    for (int s = 0; s < 4; ++s) {
      const int r = ty + 8 * s;
      P[r][tx] = Ab[(size_t)(J * kT + r) * np + kb * kT + tx];
      if (!diag) Q[r][tx] = Ab[(size_t)(I * kT + r) * np + kb * kT + tx];
    }
    __syncthreads();
    for (int s = 0; s < 4; ++s) {
      const int r = ty + 8 * s;
      double dv = Dg[r][tx], tv = diag ? 0.0 : T[r][tx];
#pragma unroll 8
      for (int k = 0; k < kT; ++k) {
        dv = fma(-P[r][k], P[tx][k], dv);
        if (!diag) tv = fma(-Q[r][k], P[tx][k], tv);
      }
      Dg[r][tx] = dv;
      if (!diag) T[r][tx] = tv;
    }
  }
  __syncthreads();
  if (ty == 0) {  // unblocked Cholesky of the diagonal block, lane = row
    const int r = tx;
    for (int j = 0; j < kT; ++j) {
      const double piv = Dg[j][j];
      const bool bad = !(piv > 0.0);
      if (bad && r == 0 && diag) atomicExch(fail, 1);
      const double ljj = sqrt(bad ? 1.0 : piv);
      __syncwarp();
      if (r > j) Dg[r][j] /= ljj;
      __syncwarp();
      if (r == j) Dg[j][j] = ljj;
      if (r > j)
        for (int c = j + 1; c <= r; ++c) Dg[r][c] = fma(-Dg[r][j], Dg[c][j], Dg[r][c]);
      __syncwarp();
    }
  }
  __syncthreads();
  if (diag) {
    for (int s = 0; s < 4; ++s) {
      const int r = ty + 8 * s;
      A[(size_t)(J * kT + r) * np + J * kT + tx] = tx <= r ? Dg[r][tx] : 0.0;
    }
    return;
  }
  if (ty == 0) {  // rows of T times L_JJ^-T: forward substitution per row
    const int r = tx;
    for (int c = 0; c < kT; ++c) {
      double x = T[r][c];
      for (int k = 0; k < c; ++k) x = fma(-T[r][k], Dg[c][k], x);
      T[r][c] = x / Dg[c][c];
    }
  }
  __syncthreads();
  for (int s = 0; s < 4; ++s) {
    const int r = ty + 8 * s;
    A[(size_t)(I * kT + r) * np + J * kT + tx] = T[r][tx];
  }
}

// X = L^-1 (lower; X is zeroed beforehand): one warp per column, the column kept in shared memory
constexpr int kInvW = 8;
__global__ void __launch_bounds__(kInvW * 32) lw_inverse_kernel(const double* L0, int np, double* X0) {
  __shared__ double xs[kInvW][512 + 32];
  const double* L = L0 + (size_t)blockIdx.y * np * np;  // setting blockIdx.y
  double* X = X0 + (size_t)blockIdx.y * np * np;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int j = blockIdx.x * kInvW + warp;
  if (j >= np) return;
  double* x = xs[warp];
  if (lane == 0) x[j] = 1.0 / L[(size_t)j * np + j];
  __syncwarp();
  for (int i = j + 1; i < np; ++i) {
    const double* Li = L + (size_t)i * np;
    double s = 0.0;
    for (int k = j + lane; k < i; k += 32) s = fma(Li[k], x[k], s);
#pragma unroll
    for (int off = 16; off; off >>= 1) s += __shfl_xor_sync(0xffffffffu, s, off);
    if (lane == 0) x[i] = -s / Li[i];
    __syncwarp();
  }
  for (int i = j + lane; i < np; i += 32) X[(size_t)i * np + j] = x[i];
}

__device__ __forceinline__ double block_sum_lw(double v, double* red) {
  for (int off = 16; off; off >>= 1) v += __shfl_xor_sync(0xffffffffu, v, off);
  __syncthreads();
  if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = v;
  __syncthreads();
  double s = 0.0;
  for (int w = 0; w < (int)(blockDim.x >> 5); ++w) s += red[w];
  return s;
}

__global__ void __launch_bounds__(512) lw_value_kernel(const double* L0, const double* X0, int n, int np, int D,
                                                       const double* z, const double* prm0, double prior_k,
                                                       double prior_rate, int use_prior, const int* fail0,
                                                       double* u0, double* al0, double* out_value0, int* out_ok0) {
  __shared__ double red[16];
  const int y = blockIdx.y;  // setting
  const double* L = L0 + (size_t)y * np * np;
  const double* X = X0 + (size_t)y * np * np;
  const double* prm = prm0 + (size_t)y * (2 + D);
  const int* fail = fail0 + y;
  double* u = u0 + (size_t)y * np;
  double* al = al0 + (size_t)y * np;
  double* out_value = out_value0 + y;
  int* out_ok = out_ok0 + y;
  const int tid = threadIdx.x;
  for (int i = tid; i < n; i += blockDim.x) {  // u = L^-1 z
    double s = 0.0;
    for (int k = 0; k <= i; ++k) s = fma(X[(size_t)i * np + k], z[k], s);
    u[i] = s;
  }
  __syncthreads();
  for (int j = tid; j < n; j += blockDim.x) {  // alpha = L^-T u
    double s = 0.0;
    for (int i = j; i < n; ++i) s = fma(X[(size_t)i * np + j], u[i], s);
    al[j] = s;
  }
  __syncthreads();
  double za = 0.0, ld = 0.0;
  for (int i = tid; i < n; i += blockDim.x) {
    za = fma(z[i], al[i], za);
    ld += log(L[(size_t)i * np + i]);
  }
  za = block_sum_lw(za, red);
  ld = block_sum_lw(ld, red);
  if (tid == 0) {
    double value = -0.5 * za - ld - 0.5 * n * log(2.0 * 3.14159265358979323846);
    if (use_prior) {  // Gamma(k, rate) log density per lengthscale (surrogate.py:380-383)
      double sl = 0.0, sll = 0.0;
      for (int k = 0; k < D; ++k) {
        sl += prm[2 + k];
        sll += log(prm[2 + k]);
      }
      value += D * (prior_k * log(prior_rate) - lgamma(prior_k)) + (prior_k - 1.0) * sll - prior_rate * sl;
    }
    const bool ok = *fail == 0;
    *out_ok = ok ? 1 : 0;
    *out_value = ok ? value : -INFINITY;
  }
}

// tile (a, b), a >= b, of K^-1 = X^T X fused with the gradient sums over its elements
__global__ void __launch_bounds__(256) lw_grad_kernel(const double* X0, const double* K0, const double* sq,
                                                      const double* al0, const double* prm0, int n, int np, int D,
                                                      double* partial0) {
  __shared__ double Xa[kT][kT + 1], Xb[kT][kT + 1];
  const int y = blockIdx.y;  // setting
  const double* X = X0 + (size_t)y * np * np;
  const double* K = K0 + (size_t)y * np * np;
  const double* al = al0 + (size_t)y * np;
  const double* prm = prm0 + (size_t)y * (2 + D);
  double* partial = partial0 + (size_t)y * gridDim.x * (2 + D);
  __shared__ double il2[BX_MAX_PARAMS];
  __shared__ double red[8];
  int t = blockIdx.x, a = 0;
  while (t > a) t -= ++a;  // blockIdx.x -> (a, b = t), b <= a
  const int b = t;
  const int tid = threadIdx.x, tx = tid & 31, ty = tid >> 5;
  for (int k = tid; k < D; k += blockDim.x) il2[k] = 1.0 / (prm[2 + k] * prm[2 + k]);
  double acc[4] = {0.0, 0.0, 0.0, 0.0};
  const int nb = np / kT;
  for (int kb = a; kb < nb; ++kb) {  // X_ka = 0 for k < a
    __syncthreads();
    for (int s = 0; s < 4; ++s) {
      const int r = ty + 8 * s;
      Xa[r][tx] = X[(size_t)(kb * kT + r) * np + a * kT + tx];
      Xb[r][tx] = X[(size_t)(kb * kT + r) * np + b * kT + tx];
    }
    __syncthreads();
    for (int s = 0; s < 4; ++s) {
      const int r = ty + 8 * s;  // element (a*32 + r, b*32 + tx)
#pragma unroll 8
      for (int k = 0; k < kT; ++k) acc[s] = fma(Xa[k][r], Xb[k][tx], acc[s]);
    }
  }
  const double w = a == b ? 1.0 : 2.0;  // the symmetric (b, a) tile
  const size_t nn = (size_t)n * n;
  double g0 = 0.0, g1 = 0.0;
  double gl[BX_MAX_PARAMS];
  for (int k = 0; k < D; ++k) gl[k] = 0.0;
  for (int s = 0; s < 4; ++s) {
    const int i = a * kT + ty + 8 * s, j = b * kT + tx;
    if (i >= n || j >= n) continue;
    const double M = w * (al[i] * al[j] - acc[s]);
    g0 = fma(M, K[(size_t)i * np + j], g0);
    if (i == j) g1 += M;
    const size_t e = (size_t)i * n + j;
    double W = 0.0;
    for (int k = 0; k < D; ++k) W = fma(sq[(size_t)k * nn + e], il2[k], W);
    const double d = sqrt(fmax(W, 0.0));
    const double MG = M * ((1.0 + kSqrt5 * d) * exp(-kSqrt5 * d));
    for (int k = 0; k < D; ++k) gl[k] = fma(MG, sq[(size_t)k * nn + e], gl[k]);
  }
  double* out = partial + (size_t)blockIdx.x * (2 + D);
  g0 = block_sum_lw(g0, red);
  if (tid == 0) out[0] = g0;
  g1 = block_sum_lw(g1, red);
  if (tid == 0) out[1] = g1;
  for (int k = 0; k < D; ++k) {
    const double v = block_sum_lw(gl[k], red);
    if (tid == 0) out[2 + k] = v;
  }
}

__global__ void lw_final_kernel(const double* partial0, int tiles, const double* prm0, int D, double prior_k,
                                double prior_rate, int use_prior, const int* fail0, double* grad0) {
  const int k = threadIdx.x, y = blockIdx.x;  // setting
  const double* partial = partial0 + (size_t)y * tiles * (2 + D);
  const double* prm = prm0 + (size_t)y * (2 + D);
  const int* fail = fail0 + y;
  double* grad = grad0 + (size_t)y * (2 + D);
  if (k >= 2 + D) return;
  if (*fail) {
    grad[k] = 0.0;
    return;
  }
  double s = 0.0;
  for (int t = 0; t < tiles; ++t) s += partial[(size_t)t * (2 + D) + k];
  const double sigma = prm[0], noise = fmax(prm[1], 1e-6);
  if (k == 0) {
    grad[0] = 0.5 * s;
  } else if (k == 1) {
    grad[1] = 0.5 * noise * s;
  } else {
    const double l = prm[k];
    double g = ((5.0 / 6.0) * sigma / (l * l)) * s;
    if (use_prior) g += (prior_k - 1.0) - prior_rate * l;
    grad[k] = g;
  }
}

// _batched_coarse_lml's value for setting blockIdx.x from its factor: u = L^-1 z by 32-row blocks
// (one warp solves the diagonal block, the CTA updates the rows below), then
// -0.5 |u|^2 - sum log L_ii - n/2 log 2 pi (surrogate.py:450-455), -inf when the factorisation failed
__global__ void __launch_bounds__(256) lw_coarse_value_kernel(const double* L0, int n, int np, const double* z,
                                                              const int* fail, double* out) {
  __shared__ double u[512];
  __shared__ double red[8];
  const double* L = L0 + (size_t)blockIdx.x * np * np;
  const int tid = threadIdx.x, lane = tid & 31;
  for (int i = tid; i < np; i += blockDim.x) u[i] = i < n ? z[i] : 0.0;
  const int nb = np / kT;
  for (int jb = 0; jb < nb; ++jb) {
    __syncthreads();
    if (tid < 32) {
      const int r = jb * kT + lane;
      double ur = u[r];
      for (int c = 0; c < kT; ++c) {
        const int col = jb * kT + c;
        const double uc = __shfl_sync(0xffffffffu, ur / L[(size_t)r * np + r], c);  // lane c holds row col
        if (lane == c) ur = uc;
        if (lane > c) ur = fma(-L[(size_t)r * np + col], uc, ur);
      }
      u[r] = ur;
    }
    __syncthreads();
    for (int i = (jb + 1) * kT + tid; i < np; i += blockDim.x) {
      double s = u[i];
      const double* Li = L + (size_t)i * np + jb * kT;
#pragma unroll 8
      for (int k = 0; k < kT; ++k) s = fma(-Li[k], u[jb * kT + k], s);
      u[i] = s;
    }
  }
  __syncthreads();
  double q = 0.0, ld = 0.0;
  for (int i = tid; i < n; i += blockDim.x) {
    q = fma(u[i], u[i], q);
    ld += log(L[(size_t)i * np + i]);
  }
  q = block_sum_lw(q, red);
  ld = block_sum_lw(ld, red);
  if (tid == 0)
    out[blockIdx.x] = fail[blockIdx.x] ? -INFINITY : -0.5 * q - ld - 0.5 * n * log(2.0 * 3.14159265358979323846);
}

}  // namespace

size_t lml_coarse_wide_scratch_doubles(int n, int c) {
  const int np = (n + kT - 1) / kT * kT;
  return (size_t)c * np * np + (size_t)c;  // factors + failure flags
}

// _batched_coarse_lml for c settings: the blocked Cholesky batched over settings (grid.y)
cudaError_t launch_lml_coarse_wide(const double* sq, int n, int D, const double* z, const double* thetas, int c,
                                   double* out, double* scratch, cudaStream_t s) {
  if (n > 512 || c <= 0) return c <= 0 ? cudaSuccess : cudaErrorInvalidValue;
  const int np = (n + kT - 1) / kT * kT, nb = np / kT;
  double* L = scratch;
  int* fail = reinterpret_cast<int*>(L + (size_t)c * np * np);
  cudaError_t e = cudaMemsetAsync(fail, 0, (size_t)c * sizeof(int), s);
  if (e != cudaSuccess) return e;
  const int gx = (int)std::min<size_t>(((size_t)np * np + 255) / 256, 64);
  lw_gram_kernel<<<dim3(gx, c), 256, 0, s>>>(sq, n, np, D, thetas, 1, nullptr, L);
  for (int J = 0; J < nb; ++J) lw_chol_kernel<<<dim3(nb - J, c), 256, 0, s>>>(L, np, J, fail);
  lw_coarse_value_kernel<<<c, 256, 0, s>>>(L, n, np, z, fail, out);
  return cudaGetLastError();
}

size_t lml_wide_scratch_doubles(int n, int D, int c) {
  const int np = (n + kT - 1) / kT * kT, nb = np / kT;
  return (size_t)c * (3 * (size_t)np * np + 2 * (size_t)np + (size_t)nb * (nb + 1) / 2 * (2 + D)) + (size_t)c + 1;
}

bool lml_wide_supported(int n) { return n <= 512; }

// c hyperparameter settings (prm = c rows of sigma, noise, l_1..l_D in natural units), each spread
// over the GPU and all of them side by side on grid.y: a setting's arithmetic does not depend on c
cudaError_t launch_lml_wide(const double* sq, int n, int D, const double* z, const double* prm, int c, double prior_k,
                            double prior_rate, int use_prior, int want_grad, double* out_value, double* out_grad,
                            int* out_ok, double* scratch, cudaStream_t s) {
  if (n > 512 || c < 1) return cudaErrorInvalidValue;
  const int np = (n + kT - 1) / kT * kT, nb = np / kT, tiles = nb * (nb + 1) / 2;
  double* K = scratch;
  double* L = K + (size_t)c * np * np;
  double* X = L + (size_t)c * np * np;
  double* u = X + (size_t)c * np * np;
  double* al = u + (size_t)c * np;
  double* partial = al + (size_t)c * np;
  int* fail = reinterpret_cast<int*>(partial + (size_t)c * tiles * (2 + D));
  cudaError_t e = cudaMemsetAsync(fail, 0, sizeof(int) * c, s);
  if (e != cudaSuccess) return e;
  e = cudaMemsetAsync(X, 0, (size_t)c * np * np * sizeof(double), s);
  if (e != cudaSuccess) return e;
  const int g = (int)std::min<size_t>(((size_t)np * np + 255) / 256, 148 * 8);
  lw_gram_kernel<<<dim3(g, c), 256, 0, s>>>(sq, n, np, D, prm, 0, K, L);
  for (int J = 0; J < nb; ++J) lw_chol_kernel<<<dim3(nb - J, c), 256, 0, s>>>(L, np, J, fail);
  lw_inverse_kernel<<<dim3((np + kInvW - 1) / kInvW, c), kInvW * 32, 0, s>>>(L, np, X);
  lw_value_kernel<<<dim3(1, c), 512, 0, s>>>(L, X, n, np, D, z, prm, prior_k, prior_rate, use_prior, fail, u, al,
                                             out_value, out_ok);
  if (want_grad) {
    lw_grad_kernel<<<dim3(tiles, c), 256, 0, s>>>(X, K, sq, al, prm, n, np, D, partial);
    lw_final_kernel<<<c, 64, 0, s>>>(partial, tiles, prm, D, prior_k, prior_rate, use_prior, fail, out_grad);
  }
  return cudaGetLastError();
}

// GPModel.__init__ (surrogate.py:286-303) on the device for one hyperparameter setting: Gram with
// noise floor + jitter, the blocked Cholesky, L^-1 and alpha = L^-T L^-1 z, in the scratch layout
// of launch_lml_wide (c = 1); the factor is left at L (row stride np), alpha at al, the failure
// flag (potrf info > 0) at fail.
cudaError_t launch_gp_factor(const double* sq, int n, int D, const double* z, const double* prm, double* scratch,
                             const double** L_out, const double** al_out, const int** fail_out,
                             const double** X_out, cudaStream_t s) {
  if (n > 512 || n < 1) return cudaErrorInvalidValue;
  const int np = (n + kT - 1) / kT * kT, nb = np / kT, tiles = nb * (nb + 1) / 2;
  double* K = scratch;
  double* L = K + (size_t)np * np;
  double* X = L + (size_t)np * np;
  double* u = X + (size_t)np * np;
  double* al = u + np;
  double* partial = al + np;
  int* fail = reinterpret_cast<int*>(partial + (size_t)tiles * (2 + D));
  double* val = partial;  // the value kernel's outputs (unused here) in the partial-sum area
  int* ok = fail + 1;
  cudaError_t e = cudaMemsetAsync(fail, 0, sizeof(int), s);
  if (e != cudaSuccess) return e;
  e = cudaMemsetAsync(X, 0, (size_t)np * np * sizeof(double), s);
  if (e != cudaSuccess) return e;
  const int g = (int)std::min<size_t>(((size_t)np * np + 255) / 256, 148 * 8);
  lw_gram_kernel<<<dim3(g, 1), 256, 0, s>>>(sq, n, np, D, prm, 0, nullptr, L);
  for (int J = 0; J < nb; ++J) lw_chol_kernel<<<dim3(nb - J, 1), 256, 0, s>>>(L, np, J, fail);
  lw_inverse_kernel<<<dim3((np + kInvW - 1) / kInvW, 1), kInvW * 32, 0, s>>>(L, np, X);
  lw_value_kernel<<<dim3(1, 1), 512, 0, s>>>(L, X, n, np, D, z, prm, 0.0, 0.0, 0, fail, u, al, val, ok);
  *L_out = L;
  *al_out = al;
  *fail_out = fail;
  *X_out = X;
  return cudaGetLastError();
}

}  // namespace bx

