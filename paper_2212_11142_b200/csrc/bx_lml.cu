// bx_lml.cu — the hyperparameter-fit objectives behind the C ABI: the batched coarse LML
// (_batched_coarse_lml), _lml_core with its gradient for c settings, and the bit-exact pairwise
// squared distances (pairwise_sq_distances) they take.
#include <cstring>

#include "bx_handle.cuh"

extern "C" {
int bx_lml_batched(bx_handle* h, const double* sq, int32_t n, int32_t D, const double* z,
                   const double* thetas, int32_t c, double* out, void* stream) {
  if (!h) return BX_ERR_ARG;
  if (n < 1 || D < 1 || D > BX_MAX_PARAMS || c < 0)
    return fail(h, BX_ERR_ARG, "bad lml shape n=%d D=%d c=%d", n, D, c);
  cudaSetDevice(h->device);
  // small n: one CTA per setting with the packed triangle in shared memory beats the blocked
  // whole-GPU pipeline (measured crossover ~ n = 100)
  if (lml_wide_supported(n) && !h->lml_narrow && n > 96) {
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

int bx_lml_core(bx_handle* h, const double* sq, int32_t n, int32_t D, const double* z,
                const double* params, int32_t c, double prior_shape, double prior_rate,
                int32_t use_prior, int32_t want_grad, double* value, double* grad, int32_t* ok,
                void* stream) {
  if (!h) return BX_ERR_ARG;
  if (n < 1 || D < 1 || D > BX_MAX_PARAMS || c < 0)
    return fail(h, BX_ERR_ARG, "bad lml shape n=%d D=%d c=%d", n, D, c);
  if (want_grad && !grad) return fail(h, BX_ERR_ARG, "want_grad needs a gradient buffer");
  cudaSetDevice(h->device);
  // small n (<= 40, the measured crossover; the kernel takes up to 232): one CTA per setting with
  // everything in its shared memory (lml_small_kernel); larger n: the whole-GPU pipeline, settings side by side on grid.y, in groups that keep the scratch
  // under 1 GiB.  Either way a setting's arithmetic does not depend on the batch (the batched
  // L-BFGS-B restarts get the values a single call gives).  BX_OPT_LML_NARROW: the one-CTA-per-
  // setting kernel with global scratch (any n; the cross-check of the other two).
  if (lml_small_supported(n) && n <= h->lml_small_max && !h->lml_narrow) {
    BX_CUDA(h, launch_lml_small(sq, n, D, z, params, c, prior_shape, prior_rate, use_prior, want_grad, value,
                                want_grad ? grad : nullptr, ok, (cudaStream_t)stream));
    return BX_OK;
  }
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

// bx_lml_core with host parameters and results (the L-BFGS-B driver's call, hyperfit.py): the
// settings go up and (values, grads, ok) come back through one pinned staging buffer and one
// device scratch, one copy each way and one stream synchronisation.
int bx_lml_core_host(bx_handle* h, const double* sq, int32_t n, int32_t D, const double* z, const double* host_params,
                     int32_t c, double prior_shape, double prior_rate, int32_t use_prior, double* host_value,
                     double* host_grad, int32_t* host_ok, void* stream) {
  if (!h) return BX_ERR_ARG;
  if (c < 0 || D < 1 || D > BX_MAX_PARAMS) return fail(h, BX_ERR_ARG, "bad lml shape D=%d c=%d", D, c);
  if (c == 0) return BX_OK;
  if (!host_params || !host_value || !host_grad || !host_ok) return fail(h, BX_ERR_ARG, "null argument");
  cudaSetDevice(h->device);
  cudaStream_t s = (cudaStream_t)stream;
  const size_t np = (size_t)c * (2 + D), nout = (size_t)c * (3 + D) + ((size_t)c + 1) / 2;  // value, grad, ok
  const size_t bytes = (np + nout) * sizeof(double);
  if (h->h_lml_stage_bytes < bytes) {
    if (h->h_lml_stage) cudaFreeHost(h->h_lml_stage);
    h->h_lml_stage = nullptr;
    h->h_lml_stage_bytes = 0;
    BX_CUDA(h, cudaMallocHost(&h->h_lml_stage, bytes));
    h->h_lml_stage_bytes = bytes;
  }
  BX_CUDA(h, h->d_lml_stage.ensure(bytes));
  double* hs = static_cast<double*>(h->h_lml_stage);
  double* ds = h->d_lml_stage.as<double>();
  std::memcpy(hs, host_params, np * sizeof(double));
  BX_CUDA(h, cudaMemcpyAsync(ds, hs, np * sizeof(double), cudaMemcpyHostToDevice, s));
  int32_t* d_ok = reinterpret_cast<int32_t*>(ds + np + (size_t)c * (3 + D));
  const int r = bx_lml_core(h, sq, n, D, z, ds, c, prior_shape, prior_rate, use_prior, 1, ds + np, ds + np + c, d_ok,
                            stream);
  if (r) return r;
  BX_CUDA(h, cudaMemcpyAsync(hs + np, ds + np, nout * sizeof(double), cudaMemcpyDeviceToHost, s));
  BX_CUDA(h, cudaStreamSynchronize(s));
  std::memcpy(host_value, hs + np, (size_t)c * sizeof(double));
  std::memcpy(host_grad, hs + np + c, (size_t)c * (2 + D) * sizeof(double));
  std::memcpy(host_ok, hs + np + (size_t)c * (3 + D), (size_t)c * sizeof(int32_t));
  return BX_OK;
}

int bx_gp_factor(bx_handle* h, const uint32_t* dev_train_rows, int32_t n, const double* host_z, double outputscale,
                 double noise_variance, const double* lengthscales, double* host_L, double* host_alpha, void* stream) {
  int r = check_space(h);
  if (r) return r;
  if (n < 1 || n > 512) return fail(h, BX_ERR_UNSUPPORTED, "bx_gp_factor: n = %d outside 1..512", n);
  if (!dev_train_rows || !host_z || !lengthscales || !host_L || !host_alpha) return fail(h, BX_ERR_ARG, "null argument");
  cudaSetDevice(h->device);
  cudaStream_t s = (cudaStream_t)stream;
  const int D = h->n_params;
  std::vector<double> prm(2 + D);
  prm[0] = outputscale;
  prm[1] = noise_variance;
  for (int k = 0; k < D; ++k) prm[2 + k] = lengthscales[k];
  // [D][n][n] squared distances | z | prm | the lml_wide scratch of one setting
  const size_t sq_d = (size_t)D * n * n;
  BX_CUDA(h, h->d_factor.ensure((sq_d + n + 2 + D + lml_wide_scratch_doubles(n, D, 1)) * sizeof(double)));
  double* sq = h->d_factor.as<double>();
  double* z = sq + sq_d;
  double* p = z + n;
  double* scratch = p + 2 + D;
  BX_CUDA(h, launch_pairwise_sq(space_dev(h), dev_train_rows, n, dev_train_rows, n, sq, s));
  BX_CUDA(h, cudaMemcpyAsync(z, host_z, (size_t)n * 8, cudaMemcpyHostToDevice, s));
  BX_CUDA(h, cudaMemcpyAsync(p, prm.data(), prm.size() * 8, cudaMemcpyHostToDevice, s));
  const double *L, *al, *X;
  const int* failed;
  BX_CUDA(h, launch_gp_factor(sq, n, D, z, p, scratch, &L, &al, &failed, &X, s));
  const int np = (n + 31) / 32 * 32;
  int fl = 0;
  BX_CUDA(h, cudaMemcpy2DAsync(host_L, (size_t)n * 8, L, (size_t)np * 8, (size_t)n * 8, n, cudaMemcpyDeviceToHost, s));
  BX_CUDA(h, cudaMemcpyAsync(host_alpha, al, (size_t)n * 8, cudaMemcpyDeviceToHost, s));
  BX_CUDA(h, cudaMemcpyAsync(&fl, failed, sizeof(int), cudaMemcpyDeviceToHost, s));
  BX_CUDA(h, cudaStreamSynchronize(s));
  if (fl) return fail(h, BX_ERR_NOT_PD, "Gram matrix is not positive definite (potrf info > 0)");
  for (int i = 0; i < n; ++i)  // the strict upper triangle of the factor is zero (np.tril)
    for (int j = i + 1; j < n; ++j) host_L[(size_t)i * n + j] = 0.0;
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
