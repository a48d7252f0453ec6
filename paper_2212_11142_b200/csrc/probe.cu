// probe.cu — live FP64 roofline denominators (DFMA pipe and DMMA m8n8k4 tensor path).
//
// MEASURED_PEAKS.json carries HBM and bf16 only; the contraction of this path runs on the FP64
// pipe, so bench.py measures that peak on the box it runs on with these two loops (the same loops
// as tools/fp64_pipes.cu, profiles/r01_fp64_pipes.txt).
#include <cuda_runtime.h>

#include "../../include/bx_sm100.h"

namespace {

constexpr int kIters = 4096;

__global__ void probe_dfma(double* out, double s) {
  double a[8];
#pragma unroll
  for (int i = 0; i < 8; i++) a[i] = threadIdx.x * 1e-3 + i;
  for (int it = 0; it < kIters; it++) {
#pragma unroll
    for (int i = 0; i < 8; i++) a[i] = fma(a[i], s, 1e-9);
  }
  double r = 0;
  for (int i = 0; i < 8; i++) r += a[i];
  if (r == 12345.0) out[0] = r;
}

__global__ void probe_dmma(double* out, double s) {
  double d[8][2];
#pragma unroll
  for (int i = 0; i < 8; i++) {
    d[i][0] = threadIdx.x;
    d[i][1] = i;
  }
  const double a = s, b = s * 0.5;
  for (int it = 0; it < kIters / 4; it++) {
#pragma unroll
    for (int i = 0; i < 8; i++)
      asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};\n"
                   : "+d"(d[i][0]), "+d"(d[i][1])
                   : "d"(a), "d"(b));
  }
  double r = 0;
  for (int i = 0; i < 8; i++) r += d[i][0] + d[i][1];
  if (r == 12345.0) out[0] = r;
}

}  // namespace

extern "C" int bx_probe_fp64(int device, double* dfma_tflops, double* dmma_tflops) {
  if (cudaSetDevice(device) != cudaSuccess) return BX_ERR_CUDA;
  int sms = 0;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, device);
  double* out = nullptr;
  if (cudaMalloc(&out, 8) != cudaSuccess) return BX_ERR_CUDA;
  cudaEvent_t a, b;
  cudaEventCreate(&a);
  cudaEventCreate(&b);
  const int blocks = sms * 8, threads = 256;
  const double nthr = (double)blocks * threads;
  float best[2] = {1e30f, 1e30f};
  for (int rep = 0; rep < 4; ++rep) {
    for (int k = 0; k < 2; ++k) {
      cudaEventRecord(a);
      if (k == 0) probe_dfma<<<blocks, threads>>>(out, 0.999999);
      else probe_dmma<<<blocks, threads>>>(out, 0.999999);
      cudaEventRecord(b);
      cudaEventSynchronize(b);
      float ms = 0;
      cudaEventElapsedTime(&ms, a, b);
      if (rep > 0 && ms < best[k]) best[k] = ms;  // rep 0 is the warm-up
    }
  }
  cudaError_t e = cudaGetLastError();
  cudaEventDestroy(a);
  cudaEventDestroy(b);
  cudaFree(out);
  if (e != cudaSuccess) return BX_ERR_CUDA;
  if (dfma_tflops) *dfma_tflops = nthr * kIters * 8 * 2 / best[0] / 1e9;
  if (dmma_tflops) *dmma_tflops = (nthr / 32) * (kIters / 4) * 8 * 512 / best[1] / 1e9;
  return BX_OK;
}
