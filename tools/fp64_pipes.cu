// Microbenchmark: FP64 SIMT (DFMA) vs FP64 tensor (DMMA m8n8k4) throughput on sm_100a,
// alone and co-issued, plus FP64 exp/sqrt cost. Guides the score_pool contraction design.
#include <cstdio>
#include <cuda_runtime.h>
#include <cmath>

#define ITERS 4096

__device__ __forceinline__ void dmma(double& d0, double& d1, double a, double b) {
  asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};\n"
               : "+d"(d0), "+d"(d1) : "d"(a), "d"(b));
}

__global__ void k_dfma(double* out, double s) {
  double a[8];
#pragma unroll
  for (int i = 0; i < 8; i++) a[i] = threadIdx.x * 1e-3 + i;
  for (int it = 0; it < ITERS; it++) {
#pragma unroll
    for (int i = 0; i < 8; i++) a[i] = fma(a[i], s, 1e-9);
  }
  double r = 0; for (int i = 0; i < 8; i++) r += a[i];
  if (r == 12345.0) out[0] = r;
}

__global__ void k_dmma(double* out, double s) {
  double d[8][2];
#pragma unroll
  for (int i = 0; i < 8; i++) { d[i][0] = threadIdx.x; d[i][1] = i; }
  double a = s, b = s * 0.5;
  for (int it = 0; it < ITERS / 4; it++) {
#pragma unroll
    for (int i = 0; i < 8; i++) dmma(d[i][0], d[i][1], a, b);
  }
  double r = 0; for (int i = 0; i < 8; i++) r += d[i][0] + d[i][1];
  if (r == 12345.0) out[0] = r;
}

// half the warps DFMA, half DMMA
__global__ void k_mixed(double* out, double s) {
  int w = threadIdx.x / 32;
  if (w & 1) {
    double d[8][2];
#pragma unroll
    for (int i = 0; i < 8; i++) { d[i][0] = threadIdx.x; d[i][1] = i; }
    double a = s, b = s * 0.5;
    for (int it = 0; it < ITERS / 4; it++) {
#pragma unroll
      for (int i = 0; i < 8; i++) dmma(d[i][0], d[i][1], a, b);
    }
    double r = 0; for (int i = 0; i < 8; i++) r += d[i][0] + d[i][1];
    if (r == 12345.0) out[0] = r;
  } else {
    double a[8];
#pragma unroll
    for (int i = 0; i < 8; i++) a[i] = threadIdx.x * 1e-3 + i;
    for (int it = 0; it < ITERS; it++) {
#pragma unroll
      for (int i = 0; i < 8; i++) a[i] = fma(a[i], s, 1e-9);
    }
    double r = 0; for (int i = 0; i < 8; i++) r += a[i];
    if (r == 12345.0) out[0] = r;
  }
}

__global__ void k_exp(double* out, double s) {
  double a[4];
  for (int i = 0; i < 4; i++) a[i] = -(threadIdx.x % 7) * 0.1 - i;
  double acc = 0;
  for (int it = 0; it < ITERS / 16; it++) {
#pragma unroll
    for (int i = 0; i < 4; i++) { acc += exp(a[i]); a[i] -= s; }
  }
  if (acc == 12345.0) out[0] = acc;
}

__global__ void k_sqrt(double* out, double s) {
  double a[4];
  for (int i = 0; i < 4; i++) a[i] = (threadIdx.x % 7) * 0.1 + i + 1;
  double acc = 0;
  for (int it = 0; it < ITERS / 16; it++) {
#pragma unroll
    for (int i = 0; i < 4; i++) { acc += sqrt(a[i]); a[i] += s; }
  }
  if (acc == 12345.0) out[0] = acc;
}

// FP32 FFMA for reference
__global__ void k_ffma(double* out, float s) {
  float a[8];
#pragma unroll
  for (int i = 0; i < 8; i++) a[i] = threadIdx.x * 1e-3f + i;
  for (int it = 0; it < ITERS; it++) {
#pragma unroll
    for (int i = 0; i < 8; i++) a[i] = fmaf(a[i], s, 1e-9f);
  }
  float r = 0; for (int i = 0; i < 8; i++) r += a[i];
  if (r == 12345.0f) out[0] = r;
}

template <typename F>
float timeit(F f, int reps = 5) {
  cudaEvent_t a, b; cudaEventCreate(&a); cudaEventCreate(&b);
  f(); cudaDeviceSynchronize();
  float best = 1e30f;
  for (int r = 0; r < reps; r++) {
    cudaEventRecord(a); f(); cudaEventRecord(b); cudaEventSynchronize(b);
    float ms; cudaEventElapsedTime(&ms, a, b); if (ms < best) best = ms;
  }
  return best;
}

int main() {
  int dev = 0; cudaDeviceProp p; cudaGetDeviceProperties(&p, dev);
  int sms = p.multiProcessorCount;
  printf("device %s sms=%d clock=%d kHz\n", p.name, sms, p.clockRate);
  double* out; cudaMalloc(&out, 8);
  int blocks = sms * 8, threads = 256;
  double nthr = (double)blocks * threads;
  float ms;
  ms = timeit([&] { k_dfma<<<blocks, threads>>>(out, 0.999999); });
  printf("DFMA   : %.3f ms  %.2f TFLOP/s\n", ms, nthr * ITERS * 8 * 2 / ms / 1e9);
  ms = timeit([&] { k_ffma<<<blocks, threads>>>(out, 0.999999f); });
  printf("FFMA   : %.3f ms  %.2f TFLOP/s\n", ms, nthr * ITERS * 8 * 2 / ms / 1e9);
  ms = timeit([&] { k_dmma<<<blocks, threads>>>(out, 0.999999); });
  // per warp per dmma: 8*8*4 FMA = 256 FMA = 512 flop
  double warps = nthr / 32;
  printf("DMMA   : %.3f ms  %.2f TFLOP/s\n", ms, warps * (ITERS / 4) * 8 * 512 / ms / 1e9);
  ms = timeit([&] { k_mixed<<<blocks, threads>>>(out, 0.999999); });
  double fl = (nthr / 2) * ITERS * 8 * 2 + (warps / 2) * (ITERS / 4) * 8 * 512;
  printf("MIXED  : %.3f ms  %.2f TFLOP/s combined (DFMA+DMMA each half the warps, equal flops)\n", ms, fl / ms / 1e9);
  ms = timeit([&] { k_exp<<<blocks, threads>>>(out, 0.001); });
  printf("exp f64: %.3f ms  %.2f Gexp/s\n", ms, nthr * (ITERS / 16) * 4 / ms / 1e6);
  ms = timeit([&] { k_sqrt<<<blocks, threads>>>(out, 0.001); });
  printf("sqrt f64: %.3f ms  %.2f Gsqrt/s\n", ms, nthr * (ITERS / 16) * 4 / ms / 1e6);
  cudaError_t e = cudaGetLastError();
  printf("status %s\n", cudaGetErrorString(e));
  return 0;
}
