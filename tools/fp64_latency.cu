// Dependent-chain latency of FP64 operations on one warp (development aid):
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o tools/fp64_latency tools/fp64_latency.cu
#include <cstdio>
#include <cuda_runtime.h>

template <int OP>
__global__ void chain(double* out, long long* clk, double a, double b, int iters) {
  double x = a + threadIdx.x;
  long long t0 = clock64();
  for (int i = 0; i < iters; ++i) {
#pragma unroll
    for (int j = 0; j < 16; ++j) {
      if (OP == 0) x = fma(x, b, a);                 // DFMA
      if (OP == 1) x = x * b;                        // DMUL
      if (OP == 2) x = x + b;                        // DADD
      if (OP == 3) { double y; asm volatile("rsqrt.approx.ftz.f64 %0, %1;" : "=d"(y) : "d"(x)); x = y; }
      if (OP == 4) x = (double)__double2ull_rz(x);   // F2I + I2F round trip
    }
  }
  long long t1 = clock64();
  out[threadIdx.x] = x;
  if (threadIdx.x == 0) *clk = t1 - t0;
}

int main() {
  double* out; long long* clk;
  cudaMalloc(&out, 1024 * 8); cudaMalloc(&clk, 8);
  const char* names[] = {"DFMA", "DMUL", "DADD", "MUFU.RSQ64H", "F2I.U64+I2F.F64"};
  for (int op = 0; op < 5; ++op) {
    for (int warps : {1, 4}) {
      long long c = 0;
      const int it = 1000;
      for (int rep = 0; rep < 2; ++rep) {
        switch (op) {
          case 0: chain<0><<<1, 32 * warps>>>(out, clk, 1.0, 0.999999, it); break;
          case 1: chain<1><<<1, 32 * warps>>>(out, clk, 1.0, 0.999999, it); break;
          case 2: chain<2><<<1, 32 * warps>>>(out, clk, 1.0, 1e-9, it); break;
          case 3: chain<3><<<1, 32 * warps>>>(out, clk, 1.0, 1.0, it); break;
          case 4: chain<4><<<1, 32 * warps>>>(out, clk, 12345.0, 1.0, it); break;
        }
        cudaMemcpy(&c, clk, 8, cudaMemcpyDeviceToHost);
      }
      printf("%-16s warps=%d  %.1f clk per dependent op\n", names[op], warps, (double)c / (16.0 * it));
    }
  }
  printf("status %s\n", cudaGetErrorString(cudaGetLastError()));
  return 0;
}
