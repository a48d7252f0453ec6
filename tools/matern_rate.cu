// matern_rate.cu — throughput of the producer's per-K* arithmetic in isolation (no tensor work):
// W accumulation over D numeric parameters, kstar_fast, 40-bit fixed point + digit packing.
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>
#include "../paper_2212_11142_b200/csrc/matern.cuh"

using namespace bx;

__device__ __forceinline__ uint32_t smem_u32(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }

template <int MODE>
__global__ void __launch_bounds__(1024) bench(const double* planes, const double* xs, int iters, int D,
                                             const double* exp2g, uint32_t* out, long long* clk, int mma) {
  __shared__ double s_exp2[64];
  __shared__ double sp[16 * 64];
  __shared__ __align__(1024) int8_t sB[96 * 32];
  __shared__ uint32_t tmem_base;
  __shared__ volatile int stop;
  __shared__ __align__(8) uint64_t bar;
  for (int i = threadIdx.x; i < 64; i += blockDim.x) s_exp2[i] = exp2g[i];
  for (int i = threadIdx.x; i < 16 * 64; i += blockDim.x) sp[i] = planes[i];
  __syncthreads();
  if (mma) {
    const int warp = threadIdx.x >> 5;
    if (threadIdx.x == 0) {
      stop = 0;
      asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(&bar)), "r"(1));
      asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    if (warp == 0) {
      asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(smem_u32(&tmem_base)), "r"(512));
      asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
    }
    asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
    __syncthreads();
    asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
    if (warp == 0) {
      const uint32_t tmem = tmem_base;
      const uint64_t bd = (uint64_t)((smem_u32(sB) >> 4) & 0x3FFF) | ((uint64_t)(128 >> 4) << 16) | ((uint64_t)(256 >> 4) << 32) | ((uint64_t)1 << 46);
      constexpr uint32_t idesc = (2u << 4) | (0u << 7) | (1u << 10) | ((uint32_t)(96 >> 3) << 17) | ((uint32_t)(128 >> 4) << 24);
      int n = 0;
      while (!stop) {
        for (int i = 0; i < 64; ++i)
          asm volatile("{\n\t.reg .pred p, e;\n\telect.sync _|e, 0xffffffff;\n\tsetp.ne.b32 p, %3, 0;\n\t"
                       "@e tcgen05.mma.cta_group::1.kind::i8 [%0], [%1], %2, %4, p;\n\t}\n"
                       ::"r"(tmem), "r"(tmem + 256), "l"(bd), "r"(1u), "n"(idesc));
        ++n;
        if (n > 20000) break;
      }
      asm volatile("{\n\t.reg .pred e;\n\telect.sync _|e, 0xffffffff;\n\t"
                   "@e tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];\n\t}\n" ::"r"(smem_u32(&bar)) : "memory");
      uint32_t done = 0;
      while (!done)
        asm volatile("{\n\t.reg .pred p;\n\tmbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\n\tselp.u32 %0, 1, 0, p;\n\t}\n"
                     : "=r"(done) : "r"(smem_u32(&bar)), "r"(0) : "memory");
      asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
    }
    if (warp == 0) {
      __syncwarp();
    }
  }
  if (mma && (threadIdx.x >> 5) == 0) {
    // wait for the others, then free TMEM
    while (stop < 1) {}
    asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem_base), "r"(512));
    return;
  }
  const MaternConst mc{1.3, 1.3 * kSqrt5, 1.3 * 5.0 / 3.0};
  uint32_t acc = 0;
  double x[16];
  for (int k = 0; k < D; ++k) x[k] = xs[(threadIdx.x + k) & 255];
  long long t0 = clock64();
  for (int it = 0; it < iters; ++it) {
    const int j0 = (it * 8) & 63;
    double W[8];
#pragma unroll
    for (int u = 0; u < 8; ++u) W[u] = 0.0;
    for (int k = 0; k < D; ++k) {
#pragma unroll
      for (int u = 0; u < 8; ++u) {
        const double d = x[k] - sp[k * 64 + j0 + u];
        W[u] = fma(d, d, W[u]);
      }
    }
#pragma unroll
    for (int u = 0; u < 8; ++u) {
      double kv;
      if (MODE == 2) kv = W[u] * 1.0000001;
      else kv = kstar_fast(W[u], mc, s_exp2);
      if (MODE == 1) acc += (uint32_t)__double_as_longlong(kv);
      else {
        unsigned long long X = __double2ull_rz(kv * 1099511627776.0);
        acc += (uint32_t)X ^ (uint32_t)(X >> 32);
      }
    }
  }
  long long t1 = clock64();
  out[blockIdx.x * blockDim.x + threadIdx.x] = acc;
  if (threadIdx.x == (mma ? 32 : 0)) clk[blockIdx.x] = t1 - t0;
  if (mma) {
    __threadfence_block();
    asm volatile("bar.sync 1, %0;" ::"r"((int)blockDim.x - 32));
    if (threadIdx.x == 32) stop = 1;
  }
}

int main() {
  setvbuf(stdout, nullptr, _IONBF, 0);
  double hp[16 * 64], hx[256], he[64];
  for (int i = 0; i < 16 * 64; ++i) hp[i] = (i % 97) * 0.013;
  for (int i = 0; i < 256; ++i) hx[i] = (i % 31) * 0.021;
  for (int j = 0; j < 64; ++j) he[j] = exp2((double)j / 64.0);
  double *dp, *dx, *de;
  uint32_t* dout;
  long long* dclk;
  cudaMalloc(&dp, sizeof hp); cudaMalloc(&dx, sizeof hx); cudaMalloc(&de, sizeof he);
  cudaMalloc(&dout, 148 * 2048 * 4); cudaMalloc(&dclk, 148 * 8);
  cudaMemcpy(dp, hp, sizeof hp, cudaMemcpyHostToDevice);
  cudaMemcpy(dx, hx, sizeof hx, cudaMemcpyHostToDevice);
  cudaMemcpy(de, he, sizeof he, cudaMemcpyHostToDevice);
  const int iters = 2000;
  for (int mode = 0; mode < 3; ++mode)
    for (int D : {10})
      for (int mma : {0, 1})
      for (int threads : {512}) {
        auto k = mode == 0 ? bench<0> : mode == 1 ? bench<1> : bench<2>;
        k<<<148, threads + 32 * mma>>>(dp, dx, iters, D, de, dout, dclk, mma);
        cudaError_t e = cudaDeviceSynchronize();
        if (e != cudaSuccess) { printf("err %s\n", cudaGetErrorString(e)); return 1; }
        long long h[148];
        cudaMemcpy(h, dclk, sizeof h, cudaMemcpyDeviceToHost);
        long long mx = 0;
        for (int i = 0; i < 148; ++i) mx = h[i] > mx ? h[i] : mx;
        const double per = (double)threads * iters * 8 / mx;
        printf("mma %d mode %d (%s) D=%2d threads=%d: %.2f K*/clk/SM  (%.1f clk per K* per SMSP-warp-lane)\n", mode,
               mma, mode == 0 ? "matern+fixed" : mode == 1 ? "matern only" : "distance only", D, threads, per, 1.0 / per);
      }
  return 0;
}
