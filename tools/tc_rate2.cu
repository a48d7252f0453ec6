// tc_rate2.cu — issue cost of unrolled tcgen05.mma kind::i8 sequences (the gp_tc pattern):
// 20 digit-pair MMAs per block with compile-time descriptor / TMEM offsets.
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>

__device__ __forceinline__ uint32_t smem_u32(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }
__device__ __forceinline__ uint64_t smem_desc(const void* p) {
  return (uint64_t)((smem_u32(p) >> 4) & 0x3FFF) | ((uint64_t)(128 >> 4) << 16) | ((uint64_t)(256 >> 4) << 32) | ((uint64_t)1 << 46);
}

template <int N, bool TS, int MODE>
__global__ void rate(int R, long long* out) {
  extern __shared__ __align__(1024) int8_t sm[];
  int8_t* sA = sm;              // 5 x 4 KB
  int8_t* sB = sm + 5 * 4096;   // 6 x N*32
  __shared__ uint32_t tmem_base;
  __shared__ __align__(8) uint64_t bar;
  const int tid = threadIdx.x, warp = tid >> 5;
  for (int i = tid; i < 5 * 4096 + 6 * N * 32; i += blockDim.x) sm[i] = (int8_t)(i * 7);
  if (warp == 0) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(smem_u32(&tmem_base)), "r"(512));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
  }
  if (tid == 0) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(&bar)), "r"(1));
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
  const uint32_t tmem = tmem_base;
  constexpr uint32_t idesc = (2u << 4) | (0u << 7) | (1u << 10) | ((uint32_t)(N >> 3) << 17) | ((uint32_t)(128 >> 4) << 24);
  if (MODE == 0 ? tid == 0 : warp == 0) {
    const uint64_t adesc0 = smem_desc(sA), bdesc0 = smem_desc(sB);
    long long t0 = clock64();
    for (int r = 0; r < R; ++r) {
#pragma unroll
      for (int da = 0; da < 6; ++da)
#pragma unroll
        for (int db = 0; db < 5; ++db)
          if (da + db < 6) {
            const uint32_t d = tmem + (uint32_t)((da + db) * N);
            const uint64_t bd = bdesc0 + (uint64_t)((da * N * 32) >> 4);
            const uint32_t acc = (r > 0 || da > 0) ? 1u : 0u;
            if (MODE == 1) {
              const uint64_t ad = adesc0 + (uint64_t)((db * 4096) >> 4);
              asm volatile("{\n\t.reg .pred p, e;\n\telect.sync _|e, 0xffffffff;\n\tsetp.ne.b32 p, %4, 0;\n\t"
                           "@e tcgen05.mma.cta_group::1.kind::i8 [%0], %1, %2, %3, p;\n\t}\n" ::"r"(d),
                           "l"(ad), "l"(bd), "n"(idesc), "r"(acc));
            } else if (TS) {
              const uint32_t a_t = tmem + 256 + db * 8;
              asm volatile("{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\t"
                           "tcgen05.mma.cta_group::1.kind::i8 [%0], [%1], %2, %3, p;\n\t}\n" ::"r"(d),
                           "r"(a_t), "l"(bd), "n"(idesc), "r"(acc));
            } else {
              const uint64_t ad = adesc0 + (uint64_t)((db * 4096) >> 4);
              asm volatile("{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\t"
                           "tcgen05.mma.cta_group::1.kind::i8 [%0], %1, %2, %3, p;\n\t}\n" ::"r"(d),
                           "l"(ad), "l"(bd), "n"(idesc), "r"(acc));
            }
          }
    }
    if (MODE == 1)
      asm volatile("{\n\t.reg .pred e;\n\telect.sync _|e, 0xffffffff;\n\t"
                   "@e tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];\n\t}\n" ::"r"(smem_u32(&bar)) : "memory");
    else
      asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(smem_u32(&bar)) : "memory");
    uint32_t done = 0;
    while (!done)
      asm volatile("{\n\t.reg .pred p;\n\tmbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\n\tselp.u32 %0, 1, 0, p;\n\t}\n"
                   : "=r"(done) : "r"(smem_u32(&bar)), "r"(0) : "memory");
    if (tid == 0) out[blockIdx.x] = clock64() - t0;
  }
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
  __syncthreads();
  if (warp == 0) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem), "r"(512));
}

template <int N, bool TS, int MODE = 0>
void run(long long* d) {
  const int R = 256, smem = 5 * 4096 + 6 * N * 32;
  cudaFuncSetAttribute(rate<N, TS, MODE>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
  rate<N, TS, MODE><<<148, 128, smem>>>(R, d);
  cudaError_t e = cudaDeviceSynchronize();
  if (e != cudaSuccess) { printf("error %s\n", cudaGetErrorString(e)); return; }
  long long h[148];
  cudaMemcpy(h, d, 148 * 8, cudaMemcpyDeviceToHost);
  long long mx = 0;
  for (int i = 0; i < 148; ++i) mx = h[i] > mx ? h[i] : mx;
  printf("%s mode %d N=%3d: %6.1f clk/MMA (floor %d), %.0f MAC/clk/SM\n", TS ? "TS" : "SS", MODE, N, (double)mx / (R * 20),
         128 * N / 256, 128.0 * N * 32 * R * 20 / mx);
}

int main() {
  setvbuf(stdout, nullptr, _IONBF, 0);
  long long* d;
  cudaMalloc(&d, 148 * 8);
  run<16, false>(d); run<32, false>(d); run<64, false>(d); run<80, false>(d);
  run<16, false, 1>(d); run<32, false, 1>(d); run<64, false, 1>(d); run<80, false, 1>(d);
  run<16, true>(d); run<32, true>(d); run<64, true>(d); run<80, true>(d);
  return 0;
}
