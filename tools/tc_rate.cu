// tc_rate.cu — cycles per tcgen05.mma kind::i8 (M = 128, K = 32) for A in SMEM (SS) or TMEM (TS)
// and several N, measured by one thread issuing R back-to-back MMAs into one accumulator.
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>

__device__ __forceinline__ uint32_t smem_u32(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }
__device__ __forceinline__ uint64_t smem_desc(const void* p) {
  return (uint64_t)((smem_u32(p) >> 4) & 0x3FFF) | ((uint64_t)(128 >> 4) << 16) | ((uint64_t)(256 >> 4) << 32) | ((uint64_t)1 << 46);
}

__global__ void rate(int N, int ts, int R, int rot, long long* out) {
  __shared__ __align__(1024) int8_t sA[4][128 * 32];
  __shared__ __align__(1024) int8_t sB[2][256 * 32];
  __shared__ uint32_t tmem_base;
  __shared__ __align__(8) uint64_t bar;
  const int tid = threadIdx.x, warp = tid >> 5;
  for (int i = tid; i < 4 * 128 * 32; i += blockDim.x) (&sA[0][0])[i] = (int8_t)(i * 7);
  for (int i = tid; i < 2 * 256 * 32; i += blockDim.x) (&sB[0][0])[i] = (int8_t)(i * 13);
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
  const uint32_t idesc = (2u << 4) | (0u << 7) | (1u << 10) | ((uint32_t)(N >> 3) << 17) | ((uint32_t)(128 >> 4) << 24);
  if (tid == 0) {
    long long t0 = clock64();
    for (int r = 0; r < R; ++r) {
      const uint64_t bd = smem_desc(sB[r & 1]);
      if (ts) {
        const uint32_t a_t = tmem + 256 + (r & 7) * 8;
        asm volatile("{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\t"
                     "tcgen05.mma.cta_group::1.kind::i8 [%0], [%1], %2, %3, p;\n\t}\n" ::"r"(tmem + (uint32_t)((r % rot) * N)),
                     "r"(a_t), "l"(bd), "r"(idesc), "r"(r > 0 ? 1u : 0u));
      } else {
        const uint64_t ad = smem_desc(sA[r & 3]);
        asm volatile("{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\t"
                     "tcgen05.mma.cta_group::1.kind::i8 [%0], %1, %2, %3, p;\n\t}\n" ::"r"(tmem + (uint32_t)((r % rot) * N)),
                     "l"(ad), "l"(bd), "r"(idesc), "r"(r > 0 ? 1u : 0u));
      }
    }
    asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(smem_u32(&bar)) : "memory");
    uint32_t done = 0;
    while (!done)
      asm volatile("{\n\t.reg .pred p;\n\tmbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\n\tselp.u32 %0, 1, 0, p;\n\t}\n"
                   : "=r"(done) : "r"(smem_u32(&bar)), "r"(0) : "memory");
    out[blockIdx.x] = clock64() - t0;
  }
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
  __syncthreads();
  if (warp == 0) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem), "r"(512));
}

int main() {
  long long* d;
  cudaMalloc(&d, 148 * 8);
  long long h[148];
  const int R = 4096;
  int Ns[] = {16, 32, 64, 128, 256};
  for (int ts = 0; ts < 2; ++ts)
    for (int N : Ns)
    for (int rot : {1, 2, 4, 8}) {
      if (rot * N > 256) continue;
      for (int grid : {148}) {
        rate<<<grid, 128>>>(N, ts, R, rot, d);
        cudaError_t e = cudaDeviceSynchronize();
        if (e != cudaSuccess) { printf("error %s\n", cudaGetErrorString(e)); return 1; }
        cudaMemcpy(h, d, grid * 8, cudaMemcpyDeviceToHost);
        long long mx = 0;
        for (int i = 0; i < grid; ++i) mx = h[i] > mx ? h[i] : mx;
        printf("%s N=%3d rot=%d grid=%3d: %6.1f clk/MMA (floor %d), %.0f MAC/clk/SM\n", ts ? "TS" : "SS", N, rot, grid,
               (double)mx / R, 128 * N / 256, 128.0 * N * 32 * R / mx);
      }
    }
  return 0;
}
