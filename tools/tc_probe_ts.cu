// tc_probe_ts.cu — validate tcgen05.mma kind::i8 with the A operand in TMEM (written by
// tcgen05.st from registers) and B in shared memory, M = 128, N = 16, unsigned A x signed B.
#include <cstdio>
#include <cstdint>
#include <cstdlib>
#include <cuda_runtime.h>

constexpr int M = 128, N = 16, KSTEPS = 4, K = 32 * KSTEPS;

__device__ __forceinline__ uint32_t smem_u32(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }
__device__ __forceinline__ int kmajor_off(int r, int kb) { return (r >> 3) * 256 + (kb >> 4) * 128 + (r & 7) * 16 + (kb & 15); }
__device__ __forceinline__ uint64_t smem_desc(const void* p) {
  return (uint64_t)((smem_u32(p) >> 4) & 0x3FFF) | ((uint64_t)(128 >> 4) << 16) | ((uint64_t)(256 >> 4) << 32) | ((uint64_t)1 << 46);
}

__global__ void probe(const uint8_t* gA, const int8_t* gB, int32_t* gD, int mode) {
  __shared__ __align__(1024) int8_t sB[KSTEPS][N * 32];
  __shared__ uint32_t tmem_base;
  __shared__ __align__(8) uint64_t bar;
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  for (int i = tid; i < KSTEPS * N * 32; i += blockDim.x) {
    const int ks = i / (N * 32), r = (i / 32) % N, kb = i % 32;
    sB[ks][kmajor_off(r, kb)] = gB[(size_t)r * K + ks * 32 + kb];
  }
  if (warp == 0) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(smem_u32(&tmem_base)), "r"(64));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
  }
  if (tid == 0) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(&bar)), "r"(1));
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
  const uint32_t tmem = tmem_base;
  // A row m = lane (32 * warp + lane) -> TMEM columns 32..63 (4 bytes per column, K-order)
  const int row = warp * 32 + lane;
  for (int c0 = 0; c0 < K / 4; c0 += 8) {
    uint32_t v[8];
    for (int j = 0; j < 8; ++j) {
      const int k = 4 * (c0 + j);
      const uint8_t* a = gA + (size_t)row * K + k;
      if (mode == 0) v[j] = a[0] | (a[1] << 8) | (a[2] << 16) | ((uint32_t)a[3] << 24);
      else v[j] = a[3] | (a[2] << 8) | (a[1] << 16) | ((uint32_t)a[0] << 24);
    }
    const uint32_t addr = tmem + ((uint32_t)(warp * 32) << 16) + 32 + c0;
    asm volatile("tcgen05.st.sync.aligned.32x32b.x8.b32 [%0], {%1,%2,%3,%4,%5,%6,%7,%8};" ::"r"(addr),
                 "r"(v[0]), "r"(v[1]), "r"(v[2]), "r"(v[3]), "r"(v[4]), "r"(v[5]), "r"(v[6]), "r"(v[7]));
  }
  asm volatile("tcgen05.wait::st.sync.aligned;" ::: "memory");
  asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
  const uint32_t idesc = (2u << 4) | (0u << 7) | (1u << 10) | ((uint32_t)(N >> 3) << 17) | ((uint32_t)(M >> 4) << 24);
  if (tid == 0) {
    for (int ks = 0; ks < KSTEPS; ++ks) {
      const uint32_t a_t = tmem + 32 + ks * 8;
      const uint64_t bd = smem_desc(sB[ks]);
      asm volatile("{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\t"
                   "tcgen05.mma.cta_group::1.kind::i8 [%0], [%1], %2, %3, p;\n\t}\n" ::"r"(tmem),
                   "r"(a_t), "l"(bd), "r"(idesc), "r"(ks > 0 ? 1u : 0u));
    }
    asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(smem_u32(&bar)) : "memory");
  }
  uint32_t done = 0;
  while (!done)
    asm volatile("{\n\t.reg .pred p;\n\tmbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\n\tselp.u32 %0, 1, 0, p;\n\t}\n"
                 : "=r"(done) : "r"(smem_u32(&bar)), "r"(0) : "memory");
  asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
  for (int c0 = 0; c0 < N; c0 += 8) {
    uint32_t v[8];
    const uint32_t addr = tmem + ((uint32_t)(warp * 32) << 16) + c0;
    asm volatile("tcgen05.ld.sync.aligned.32x32b.x8.b32 {%0, %1, %2, %3, %4, %5, %6, %7}, [%8];"
                 : "=r"(v[0]), "=r"(v[1]), "=r"(v[2]), "=r"(v[3]), "=r"(v[4]), "=r"(v[5]), "=r"(v[6]), "=r"(v[7])
                 : "r"(addr));
    asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
    for (int j = 0; j < 8; ++j) gD[row * N + c0 + j] = (int32_t)v[j];
  }
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
  __syncthreads();
  if (warp == 0) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem), "r"(64));
}

int main() {
  uint8_t* hA = (uint8_t*)malloc(M * K);
  int8_t* hB = (int8_t*)malloc(N * K);
  srand(1);
  for (int i = 0; i < M * K; ++i) hA[i] = (uint8_t)(rand() % 256);
  for (int i = 0; i < N * K; ++i) hB[i] = (int8_t)(rand() % 256 - 128);
  uint8_t* dA;
  int8_t* dB;
  int32_t* dD;
  cudaMalloc(&dA, M * K);
  cudaMalloc(&dB, N * K);
  cudaMalloc(&dD, M * N * 4);
  cudaMemcpy(dA, hA, M * K, cudaMemcpyHostToDevice);
  cudaMemcpy(dB, hB, N * K, cudaMemcpyHostToDevice);
  int32_t* hD = (int32_t*)malloc(M * N * 4);
  int rc = 1;
  for (int mode = 0; mode < 2; ++mode) {
    cudaMemset(dD, 0, M * N * 4);
    probe<<<1, 128>>>(dA, dB, dD, mode);
    cudaError_t e = cudaDeviceSynchronize();
    printf("mode %d kernel: %s\n", mode, cudaGetErrorString(e));
    if (e != cudaSuccess) return 2;
    cudaMemcpy(hD, dD, M * N * 4, cudaMemcpyDeviceToHost);
    int bad = 0;
    for (int i = 0; i < M; ++i)
      for (int j = 0; j < N; ++j) {
        int32_t ref = 0;
        for (int k = 0; k < K; ++k) ref += (int32_t)hA[i * K + k] * (int32_t)hB[j * K + k];
        if (ref != hD[i * N + j] && bad++ < 3) printf("  mismatch D[%d][%d] = %d, want %d\n", i, j, hD[i * N + j], ref);
      }
    printf("A-in-TMEM kind::i8 u8 x s8, N=%d, byte order %d: %s (%d mismatches of %d)\n", N, mode, bad ? "FAIL" : "PASS", bad, M * N);
    if (!bad) rc = 0;
  }
  return rc;
}
