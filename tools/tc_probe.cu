// tc_probe.cu — validate the tcgen05.mma kind::i8 encoding used by the Ozaki contraction:
// K-major SWIZZLE_NONE smem descriptors, the instruction descriptor, TMEM alloc / ld, commit.
// D[M=128][N=64] (s32, TMEM) = sum over KSTEPS of A[128 x 32k] (s8) * B[64 x 32k]^T (s8).
#include <cstdio>
#include <cstdint>
#include <cstdlib>
#include <cuda_runtime.h>

constexpr int M = 128, N = 64, KSTEPS = 4;

__device__ __forceinline__ uint32_t smem_u32(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }

// K-major, no swizzle: core matrix = 8 rows x 16 bytes (128 B contiguous); layout per K-step
// [row group][k half][8 rows][16 B]  ->  SBO (row-group stride) = 256 B, LBO (k-half stride) = 128 B
__device__ __forceinline__ int kmajor_off(int r, int kb) {
  return (r >> 3) * 256 + (kb >> 4) * 128 + (r & 7) * 16 + (kb & 15);
}

__device__ __forceinline__ uint64_t smem_desc(const void* p, uint32_t lbo, uint32_t sbo) {
  uint64_t d = 0;
  d |= (uint64_t)((smem_u32(p) >> 4) & 0x3FFF);
  d |= (uint64_t)((lbo >> 4) & 0x3FFF) << 16;
  d |= (uint64_t)((sbo >> 4) & 0x3FFF) << 32;
  d |= (uint64_t)1 << 46;  // version 1 (sm100)
  return d;                 // base offset 0, lbo mode 0, layout SWIZZLE_NONE (0)
}

__global__ void probe(const int8_t* gA, const int8_t* gB, int32_t* gD) {
  __shared__ __align__(1024) int8_t sA[KSTEPS][M * 32];
  __shared__ __align__(1024) int8_t sB[KSTEPS][N * 32];
  __shared__ uint32_t tmem_base;
  __shared__ __align__(8) uint64_t bar;
  const int tid = threadIdx.x, warp = tid >> 5;
  for (int i = tid; i < KSTEPS * M * 32; i += blockDim.x) {
    const int ks = i / (M * 32), r = (i / 32) % M, kb = i % 32;
    sA[ks][kmajor_off(r, kb)] = gA[(size_t)r * (32 * KSTEPS) + ks * 32 + kb];
  }
  for (int i = tid; i < KSTEPS * N * 32; i += blockDim.x) {
    const int ks = i / (N * 32), r = (i / 32) % N, kb = i % 32;
    sB[ks][kmajor_off(r, kb)] = gB[(size_t)r * (32 * KSTEPS) + ks * 32 + kb];
  }
  if (warp == 0) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(smem_u32(&tmem_base)), "r"(64));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
  }
  if (tid == 0) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(&bar)), "r"(1));
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  asm volatile("fence.proxy.async.shared::cta;" ::: "memory");  // smem writes -> async proxy
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
  const uint32_t tmem = tmem_base;
  const uint32_t idesc = (2u << 4) | (1u << 7) | (1u << 10) | ((uint32_t)(N >> 3) << 17) | ((uint32_t)(M >> 4) << 24);
  if (tid == 0) {
    for (int ks = 0; ks < KSTEPS; ++ks) {
      const uint64_t ad = smem_desc(sA[ks], 128, 256), bd = smem_desc(sB[ks], 128, 256);
      const uint32_t acc = ks > 0 ? 1u : 0u;
      asm volatile(
          "{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\t"
          "tcgen05.mma.cta_group::1.kind::i8 [%0], %1, %2, %3, p;\n\t}\n" ::"r"(tmem),
          "l"(ad), "l"(bd), "r"(idesc), "r"(acc));
    }
    asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(smem_u32(&bar)) : "memory");
  }
  // wait for the MMAs
  uint32_t done = 0;
  while (!done)
    asm volatile("{\n\t.reg .pred p;\n\tmbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\n\tselp.u32 %0, 1, 0, p;\n\t}\n"
                 : "=r"(done) : "r"(smem_u32(&bar)), "r"(0) : "memory");
  asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
  // each warp w (0..3) reads TMEM lanes 32w..32w+31 (rows of D), 64 columns in 8 chunks of 8
  const int row = warp * 32 + (tid & 31);
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
  const int K = 32 * KSTEPS;
  int8_t *hA = (int8_t*)malloc(M * K), *hB = (int8_t*)malloc(N * K);
  srand(1);
  for (int i = 0; i < M * K; ++i) hA[i] = (int8_t)(rand() % 129 - 64);
  for (int i = 0; i < N * K; ++i) hB[i] = (int8_t)(rand() % 129 - 64);
  int8_t *dA, *dB;
  int32_t* dD;
  cudaMalloc(&dA, M * K);
  cudaMalloc(&dB, N * K);
  cudaMalloc(&dD, M * N * 4);
  cudaMemcpy(dA, hA, M * K, cudaMemcpyHostToDevice);
  cudaMemcpy(dB, hB, N * K, cudaMemcpyHostToDevice);
  cudaMemset(dD, 0, M * N * 4);
  probe<<<1, 128>>>(dA, dB, dD);
  cudaError_t e = cudaDeviceSynchronize();
  printf("kernel: %s\n", cudaGetErrorString(e));
  int32_t* hD = (int32_t*)malloc(M * N * 4);
  cudaMemcpy(hD, dD, M * N * 4, cudaMemcpyDeviceToHost);
  int bad = 0;
  for (int i = 0; i < M; ++i)
    for (int j = 0; j < N; ++j) {
      int32_t ref = 0;
      for (int k = 0; k < K; ++k) ref += (int32_t)hA[i * K + k] * (int32_t)hB[j * K + k];
      if (ref != hD[i * N + j] && bad++ < 5) printf("mismatch D[%d][%d] = %d, want %d\n", i, j, hD[i * N + j], ref);
    }
  printf("tcgen05 kind::i8 probe: %s (%d mismatches of %d)\n", bad ? "FAIL" : "PASS", bad, M * N);
  return bad != 0;
}
