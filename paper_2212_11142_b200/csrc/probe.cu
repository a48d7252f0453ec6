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

// ---- int8 tcgen05.mma rate (the denominator of the posterior's split-product contraction) -------
// One CTA per SM, one elected thread issues R back-to-back tcgen05.mma.kind::i8 (M = 128, K = 32)
// into TMEM accumulators.  shape 0: the dense peak shape (A and B from shared memory, N = 256);
// shape 1: the posterior's own per-(chunk, slice) block — A (candidate digits) from TMEM, five MMAs
// with N = 96, 80, 64, 48, 32 (gp_tc.cu MMA issuer).
namespace {

__device__ __forceinline__ uint32_t p_su32(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }
__device__ __forceinline__ uint64_t p_sdesc(const void* p) {
  return (uint64_t)((p_su32(p) >> 4) & 0x3FFF) | ((uint64_t)(128 >> 4) << 16) | ((uint64_t)(256 >> 4) << 32) |
         ((uint64_t)1 << 46);
}
template <int N>
constexpr uint32_t p_idesc() {
  return (2u << 4) | (0u << 7) | (1u << 10) | ((uint32_t)(N >> 3) << 17) | ((uint32_t)(128 >> 4) << 24);
}
__device__ __forceinline__ void p_mma_ss(uint32_t d, uint64_t a, uint64_t b, uint32_t idesc, uint32_t acc) {
  asm volatile("{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\t"
               "tcgen05.mma.cta_group::1.kind::i8 [%0], %1, %2, %3, p;\n\t}\n" ::"r"(d), "l"(a), "l"(b), "r"(idesc),
               "r"(acc));
}
__device__ __forceinline__ void p_mma_ts(uint32_t d, uint32_t a, uint64_t b, uint32_t idesc, uint32_t acc) {
  asm volatile("{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\t"
               "tcgen05.mma.cta_group::1.kind::i8 [%0], [%1], %2, %3, p;\n\t}\n" ::"r"(d), "r"(a), "l"(b), "r"(idesc),
               "r"(acc));
}

__global__ void probe_i8(int shape, int R) {
  __shared__ __align__(1024) int8_t sA[128 * 32];
  __shared__ __align__(1024) int8_t sB[256 * 32];
  __shared__ uint32_t tmem_base;
  __shared__ __align__(8) uint64_t bar;
  const int tid = threadIdx.x, warp = tid >> 5;
  for (int i = tid; i < 128 * 32; i += blockDim.x) sA[i] = (int8_t)(i * 7);
  for (int i = tid; i < 256 * 32; i += blockDim.x) sB[i] = (int8_t)(i * 13);
  if (warp == 0) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(p_su32(&tmem_base)), "r"(512));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
  }
  if (tid == 0) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(p_su32(&bar)), "r"(1));
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
  const uint32_t tmem = tmem_base;
  if (tid == 0) {
    const uint64_t ad = p_sdesc(sA), bd = p_sdesc(sB);
    for (int r = 0; r < R; ++r) {
      if (shape == 0) {
        p_mma_ss(tmem, ad, bd, p_idesc<256>(), r > 0 ? 1u : 0u);
      } else {  // accumulators at columns 0.., candidate digits at 256.. (as in the posterior)
        const uint32_t at = tmem + 256 + (uint32_t)((r & 3) * 40);
        p_mma_ts(tmem, at, bd, p_idesc<96>(), r > 0 ? 1u : 0u);
        p_mma_ts(tmem + 16, at + 8, bd, p_idesc<80>(), 1u);
        p_mma_ts(tmem + 32, at + 16, bd, p_idesc<64>(), 1u);
        p_mma_ts(tmem + 48, at + 24, bd, p_idesc<48>(), 1u);
        p_mma_ts(tmem + 64, at + 32, bd, p_idesc<32>(), 1u);
      }
    }
    asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(p_su32(&bar))
                 : "memory");
    uint32_t done = 0;
    while (!done)
      asm volatile("{\n\t.reg .pred p;\n\tmbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\n\tselp.u32 %0, 1, 0, p;\n\t}\n"
                   : "=r"(done) : "r"(p_su32(&bar)), "r"(0) : "memory");
  }
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
  __syncthreads();
  if (warp == 0) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem), "r"(512));
}

}  // namespace

// dense_mac_s: int8 MACs per second of the peak shape over all SMs; block_ns: time of one of the
// posterior's (chunk, slice) blocks (five MMAs, 1.31 M MACs) on one SM
extern "C" int bx_probe_int8(int device, double* dense_mac_s, double* block_ns) {
  if (cudaSetDevice(device) != cudaSuccess) return BX_ERR_CUDA;
  int sms = 0;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, device);
  cudaEvent_t a, b;
  cudaEventCreate(&a);
  cudaEventCreate(&b);
  const int R = 8192;
  float best[2] = {1e30f, 1e30f};
  for (int rep = 0; rep < 4; ++rep)
    for (int shape = 0; shape < 2; ++shape) {
      cudaEventRecord(a);
      probe_i8<<<sms, 128>>>(shape, shape == 0 ? R : R / 4);
      cudaEventRecord(b);
      cudaEventSynchronize(b);
      float ms = 0;
      cudaEventElapsedTime(&ms, a, b);
      if (rep > 0 && ms < best[shape]) best[shape] = ms;
    }
  cudaError_t e = cudaGetLastError();
  cudaEventDestroy(a);
  cudaEventDestroy(b);
  if (e != cudaSuccess) return BX_ERR_CUDA;
  if (dense_mac_s) *dense_mac_s = (double)sms * R * 128.0 * 256 * 32 / (best[0] * 1e-3);
  if (block_ns) *block_ns = best[1] * 1e6 / (R / 4);
  return BX_OK;
}
