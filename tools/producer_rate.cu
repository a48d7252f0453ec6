// producer_rate.cu — the tensor-core posterior's producer loop in isolation (development aid):
// centred dot-product distances over D = 10 coordinates (broadcast 16-byte shared loads), the
// Matérn K* in 40-bit fixed point (kstar_fixed of gp_tc.cu), digit packing; no tensor memory.
// Variants knock out one ingredient at a time to find what bounds the loop.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o tools/producer_rate tools/producer_rate.cu
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>

__device__ __forceinline__ double rsqrt_approx(double x) {
  double y;
  asm("rsqrt.approx.ftz.f64 %0, %1;" : "=d"(y) : "d"(x));
  return y;
}

template <int V>
__device__ __forceinline__ unsigned long long kstar_fixed(double W, double s0, double s1, double s2, const double* tab) {
  const double w = W + 1e-300;
  double y0;
  if (V == 8) y0 = __hiloint2double(0x5fe6eb50 - (__double2hiint(w) >> 1), 0);  // timing only: integer seed
  else y0 = rsqrt_approx(w);
  const double y0h = __hiloint2double(__double2hiint(y0) - (1 << 20), __double2loint(y0));
  const double d0 = w * y0;
  const double e0h = fma(-d0, y0h, 0.5);
  const double d = fma(d0, e0h, d0);
  const double t = fma(d, -825.8468306507675, 6755399441055744.0);
  const int k = max(__double2loint(t), -256 * 900);
  const double kf = t - 6755399441055744.0;
  double r = fma(kf, 0.0012108782921131933, d);
  r = fma(kf, 1.8708673154509723e-13, r);
  double p = fma(r, 25.0 / 24.0, -1.8633899812498247);
  p = fma(r, p, 2.5);
  p = fma(r, p, -2.23606797749979);
  p = fma(r, p, 1.0);
  double tj;
  if (V == 1) tj = 1.0 + (k & 255) * 1e-3;   // no table load
  else tj = tab[k & 255];
  const double scale = __hiloint2double(__double2hiint(tj) + ((k >> 8) << 20), __double2loint(tj));
  const double X = fma(fma(s2, W, fma(s1, d, s0)), p * scale, 4503599627370496.0);
  return (unsigned long long)__double_as_longlong(X);
}

// V: 0 full loop, 1 no exp table load, 2 distances from registers (no plane loads),
//    3 distance only (no Matérn), 4 Matérn only (W from a register recurrence)
template <int V>
__global__ void __launch_bounds__(512, 1) bench(const double* planes, const double* xs, const double* tabg, int iters,
                                                uint32_t* out, long long* clk) {
  __shared__ __align__(16) double sp[10 * 256 + 256];
  __shared__ double tab[256];
  for (int i = threadIdx.x; i < 10 * 256 + 256; i += blockDim.x) sp[i] = planes[i % 2560] * 0.01;
  for (int i = threadIdx.x; i < 256; i += blockDim.x) tab[i] = tabg[i];
  __syncthreads();
  double xr[10], xx = 0.0;
#pragma unroll
  for (int k = 0; k < 10; ++k) {
    xr[k] = xs[(threadIdx.x * 7 + k) & 255] * 0.1;
    xx = fma(xr[k], xr[k], xx);
  }
  double xr2[10], xx2 = 0.0;
#pragma unroll
  for (int k = 0; k < 10; ++k) {
    xr2[k] = xs[(threadIdx.x * 5 + k + 3) & 255] * 0.1;
    xx2 = fma(xr2[k], xr2[k], xx2);
  }
  const double s0 = 1099511627776.0 * 0.7, s1 = s0 * 2.2360679774997896, s2 = s0 * 5.0 / 3.0;
  uint32_t acc = 0;
  const int part = (threadIdx.x >> 7) & 3;
  long long t0 = clock64();
  for (int it = 0; it < iters; ++it) {
    const int j0 = ((it * 32) & 255) + 8 * part;
    double W[8];
#pragma unroll
    for (int u = 0; u < 8; ++u) W[u] = 0.0;
    if (V == 2) {
#pragma unroll
      for (int k = 0; k < 10; ++k)
#pragma unroll
        for (int u = 0; u < 8; ++u) W[u] = fma(xr[k], xr[(k + u) % 10] + it, W[u]);
    } else if (V != 4) {
#pragma unroll
      for (int k = 0; k < 10; ++k) {
        const double2* pl = reinterpret_cast<const double2*>(sp + k * 256 + j0);
#pragma unroll
        for (int u = 0; u < 4; ++u) {
          const double2 y = pl[u];
          W[2 * u] = fma(xr[k], y.x, W[2 * u]);
          W[2 * u + 1] = fma(xr[k], y.y, W[2 * u + 1]);
        }
      }
    } else {
#pragma unroll
      for (int u = 0; u < 8; ++u) W[u] = xx + u + (it & 7);
    }
    if (V == 5) {  // lane pairs: 2 candidates x 4 columns per thread, half the plane loads
      const int jh = j0 + 4 * (threadIdx.x & 1);
      double Wb[8];
      const double2* yyp = reinterpret_cast<const double2*>(sp + 2560 + jh);
#pragma unroll
      for (int u = 0; u < 2; ++u) {
        const double2 y = yyp[u];
        Wb[2 * u] = xx + y.x; Wb[2 * u + 1] = xx + y.y;
        Wb[4 + 2 * u] = xx2 + y.x; Wb[4 + 2 * u + 1] = xx2 + y.y;
      }
#pragma unroll
      for (int k = 0; k < 10; ++k) {
        const double2* pl = reinterpret_cast<const double2*>(sp + k * 256 + jh);
#pragma unroll
        for (int u = 0; u < 2; ++u) {
          const double2 y = pl[u];
          Wb[2 * u] = fma(xr[k], y.x, Wb[2 * u]);
          Wb[2 * u + 1] = fma(xr[k], y.y, Wb[2 * u + 1]);
          Wb[4 + 2 * u] = fma(xr2[k], y.x, Wb[4 + 2 * u]);
          Wb[4 + 2 * u + 1] = fma(xr2[k], y.y, Wb[4 + 2 * u + 1]);
        }
      }
      uint32_t lo[8], hi[8];
#pragma unroll
      for (int u = 0; u < 8; ++u) {
        const unsigned long long X = kstar_fixed<0>(fabs(Wb[u]), s0, s1, s2, tab);
        lo[u] = (uint32_t)X;
        hi[u] = (uint32_t)(X >> 32);
      }
      uint32_t dw[2][5];
#pragma unroll
      for (int qd = 0; qd < 2; ++qd) {
        const uint32_t p01 = __byte_perm(lo[4 * qd], lo[4 * qd + 1], 0x5140), p23 = __byte_perm(lo[4 * qd + 2], lo[4 * qd + 3], 0x5140);
        const uint32_t q01 = __byte_perm(lo[4 * qd], lo[4 * qd + 1], 0x7362), q23 = __byte_perm(lo[4 * qd + 2], lo[4 * qd + 3], 0x7362);
        const uint32_t h01 = __byte_perm(hi[4 * qd], hi[4 * qd + 1], 0x5140), h23 = __byte_perm(hi[4 * qd + 2], hi[4 * qd + 3], 0x5140);
        dw[qd][0] = __byte_perm(h01, h23, 0x5410); dw[qd][1] = __byte_perm(q01, q23, 0x7632);
        dw[qd][2] = __byte_perm(q01, q23, 0x5410); dw[qd][3] = __byte_perm(p01, p23, 0x7632);
        dw[qd][4] = __byte_perm(p01, p23, 0x5410);
      }
      // even lanes keep candidate 0's words and send candidate 1's; odd lanes the reverse
      const bool odd = threadIdx.x & 1;
#pragma unroll
      for (int b = 0; b < 5; ++b) {
        const uint32_t send = odd ? dw[0][b] : dw[1][b];
        const uint32_t got = __shfl_xor_sync(0xffffffffu, send, 1);
        acc += (odd ? dw[1][b] : dw[0][b]) ^ got;
      }
      continue;
    }
    const double2* yy2 = reinterpret_cast<const double2*>(sp + 2560 + j0);
#pragma unroll
    for (int u = 0; u < 4; ++u) {
      const double2 y = V == 4 ? make_double2(0.1, 0.2) : yy2[u];
      W[2 * u] = fma(-2.0, W[2 * u], xx + y.x);
      W[2 * u + 1] = fma(-2.0, W[2 * u + 1], xx + y.y);
    }
    uint32_t lo[8], hi[8];
#pragma unroll
    for (int u = 0; u < 8; ++u) {
      unsigned long long X;
      if (V == 3) X = (unsigned long long)__double_as_longlong(W[u]);
      else X = kstar_fixed<V == 1 ? 1 : (V == 8 ? 8 : 0)>(fabs(W[u]), s0, s1, s2, tab);
      lo[u] = (uint32_t)X;
      hi[u] = (uint32_t)(X >> 32);
    }
#pragma unroll
    for (int qd = 0; qd < 2; ++qd) {
      const uint32_t p01 = __byte_perm(lo[4 * qd], lo[4 * qd + 1], 0x5140), p23 = __byte_perm(lo[4 * qd + 2], lo[4 * qd + 3], 0x5140);
      const uint32_t q01 = __byte_perm(lo[4 * qd], lo[4 * qd + 1], 0x7362), q23 = __byte_perm(lo[4 * qd + 2], lo[4 * qd + 3], 0x7362);
      const uint32_t h01 = __byte_perm(hi[4 * qd], hi[4 * qd + 1], 0x5140), h23 = __byte_perm(hi[4 * qd + 2], hi[4 * qd + 3], 0x5140);
      acc += __byte_perm(h01, h23, 0x5410) ^ __byte_perm(q01, q23, 0x7632) ^ __byte_perm(q01, q23, 0x5410) ^
             __byte_perm(p01, p23, 0x7632) ^ __byte_perm(p01, p23, 0x5410);
    }
  }
  long long t1 = clock64();
  out[blockIdx.x * blockDim.x + threadIdx.x] = acc;
  if (threadIdx.x == 0) clk[blockIdx.x] = t1 - t0;
}

int main() {
  static double hp[2560], hx[256], he[256];
  for (int i = 0; i < 2560; ++i) hp[i] = (i % 97) * 0.013 - 0.6;
  for (int i = 0; i < 256; ++i) hx[i] = (i % 31) * 0.021 - 0.3;
  for (int j = 0; j < 256; ++j) he[j] = exp2((double)j / 256.0);
  double *dp, *dx, *de;
  uint32_t* dout;
  long long* dclk;
  cudaMalloc(&dp, sizeof hp); cudaMalloc(&dx, sizeof hx); cudaMalloc(&de, sizeof he);
  cudaMalloc(&dout, 148 * 512 * 4); cudaMalloc(&dclk, 148 * 8);
  cudaMemcpy(dp, hp, sizeof hp, cudaMemcpyHostToDevice);
  cudaMemcpy(dx, hx, sizeof hx, cudaMemcpyHostToDevice);
  cudaMemcpy(de, he, sizeof he, cudaMemcpyHostToDevice);
  const char* names[] = {"full loop", "no exp-table load", "distances from registers", "distance only",
                         "Matern only", "lane pairs (2 cand x 4 col)", "full loop, 8 warps", "lane pairs, 8 warps", "no MUFU (integer seed)"};
  const int iters = 4000;
  for (int v = 0; v < 9; ++v) {
    for (int rep = 0; rep < 2; ++rep) {
      switch (v) {
        case 0: bench<0><<<148, 512>>>(dp, dx, de, iters, dout, dclk); break;
        case 1: bench<1><<<148, 512>>>(dp, dx, de, iters, dout, dclk); break;
        case 2: bench<2><<<148, 512>>>(dp, dx, de, iters, dout, dclk); break;
        case 3: bench<3><<<148, 512>>>(dp, dx, de, iters, dout, dclk); break;
        case 4: bench<4><<<148, 512>>>(dp, dx, de, iters, dout, dclk); break;
        case 5: bench<5><<<148, 512>>>(dp, dx, de, iters, dout, dclk); break;
        case 6: bench<0><<<148, 256>>>(dp, dx, de, iters, dout, dclk); break;
        case 7: bench<5><<<148, 256>>>(dp, dx, de, iters, dout, dclk); break;
        case 8: bench<8><<<148, 512>>>(dp, dx, de, iters, dout, dclk); break;
      }
      cudaDeviceSynchronize();
    }
    long long h[148];
    cudaMemcpy(h, dclk, sizeof h, cudaMemcpyDeviceToHost);
    long long mx = 0;
    for (int i = 0; i < 148; ++i) mx = h[i] > mx ? h[i] : mx;
    const double per = (v >= 6 ? 256.0 : 512.0) * iters * 8 / mx;
    printf("%-26s %.3f K*/clk/SM  (%.1f SMSP clk per 32 K*)\n", names[v], per, 4 * 32 / per);
  }
  printf("status %s\n", cudaGetErrorString(cudaGetLastError()));
  return 0;
}
