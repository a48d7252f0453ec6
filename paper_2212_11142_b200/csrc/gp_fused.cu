// gp_fused.cu — register-resident posterior + EI kernel (n <= 8*MT - 1 training points).
//
// Per warp: 8 candidates = one DMMA n-tile.  The whole output column block [v ; mean] for those 8
// candidates (rows 0..8*MT-1 of A = [L^-1 ; alpha^T]) lives in registers, so K* never touches
// shared memory: every k-step (4 training columns) each lane evaluates exactly the Matérn value its
// B fragment needs, K*[c = lane/4][j = k0 + lane%4] (surrogate.py:318-321), and the warp issues one
// DMMA per m-tile that intersects the lower triangle (surrogate.py:322-325).
//
// A is streamed through shared memory in 16-column panels by one-dimensional TMA bulk copies
// (cp.async.bulk + mbarrier complete_tx), double-buffered and shared by every warp of the CTA;
// rows above the diagonal block of a panel are never copied.  The epilogue de-standardises, takes
// max(σ - Σv², 0) and the expected improvement (acquisition.py:40-51) and writes EI (or mean /
// variance for predict_batch).  The feasibility weight, eps_f filter and summaries are applied by
// the forest / summary kernels after it (score_summary.cu, forest.cu).
#include "bx_common.cuh"
#include "matern.cuh"

namespace bx {

namespace {

constexpr int kKC = 16;        // panel width (columns of A per TMA copy; 32 measured no faster)
constexpr int kKCP = kKC + 4;  // padded panel row (doubles): == 4 (mod 16), fragment loads hit 2 wavefronts

__device__ __forceinline__ uint32_t smem_u32(const void* p) {
  return (uint32_t)__cvta_generic_to_shared(p);
}

__device__ __forceinline__ void mbar_init(uint64_t* bar, uint32_t count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;\n" ::"r"(smem_u32(bar)), "r"(count));
}

__device__ __forceinline__ void mbar_expect_tx(uint64_t* bar, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;\n" ::"r"(smem_u32(bar)),
               "r"(bytes)
               : "memory");
}

__device__ __forceinline__ void mbar_wait(uint64_t* bar, uint32_t phase) {
  uint32_t done = 0;
  while (!done) {
    asm volatile(
        "{\n\t.reg .pred p;\n\t"
        "mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\n\t"
        "selp.u32 %0, 1, 0, p;\n\t}\n"
        : "=r"(done)
        : "r"(smem_u32(bar)), "r"(phase)
        : "memory");
  }
}

__device__ __forceinline__ void tma_bulk_g2s(void* dst, const void* src, uint32_t bytes, uint64_t* bar) {
  asm volatile(
      "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];\n" ::"r"(
          smem_u32(dst)),
      "l"(src), "r"(bytes), "r"(smem_u32(bar))
      : "memory");
}

__device__ __forceinline__ void dmma(double& d0, double& d1, double a, double b) {
  asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};\n"
               : "+d"(d0), "+d"(d1)
               : "d"(a), "d"(b));
}

struct FusedLayout {
  int par, planes, kmask, abuf, cand, tile, bar, exp2, total;
};

__host__ __device__ inline FusedLayout fused_layout(int nw, int n, int n_params, int n_kendall, int rows8) {
  FusedLayout L;
  int off = 0;
  L.par = off;
  off += n_params * (int)sizeof(bx_param_desc);
  off = (off + 15) & ~15;
  L.planes = off;
  off += n_params * n * 8;
  L.kmask = off;
  off += n_kendall * n * 16;
  off = (off + 127) & ~127;
  L.abuf = off;
  off += 2 * rows8 * kKCP * 8;
  L.cand = off;  // per warp: [n_params][8] values + [n_params][8][2] Kendall masks
  off += nw * n_params * 8 * 24;
  L.tile = off;  // per warp: ss[8], mean[8]
  off += nw * 16 * 8;
  L.bar = off;
  off += 2 * 8;
  L.exp2 = off;
  off += 64 * 8;
  L.total = off;
  return L;
}

// Warps per CTA: as many as the register file allows with the MT-tile accumulator resident
// (one CTA per SM): 16 warps up to 20 m-tiles, 12 beyond (ptxas: no spills in either case).
template <int MT>
constexpr int warps_for() { return MT <= 20 ? 16 : 12; }

template <int MT>
__global__ void __launch_bounds__(warps_for<MT>() * 32, 1) gp_fused_kernel(FusedArgs a) {
  extern __shared__ __align__(128) unsigned char smem[];
  constexpr int nw = warps_for<MT>();
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  const int n_params = a.space.n_params, words = a.space.row_words;
  const int n = a.gp.n;
  const int rows8 = 8 * MT;
  const FusedLayout L = fused_layout(nw, n, n_params, a.n_kendall, rows8);
  bx_param_desc* params = reinterpret_cast<bx_param_desc*>(smem + L.par);
  uint64_t* planes = reinterpret_cast<uint64_t*>(smem + L.planes);
  uint64_t* kmask = reinterpret_cast<uint64_t*>(smem + L.kmask);
  double* abuf = reinterpret_cast<double*>(smem + L.abuf);
  uint64_t* cval = reinterpret_cast<uint64_t*>(smem + L.cand) + (size_t)warp * n_params * 24;
  uint64_t* cmask = cval + n_params * 8;
  double* t_ss = reinterpret_cast<double*>(smem + L.tile) + warp * 16;
  double* t_mean = t_ss + 8;
  uint64_t* bars = reinterpret_cast<uint64_t*>(smem + L.bar);
  double* s_exp2 = reinterpret_cast<double*>(smem + L.exp2);
  for (int i = tid; i < 64; i += blockDim.x) s_exp2[i] = a.exp2tab[i];
  const MaternConst mc{a.gp.outputscale, a.gp.outputscale * kSqrt5, a.gp.outputscale * (5.0 / 3.0)};

  for (int i = tid; i < n_params * (int)sizeof(bx_param_desc) / 4; i += blockDim.x)
    reinterpret_cast<int32_t*>(params)[i] = reinterpret_cast<const int32_t*>(a.space.params)[i];
  for (int i = tid; i < n_params * n; i += blockDim.x) planes[i] = a.gp.planes[i];
  for (int i = tid; i < a.n_kendall * n * 2; i += blockDim.x) {
    const int kk = i / (2 * n), rest = i % (2 * n);
    kmask[i] = a.gp.kmask[((size_t)a.kendall_param[kk] * n) * 2 + rest];
  }
  if (tid == 0) {
    mbar_init(&bars[0], 1);
    mbar_init(&bars[1], 1);
    asm volatile("fence.mbarrier_init.release.cluster;\n" ::: "memory");
  }
  __syncthreads();

  const double sigma = a.gp.outputscale;
  const int n_chunks = (a.gp.ncols_pad + kKC - 1) / kKC;
  const int64_t n_tiles = (a.q + 8 * nw - 1) / (8 * nw);
  const int c = lane >> 2, fk = lane & 3;
  uint32_t phase[2] = {0, 0};

  // panel c: rows [16c, rows8) of the padded panel-major copy of A
  auto issue = [&](int chunk, int buf) {
    const int r0 = kKC * chunk;
    const uint32_t bytes = (uint32_t)(rows8 - r0) * kKCP * 8;
    mbar_expect_tx(&bars[buf], bytes);
    tma_bulk_g2s(abuf + (size_t)buf * rows8 * kKCP + (size_t)r0 * kKCP,
                 a.panels + (size_t)chunk * rows8 * kKCP + (size_t)r0 * kKCP, bytes, &bars[buf]);
  };

  for (int64_t tile = blockIdx.x; tile < n_tiles; tile += gridDim.x) {
    const int64_t cbase = tile * 8 * nw + (int64_t)warp * 8;
    if (tid == 0) {
      issue(0, 0);
      if (n_chunks > 1) issue(1, 1);
    }
    // decode the warp's 8 candidates
    for (int idx = lane; idx < n_params * 8; idx += 32) {
      const int k = idx >> 3, cc = idx & 7;
      const int64_t gi = cbase + cc;
      const bx_param_desc& p = params[k];
      uint64_t v = 0, lo = 0, hi = 0;
      if (gi < a.q) {
        const uint32_t* row = a.rows + (size_t)gi * words;
        if (p.kind == BX_PERMUTATION) {
          v = row_u64(row, p.word);
          if (p.metric == BX_KENDALL) kendall_mask(v, p.size, lo, hi);
        } else if (p.kind == BX_CATEGORICAL) {
          v = row[p.word];
        } else {
          v = (uint64_t)__double_as_longlong(row_coord(p, a.space.coord_lut, row) * a.gp.inv_l[k]);
        }
      }
      cval[k * 8 + cc] = v;
      cmask[(k * 8 + cc) * 2] = lo;
      cmask[(k * 8 + cc) * 2 + 1] = hi;
    }
    __syncwarp();

    double acc[MT][2];
#pragma unroll
    for (int m = 0; m < MT; ++m) acc[m][0] = acc[m][1] = 0.0;
    for (int chunk = 0; chunk < n_chunks; ++chunk) {
      const int buf = chunk & 1;
      for (int half = 0; half < kKC / 16; ++half) {
      const int jb = chunk * kKC + 16 * half;
      // K* for this lane's four columns of the half panel: j = jb + 4 ks + fk (B fragments)
      double W[4] = {0.0, 0.0, 0.0, 0.0};
      int jj[4];
#pragma unroll
      for (int s = 0; s < 4; ++s) {
        const int j = jb + 4 * s + fk;
        jj[s] = j < n ? j : 0;
      }
      for (int i = 0; i < a.n_num; ++i) {
        const int k = a.num_param[i];
        const double x = __longlong_as_double((long long)cval[k * 8 + c]);
        const uint64_t* pl = planes + (size_t)k * n;
#pragma unroll
        for (int s = 0; s < 4; ++s) {
          const double d = x - __longlong_as_double((long long)pl[jj[s]]);
          W[s] = fma(d, d, W[s]);
        }
      }
      for (int i = 0; i < a.n_cat; ++i) {
        const int k = a.cat_param[i];
        const uint64_t x = cval[k * 8 + c];
        const double wl = a.gp.inv_l2[k];
        const uint64_t* pl = planes + (size_t)k * n;
#pragma unroll
        for (int s = 0; s < 4; ++s) W[s] += (x != pl[jj[s]]) ? wl : 0.0;
      }
      for (int i = 0, kend = 0; i < a.n_perm; ++i) {
        const int k = a.perm_param[i];
        const bx_param_desc& p = params[k];
        const uint64_t x = cval[k * 8 + c];
        const uint64_t xl = cmask[(k * 8 + c) * 2], xh = cmask[(k * 8 + c) * 2 + 1];
        const double* tab = a.gp.disc_tab + a.gp.disc_off[k];
        const bool kd = p.metric == BX_KENDALL;
#pragma unroll
        for (int s = 0; s < 4; ++s) {
          const uint64_t bl = kd ? kmask[((size_t)kend * n + jj[s]) * 2] : 0;
          const uint64_t bh = kd ? kmask[((size_t)kend * n + jj[s]) * 2 + 1] : 0;
          W[s] += __ldg(tab + perm_raw(p.metric, p.size, x, planes[(size_t)k * n + jj[s]], xl, xh, bl, bh));
        }
        kend += kd ? 1 : 0;
      }
      double kv[4];
#pragma unroll
      for (int s = 0; s < 4; ++s)
        kv[s] = (jb + 4 * s + fk < n)
                    ? (a.precise ? kstar(W[s], sigma) : kstar_fast(W[s], mc, s_exp2))
                    : 0.0;

      if (half == 0) {
        mbar_wait(&bars[buf], phase[buf]);
        phase[buf] ^= 1u;
      }
      const double* As = abuf + (size_t)buf * rows8 * kKCP;
#pragma unroll
      for (int ks = 0; ks < 4; ++ks) {
        const int mt_lo = (jb + ks * 4) >> 3;  // m-tiles above are zero in these columns
        const double* Af = As + (size_t)c * kKCP + 16 * half + ks * 4 + fk;  // A row 8*m + c
        const double b = kv[ks];
        // enter the unrolled m-tile sequence at mt_lo (Duff's device: one indirect branch)
#define BX_DM(m)                                                              \
  case m:                                                                     \
    if constexpr ((m) < MT) dmma(acc[m][0], acc[m][1], Af[(size_t)(m) * 8 * kKCP], b); \
    [[fallthrough]];
        switch (mt_lo) {
          BX_DM(0) BX_DM(1) BX_DM(2) BX_DM(3) BX_DM(4) BX_DM(5) BX_DM(6) BX_DM(7)
          BX_DM(8) BX_DM(9) BX_DM(10) BX_DM(11) BX_DM(12) BX_DM(13) BX_DM(14) BX_DM(15)
          BX_DM(16) BX_DM(17) BX_DM(18) BX_DM(19) BX_DM(20) BX_DM(21) BX_DM(22) BX_DM(23)
          BX_DM(24) BX_DM(25) BX_DM(26) BX_DM(27) BX_DM(28) BX_DM(29) BX_DM(30) BX_DM(31)
          default:
            break;
        }
#undef BX_DM
      }
      }  // half
      __syncthreads();  // everyone is done with this buffer
      if (tid == 0 && chunk + 2 < n_chunks) issue(chunk + 2, buf);
    }

    // reduce: rows < n -> sum of squares, row n -> mean
    double ss0 = 0.0, ss1 = 0.0, mn0 = 0.0, mn1 = 0.0;
#pragma unroll
    for (int m = 0; m < MT; ++m) {
      const int row = 8 * m + c;
      if (row < n) {
        ss0 = fma(acc[m][0], acc[m][0], ss0);
        ss1 = fma(acc[m][1], acc[m][1], ss1);
      } else if (row == n) {
        mn0 = acc[m][0];
        mn1 = acc[m][1];
      }
    }
#pragma unroll
    for (int off = 4; off < 32; off <<= 1) {
      ss0 += __shfl_xor_sync(0xffffffffu, ss0, off);
      ss1 += __shfl_xor_sync(0xffffffffu, ss1, off);
      mn0 += __shfl_xor_sync(0xffffffffu, mn0, off);
      mn1 += __shfl_xor_sync(0xffffffffu, mn1, off);
    }
    if (c == 0) {
      t_ss[2 * fk] = ss0;
      t_ss[2 * fk + 1] = ss1;
      t_mean[2 * fk] = mn0;
      t_mean[2 * fk + 1] = mn1;
    }
    __syncwarp();
    if (lane < 8) {
      const int64_t gi = cbase + lane;
      if (gi < a.q) {
        const double var_s = fmax(sigma - t_ss[lane], 0.0);          // surrogate.py:324-325
        const double mean = a.gp.y_mean + a.gp.y_std * t_mean[lane];  // :328
        const double var = (a.gp.y_std * a.gp.y_std) * var_s;
        if (a.mean_out) a.mean_out[gi] = mean;
        if (a.var_out) a.var_out[gi] = var;
        if (a.ei_out) a.ei_out[gi] = ei_value(mean, var, a.f_model);  // acquisition.py:40-51
      }
    }
    __syncwarp();
  }
}

template <int MT>
cudaError_t launch_mt(const FusedArgs& a, int sm_count, cudaStream_t s) {
  constexpr int nw = warps_for<MT>();
  const FusedLayout L = fused_layout(nw, a.gp.n, a.space.n_params, a.n_kendall, 8 * MT);
  if (L.total > 227 * 1024) return cudaErrorInvalidValue;
  cudaError_t e = set_smem(gp_fused_kernel<MT>, L.total);
  if (e != cudaSuccess) return e;
  int per_sm = 0;
  e = cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, gp_fused_kernel<MT>, nw * 32, L.total);
  if (e != cudaSuccess) return e;
  if (per_sm < 1) return cudaErrorInvalidConfiguration;
  int64_t tiles = (a.q + 8 * nw - 1) / (8 * nw);
  int64_t grid = (int64_t)sm_count * per_sm;
  if (tiles < grid) grid = tiles;
  if (grid < 1) grid = 1;
  gp_fused_kernel<MT><<<(int)grid, nw * 32, L.total, s>>>(a);
  return cudaGetLastError();
}

}  // namespace

int fused_max_rows() { return 8 * 32; }

size_t fused_smem_bytes(int n, int n_params, int n_kendall, int rows8) {
  return fused_layout(16, n, n_params, n_kendall, rows8).total;  // upper bound over warp counts
}

// Panel-major padded copy of A for the TMA stream: panel c holds columns [16c, 16c+16) of rows
// [0, rows8), each row padded to kKCP doubles.
__global__ void build_panels_kernel(const double* A, int lda, int rows_src, int ncols_pad, int rows8,
                                    double* panels) {
  const int64_t total = (int64_t)((ncols_pad + kKC - 1) / kKC) * rows8 * kKCP;
  for (int64_t t = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; t < total;
       t += (int64_t)gridDim.x * blockDim.x) {
    const int chunk = (int)(t / ((int64_t)rows8 * kKCP));
    const int rem = (int)(t % ((int64_t)rows8 * kKCP));
    const int r = rem / kKCP, cc = rem % kKCP;
    double v = 0.0;
    if (cc < kKC && r < rows_src && chunk * kKC + cc < ncols_pad) v = A[(size_t)r * lda + chunk * kKC + cc];
    panels[t] = v;
  }
}

cudaError_t launch_build_panels(const double* A, int lda, int rows_src, int ncols_pad, int rows8,
                                double* panels, cudaStream_t s) {
  build_panels_kernel<<<148 * 4, 256, 0, s>>>(A, lda, rows_src, ncols_pad, rows8, panels);
  return cudaGetLastError();
}

size_t panels_doubles(int ncols_pad, int rows8) {
  return (size_t)((ncols_pad + kKC - 1) / kKC) * rows8 * kKCP;
}

cudaError_t launch_gp_fused(const FusedArgs& a, int sm_count, cudaStream_t s) {
  switch (a.mt) {
    case 2: return launch_mt<2>(a, sm_count, s);
    case 4: return launch_mt<4>(a, sm_count, s);
    case 6: return launch_mt<6>(a, sm_count, s);
    case 8: return launch_mt<8>(a, sm_count, s);
    case 10: return launch_mt<10>(a, sm_count, s);
    case 12: return launch_mt<12>(a, sm_count, s);
    case 14: return launch_mt<14>(a, sm_count, s);
    case 16: return launch_mt<16>(a, sm_count, s);
    case 18: return launch_mt<18>(a, sm_count, s);
    case 20: return launch_mt<20>(a, sm_count, s);
    case 22: return launch_mt<22>(a, sm_count, s);
    case 24: return launch_mt<24>(a, sm_count, s);
    case 26: return launch_mt<26>(a, sm_count, s);
    case 28: return launch_mt<28>(a, sm_count, s);
    case 30: return launch_mt<30>(a, sm_count, s);
    case 32: return launch_mt<32>(a, sm_count, s);
    default: return cudaErrorInvalidValue;
  }
}

}  // namespace bx
