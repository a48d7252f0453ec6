// score.cu — fused candidate scoring on sm_100a.
//
// One persistent CTA of 4 warps walks tiles of 4*CPW candidates.  Per warp (CPW candidates):
//   phase 0  decode the candidate rows into smem (scaled coordinates, labels, permutations)
//   phase A  K*[c][j] = sigma * matern52(sqrt(sum_k d_k^2 / l_k^2))       (surrogate.py:318-321)
//            FP64 on the DFMA pipe, lane tile = CPW candidates x 2 training points
//   phase B  [v ; mean] = [L^-1 ; alpha^T] K*^T on the FP64 tensor pipe (DMMA m8n8k4),
//            block-triangular over 16-row blocks, ss = sum_i v_i^2             (:322-325)
//   phase C  de-standardise, EI (acquisition.py:40-51), x p, -inf below eps_f (:70-79)
// then the warp folds its candidates into a warp-private summary: stable top-k by
// (value desc, index asc) (acquisition.py:188) and the two _Tracker reductions (value desc /
// prob desc, ties -> smallest configuration, evaluated skipped; :97-111).  A ballot against the
// warp's current thresholds skips the sequential insert for almost every candidate.  The partial
// summaries are merged by merge_kernel.
#include "summary.cuh"

namespace bx {

namespace {

constexpr int kWarps = 4;
constexpr int kThreads = kWarps * 32;

__device__ __forceinline__ void dmma8x8x4(double& d0, double& d1, double a, double b) {
  asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};\n"
               : "+d"(d0), "+d"(d1)
               : "d"(a), "d"(b));
}

// smem row stride (doubles) for a K* row of `ncols` entries: == 4 (mod 16) so that the 8x4 DMMA
// fragment loads of 8 candidates hit 32 distinct banks in two wavefronts.
__host__ __device__ __forceinline__ int ks_stride(int ncols) { return ((ncols + 15) / 16) * 16 + 4; }

struct SmemLayout {
  int par_off, ks_off, cand_off, tile_off, sum_off, total;
};

__host__ __device__ inline SmemLayout smem_layout(int cpw, int ncols, int n_params) {
  SmemLayout L;
  int off = 0;
  L.par_off = off;
  off += n_params * (int)sizeof(bx_param_desc);
  off = (off + 15) & ~15;
  L.ks_off = off;
  off += kWarps * cpw * ks_stride(ncols) * 8;
  L.cand_off = off;  // per warp: [n_params][cpw] 8-byte values + Kendall masks [n_params][cpw][2]
  off += kWarps * n_params * cpw * 8 * 3;
  L.tile_off = off;  // per warp tile: ss, mean (doubles)
  off += kWarps * cpw * 16;
  off = (off + 15) & ~15;
  L.sum_off = off;
  off += kWarps * (int)sizeof(Partial);
  L.total = off;
  return L;
}

// Matern-5/2 correlation times outputscale at squared weighted distance W (surrogate.py:142-145,
// 321: sigma * matern52(sqrt(max(W, 0)))).
__device__ __forceinline__ double kstar_from_w(double W, double sigma) {
  double d = sqrt(fmax(W, 0.0));
  double e = exp(-kSqrt5 * d);
  return sigma * ((1.0 + kSqrt5 * d + (5.0 / 3.0) * d * d) * e);
}

template <int CPW>
__global__ void __launch_bounds__(kThreads) score_kernel(ScoreArgs a) {
  extern __shared__ __align__(16) unsigned char smem[];
  const int n_params = a.space.n_params;
  const int words = a.space.row_words;
  const int n = a.gp.n;
  const int ncols = a.gp.ncols_pad;  // multiple of 16
  const int S = ks_stride(ncols);
  const SmemLayout L = smem_layout(CPW, ncols, n_params);
  bx_param_desc* params = reinterpret_cast<bx_param_desc*>(smem + L.par_off);
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;

  for (int i = tid; i < n_params * (int)sizeof(bx_param_desc) / 4; i += kThreads)
    reinterpret_cast<int32_t*>(params)[i] = reinterpret_cast<const int32_t*>(a.space.params)[i];

  double* ks = reinterpret_cast<double*>(smem + L.ks_off) + (size_t)warp * CPW * S;
  uint64_t* cval = reinterpret_cast<uint64_t*>(smem + L.cand_off) + (size_t)warp * n_params * CPW * 3;
  uint64_t* cmask = cval + n_params * CPW;  // [n_params][CPW][2]
  double* t_ss = reinterpret_cast<double*>(smem + L.tile_off) + warp * CPW * 2;
  double* t_mean = t_ss + CPW;
  Partial* summ = reinterpret_cast<Partial*>(smem + L.sum_off) + warp;
  const bool want_summary = a.partials != nullptr;
  if (want_summary && lane == 0) partial_init(summ);
  __syncthreads();

  const double sigma = a.gp.outputscale;
  constexpr int TC = kWarps * CPW;
  const int64_t n_tiles = (a.q + TC - 1) / TC;

  for (int64_t tile = blockIdx.x; tile < n_tiles; tile += gridDim.x) {
    const int64_t cbase = tile * TC + (int64_t)warp * CPW;

    // ---- phase 0: decode this warp's candidates --------------------------------------------
    for (int idx = lane; idx < n_params * CPW; idx += 32) {
      int k = idx / CPW, c = idx % CPW;
      int64_t gi = cbase + c;
      const bx_param_desc& p = params[k];
      uint64_t v = 0, mlo = 0, mhi = 0;
      if (gi < a.q) {
        const uint32_t* row = a.rows + (size_t)gi * words;
        if (p.kind == BX_PERMUTATION) {
          v = row_u64(row, p.word);
          if (p.metric == BX_KENDALL) kendall_mask(v, p.size, mlo, mhi);
        } else if (p.kind == BX_CATEGORICAL) {
          v = row[p.word];
        } else {
          double x = row_coord(p, a.space.coord_lut, row) * a.gp.inv_l[k];
          v = (uint64_t)__double_as_longlong(x);
        }
      }
      cval[k * CPW + c] = v;
      cmask[(k * CPW + c) * 2] = mlo;
      cmask[(k * CPW + c) * 2 + 1] = mhi;
    }
    __syncwarp();

    // ---- phase A: K* into smem; lane covers training columns 2*lane, 2*lane+1 (+64 r) ---------
    for (int j0 = 2 * lane; j0 < ncols; j0 += 64) {
      double w[CPW][2];
#pragma unroll
      for (int c = 0; c < CPW; ++c) w[c][0] = w[c][1] = 0.0;
      const int ja = j0 < n ? j0 : 0, jb = (j0 + 1) < n ? j0 + 1 : 0;
      for (int k = 0; k < n_params; ++k) {
        const bx_param_desc& p = params[k];
        const uint64_t* plane = a.gp.planes + (size_t)k * n;
        if (p.kind == BX_CATEGORICAL) {
          const uint64_t ta = __ldg(plane + ja), tb = __ldg(plane + jb);
          const double wl = a.gp.inv_l2[k];
#pragma unroll
          for (int c = 0; c < CPW; ++c) {
            const uint64_t x = cval[k * CPW + c];
            w[c][0] += (x != ta) ? wl : 0.0;
            w[c][1] += (x != tb) ? wl : 0.0;
          }
        } else if (p.kind == BX_PERMUTATION) {
          const uint64_t ta = __ldg(plane + ja), tb = __ldg(plane + jb);
          uint64_t al = 0, ah = 0, bl = 0, bh = 0;
          if (p.metric == BX_KENDALL) {
            const uint64_t* km = a.gp.kmask + (size_t)k * n * 2;
            al = __ldg(km + 2 * ja); ah = __ldg(km + 2 * ja + 1);
            bl = __ldg(km + 2 * jb); bh = __ldg(km + 2 * jb + 1);
          }
          const double* tab = a.gp.disc_tab + a.gp.disc_off[k];
#pragma unroll
          for (int c = 0; c < CPW; ++c) {
            const uint64_t x = cval[k * CPW + c];
            const uint64_t xl = cmask[(k * CPW + c) * 2], xh = cmask[(k * CPW + c) * 2 + 1];
            w[c][0] += __ldg(tab + perm_raw(p.metric, p.size, x, ta, xl, xh, al, ah));
            w[c][1] += __ldg(tab + perm_raw(p.metric, p.size, x, tb, xl, xh, bl, bh));
          }
        } else {
          const double ta = __longlong_as_double((long long)__ldg(plane + ja));
          const double tb = __longlong_as_double((long long)__ldg(plane + jb));
#pragma unroll
          for (int c = 0; c < CPW; ++c) {
            const double x = __longlong_as_double((long long)cval[k * CPW + c]);
            const double da = x - ta, db = x - tb;
            w[c][0] = fma(da, da, w[c][0]);
            w[c][1] = fma(db, db, w[c][1]);
          }
        }
      }
#pragma unroll
      for (int c = 0; c < CPW; ++c) {
        double k0 = j0 < n ? kstar_from_w(w[c][0], sigma) : 0.0;
        double k1 = (j0 + 1) < n ? kstar_from_w(w[c][1], sigma) : 0.0;
        *reinterpret_cast<double2*>(ks + c * S + j0) = make_double2(k0, k1);
      }
    }
    __syncwarp();

    // ---- phase B: [L^-1; alpha] K*^T with DMMA, block-triangular ------------------------------
    // Two accumulator sets (even / odd k-steps) double the independent DMMA chains.
    constexpr int NT = CPW / 8;
    double ss[NT][2], mn[NT][2];
#pragma unroll
    for (int t = 0; t < NT; ++t) ss[t][0] = ss[t][1] = mn[t][0] = mn[t][1] = 0.0;
    const int fr = lane >> 2, fk = lane & 3;
    const int n_rb = a.gp.rows_pad / 16;
    for (int rb = 0; rb < n_rb; ++rb) {
      const int ext = min(ncols, 16 * (rb + 1));
      double acc[2][2][NT][2];
#pragma unroll
      for (int h = 0; h < 2; ++h)
#pragma unroll
        for (int m = 0; m < 2; ++m)
#pragma unroll
          for (int t = 0; t < NT; ++t) acc[h][m][t][0] = acc[h][m][t][1] = 0.0;
      const double* A0 = a.gp.A + (size_t)(16 * rb + fr) * a.gp.lda + fk;
      const double* A1 = A0 + (size_t)8 * a.gp.lda;
      const double* B0 = ks + fr * S + fk;
      for (int k0 = 0; k0 < ext; k0 += 16) {
        double ra[2][4], rbv[NT][4];
#pragma unroll
        for (int s = 0; s < 4; ++s) {
          ra[0][s] = __ldg(A0 + k0 + 4 * s);
          ra[1][s] = __ldg(A1 + k0 + 4 * s);
#pragma unroll
          for (int t = 0; t < NT; ++t) rbv[t][s] = B0[t * 8 * S + k0 + 4 * s];
        }
#pragma unroll
        for (int s = 0; s < 4; ++s)
#pragma unroll
          for (int m = 0; m < 2; ++m)
#pragma unroll
            for (int t = 0; t < NT; ++t)
              dmma8x8x4(acc[s & 1][m][t][0], acc[s & 1][m][t][1], ra[m][s], rbv[t][s]);
      }
#pragma unroll
      for (int m = 0; m < 2; ++m) {
        const int row = 16 * rb + 8 * m + fr;
#pragma unroll
        for (int t = 0; t < NT; ++t) {
          const double v0 = acc[0][m][t][0] + acc[1][m][t][0];
          const double v1 = acc[0][m][t][1] + acc[1][m][t][1];
          if (row < n) {
            ss[t][0] = fma(v0, v0, ss[t][0]);
            ss[t][1] = fma(v1, v1, ss[t][1]);
          } else if (row == n) {
            mn[t][0] = v0;
            mn[t][1] = v1;
          }
        }
      }
    }
#pragma unroll
    for (int t = 0; t < NT; ++t)
#pragma unroll
      for (int e = 0; e < 2; ++e) {
#pragma unroll
        for (int off = 4; off < 32; off <<= 1) {
          ss[t][e] += __shfl_xor_sync(0xffffffffu, ss[t][e], off);
          mn[t][e] += __shfl_xor_sync(0xffffffffu, mn[t][e], off);
        }
      }
    if (fr == 0) {
#pragma unroll
      for (int t = 0; t < NT; ++t)
#pragma unroll
        for (int e = 0; e < 2; ++e) {
          const int c = t * 8 + 2 * fk + e;
          t_ss[c] = ss[t][e];
          t_mean[c] = mn[t][e];
        }
    }
    __syncwarp();

    // ---- phase C: epilogue per candidate (lane c < CPW) ------------------------------------
    const int64_t gi = cbase + lane;
    double value = -INFINITY, prob = -INFINITY;
    bool valid = false, evaluated = false;
    if (lane < CPW && gi < a.q) {
      valid = true;
      const double var_s = fmax(sigma - t_ss[lane], 0.0);          // surrogate.py:324-325
      const double mean = a.gp.y_mean + a.gp.y_std * t_mean[lane];  // :328
      const double var = (a.gp.y_std * a.gp.y_std) * var_s;
      if (a.mean_out) a.mean_out[gi] = mean;
      if (a.var_out) a.var_out[gi] = var;
      // expected_improvement_vec (acquisition.py:40-51)
      const double s = sqrt(fmax(var, 0.0));
      const double delta = a.f_model - mean;
      double ei = fmax(delta, 0.0);
      if (s > 0.0) {
        const double z = delta / s;
        const double phi = kInvSqrt2Pi * exp(-0.5 * z * z);
        ei = delta * normcdf(z) + s * phi;
      }
      ei = fmax(ei, 0.0);
      if (a.use_forest) {
        prob = a.forest.has_trees ? a.probs_in[gi] : a.forest.constant;
        value = (prob < a.eps_f) ? -INFINITY : ei * prob;  // acquisition.py:78
      } else {
        prob = 1.0;
        value = ei;
      }
      if (a.values_out) a.values_out[gi] = value;
      if (a.probs_out) a.probs_out[gi] = prob;
      if (want_summary) evaluated = is_evaluated(a.evald, a.rows + (size_t)gi * words, words);
    }
    if (want_summary) {
      // conservative filter against the warp's current thresholds (they only tighten)
      bool pass = false;
      if (valid) {
        const bool fin = value != -INFINITY;
        const bool top_ok = fin && a.k > 0 && (summ->n_top < a.k || value >= summ->top[a.k - 1].value);
        const bool best_ok = fin && !evaluated && value >= summ->best.value;
        const bool prob_ok = !evaluated && prob >= summ->best_prob.prob;
        pass = top_ok || best_ok || prob_ok;
      }
      const unsigned vmask = __ballot_sync(0xffffffffu, valid);
      const unsigned fmask = __ballot_sync(0xffffffffu, valid && value != -INFINITY);
      const unsigned pmask = __ballot_sync(0xffffffffu, pass);
      const unsigned emask = __ballot_sync(0xffffffffu, evaluated);
      if (lane == 0) {
        summ->n_scored += __popc(vmask);
        summ->n_finite += __popc(fmask);
      }
      unsigned m = pmask;
      while (m) {
        const int c = __ffs(m) - 1;
        m &= m - 1;
        const double vc = __shfl_sync(0xffffffffu, value, c);
        const double pc = __shfl_sync(0xffffffffu, prob, c);
        if (lane == 0)
          partial_add(summ, a.k, params, n_params, a.space.rank_lut, words, vc, pc,
                      a.index_base + cbase + c, (emask >> c) & 1u, a.rows + (size_t)(cbase + c) * words);
        __syncwarp();
      }
    }
    __syncwarp();
  }

  if (want_summary) {
    __syncwarp();
    const int32_t* src = reinterpret_cast<const int32_t*>(summ);
    int32_t* dst = reinterpret_cast<int32_t*>(a.partials + (size_t)blockIdx.x * kWarps + warp);
    for (int i = lane; i < (int)(sizeof(Partial) / 4); i += 32) dst[i] = src[i];
  }
}

template <int CPW>
cudaError_t launch_score_t(const ScoreArgs& a, int sm_count, cudaStream_t s, int* n_partials) {
  const SmemLayout L = smem_layout(CPW, a.gp.ncols_pad, a.space.n_params);
  cudaError_t e = set_smem(score_kernel<CPW>, L.total);
  if (e != cudaSuccess) return e;
  int per_sm = 0;
  e = cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, score_kernel<CPW>, kThreads, L.total);
  if (e != cudaSuccess) return e;
  if (per_sm < 1) return cudaErrorInvalidConfiguration;
  constexpr int TC = kWarps * CPW;
  int64_t tiles = (a.q + TC - 1) / TC;
  int64_t grid = (int64_t)sm_count * per_sm;
  if (tiles < grid) grid = tiles;
  if (grid < 1) grid = 1;
  *n_partials = (int)grid * kWarps;
  score_kernel<CPW><<<(int)grid, kThreads, L.total, s>>>(a);
  return cudaGetLastError();
}

}  // namespace

int score_smem_bytes(int cpw, int ncols, int n_params) {
  return smem_layout(cpw, ncols, n_params).total;
}

int score_max_partials(int sm_count) { return sm_count * 16 * kWarps; }

cudaError_t launch_score(const ScoreArgs& a, int sm_count, cudaStream_t s, int* n_partials) {
  if (score_smem_bytes(8, a.gp.ncols_pad, a.space.n_params) > 227 * 1024) return cudaErrorInvalidValue;
  return launch_score_t<8>(a, sm_count, s, n_partials);
}


}  // namespace bx
