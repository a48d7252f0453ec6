// score.cu — fused candidate scoring on sm_100a.
//
// One persistent CTA of 4 warps walks tiles of 4*CPW candidates.  Per warp (CPW candidates):
//   phase 0  decode the candidate rows into smem (scaled coordinates, labels, permutations)
//   phase A  K*[c][j] = sigma * matern52(sqrt(sum_k d_k^2 / l_k^2))       (surrogate.py:318-321)
//            FP64 on the DFMA pipe, lane tile = CPW candidates x 2 training points
//   phase B  [v ; mean] = [L^-1 ; alpha^T] K*^T on the FP64 tensor pipe (DMMA m8n8k4),
//            block-triangular over 16-row blocks, ss = sum_i v_i^2             (:322-325)
//   phase C  de-standardise, EI (acquisition.py:40-51), x p, -inf below eps_f (:70-79)
// then one thread folds the tile into the CTA's running summary: stable top-k by
// (value desc, index asc) (acquisition.py:188), and the two _Tracker reductions
// (value desc / prob desc, ties -> smallest configuration, evaluated skipped; :97-111).
#include "bx_common.cuh"

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
  int ks_off, cand_off, tile_off, sum_off, par_off, total;
};

__host__ __device__ inline SmemLayout smem_layout(int cpw, int ncols, int n_params, int row_words) {
  SmemLayout L;
  int off = 0;
  L.par_off = off;
  off += n_params * (int)sizeof(bx_param_desc);
  off = (off + 15) & ~15;
  L.ks_off = off;
  off += kWarps * cpw * ks_stride(ncols) * 8;
  L.cand_off = off;  // per warp: [n_params][cpw] 8-byte values + Kendall masks [n_params][cpw][2]
  off += kWarps * n_params * cpw * 8 * 3;
  L.tile_off = off;  // per tile: value, prob (doubles), flags (int) for 4*cpw candidates
  off += kWarps * cpw * (8 + 8 + 8 + 8 + 4);
  off = (off + 15) & ~15;
  L.sum_off = off;
  off += (int)sizeof(bx_score_summary);
  L.total = off;
  (void)row_words;
  return L;
}

__device__ void summary_init(bx_score_summary* s, int k) {
  s->n_scored = 0;
  s->n_finite = 0;
  s->k = k;
  s->n_top = 0;
  s->best.value = -INFINITY;
  s->best.prob = -INFINITY;
  s->best.index = -1;
  s->best_prob.value = -INFINITY;
  s->best_prob.prob = -INFINITY;
  s->best_prob.index = -1;
}

__device__ __forceinline__ void copy_row(uint32_t* dst, const uint32_t* src, int words) {
  for (int w = 0; w < words; ++w) dst[w] = src[w];
}

// Fold one scored candidate into a summary (single thread).
__device__ void summary_add(bx_score_summary* s, const bx_param_desc* params, int n_params,
                            const int32_t* rank_lut, int words, double v, double p, int64_t g,
                            bool evaluated, const uint32_t* row) {
  s->n_scored += 1;
  if (v != -INFINITY) {
    s->n_finite += 1;
    // stable top-k by (value desc, index asc)
    int k = s->k, nt = s->n_top;
    bool enters = nt < k;
    if (!enters) {
      const bx_cand& last = s->top[nt - 1];
      enters = v > last.value || (v == last.value && g < last.index);
    }
    if (enters) {
      int pos = nt < k ? nt : k - 1;
      while (pos > 0) {
        const bx_cand& prev = s->top[pos - 1];
        if (v > prev.value || (v == prev.value && g < prev.index)) {
          s->top[pos] = prev;
          --pos;
        } else {
          break;
        }
      }
      s->top[pos].value = v;
      s->top[pos].prob = p;
      s->top[pos].index = g;
      copy_row(s->top[pos].row, row, words);
      if (nt < k) s->n_top = nt + 1;
    }
    if (!evaluated) {
      bool take = v > s->best.value;
      if (!take && v == s->best.value)
        take = s->best.index < 0 || key_cmp(params, n_params, rank_lut, row, s->best.row) < 0;
      if (take) {
        s->best.value = v;
        s->best.prob = p;
        s->best.index = g;
        copy_row(s->best.row, row, words);
      }
    }
  }
  if (!evaluated && p != -INFINITY) {
    bool take = p > s->best_prob.prob;
    if (!take && p == s->best_prob.prob)
      take = s->best_prob.index < 0 ||
             key_cmp(params, n_params, rank_lut, row, s->best_prob.row) < 0;
    if (take) {
      s->best_prob.value = v;
      s->best_prob.prob = p;
      s->best_prob.index = g;
      copy_row(s->best_prob.row, row, words);
    }
  }
}

// Merge summary `b` into `a` (single thread).  Same orders as summary_add.
__device__ void summary_merge(bx_score_summary* a, const bx_score_summary* b,
                              const bx_param_desc* params, int n_params, const int32_t* rank_lut,
                              int words) {
  a->n_scored += b->n_scored;
  a->n_finite += b->n_finite;
  for (int i = 0; i < b->n_top; ++i) {
    const bx_cand& c = b->top[i];
    int k = a->k, nt = a->n_top;
    bool enters = nt < k;
    if (!enters) {
      const bx_cand& last = a->top[nt - 1];
      enters = c.value > last.value || (c.value == last.value && c.index < last.index);
    }
    if (!enters) break;  // b->top is sorted: nothing later can enter
    int pos = nt < k ? nt : k - 1;
    while (pos > 0) {
      const bx_cand& prev = a->top[pos - 1];
      if (c.value > prev.value || (c.value == prev.value && c.index < prev.index)) {
        a->top[pos] = prev;
        --pos;
      } else {
        break;
      }
    }
    a->top[pos] = c;
    if (nt < k) a->n_top = nt + 1;
  }
  if (b->best.index >= 0) {
    bool take = b->best.value > a->best.value;
    if (!take && b->best.value == a->best.value)
      take = a->best.index < 0 ||
             key_cmp(params, n_params, rank_lut, b->best.row, a->best.row) < 0;
    if (take) a->best = b->best;
  }
  if (b->best_prob.index >= 0) {
    bool take = b->best_prob.prob > a->best_prob.prob;
    if (!take && b->best_prob.prob == a->best_prob.prob)
      take = a->best_prob.index < 0 ||
             key_cmp(params, n_params, rank_lut, b->best_prob.row, a->best_prob.row) < 0;
    if (take) a->best_prob = b->best_prob;
  }
  (void)words;
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
  const SmemLayout L = smem_layout(CPW, ncols, n_params, words);
  bx_param_desc* params = reinterpret_cast<bx_param_desc*>(smem + L.par_off);
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;

  for (int i = tid; i < n_params * (int)sizeof(bx_param_desc) / 4; i += kThreads)
    reinterpret_cast<int32_t*>(params)[i] = reinterpret_cast<const int32_t*>(a.space.params)[i];

  double* ks = reinterpret_cast<double*>(smem + L.ks_off) + (size_t)warp * CPW * S;
  uint64_t* cval = reinterpret_cast<uint64_t*>(smem + L.cand_off) + (size_t)warp * n_params * CPW * 3;
  uint64_t* cmask = cval + n_params * CPW;  // [n_params][CPW][2]
  constexpr int TC = kWarps * CPW;
  double* t_value = reinterpret_cast<double*>(smem + L.tile_off);
  double* t_prob = t_value + TC;
  double* t_ss = t_prob + TC;
  double* t_mean = t_ss + TC;
  int* t_flag = reinterpret_cast<int*>(t_mean + TC);
  bx_score_summary* summ = reinterpret_cast<bx_score_summary*>(smem + L.sum_off);
  const bool want_summary = a.partials != nullptr;
  if (want_summary && tid == 0) summary_init(summ, a.k);
  __syncthreads();

  const double sigma = a.gp.outputscale;
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
    constexpr int NT = CPW / 8;
    double ss[NT][2], mn[NT][2];
#pragma unroll
    for (int t = 0; t < NT; ++t) ss[t][0] = ss[t][1] = mn[t][0] = mn[t][1] = 0.0;
    const int fr = lane >> 2, fk = lane & 3;
    const int n_rb = a.gp.rows_pad / 16;
    for (int rb = 0; rb < n_rb; ++rb) {
      const int ext = min(ncols, 16 * (rb + 1));
      double acc[2][NT][2];
#pragma unroll
      for (int m = 0; m < 2; ++m)
#pragma unroll
        for (int t = 0; t < NT; ++t) acc[m][t][0] = acc[m][t][1] = 0.0;
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
            for (int t = 0; t < NT; ++t) dmma8x8x4(acc[m][t][0], acc[m][t][1], ra[m][s], rbv[t][s]);
      }
#pragma unroll
      for (int m = 0; m < 2; ++m) {
        const int row = 16 * rb + 8 * m + fr;
#pragma unroll
        for (int t = 0; t < NT; ++t) {
          if (row < n) {
            ss[t][0] = fma(acc[m][t][0], acc[m][t][0], ss[t][0]);
            ss[t][1] = fma(acc[m][t][1], acc[m][t][1], ss[t][1]);
          } else if (row == n) {
            mn[t][0] = acc[m][t][0];
            mn[t][1] = acc[m][t][1];
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
          const int c = warp * CPW + t * 8 + 2 * fk + e;
          t_ss[c] = ss[t][e];
          t_mean[c] = mn[t][e];
        }
    }
    __syncwarp();

    // ---- phase C: epilogue per candidate ----------------------------------------------------
    if (lane < CPW) {
      const int c = warp * CPW + lane;
      const int64_t gi = cbase + lane;
      double value = -INFINITY, prob = -INFINITY;
      int flag = 0;
      if (gi < a.q) {
        flag = 1;
        const double var_s = fmax(sigma - t_ss[c], 0.0);          // surrogate.py:324-325
        const double mean = a.gp.y_mean + a.gp.y_std * t_mean[c];  // :328
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
        if (want_summary && is_evaluated(a.evald, a.rows + (size_t)gi * words, words)) flag = 2;
      }
      t_value[c] = value;
      t_prob[c] = prob;
      t_flag[c] = flag;
    }
    if (want_summary) {
      __syncthreads();
      if (tid == 0) {
        const int64_t tbase = tile * TC;
        for (int c = 0; c < TC; ++c) {
          if (t_flag[c] == 0) continue;
          const int64_t gi = tbase + c;
          summary_add(summ, params, n_params, a.space.rank_lut, words, t_value[c], t_prob[c],
                      a.index_base + gi, t_flag[c] == 2, a.rows + (size_t)gi * words);
        }
      }
      __syncthreads();
    } else {
      __syncwarp();
    }
  }

  if (want_summary) {
    __syncthreads();
    // copy the CTA summary out (int32 granularity)
    const int32_t* src = reinterpret_cast<const int32_t*>(summ);
    int32_t* dst = reinterpret_cast<int32_t*>(a.partials + blockIdx.x);
    for (int i = tid; i < (int)(sizeof(bx_score_summary) / 4); i += kThreads) dst[i] = src[i];
  }
}

__global__ void merge_kernel(const bx_score_summary* partials, int n_partials, SpaceDev space, int k,
                             bx_score_summary* out) {
  __shared__ bx_score_summary acc;
  __shared__ bx_param_desc params[BX_MAX_PARAMS];
  for (int i = threadIdx.x; i < space.n_params * (int)sizeof(bx_param_desc) / 4; i += blockDim.x)
    reinterpret_cast<int32_t*>(params)[i] = reinterpret_cast<const int32_t*>(space.params)[i];
  __syncthreads();
  if (threadIdx.x == 0) {
    summary_init(&acc, k);
    for (int p = 0; p < n_partials; ++p)
      summary_merge(&acc, partials + p, params, space.n_params, space.rank_lut, space.row_words);
  }
  __syncthreads();
  const int32_t* src = reinterpret_cast<const int32_t*>(&acc);
  int32_t* dst = reinterpret_cast<int32_t*>(out);
  for (int i = threadIdx.x; i < (int)(sizeof(bx_score_summary) / 4); i += blockDim.x) dst[i] = src[i];
}

template <int CPW>
cudaError_t launch_score_t(const ScoreArgs& a, int sm_count, cudaStream_t s, int* grid_used) {
  const SmemLayout L = smem_layout(CPW, a.gp.ncols_pad, a.space.n_params, a.space.row_words);
  cudaError_t e = cudaFuncSetAttribute(score_kernel<CPW>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                       L.total);
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
  *grid_used = (int)grid;
  score_kernel<CPW><<<(int)grid, kThreads, L.total, s>>>(a);
  return cudaGetLastError();
}

}  // namespace

int score_smem_bytes(int cpw, int ncols, int n_params, int row_words) {
  return smem_layout(cpw, ncols, n_params, row_words).total;
}

cudaError_t launch_score(const ScoreArgs& a, int sm_count, cudaStream_t s, int* grid_used) {
  // 8 candidates per warp keeps two CTAs per SM resident up to n ~ 300; 16 per warp halves the
  // B-fragment traffic per DMMA when the tile still fits.
  const int big = score_smem_bytes(16, a.gp.ncols_pad, a.space.n_params, a.space.row_words);
  const int small = score_smem_bytes(8, a.gp.ncols_pad, a.space.n_params, a.space.row_words);
  if (small > 227 * 1024) return cudaErrorInvalidValue;
  (void)big;
  return launch_score_t<8>(a, sm_count, s, grid_used);
}

cudaError_t launch_summary_merge(const bx_score_summary* partials, int n_partials,
                                 const SpaceDev& space, int k, int64_t q, bx_score_summary* out,
                                 cudaStream_t s) {
  (void)q;
  merge_kernel<<<1, 32, 0, s>>>(partials, n_partials, space, k, out);
  return cudaGetLastError();
}

}  // namespace bx
