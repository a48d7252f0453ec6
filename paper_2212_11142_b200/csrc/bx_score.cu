// bx_score.cu — scoring behind the C ABI: the step (posterior -> forest + summary -> merge) for
// device pools (bx_score), streamed host pools encoded or packed (bx_score_host), device-generated
// pools (bx_generate, bx_score_generated), the predict entry points and the device hill climb
// (bx_climb).
#include <algorithm>
#include "bx_handle.cuh"

namespace bx {
__global__ void unpack_kernel(PackSpec spec, const uint32_t* packed, int64_t q, int words, uint32_t* rows) {
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < q; i += (int64_t)gridDim.x * blockDim.x)
    unpack_row(spec, packed + (size_t)i * spec.pw, rows + (size_t)i * words, words);
}
cudaError_t launch_unpack(const PackSpec& spec, const uint32_t* packed, int64_t q, int words, uint32_t* rows,
                          cudaStream_t s) {
  int64_t blocks = (q + 255) / 256;
  if (blocks > 148 * 16) blocks = 148 * 16;
  unpack_kernel<<<(int)blocks, 256, 0, s>>>(spec, packed, q, words, rows);
  return cudaGetLastError();
}
}  // namespace bx


namespace bx {
// bx_climb state on the device: per start the current row, value and an active flag; the tracker
struct ClimbState {
  int32_t n_active;
  int32_t steps;                     // steps that had an active start (the host's loop count)
  TopRec best;                       // index >= 0 once set
  uint32_t best_row[BX_MAX_ROW_WORDS];
};

// per-row forest order: a start whose CoT-filtered list has exactly one neighbour is scored like
// the reference's _scores on one configuration (q == 1: numpy's pairwise tree sum)
__global__ void climb_flags_kernel(int A, int S, const int32_t* active, const uint8_t* valid, uint8_t* pw) {
  for (int a = threadIdx.x; a < A; a += blockDim.x) {
    int cnt = 0;
    for (int s = 0; s < S; ++s) cnt += valid[a * S + s] ? 1 : 0;
    for (int s = 0; s < S; ++s) pw[a * S + s] = (active[a] && cnt == 1) ? 1 : 0;
  }
}

// one step's bookkeeping (acquisition.py:193-201): per active start the argbest neighbour under
// (value desc, configuration asc) (_argbest, :87-94), moved to iff strictly better; every scored
// neighbour folded into the tracker (_Tracker.update, :105-111).  Warp a = start a: its lanes scan
// the slots, then a shuffle reduction under the same total orders; thread 0 folds the starts'
// tracker candidates.
__device__ __forceinline__ bool climb_better(const SpaceDev& sp, const uint32_t* nb, int W, double v1, int r1, double v2,
                                             int r2) {
  if (r1 < 0) return false;
  if (r2 < 0) return true;
  if (v1 != v2) return v1 > v2;
  return key_cmp(sp.params, sp.n_params, sp.rank_lut, nb + (size_t)r1 * W, nb + (size_t)r2 * W) < 0;
}

__global__ void climb_update_kernel(SpaceDev sp, EvalSetDev ev, int A, int S, int32_t* active, uint32_t* cur,
                                    double* curv, const uint32_t* nb, const uint8_t* valid, const double* vals,
                                    ClimbState* st) {
  __shared__ int s_trk[BX_MAX_K];
  __shared__ int s_moved[BX_MAX_K];
  __shared__ int s_any;
  const int W = sp.row_words;
  const int a = threadIdx.x >> 5, lane = threadIdx.x & 31;
  if (threadIdx.x == 0) s_any = 0;
  __syncthreads();
  if (a < A && lane == 0 && active[a]) s_any = 1;
  if (a < A) {
    int br = -1, tr = -1;  // argbest row and tracker-candidate row of this lane
    double bv = -INFINITY, tv = -INFINITY;
    if (active[a])
      for (int s2 = lane; s2 < S; s2 += 32) {
        const int r = a * S + s2;
        if (!valid[r]) continue;
        const double v = vals[r];
        if (climb_better(sp, nb, W, v, r, bv, br)) {
          bv = v;
          br = r;
        }
        if (v != -INFINITY && !(ev.count > 0 && is_evaluated(ev, nb + (size_t)r * W, W)) &&
            climb_better(sp, nb, W, v, r, tv, tr)) {
          tv = v;
          tr = r;
        }
      }
#pragma unroll
    for (int o = 16; o; o >>= 1) {
      const double ov = __shfl_xor_sync(0xffffffffu, bv, o), otv = __shfl_xor_sync(0xffffffffu, tv, o);
      const int orow = __shfl_xor_sync(0xffffffffu, br, o), otr = __shfl_xor_sync(0xffffffffu, tr, o);
      if (climb_better(sp, nb, W, ov, orow, bv, br)) {
        bv = ov;
        br = orow;
      }
      if (climb_better(sp, nb, W, otv, otr, tv, tr)) {
        tv = otv;
        tr = otr;
      }
    }
    if (lane == 0) {
      s_trk[a] = tr;
      int moved = 0;
      if (active[a]) {
        if (br >= 0 && bv > curv[a]) {  // acquisition.py:200
          curv[a] = bv;
          moved = 1;
        } else {
          active[a] = 0;  // no neighbours, or no improvement: this start stops
        }
      }
      s_moved[a] = moved ? br : -1;
    }
    __syncwarp();
    const int mr = __shfl_sync(0xffffffffu, lane == 0 ? s_moved[a] : 0, 0);
    if (mr >= 0)
      for (int w = lane; w < W; w += 32) cur[(size_t)a * W + w] = nb[(size_t)mr * W + w];
  }
  __syncthreads();
  if (threadIdx.x < 32) {
    // warp 0: the starts' tracker candidates reduced under the tracker's total order (value desc,
    // configuration asc) - the maximum the start-by-start fold reaches - then one fold into it
    const int i = threadIdx.x;
    int r = i < A ? s_trk[i] : -1;
    double v = r >= 0 ? vals[r] : -INFINITY;
#pragma unroll
    for (int o = 16; o; o >>= 1) {
      const double ov = __shfl_xor_sync(0xffffffffu, v, o);
      const int orow = __shfl_xor_sync(0xffffffffu, r, o);
      if (climb_better(sp, nb, W, ov, orow, v, r)) {
        v = ov;
        r = orow;
      }
    }
    const unsigned moved = __ballot_sync(0xffffffffu, i < A && s_moved[i] >= 0);
    if (i == 0) {
      if (r >= 0) {
        const uint32_t* row = nb + (size_t)r * W;
        bool take = st->best.index < 0 || v > st->best.value;
        if (!take && v == st->best.value) take = key_cmp(sp.params, sp.n_params, sp.rank_lut, row, st->best_row) < 0;
        if (take) {
          st->best = TopRec{v, 0.0, 0};
          for (int w = 0; w < W; ++w) st->best_row[w] = row[w];
        }
      }
      st->n_active = __popc(moved);
      st->steps += s_any;  // a step after every start stopped (a batched launch) changes nothing
    }
  }
}
}  // namespace bx


static SummaryArgs last_summary_args(bx_handle* h, const uint32_t* rows, int64_t q,
                                     int64_t index_base, double eps_f, int32_t k, double* values,
                                     double* probs_out, Partial* partials) {
  const bool forest = h->has_forest && h->forest.has_trees;
  SummaryArgs m{};
  m.space = space_dev(h);
  m.evald = eval_dev(h);
  m.rows = rows;
  m.q = q;
  m.index_base = index_base;
  m.ei = h->d_ei.as<double>();
  m.probs_in = forest ? h->d_probs.as<double>() : nullptr;
  m.use_forest = h->has_forest ? 1 : 0;
  m.has_trees = forest ? 1 : 0;
  m.constant = h->forest.constant;
  m.eps_f = eps_f;
  m.k = k;
  m.values_out = values;
  m.probs_out = probs_out;
  m.partials = partials;
  return m;
}

int score_impl(bx_handle* h, const uint32_t* rows, int64_t q, int64_t index_base,
                      double f_model, double eps_f, int32_t k, int32_t flags, double* values,
                      double* probs_out, Partial* partials, int* n_partials, cudaStream_t s,
                      int timing, bool track_prob, cudaEvent_t rows_ready) {
  ScoreArgs a{};
  a.space = space_dev(h);
  a.gp = gp_dev(h);
  a.evald = eval_dev(h);
  a.rows = rows;
  a.q = q;
  a.index_base = index_base;
  a.f_model = f_model;
  a.eps_f = eps_f;
  a.k = k;
  a.flags = flags;
  a.use_forest = h->has_forest ? 1 : 0;
  a.forest = h->forest;
  a.values_out = values;
  a.probs_out = probs_out;
  a.partials = partials;
  const bool forest = h->has_forest && h->forest.has_trees;
  if (forest) BX_CUDA(h, h->d_probs.ensure((size_t)q * 8));
  if (fused_path(h)) {
    // posterior (mean / var) -> forest -> summary.  With a summary wanted and QuickScorer tables
    // that fit, the forest and the summary are one kernel after the posterior (it evaluates the EI
    // only for the candidates whose probability passes eps_f); otherwise the stand-alone forest
    // kernel runs before the posterior and the summary kernel after it.  The forest and posterior
    // kernels each fill every SM's shared memory, so they run back to back on the caller's stream
    // (which also makes the per-kernel CUDA-event timing exact).
    const bool rf_summ = forest && !(flags & BX_SCORE_RF_PAIRWISE) && !h->pw_rows && partials != nullptr &&
                         qs_summary_available(h->forest);
    h->rf_after_gp = rf_summ;
    // a stand-alone forest kernel before the posterior reads the rows: a streaming pool must be in
    if (rows_ready && forest && !rf_summ) BX_CUDA(h, cudaStreamWaitEvent(s, rows_ready, 0));
    if (timing == 1 && !rf_summ) BX_CUDA(h, cudaEventRecord(h->ev_t[0], s));
    if (forest && !rf_summ)
      BX_CUDA(h, launch_rf(a.space, h->forest, rows, q, (flags & BX_SCORE_RF_PAIRWISE) ? 1 : 0,
                           h->d_probs.as<double>(), s, h->pw_rows));
    if (timing == 1 && !rf_summ) BX_CUDA(h, cudaEventRecord(h->ev_t[1], s));
    BX_CUDA(h, h->d_ei.ensure((size_t)q * 16));
    FusedArgs f = fused_args(h, rows, q, f_model);
    f.mean_out = h->d_ei.as<double>();
    f.var_out = h->d_ei.as<double>() + q;
    if (timing) BX_CUDA(h, cudaEventRecord(h->ev_t[2], s));
    BX_CUDA(h, launch_posterior(h, f, s));
    if (timing) BX_CUDA(h, cudaEventRecord(h->ev_t[3], s));
    SummaryArgs m = last_summary_args(h, rows, q, index_base, eps_f, k, values, probs_out, partials);
    m.track_prob = track_prob ? 1 : 0;
    m.mean = h->d_ei.as<double>();
    m.var = h->d_ei.as<double>() + q;
    m.f_model = f_model;
    if (rows_ready) BX_CUDA(h, cudaStreamWaitEvent(s, rows_ready, 0));  // streaming pool fully copied
    if (rf_summ) {
      if (timing == 1) BX_CUDA(h, cudaEventRecord(h->ev_t[0], s));
      BX_CUDA(h, launch_rf_summary(a.space, h->forest, m, h->sm_count, s, n_partials));
      if (timing == 1) BX_CUDA(h, cudaEventRecord(h->ev_t[1], s));
      return BX_OK;
    }
    BX_CUDA(h, launch_summary(m, h->sm_count, s, n_partials));
    return BX_OK;
  }
  if (timing == 1) BX_CUDA(h, cudaEventRecord(h->ev_t[0], s));
  if (forest) {
    BX_CUDA(h, launch_rf(a.space, h->forest, rows, q, (flags & BX_SCORE_RF_PAIRWISE) ? 1 : 0,
                         h->d_probs.as<double>(), s, h->pw_rows));
    a.probs_in = h->d_probs.as<double>();
  }
  if (timing == 1) BX_CUDA(h, cudaEventRecord(h->ev_t[1], s));
  if (timing) BX_CUDA(h, cudaEventRecord(h->ev_t[2], s));
  BX_CUDA(h, launch_score(a, h->sm_count, s, n_partials));
  if (timing) BX_CUDA(h, cudaEventRecord(h->ev_t[3], s));
  return BX_OK;
}

extern "C" {

int bx_score(bx_handle* h, const uint32_t* rows, int64_t q, int64_t index_base, double f_model,
             double eps_f, int32_t k, int32_t flags, double* values, double* probs,
             bx_score_summary* summary, void* stream) {
  int r = check_gp(h);
  if (r) return r;
  if (q < 1) return fail(h, BX_ERR_ARG, "empty candidate pool");
  if (k < 0 || k > BX_MAX_K) return fail(h, BX_ERR_ARG, "k=%d outside [0, %d]", k, BX_MAX_K);
  cudaSetDevice(h->device);
  cudaStream_t s = (cudaStream_t)stream;
  const bool want = !(flags & BX_SCORE_NO_SUMMARY) && summary != nullptr;
  const int timing = (flags & BX_SCORE_TIMING) ? 1 : ((flags & BX_SCORE_TIMING_POSTERIOR) ? 2 : 0);
  Partial* partials = nullptr;
  if (want) {
    BX_CUDA(h, h->d_partials.ensure(sizeof(Partial) * (size_t)max_partials(h->sm_count)));
    BX_CUDA(h, h->d_summary.ensure(sizeof(bx_score_summary)));
    partials = h->d_partials.as<Partial>();
  }
  int np = 0;
  r = score_impl(h, rows, q, index_base, f_model, eps_f, k, flags, values, probs, partials, &np, s,
                 timing);
  if (r) return r;
  if (want) {
    BX_CUDA(h, launch_summary_merge(partials, np, space_dev(h), k, rows, index_base,
                                    h->d_summary.as<bx_score_summary>(), s));
    if (timing == 1) BX_CUDA(h, cudaEventRecord(h->ev_t[4], s));
    BX_CUDA(h, cudaMemcpyAsync(summary, h->d_summary.p, sizeof(bx_score_summary),
                               cudaMemcpyDeviceToHost, s));
  } else if (timing == 1) {
    BX_CUDA(h, cudaEventRecord(h->ev_t[4], s));
  }
  if (want || timing) BX_CUDA(h, cudaStreamSynchronize(s));
  if (want && summary->n_finite == 0 && fused_path(h)) {
    // every value is -inf: only now is the probability tracker needed (acquisition.py:179-184)
    // rerun the step with the tracker on (it is the only rare path, so no state is kept for it)
    r = score_impl(h, rows, q, index_base, f_model, eps_f, k, flags & ~(BX_SCORE_TIMING | BX_SCORE_TIMING_POSTERIOR),
                   values, probs, partials, &np, s, 0, true);
    if (r) return r;
    BX_CUDA(h, launch_summary_merge(partials, np, space_dev(h), k, rows, index_base,
                                    h->d_summary.as<bx_score_summary>(), s));
    BX_CUDA(h, cudaMemcpyAsync(summary, h->d_summary.p, sizeof(bx_score_summary),
                               cudaMemcpyDeviceToHost, s));
    BX_CUDA(h, cudaStreamSynchronize(s));
  }
  if (timing == 1) {
    cudaEventElapsedTime(&h->t_ms[0], h->ev_t[0], h->ev_t[1]);
    cudaEventElapsedTime(&h->t_ms[1], h->ev_t[2], h->ev_t[3]);
    cudaEventElapsedTime(&h->t_ms[2], h->rf_after_gp ? h->ev_t[1] : h->ev_t[3], h->ev_t[4]);
  } else if (timing == 2) {  // the posterior only: the other kernels run back to back, unobserved
    cudaEventElapsedTime(&h->t_ms[1], h->ev_t[2], h->ev_t[3]);
    h->t_ms[0] = h->t_ms[2] = -1.0f;
  }
  return BX_OK;
}

int bx_last_timing(bx_handle* h, float* rf_ms, float* score_ms, float* merge_ms) {
  if (!h) return BX_ERR_ARG;
  if (rf_ms) *rf_ms = h->t_ms[0];
  if (score_ms) *score_ms = h->t_ms[1];
  if (merge_ms) *merge_ms = h->t_ms[2];
  return BX_OK;
}

int bx_score_host(bx_handle* h, const uint32_t* host_rows, int64_t q, int64_t index_base,
                  double f_model, double eps_f, int32_t k, int32_t flags,
                  bx_score_summary* summary, void* stream) {
  int r = check_gp(h);
  if (r) return r;
  if (q < 1) return fail(h, BX_ERR_ARG, "empty candidate pool");
  if (!summary) return fail(h, BX_ERR_ARG, "bx_score_host needs a summary");
  if (k < 0 || k > BX_MAX_K) return fail(h, BX_ERR_ARG, "k=%d outside [0, %d]", k, BX_MAX_K);
  cudaSetDevice(h->device);
  cudaStream_t s = (cudaStream_t)stream;
  const int W = h->row_words;
  const bool packed = (flags & BX_SCORE_PACKED) != 0;
  const int HW = packed ? h->pack.pw : W;  // words per host row
  flags &= ~(BX_SCORE_PACKED | BX_SCORE_NO_SUMMARY);
  BX_CUDA(h, h->d_pool.ensure((size_t)q * W * 4));
  if (packed) BX_CUDA(h, h->d_packed.ensure((size_t)q * HW * 4));
  BX_CUDA(h, h->d_partials.ensure(sizeof(Partial) * (size_t)max_partials(h->sm_count)));
  BX_CUDA(h, h->d_summary.ensure(sizeof(bx_score_summary)));
  uint32_t* pool = h->d_pool.as<uint32_t>();
  uint32_t* dst = packed ? h->d_packed.as<uint32_t>() : pool;  // where the host rows land
  Partial* parts = h->d_partials.as<Partial>();
  const bool forest = h->has_forest && h->forest.has_trees;
  // Packed rows in pinned (hence mapped) host memory: the posterior's row prefetcher bulk-copies
  // each tile's packed rows straight from host memory over the bus - no copy engine, no ready
  // flags, nothing that depends on the copy running concurrently with the kernel (profilers and
  // CUDA_LAUNCH_BLOCKING serialise the two).  BX_TC_DEBUG bit 64: always the copy path.
  const uint32_t* mapped = nullptr;
  if (packed && h->use_tc && !(h->tc_debug & 64)) {
    cudaPointerAttributes at{};
    if (cudaPointerGetAttributes(&at, host_rows) == cudaSuccess && at.type == cudaMemoryTypeHost && at.devicePointer)
      mapped = static_cast<const uint32_t*>(at.devicePointer);
    cudaGetLastError();  // pageable memory: clear the attribute query's error, take the copy path
    if (mapped && (h->tc_debug & 128)) {  // timing experiment: the same path over a device copy
      BX_CUDA(h, cudaMemcpyAsync(dst, host_rows, (size_t)q * HW * 4, cudaMemcpyHostToDevice, s));
      mapped = dst;
    }
  }
  if (mapped && (!forest || qs_summary_available(h->forest)) && !(flags & BX_SCORE_RF_PAIRWISE) &&
      h->pack.pw <= 16) {
    for (int pass = 0; pass < 2; ++pass) {  // pass 2 (probability tracker) only if every value is -inf
      int np = 0;
      h->stream_packed = pass == 0 ? mapped : nullptr;  // pass 2 reads the pool the decoders unpacked
      r = score_impl(h, pool, q, index_base, f_model, eps_f, k, flags, nullptr, nullptr, parts, &np, s, false,
                     pass == 1);
      h->stream_packed = nullptr;
      if (r) return r;
      BX_CUDA(h, launch_summary_merge(parts, np, space_dev(h), k, nullptr, 0,
                                      h->d_summary.as<bx_score_summary>(), s));
      BX_CUDA(h, cudaMemcpyAsync(summary, h->d_summary.p, sizeof(bx_score_summary), cudaMemcpyDeviceToHost, s));
      BX_CUDA(h, cudaStreamSynchronize(s));
      if (summary->n_finite != 0) break;
    }
  } else if (h->use_tc && (!forest || qs_summary_available(h->forest)) && !(flags & BX_SCORE_RF_PAIRWISE) &&
             (!packed || h->pack.pw <= 16)) {
    // Streaming: the whole pool is copied in 2^16-row chunks on the copy stream, each followed by a
    // 4-byte ready flag written by the copy engine; one posterior launch consumes tiles as their
    // chunk lands (the row prefetcher waits on the flag; packed rows are unpacked by its decoders,
    // which write the full rows for the kernels after it), so only the first chunk's copy is
    // exposed and there is no per-chunk launch cost.  The forest + summary kernel runs after the
    // last copy.
    const int shift = 16;
    const int64_t n_chunks = (q + (1 << shift) - 1) >> shift;
    BX_CUDA(h, h->d_ready.ensure((size_t)n_chunks * 4));
    if (h->h_ones_len < n_chunks) {
      if (h->h_ones) cudaFreeHost(h->h_ones);
      h->h_ones = nullptr;
      BX_CUDA(h, cudaMallocHost(&h->h_ones, (size_t)n_chunks * 4));
      for (int64_t i = 0; i < n_chunks; ++i) h->h_ones[i] = 1u;
      h->h_ones_len = n_chunks;
    }
    uint32_t* ready = h->d_ready.as<uint32_t>();
    BX_CUDA(h, cudaMemsetAsync(ready, 0, (size_t)n_chunks * 4, s));
    BX_CUDA(h, cudaEventRecord(h->ev_done, s));
    BX_CUDA(h, cudaStreamWaitEvent(h->copy_stream, h->ev_done, 0));
    for (int64_t c = 0; c < n_chunks; ++c) {
      const int64_t off = c << shift, len = std::min<int64_t>((int64_t)1 << shift, q - off);
      BX_CUDA(h, cudaMemcpyAsync(dst + (size_t)off * HW, host_rows + (size_t)off * HW, (size_t)len * HW * 4,
                                 cudaMemcpyHostToDevice, h->copy_stream));
      BX_CUDA(h, cudaMemcpyAsync(ready + c, h->h_ones + c, 4, cudaMemcpyHostToDevice, h->copy_stream));
    }
    BX_CUDA(h, cudaEventRecord(h->ev_copy, h->copy_stream));
    for (int pass = 0; pass < 2; ++pass) {  // pass 2 (probability tracker) only if every value is -inf
      int np = 0;
      h->stream_ready = pass == 0 ? ready : nullptr;
      h->stream_shift = shift;
      h->stream_packed = (pass == 0 && packed) ? dst : nullptr;  // pass 2 reads the unpacked pool
      r = score_impl(h, pool, q, index_base, f_model, eps_f, k, flags, nullptr, nullptr, parts, &np, s, false,
                     pass == 1, pass == 0 ? h->ev_copy : nullptr);
      h->stream_ready = nullptr;
      h->stream_packed = nullptr;
      if (r) return r;
      BX_CUDA(h, launch_summary_merge(parts, np, space_dev(h), k, nullptr, 0,
                                      h->d_summary.as<bx_score_summary>(), s));
      BX_CUDA(h, cudaMemcpyAsync(summary, h->d_summary.p, sizeof(bx_score_summary), cudaMemcpyDeviceToHost, s));
      BX_CUDA(h, cudaStreamSynchronize(s));
      if (summary->n_finite != 0) break;
    }
  } else {
    // the other kernel paths: one copy (and a device unpack), then the device-resident path
    BX_CUDA(h, cudaMemcpyAsync(dst, host_rows, (size_t)q * HW * 4, cudaMemcpyHostToDevice, s));
    if (packed) BX_CUDA(h, launch_unpack(h->pack, dst, q, W, pool, s));
    r = bx_score(h, pool, q, index_base, f_model, eps_f, k, flags, nullptr, nullptr, summary, stream);
    if (r) return r;
  }
  // the pool is host-resident: the top-k rows come straight from the caller's buffer
  for (int i = 0; i < summary->n_top; ++i) {
    const uint32_t* src = host_rows + (size_t)(summary->top[i].index - index_base) * HW;
    if (packed) unpack_row(h->pack, src, summary->top[i].row, W);
    else std::memcpy(summary->top[i].row, src, (size_t)W * 4);
  }
  return BX_OK;
}

int bx_gp_predict(bx_handle* h, const uint32_t* rows, int64_t q, double* mean, double* var,
                  void* stream) {
  int r = check_gp(h);
  if (r) return r;
  if (q < 1) return BX_OK;
  cudaSetDevice(h->device);
  ScoreArgs a{};
  a.space = space_dev(h);
  a.gp = gp_dev(h);
  a.evald = EvalSetDev{};
  a.rows = rows;
  a.q = q;
  a.f_model = 0.0;
  a.mean_out = mean;
  a.var_out = var;
  int np = 0;
  if (fused_path(h)) {
    FusedArgs f = fused_args(h, rows, q, 0.0);
    f.mean_out = mean;
    f.var_out = var;
    BX_CUDA(h, launch_posterior(h, f, (cudaStream_t)stream));
    return BX_OK;
  }
  BX_CUDA(h, launch_score(a, h->sm_count, (cudaStream_t)stream, &np));
  return BX_OK;
}

int bx_rf_predict(bx_handle* h, const uint32_t* rows, int64_t q, int32_t flags, double* probs,
                  void* stream) {
  int r = check_space(h);
  if (r) return r;
  if (!h->has_forest) return fail(h, BX_ERR_STATE, "bx_set_forest has not been called");
  if (q < 1) return BX_OK;
  cudaSetDevice(h->device);
  cudaStream_t s = (cudaStream_t)stream;
  if (!h->forest.has_trees) {
    std::vector<double> c((size_t)q, h->forest.constant);
    BX_CUDA(h, cudaMemcpyAsync(probs, c.data(), (size_t)q * 8, cudaMemcpyHostToDevice, s));
    BX_CUDA(h, cudaStreamSynchronize(s));
    return BX_OK;
  }
  BX_CUDA(h, launch_rf(space_dev(h), h->forest, rows, q, (flags & BX_SCORE_RF_PAIRWISE) ? 1 : 0,
                       probs, s));
  return BX_OK;
}

int bx_climb(bx_handle* h, const uint32_t* dev_pool_rows, const int64_t* host_start_index,
             const double* host_start_values, int32_t n_starts, int32_t use_cot, double f_model, double eps_f,
             int32_t max_steps, bx_cand* host_best, int32_t* host_steps, void* stream) {
  int r = check_gp(h);
  if (r) return r;
  if (n_starts < 0 || n_starts > BX_MAX_K || !host_best) return fail(h, BX_ERR_ARG, "bad climb arguments");
  if (use_cot && !h->has_cot) return fail(h, BX_ERR_STATE, "bx_set_cot has not been called");
  if (host_steps) *host_steps = 0;
  if (n_starts == 0) return BX_OK;
  cudaSetDevice(h->device);
  cudaStream_t s = (cudaStream_t)stream;
  const int A = n_starts, S = h->n_slots, W = h->row_words;
  // scratch: cur rows, values, active flags, neighbour rows, valid, pairwise flags, values, state
  size_t off = 0;
  auto take = [&](size_t bytes) { const size_t o = off; off += (bytes + 255) & ~(size_t)255; return o; };
  const size_t o_cur = take((size_t)A * W * 4), o_curv = take((size_t)A * 8), o_act = take((size_t)A * 4),
               o_nb = take((size_t)A * S * W * 4), o_val = take((size_t)A * S), o_pw = take((size_t)A * S),
               o_vals = take((size_t)A * S * 8), o_probs = take((size_t)A * S * 8), o_st = take(sizeof(ClimbState));
  BX_CUDA(h, h->d_climb.ensure(off));
  unsigned char* base = h->d_climb.as<unsigned char>();
  uint32_t* cur = reinterpret_cast<uint32_t*>(base + o_cur);
  double* curv = reinterpret_cast<double*>(base + o_curv);
  int32_t* act = reinterpret_cast<int32_t*>(base + o_act);
  uint32_t* nb = reinterpret_cast<uint32_t*>(base + o_nb);
  uint8_t* valid = base + o_val;
  uint8_t* pw = base + o_pw;
  double* vals = reinterpret_cast<double*>(base + o_vals);
  double* probs = reinterpret_cast<double*>(base + o_probs);
  ClimbState* st = reinterpret_cast<ClimbState*>(base + o_st);
  ClimbState hs{};
  hs.n_active = A;
  hs.best = TopRec{host_best->value, host_best->prob, host_best->index};
  std::memcpy(hs.best_row, host_best->row, sizeof(hs.best_row));
  std::vector<int32_t> ones(A, 1);
  for (int a = 0; a < A; ++a)  // the start rows, gathered from the pool
    BX_CUDA(h, cudaMemcpyAsync(cur + (size_t)a * W, dev_pool_rows + (size_t)host_start_index[a] * W, (size_t)W * 4,
                               cudaMemcpyDeviceToDevice, s));
  BX_CUDA(h, cudaMemcpyAsync(curv, host_start_values, (size_t)A * 8, cudaMemcpyHostToDevice, s));
  BX_CUDA(h, cudaMemcpyAsync(act, ones.data(), (size_t)A * 4, cudaMemcpyHostToDevice, s));
  BX_CUDA(h, cudaMemcpyAsync(st, &hs, sizeof(ClimbState), cudaMemcpyHostToDevice, s));
  if (!h->h_climb_flag) BX_CUDA(h, cudaMallocHost(&h->h_climb_flag, 64));
  // Steps go out in batches of kClimbBatch with one 4-byte read of the active count per batch: a
  // step whose starts have all stopped is a no-op (no start moves, nothing is folded, the step
  // count does not advance), so the batch's tail changes nothing, and the host stays ahead of the
  // device instead of waiting on every step.
  constexpr int kClimbBatch = 4;
  for (int step = 0; step < max_steps && hs.n_active > 0;) {
    const int batch = std::min(kClimbBatch, max_steps - step);
    for (int b = 0; b < batch; ++b) {
      BX_CUDA(h, launch_neighbors(space_dev(h), use_cot ? &h->cot : nullptr, cur, A, nb, valid, s));
      climb_flags_kernel<<<1, 32, 0, s>>>(A, S, act, valid, pw);
      BX_CUDA(h, cudaGetLastError());
      h->pw_rows = pw;
      int np = 0;
      r = score_impl(h, nb, (int64_t)A * S, 0, f_model, eps_f, 0, 0, vals, probs, nullptr, &np, s, 0);
      h->pw_rows = nullptr;
      if (r) return r;
      climb_update_kernel<<<1, 32 * A, 0, s>>>(space_dev(h), eval_dev(h), A, S, act, cur, curv, nb, valid, vals,
                                               st);
      BX_CUDA(h, cudaGetLastError());
    }
    step += batch;
    BX_CUDA(h, cudaMemcpyAsync(h->h_climb_flag, &st->n_active, 4, cudaMemcpyDeviceToHost, s));
    BX_CUDA(h, cudaStreamSynchronize(s));  // the one device -> host read per batch
    hs.n_active = *h->h_climb_flag;
  }
  BX_CUDA(h, cudaMemcpyAsync(&hs, st, sizeof(ClimbState), cudaMemcpyDeviceToHost, s));
  BX_CUDA(h, cudaStreamSynchronize(s));
  host_best->value = hs.best.value;
  host_best->prob = hs.best.prob;
  host_best->index = hs.best.index;
  std::memcpy(host_best->row, hs.best_row, sizeof(hs.best_row));
  if (host_steps) *host_steps = hs.steps;
  return BX_OK;
}

static int check_generate(bx_handle* h, int32_t mode) {
  int r = check_space(h);
  if (r) return r;
  if (mode < 0 || mode > 2) return fail(h, BX_ERR_ARG, "generation mode %d not in {0, 1, 2}", mode);
  if (mode == 1 && !(h->has_cot && h->has_leaf_count))
    return fail(h, BX_ERR_STATE, "mode 1 needs bx_set_cot with node leaf counts");
  if (mode == 2 && !h->has_cot) return fail(h, BX_ERR_STATE, "mode 2 needs bx_set_cot");
  return BX_OK;
}

int bx_generate(bx_handle* h, uint64_t seed, int64_t index_base, int64_t q, int32_t mode,
                uint32_t* rows, void* stream) {
  int r = check_generate(h, mode);
  if (r) return r;
  cudaSetDevice(h->device);
  CotDev cot = h->has_cot ? h->cot : CotDev{};
  BX_CUDA(h, launch_generate(space_dev(h), cot, h->d_leaf_count.as<int64_t>(), mode, seed, index_base,
                             q, rows, (cudaStream_t)stream));
  return BX_OK;
}

int bx_score_generated(bx_handle* h, uint64_t seed, int64_t index_base, int64_t q, int32_t mode,
                       double f_model, double eps_f, int32_t k, bx_score_summary* summary,
                       void* stream) {
  int r = check_gp(h);
  if (r) return r;
  r = check_generate(h, mode);
  if (r) return r;
  if (q < 1) return fail(h, BX_ERR_ARG, "empty candidate pool");
  if (!summary) return fail(h, BX_ERR_ARG, "bx_score_generated needs a summary");
  if (k < 0 || k > BX_MAX_K) return fail(h, BX_ERR_ARG, "k=%d outside [0, %d]", k, BX_MAX_K);
  cudaSetDevice(h->device);
  cudaStream_t s = (cudaStream_t)stream;
  const int W = h->row_words;
  const int64_t chunk = 1 << 22;
  const int64_t n_chunks = (q + chunk - 1) / chunk;
  const size_t per_chunk = (size_t)max_partials(h->sm_count);
  BX_CUDA(h, h->d_partials.ensure(sizeof(Partial) * per_chunk * (size_t)n_chunks));
  BX_CUDA(h, h->d_summary.ensure(sizeof(bx_score_summary)));
  BX_CUDA(h, h->d_gen_rows.ensure((size_t)chunk * W * 4));
  CotDev cot = h->has_cot ? h->cot : CotDev{};
  Partial* base = h->d_partials.as<Partial>();
  // Partials per chunk: one per SM (forest + summary kernel) or two (summary kernel).  They are
  // merged once at the end when all of them fit the fast merge, else folded into a running
  // partial after every chunk.
  const bool rf_summ = h->use_tc && h->has_forest && h->forest.has_trees && qs_summary_available(h->forest);
  const int64_t np_max = fused_path(h) ? (rf_summ ? 1 : 2) * (int64_t)h->sm_count : (int64_t)per_chunk;
  const bool fits_once = np_max * n_chunks <= 1024 &&
                         np_max * n_chunks * (k > 0 ? k : 1) * (int64_t)sizeof(TopRec) <= 200 * 1024;
  const bool running = !fits_once && np_max + 1 <= 1024 &&
                       (np_max + 1) * (k > 0 ? k : 1) * (int64_t)sizeof(TopRec) <= 200 * 1024;
  for (int pass = 0; pass < 2; ++pass) {
    int total = 0;
    for (int64_t c = 0; c < n_chunks; ++c) {
      const int64_t off = c * chunk;
      const int64_t len = (q - off) < chunk ? (q - off) : chunk;
      BX_CUDA(h, launch_generate(space_dev(h), cot, h->d_leaf_count.as<int64_t>(), mode, seed,
                                 index_base + off, len, h->d_gen_rows.as<uint32_t>(), s));
      int np = 0;
      Partial* dst = running ? base + 1 : base + total;
      r = score_impl(h, h->d_gen_rows.as<uint32_t>(), len, index_base + off, f_model, eps_f, k, 0,
                     nullptr, nullptr, dst, &np, s, false, pass == 1);
      if (r) return r;
      if (running)
        BX_CUDA(h, c == 0 ? launch_partial_merge(base + 1, np, space_dev(h), k, base, s)
                          : launch_partial_merge(base, np + 1, space_dev(h), k, base, s));
      total = running ? 1 : total + np;
    }
    BX_CUDA(h, launch_summary_merge(base, total, space_dev(h), k, nullptr, 0,
                                    h->d_summary.as<bx_score_summary>(), s));
    BX_CUDA(h, cudaMemcpyAsync(summary, h->d_summary.p, sizeof(bx_score_summary),
                               cudaMemcpyDeviceToHost, s));
    BX_CUDA(h, cudaStreamSynchronize(s));
    if (summary->n_finite != 0 || !fused_path(h)) break;
  }
  // regenerate the top-k rows from their global indices
  int64_t idx[BX_MAX_K];
  for (int i = 0; i < summary->n_top; ++i) idx[i] = summary->top[i].index;
  if (summary->n_top > 0) {
    BX_CUDA(h, launch_generate_indexed(space_dev(h), cot, h->d_leaf_count.as<int64_t>(), mode, seed,
                                       idx, summary->n_top, h->d_gen_rows.as<uint32_t>(), s));
    std::vector<uint32_t> rows((size_t)summary->n_top * W);
    BX_CUDA(h, cudaMemcpyAsync(rows.data(), h->d_gen_rows.p, rows.size() * 4, cudaMemcpyDeviceToHost, s));
    BX_CUDA(h, cudaStreamSynchronize(s));
    for (int i = 0; i < summary->n_top; ++i)
      std::memcpy(summary->top[i].row, rows.data() + (size_t)i * W, (size_t)W * 4);
  }
  return BX_OK;
}

}  // extern "C"
