// summary.cuh — per-warp partial summaries: stable top-k by (value desc, index asc)
// (acquisition.py:188) and the _Tracker reductions (acquisition.py:97-111).
#pragma once
#include "bx_common.cuh"
namespace bx {
__device__ inline void partial_init(Partial* s) {
  s->n_scored = 0;
  s->n_finite = 0;
  s->n_top = 0;
  s->best = TopRec{-INFINITY, -INFINITY, -1};
  s->best_prob = TopRec{-INFINITY, -INFINITY, -1};
}

__device__ __forceinline__ bool top_before(double v, int64_t g, const TopRec& r) {
  return v > r.value || (v == r.value && g < r.index);
}

__device__ inline void top_insert(TopRec* top, int& n_top, int k, const TopRec& rec) {
  if (k <= 0) return;
  if (n_top == k && !top_before(rec.value, rec.index, top[k - 1])) return;
  int pos = n_top < k ? n_top : k - 1;
  while (pos > 0 && top_before(rec.value, rec.index, top[pos - 1])) {
    top[pos] = top[pos - 1];
    --pos;
  }
  top[pos] = rec;
  if (n_top < k) ++n_top;
}

// Fold one scored candidate into a partial (single lane).
__device__ inline void partial_add(Partial* s, int k, const bx_param_desc* params, int n_params,
                            const int32_t* rank_lut, int words, double v, double p, int64_t g,
                            bool evaluated, const uint32_t* row, bool track_prob = true) {
  if (v != -INFINITY) {
    int nt = s->n_top;
    top_insert(s->top, nt, k, TopRec{v, p, g});
    s->n_top = nt;
    if (!evaluated) {
      bool take = v > s->best.value;
      if (!take && v == s->best.value)
        take = s->best.index < 0 || key_cmp(params, n_params, rank_lut, row, s->best_row) < 0;
      if (take) {
        s->best = TopRec{v, p, g};
        for (int w = 0; w < words; ++w) s->best_row[w] = row[w];
      }
    }
  }
  if (track_prob && !evaluated && p != -INFINITY) {
    bool take = p > s->best_prob.prob;
    if (!take && p == s->best_prob.prob)
      take = s->best_prob.index < 0 || key_cmp(params, n_params, rank_lut, row, s->best_prob_row) < 0;
    if (take) {
      s->best_prob = TopRec{v, p, g};
      for (int w = 0; w < words; ++w) s->best_prob_row[w] = row[w];
    }
  }
}

}  // namespace bx

namespace bx {
// Merge partial `b` into `a` (single lane); same total orders as partial_add.
__device__ inline void partial_merge(Partial* a, const Partial* b, int k, const bx_param_desc* params,
                                     int n_params, const int32_t* rank_lut, int words) {
  a->n_scored += b->n_scored;
  a->n_finite += b->n_finite;
  int nt = a->n_top;
  for (int i = 0; i < b->n_top; ++i) {
    if (nt == k && !top_before(b->top[i].value, b->top[i].index, a->top[k - 1])) break;
    top_insert(a->top, nt, k, b->top[i]);
  }
  a->n_top = nt;
  if (b->best.index >= 0) {
    bool take = a->best.index < 0 || b->best.value > a->best.value;
    if (!take && b->best.value == a->best.value)
      take = key_cmp(params, n_params, rank_lut, b->best_row, a->best_row) < 0;
    if (take) {
      a->best = b->best;
      for (int w = 0; w < words; ++w) a->best_row[w] = b->best_row[w];
    }
  }
  if (b->best_prob.index >= 0) {
    bool take = a->best_prob.index < 0 || b->best_prob.prob > a->best_prob.prob;
    if (!take && b->best_prob.prob == a->best_prob.prob)
      take = key_cmp(params, n_params, rank_lut, b->best_prob_row, a->best_prob_row) < 0;
    if (take) {
      a->best_prob = b->best_prob;
      for (int w = 0; w < words; ++w) a->best_prob_row[w] = b->best_prob_row[w];
    }
  }
}
}  // namespace bx
