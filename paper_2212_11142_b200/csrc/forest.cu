// forest.cu — random-forest feasibility probability (FeasibilityModel.predict_proba_batch,
// feasibility.py:72-89) over encoded rows, bit-exact.
//
// Kernels:
//  * rf_qs_kernel / rf_qs_summary_kernel (fast path): QuickScorer tables (QsForestDev) — per tree
//    and code value the AND of the leaf-elimination masks of the right-going splits on that code;
//    a candidate's exit leaf is the lowest set bit of the AND of its codes' masks.  Codes: an
//    integer / ordinal index, a permutation element's position, a categorical label index (its
//    one-hot masks pre-ANDed), a real coordinate's rank among the parameter's split thresholds.
//    The summary variant also forms p * EI, the eps_f filter and per-warp top-k / trackers.
//  * rf_coded_kernel: the forest is integer-coded on the host (CodedForestDev): each
//    split is `code < cut` on a per-candidate integer code, the node table and leaf values sit in
//    shared memory, leaves point at themselves so two trees can be walked in lockstep with no
//    per-tree exit branch.  One 512-thread CTA per SM.
//  * rf_kernel (generic): f64 comparisons on features produced on the fly from the row exactly as
//    encode_configs builds them (feasibility.py:33-51); used when the coding preconditions fail.
// Both reproduce `x <= threshold` (feasibility.py:86) exactly and numpy's summation order for the
// mean over trees: sequential over trees for q >= 2 (the (T, q) reduction over axis 0), numpy's
// pairwise_sum (8 accumulators, 128-element blocks) for q == 1.
#include "bx_common.cuh"
#include "summary.cuh"

namespace bx {

namespace {

// ---- generic path --------------------------------------------------------------------------
__device__ __forceinline__ double feature_value(const SpaceDev& sp, const bx_param_desc* params,
                                                const uint32_t* row, int f) {
  const int k = sp.feat_param[f];
  const int sub = sp.feat_sub[f];
  const bx_param_desc& p = params[k];
  if (p.kind == BX_CATEGORICAL) return (int)row[p.word] == sub ? 1.0 : 0.0;
  if (p.kind == BX_PERMUTATION) return (double)perm_pos(row_u64(row, p.word), p.size, sub);
  return row_coord(p, sp.coord_lut, row);
}

__device__ __forceinline__ double leaf_value(const SpaceDev& sp, const bx_param_desc* params,
                                             const ForestDev& f, const uint32_t* row, int tree) {
  int cur = f.roots[tree];
  for (int it = 0; it <= f.max_depth; ++it) {  // feasibility.py:80: max_depth + 1 descents
    const RfNode nd = f.nodes[cur];
    if (nd.feat < 0) break;
    const double x = feature_value(sp, params, row, nd.feat);
    cur = (x <= nd.thr) ? nd.child : nd.child + 1;
  }
  return f.nodes[cur].val;
}

// numpy pairwise_sum (numpy/_core/src/umath/loops_utils.h.src) over values v(t0 .. t0+cnt-1)
template <typename F>
__device__ double pairwise(const F& v, int t0, int cnt) {
  if (cnt < 8) {
    double res = 0.0;
    for (int i = 0; i < cnt; ++i) res = __dadd_rn(res, v(t0 + i));
    return res;
  }
  if (cnt <= 128) {
    double r[8];
    for (int i = 0; i < 8; ++i) r[i] = v(t0 + i);
    int i = 8;
    for (; i < cnt - (cnt % 8); i += 8)
      for (int j = 0; j < 8; ++j) r[j] = __dadd_rn(r[j], v(t0 + i + j));
    double res = __dadd_rn(__dadd_rn(__dadd_rn(r[0], r[1]), __dadd_rn(r[2], r[3])),
                           __dadd_rn(__dadd_rn(r[4], r[5]), __dadd_rn(r[6], r[7])));
    for (; i < cnt; ++i) res = __dadd_rn(res, v(t0 + i));
    return res;
  }
  int n2 = cnt / 2;
  n2 -= n2 % 8;
  return __dadd_rn(pairwise(v, t0, n2), pairwise(v, t0 + n2, cnt - n2));
}

__global__ void __launch_bounds__(256) rf_kernel(SpaceDev sp, ForestDev f, const uint32_t* rows,
                                                 int64_t q, int use_pairwise, double* probs, const uint8_t* pw_rows) {
  __shared__ bx_param_desc params[BX_MAX_PARAMS];
  for (int i = threadIdx.x; i < sp.n_params * (int)sizeof(bx_param_desc) / 4; i += blockDim.x)
    reinterpret_cast<int32_t*>(params)[i] = reinterpret_cast<const int32_t*>(sp.params)[i];
  __syncthreads();
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < q;
       i += (int64_t)gridDim.x * blockDim.x) {
    const uint32_t* row = rows + (size_t)i * sp.row_words;
    double sum;
    if (pw_rows ? pw_rows[i] != 0 : use_pairwise != 0) {
      sum = pairwise([&](int t) { return leaf_value(sp, params, f, row, t); }, 0, f.n_trees);
    } else {
      sum = leaf_value(sp, params, f, row, 0);
      for (int t = 1; t < f.n_trees; ++t) sum = __dadd_rn(sum, leaf_value(sp, params, f, row, t));
    }
    probs[i] = __ddiv_rn(sum, (double)f.n_trees);  // np.mean: sum / count
  }
}

// ---- integer-coded fast path -----------------------------------------------------------------
constexpr int kRfThreads = 512;

struct CodedView {
  const uint2* nodes;       // .x = arg | slot << 24 | type << 30, .y = left child
  const uint32_t* leaf_idx;
  const double* leaf;
  const int32_t* code;      // [n_codes][kRfThreads] (shared): column t of this thread
  const double* real;       // [n_codes][kRfThreads] (shared, only with real splits)
  const double* real_thr;
};

// one descent step; a leaf maps to itself (its argument 0xFFFFFF exceeds every code)
template <bool REAL>
__device__ __forceinline__ int step(const CodedView& v, int cur) {
  const uint2 nd = v.nodes[cur];
  const int slot = (int)((nd.x >> 24) & 63u);
  const int arg = (int)(nd.x & 0xFFFFFFu);
  bool right = v.code[slot * kRfThreads] >= arg;
  if (REAL && (nd.x >> 30) == 1u) right = !(v.real[slot * kRfThreads] <= v.real_thr[arg]);
  return (int)nd.y + (right ? 1 : 0);
}

__device__ __forceinline__ double leaf_of(const CodedView& v, int cur) {
  return v.leaf[v.leaf_idx[cur]];
}

template <bool REAL>
__device__ __forceinline__ double walk1(const CodedView& v, int root, int max_depth) {
  int cur = root;
  for (int it = 0; it <= max_depth; ++it) {
    const int nxt = step<REAL>(v, cur);
    if (nxt == cur) break;
    cur = nxt;
  }
  return leaf_of(v, cur);
}

template <bool SMEM, bool REAL>
__global__ void __launch_bounds__(kRfThreads, 1) rf_coded_kernel(SpaceDev sp, CodedForestDev cf,
                                                                 const uint32_t* rows, int64_t q,
                                                                 int use_pairwise, double* probs,
                                                                 const uint8_t* pw_rows) {
  extern __shared__ __align__(16) unsigned char smem[];
  __shared__ bx_param_desc params[BX_MAX_PARAMS];
  size_t off = 0;
  uint64_t* s_nodes = reinterpret_cast<uint64_t*>(smem);
  double* s_leaf = reinterpret_cast<double*>(smem + (SMEM ? (size_t)cf.n_nodes * 8 : 0));
  uint32_t* s_lidx = reinterpret_cast<uint32_t*>(smem + (SMEM ? ((size_t)cf.n_nodes + cf.n_leaves) * 8 : 0));
  off = SMEM ? ((size_t)cf.n_nodes + cf.n_leaves) * 8 + (((size_t)cf.n_nodes * 4 + 15) & ~(size_t)15) : 0;
  int32_t* s_roots = reinterpret_cast<int32_t*>(smem + off);
  off += ((size_t)cf.n_trees * 4 + 15) & ~(size_t)15;
  int32_t* code = reinterpret_cast<int32_t*>(smem + off);
  off += (size_t)cf.n_codes * kRfThreads * 4;
  double* real = reinterpret_cast<double*>(smem + off);
  for (int i = threadIdx.x; i < sp.n_params * (int)sizeof(bx_param_desc) / 4; i += blockDim.x)
    reinterpret_cast<int32_t*>(params)[i] = reinterpret_cast<const int32_t*>(sp.params)[i];
  if (SMEM) {
    for (int i = threadIdx.x; i < cf.n_nodes; i += blockDim.x) s_nodes[i] = cf.nodes[i];
    for (int i = threadIdx.x; i < cf.n_leaves; i += blockDim.x) s_leaf[i] = cf.leaf_val[i];
    for (int i = threadIdx.x; i < cf.n_nodes; i += blockDim.x) s_lidx[i] = cf.leaf_idx[i];
  }
  for (int i = threadIdx.x; i < cf.n_trees; i += blockDim.x) s_roots[i] = cf.roots[i];
  __syncthreads();
  const CodedView v{reinterpret_cast<const uint2*>(SMEM ? s_nodes : cf.nodes),
                    SMEM ? s_lidx : cf.leaf_idx, SMEM ? s_leaf : cf.leaf_val,
                    code + threadIdx.x, real + threadIdx.x, cf.real_thr};
  const int64_t stride = (int64_t)gridDim.x * blockDim.x;
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < q; i += stride) {
    const uint32_t* row = rows + (size_t)i * sp.row_words;
    for (int c = 0; c < cf.n_codes; ++c) {
      const bx_param_desc& p = params[cf.code_param[c]];
      int val = 0;
      if (p.kind == BX_PERMUTATION) {
        val = perm_pos(row_u64(row, p.word), p.size, cf.code_sub[c]);
      } else if (p.kind == BX_CATEGORICAL) {
        val = (int)row[p.word] == cf.code_sub[c] ? 1 : 0;
      } else if (p.kind == BX_REAL) {
        real[c * kRfThreads + threadIdx.x] = row_f64(row, p.word + 2);
      } else {
        val = (int)row[p.word];
      }
      code[c * kRfThreads + threadIdx.x] = val;
    }
    double sum;
    if (pw_rows ? pw_rows[i] != 0 : use_pairwise != 0) {
      sum = pairwise([&](int t) { return walk1<REAL>(v, s_roots[t], cf.max_depth); }, 0, cf.n_trees);
    } else {
      // two trees in lockstep (independent load chains); leaves added strictly in tree order
      sum = 0.0;
      int t = 0;
      for (; t + 2 <= cf.n_trees; t += 2) {
        int a = s_roots[t], b = s_roots[t + 1];
        for (int it = 0; it <= cf.max_depth; ++it) {
          const int na = step<REAL>(v, a), nb = step<REAL>(v, b);
          if (na == a && nb == b) break;
          a = na;
          b = nb;
        }
        const double la = leaf_of(v, a), lb = leaf_of(v, b);
        sum = (t == 0) ? la : __dadd_rn(sum, la);
        sum = __dadd_rn(sum, lb);
      }
      if (t < cf.n_trees) {
        const double l = walk1<REAL>(v, s_roots[t], cf.max_depth);
        sum = (t == 0) ? l : __dadd_rn(sum, l);
      }
    }
    probs[i] = __ddiv_rn(sum, (double)cf.n_trees);
  }
}

// ---- QuickScorer path (QsForestDev) -----------------------------------------------------------
constexpr int kQsThreads = 1024;
constexpr int kQsGroup = 8;  // trees evaluated together (8 masks in registers)

// explicit shared-space loads (the mask table is indexed through computed offsets, which otherwise
// compile to generic loads)
__device__ __forceinline__ ulonglong2 lds_u64x2(uint32_t saddr) {
  // two 8-byte loads, not one 16-byte load: with an odd mask-row length the <= 16 distinct rows a
  // half-warp touches fall in distinct banks, so each load is a single wavefront per half-warp
  ulonglong2 v;
  asm volatile("ld.shared.u64 %0, [%1];" : "=l"(v.x) : "r"(saddr));
  asm volatile("ld.shared.u64 %0, [%1];" : "=l"(v.y) : "r"(saddr + 8u));
  return v;
}

__device__ __forceinline__ int qs_code(const bx_param_desc& p, const uint32_t* row, int sub,
                                       const double* rthr) {
  if (p.kind == BX_REAL) {  // thresholds strictly below the coordinate (binary search, L1-resident)
    const double x = row_f64(row, p.word + 2);
    const double* t = rthr + (sub & 0xFFFF);
    int lo = 0, hi = sub >> 16;
    while (lo < hi) {
      const int mid = (lo + hi) >> 1;
      if (__ldg(t + mid) < x) lo = mid + 1;
      else hi = mid;
    }
    return lo;
  }
  if (p.kind == BX_PERMUTATION) {
    const uint64_t x = row_u64(row, p.word);
    if (sub >= 0) return perm_pos(x, p.size, sub);
    int r = 0;  // rank (Lehmer code) of the permutation, elements in position order
    for (int i = 0; i < p.size; ++i) {
      const int ai = (int)((x >> (4 * (p.size - 1 - i))) & 15u);
      int c = 0;
      for (int j = i + 1; j < p.size; ++j) c += (int)((x >> (4 * (p.size - 1 - j))) & 15u) < ai ? 1 : 0;
      r = r * (p.size - i) + c;
    }
    return r;
  }
  // sub < 0: one code for the whole categorical parameter (its label index; the per-label masks
  // are the ANDs of the one-hot features' masks), else the one-hot feature [label == sub]
  if (p.kind == BX_CATEGORICAL) return sub < 0 ? (int)row[p.word] : ((int)row[p.word] == sub ? 1 : 0);
  return (int)row[p.word];
}

// a direct slot's code: single, or a pair code_a * mul + code_b (QsForestDev.code_param2)
__device__ __forceinline__ int qs_slot_code(const bx_param_desc* params, const uint32_t* row, int p1, int s1, int p2,
                                            int s2, int mul, const double* rthr) {
  int c = qs_code(params[p1], row, s1, rthr);
  if (p2 >= 0) c = c * mul + qs_code(params[p2], row, s2, rthr);
  return c;
}

__device__ __forceinline__ int32_t lds_s32(uint32_t a) {
  int32_t v;
  asm volatile("ld.shared.s32 %0, [%1];" : "=r"(v) : "r"(a));
  return v;
}
__device__ __forceinline__ uint64_t lds_u64(uint32_t a) {
  uint64_t v;
  asm volatile("ld.shared.u64 %0, [%1];" : "=l"(v) : "r"(a));
  return v;
}
__device__ __forceinline__ uint32_t lds_u16(uint32_t a) {
  uint16_t v;
  asm volatile("ld.shared.u16 %0, [%1];" : "=h"(v) : "r"(a));
  return v;
}
__device__ __forceinline__ void sts_s32(uint32_t a, int32_t v) {
  asm volatile("st.shared.s32 [%0], %1;" ::"r"(a), "r"(v) : "memory");
}

// Shared-memory image of the QuickScorer tables: masks [stride][tpad] u64, distinct leaf values,
// leaf value ids [n_trees][64] u16, indirect-slot indices [rows][itpad] u16 and masks, then (when
// `offs`) the per-thread mask-row offsets [n_codes][kQsThreads]
struct QsSmem {
  size_t mask, uval, vid, iidx, imask, offs, end;
};
__host__ __device__ inline QsSmem qs_smem_layout(const QsForestDev& f, bool offs) {
  QsSmem L;
  size_t o = 0;
  // every region starts on 16 bytes and is copied in whole 16-byte units (qs_load_tables)
  L.mask = o;
  o += ((size_t)f.stride * f.tpad * 8 + 15) & ~(size_t)15;
  L.uval = o;
  o += ((size_t)f.n_uvals * 8 + 15) & ~(size_t)15;
  L.vid = o;
  o += ((size_t)f.n_trees * 64 * 2 + 15) & ~(size_t)15;
  L.iidx = o;
  o += f.n_ind ? (((size_t)f.n_iidx_rows * f.itpad * 2 + 15) & ~(size_t)15) : 0;
  L.imask = o;
  o += f.n_ind ? (((size_t)f.n_imask * 8 + 15) & ~(size_t)15) : 0;
  L.offs = o;
  o += offs ? (size_t)f.n_codes * kQsThreads * 4 : 0;
  L.end = (o + 15) & ~(size_t)15;
  return L;
}

// The tables go to shared memory as bulk asynchronous copies (cp.async.bulk, one elected thread,
// completion counted on an mbarrier): ~165 KB arrive in ~2 us where the element-wise loop took ~30
// us per CTA (a round of L2 latency per 8 KB).  Every region is a whole number of 16-byte units;
// the device arrays are allocated 16 bytes past their ends (upload()), so the rounded copies stay
// inside them.  Ends with a __syncthreads (the barrier also orders the callers' own shared stores).
__device__ void qs_load_tables(const QsForestDev& f, unsigned char* smem, const QsSmem& L) {
  __shared__ __align__(8) uint64_t bar;
  const uint32_t b = (uint32_t)__cvta_generic_to_shared(&bar);
  if (threadIdx.x == 0) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(b));
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  __syncthreads();
  const uint32_t sizes[5] = {(uint32_t)(L.uval - L.mask), (uint32_t)(L.vid - L.uval), (uint32_t)(L.iidx - L.vid),
                             (uint32_t)(L.imask - L.iidx), (uint32_t)(L.offs - L.imask)};
  if (threadIdx.x == 0) {
    const void* src[5] = {f.mask, f.uval, f.vid, f.iidx, f.imask};
    const size_t dst[5] = {L.mask, L.uval, L.vid, L.iidx, L.imask};
    uint32_t total = 0;
    for (int r = 0; r < 5; ++r) total += sizes[r];
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(b), "r"(total) : "memory");
    for (int r = 0; r < 5; ++r)
      if (sizes[r])
        asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];"
                     ::"r"((uint32_t)__cvta_generic_to_shared(smem + dst[r])), "l"(src[r]), "r"(sizes[r]), "r"(b)
                     : "memory");
  }
  uint32_t done = 0;
  while (!done)
    asm volatile("{\n\t.reg .pred p;\n\tmbarrier.try_wait.parity.shared::cta.b64 p, [%1], 0;\n\t"
                 "selp.u32 %0, 1, 0, p;\n\t}\n"
                 : "=r"(done) : "r"(b) : "memory");
  __syncthreads();
}

// indirect slots of one candidate: the shared address of its index row (tree 0)
__device__ __forceinline__ void qs_ind_rows(const QsForestDev& f, const bx_param_desc* params, const uint32_t* row,
                                            uint32_t iidx_s, uint32_t (&irow)[4]) {
  for (int i = 0; i < 4; ++i)
    irow[i] = i < f.n_ind
                  ? iidx_s + 2u * (uint32_t)((f.ind_off[i] + qs_code(params[f.ind_param[i]], row, f.ind_sub[i], f.rthr)) * f.itpad)
                  : 0u;
}

// the indirect slots' masks of trees g0 .. g0 + 7 ANDed into m
__device__ __forceinline__ void qs_ind_and(const QsForestDev& f, const uint32_t (&irow)[4], uint32_t imask_s, int g0,
                                           uint64_t (&m)[kQsGroup]) {
  for (int i = 0; i < f.n_ind; ++i) {
    const uint32_t ir = irow[i] + 2u * (uint32_t)g0;
    const uint64_t w0 = lds_u64(ir), w1 = lds_u64(ir + 8u);
#pragma unroll
    for (int j = 0; j < 4; ++j) {
      m[j] &= lds_u64(imask_s + 8u * (uint32_t)((w0 >> (16 * j)) & 0xFFFFu));
      m[4 + j] &= lds_u64(imask_s + 8u * (uint32_t)((w1 >> (16 * j)) & 0xFFFFu));
    }
  }
}

// Stand-alone probabilities (predict_proba_batch) in either numpy summation order.
__global__ void __launch_bounds__(kQsThreads) rf_qs_kernel(SpaceDev sp, QsForestDev f, const uint32_t* rows,
                                                           int64_t q, int use_pairwise, double* probs,
                                                           const uint8_t* pw_rows) {
  extern __shared__ __align__(16) unsigned char smem[];
  __shared__ bx_param_desc params[BX_MAX_PARAMS];
  const QsSmem L = qs_smem_layout(f, true);
  for (int i = threadIdx.x; i < sp.n_params * (int)sizeof(bx_param_desc) / 4; i += blockDim.x)
    reinterpret_cast<int32_t*>(params)[i] = reinterpret_cast<const int32_t*>(sp.params)[i];
  qs_load_tables(f, smem, L);
  __syncthreads();
  const uint32_t mask_s = (uint32_t)__cvta_generic_to_shared(smem + L.mask);
  const uint32_t uval_s = (uint32_t)__cvta_generic_to_shared(smem + L.uval);
  const uint32_t vid_s = (uint32_t)__cvta_generic_to_shared(smem + L.vid);
  const uint32_t iidx_s = (uint32_t)__cvta_generic_to_shared(smem + L.iidx);
  const uint32_t imask_s = (uint32_t)__cvta_generic_to_shared(smem + L.imask);
  const uint32_t off_s = (uint32_t)__cvta_generic_to_shared(smem + L.offs) + 4u * threadIdx.x;
  auto leaf = [=](int t, uint64_t m) {
    const uint32_t id = lds_u16(vid_s + 2u * (uint32_t)(t * 64 + __ffsll((long long)m) - 1));
    return __longlong_as_double((long long)lds_u64(uval_s + 8u * id));
  };
  const int64_t stride = (int64_t)gridDim.x * blockDim.x;
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < q; i += stride) {
    const uint32_t* row = rows + (size_t)i * sp.row_words;
    for (int c = 0; c < f.n_codes; ++c)
      sts_s32(off_s + 4u * kQsThreads * c,
              (f.soff[c] + qs_slot_code(params, row, f.code_param[c], f.code_sub[c], f.code_param2[c], f.code_sub2[c],
                                        f.code_mul[c], f.rthr)) * f.tpad);
    uint32_t irow[4];
    qs_ind_rows(f, params, row, iidx_s, irow);
    double sum = 0.0;
    if (pw_rows ? pw_rows[i] != 0 : use_pairwise != 0) {
      sum = pairwise(
          [=](int t) {
            uint64_t m = ~0ull;
            for (int c = 0; c < f.n_codes; ++c)
              m &= lds_u64(mask_s + 8u * (uint32_t)(lds_s32(off_s + 4u * kQsThreads * c) + t));
            for (int k = 0; k < f.n_ind; ++k)
              m &= lds_u64(imask_s + 8u * lds_u16(irow[k] + 2u * (uint32_t)t));
            return leaf(t, m);
          },
          0, f.n_trees);
    } else {
      for (int g0 = 0; g0 < f.n_trees; g0 += kQsGroup) {
        uint64_t m[kQsGroup];
#pragma unroll
        for (int j = 0; j < kQsGroup; ++j) m[j] = ~0ull;
        for (int c = 0; c < f.n_codes; ++c) {
          const uint32_t col = mask_s + (uint32_t)(lds_s32(off_s + 4u * kQsThreads * c) + g0) * 8u;
#pragma unroll
          for (int j = 0; j < kQsGroup / 2; ++j) {
            const ulonglong2 w = lds_u64x2(col + 16u * j);
            m[2 * j] &= w.x;
            m[2 * j + 1] &= w.y;
          }
        }
        qs_ind_and(f, irow, imask_s, g0, m);
#pragma unroll
        for (int j = 0; j < kQsGroup; ++j)
          if (g0 + j < f.n_trees) {
            const double v = leaf(g0 + j, m[j]);
            sum = (g0 + j == 0) ? v : __dadd_rn(sum, v);  // tree order (feasibility.py:89)
          }
      }
    }
    probs[i] = __ddiv_rn(sum, (double)f.n_trees);
  }
}

// QuickScorer forest fused with the acquisition summary (the work of summary_kernel): runs after the
// posterior kernel, reads its mean / variance, applies value = -inf if p < eps_f else EI * p
// (acquisition.py:77-79; the EI only for the candidates that pass) and keeps per-warp partials
// (stable top-k, trackers) merged into one per block.  NC > 0: exactly NC direct code slots, the
// candidate's mask-row addresses held in registers and two slots' loads issued back to back;
// NC == 0: any slot count (offsets through shared memory).
template <int NC>
__global__ void __launch_bounds__(kQsThreads) rf_qs_summary_kernel(SpaceDev sp, QsForestDev f, SummaryArgs a) {
  extern __shared__ __align__(16) unsigned char smem[];
  __shared__ bx_param_desc params[BX_MAX_PARAMS];
  const QsSmem L = qs_smem_layout(f, NC == 0);
  Partial* parts = reinterpret_cast<Partial*>(smem + L.end);  // [warps]
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  for (int i = tid; i < sp.n_params * (int)sizeof(bx_param_desc) / 4; i += blockDim.x)
    reinterpret_cast<int32_t*>(params)[i] = reinterpret_cast<const int32_t*>(sp.params)[i];
  qs_load_tables(f, smem, L);
  Partial* summ = &parts[warp];
  if (lane == 0) partial_init(summ);
  // per-slot constants in shared memory (broadcast loads instead of a global load per candidate)
  __shared__ int32_t s_soff[64], s_cpar[64], s_csub[64], s_cpar2[64], s_csub2[64], s_cmul[64];
  for (int c = tid; c < f.n_codes && c < 64; c += blockDim.x) {
    s_soff[c] = f.soff[c];
    s_cpar[c] = f.code_param[c];
    s_csub[c] = f.code_sub[c];
    s_cpar2[c] = f.code_param2[c];
    s_csub2[c] = f.code_sub2[c];
    s_cmul[c] = f.code_mul[c];
  }
  __syncthreads();
  const uint32_t mask_s = (uint32_t)__cvta_generic_to_shared(smem + L.mask);
  const uint32_t uval_s = (uint32_t)__cvta_generic_to_shared(smem + L.uval);
  const uint32_t vid_s = (uint32_t)__cvta_generic_to_shared(smem + L.vid);
  const uint32_t iidx_s = (uint32_t)__cvta_generic_to_shared(smem + L.iidx);
  const uint32_t imask_s = (uint32_t)__cvta_generic_to_shared(smem + L.imask);
  const uint32_t off_s = (uint32_t)__cvta_generic_to_shared(smem + L.offs) + 4u * tid;
  const int words = sp.row_words;
  const int64_t stride = (int64_t)gridDim.x * blockDim.x;
  for (int64_t base = (int64_t)blockIdx.x * blockDim.x + warp * 32; base < a.q; base += stride) {
    const int64_t i = base + lane;
    const bool valid = i < a.q;
    double value = -INFINITY, prob = -INFINITY;
    if (valid) {
      const uint32_t* row = a.rows + (size_t)i * words;
      uint32_t colr[NC > 0 ? NC : 1];
      if constexpr (NC > 0) {
#pragma unroll
        for (int c = 0; c < NC; ++c)
          colr[c] = mask_s + 8u * (uint32_t)((s_soff[c] + qs_slot_code(params, row, s_cpar[c], s_csub[c], s_cpar2[c],
                                                                        s_csub2[c], s_cmul[c], f.rthr)) * f.tpad);
      } else {
        for (int c = 0; c < f.n_codes; ++c)
          sts_s32(off_s + 4u * kQsThreads * c,
                  (f.soff[c] + qs_slot_code(params, row, f.code_param[c], f.code_sub[c], f.code_param2[c], f.code_sub2[c],
                                            f.code_mul[c], f.rthr)) * f.tpad);
      }
      uint32_t irow[4];
      qs_ind_rows(f, params, row, iidx_s, irow);
      double sum = 0.0;
      for (int g0 = 0; g0 < f.n_trees; g0 += kQsGroup) {
        uint64_t m[kQsGroup];
#pragma unroll
        for (int j = 0; j < kQsGroup; ++j) m[j] = ~0ull;
        if constexpr (NC > 0) {
#pragma unroll
          for (int c = 0; c < NC; c += 2) {
            ulonglong2 w0[kQsGroup / 2], w1[kQsGroup / 2];
#pragma unroll
            for (int j = 0; j < kQsGroup / 2; ++j) w0[j] = lds_u64x2(colr[c] + 8u * g0 + 16u * j);
            if (c + 1 < NC) {
#pragma unroll
              for (int j = 0; j < kQsGroup / 2; ++j) w1[j] = lds_u64x2(colr[c + 1] + 8u * g0 + 16u * j);
            }
#pragma unroll
            for (int j = 0; j < kQsGroup / 2; ++j) {
              m[2 * j] &= w0[j].x;
              m[2 * j + 1] &= w0[j].y;
              if (c + 1 < NC) {
                m[2 * j] &= w1[j].x;
                m[2 * j + 1] &= w1[j].y;
              }
            }
          }
        } else {
          for (int c = 0; c < f.n_codes; ++c) {
            const uint32_t col = mask_s + (uint32_t)(lds_s32(off_s + 4u * kQsThreads * c) + g0) * 8u;
#pragma unroll
            for (int j = 0; j < kQsGroup / 2; ++j) {
              const ulonglong2 w = lds_u64x2(col + 16u * j);
              m[2 * j] &= w.x;
              m[2 * j + 1] &= w.y;
            }
          }
        }
        qs_ind_and(f, irow, imask_s, g0, m);
#pragma unroll
        for (int j = 0; j < kQsGroup; ++j)
          if (g0 + j < f.n_trees) {
            const uint32_t id = lds_u16(vid_s + 2u * (uint32_t)((g0 + j) * 64 + __ffsll((long long)m[j]) - 1));
            const double v = __longlong_as_double((long long)lds_u64(uval_s + 8u * id));
            sum = (g0 + j == 0) ? v : __dadd_rn(sum, v);  // tree order (feasibility.py:89)
          }
      }
      prob = __ddiv_rn(sum, (double)f.n_trees);
      value = (prob < a.eps_f) ? -INFINITY : (a.mean ? ei_value(a.mean[i], a.var[i], a.f_model) : a.ei[i]) * prob;
      if (a.values_out) a.values_out[i] = value;
      if (a.probs_out) a.probs_out[i] = prob;
    }
    const bool fin = valid && value != -INFINITY;
    const bool top_open = a.k > 0 && summ->n_top < a.k;
    const double kth = (a.k > 0 && !top_open) ? summ->top[a.k - 1].value : -INFINITY;
    const bool prob_ok = a.track_prob && prob >= summ->best_prob.prob;
    const bool maybe = valid && ((fin && a.k > 0 && (top_open || value >= kth)) ||
                                 (fin && value >= summ->best.value) || prob_ok);
    bool evaluated = false;
    if (maybe && a.evald.count > 0) evaluated = is_evaluated(a.evald, a.rows + (size_t)i * words, words);
    const bool pass = maybe && ((fin && a.k > 0 && (top_open || value >= kth)) ||
                                (!evaluated && ((fin && value >= summ->best.value) || prob_ok)));
    const unsigned vmask = __ballot_sync(0xffffffffu, valid);
    const unsigned fmask = __ballot_sync(0xffffffffu, fin);
    unsigned pmask = __ballot_sync(0xffffffffu, pass);
    const unsigned emask = __ballot_sync(0xffffffffu, evaluated);
    if (lane == 0) {
      summ->n_scored += __popc(vmask);
      summ->n_finite += __popc(fmask);
    }
    while (pmask) {
      const int c = __ffs(pmask) - 1;
      pmask &= pmask - 1;
      const double vc = __shfl_sync(0xffffffffu, value, c);
      const double pc = __shfl_sync(0xffffffffu, prob, c);
      if (lane == 0)
        partial_add(summ, a.k, params, sp.n_params, sp.rank_lut, words, vc, pc, a.index_base + base + c,
                    (emask >> c) & 1u, a.rows + (size_t)(base + c) * words, a.track_prob != 0);
      __syncwarp();
    }
  }
  __syncthreads();  // fold the block's warp partials into one
  if (tid == 0)
    for (int w = 1; w < kQsThreads / 32; ++w)
      partial_merge(&parts[0], &parts[w], a.k, params, sp.n_params, sp.rank_lut, words);
  __syncthreads();
  const int32_t* src = reinterpret_cast<const int32_t*>(&parts[0]);
  int32_t* dst = reinterpret_cast<int32_t*>(a.partials + blockIdx.x);
  for (int i = tid; i < (int)(sizeof(Partial) / 4); i += kQsThreads) dst[i] = src[i];
}

size_t qs_smem(const QsForestDev& f) { return qs_smem_layout(f, true).end; }

size_t coded_smem(const CodedForestDev& cf, bool in_smem) {
  return (in_smem ? ((size_t)cf.n_nodes + cf.n_leaves) * 8 + (((size_t)cf.n_nodes * 4 + 15) & ~(size_t)15) : 0) +
         (((size_t)cf.n_trees * 4 + 15) & ~(size_t)15) + (size_t)cf.n_codes * kRfThreads * 4 +
         (cf.has_real ? (size_t)cf.n_codes * kRfThreads * 8 : 0);
}

template <bool SMEM>
auto pick_real(bool real) {
  return real ? rf_coded_kernel<SMEM, true> : rf_coded_kernel<SMEM, false>;
}

// code counts up to kQsMaxNC keep each thread's table offsets in registers (no offset array)
constexpr int kQsMaxNC = 24;

size_t qs_summary_smem(const QsForestDev& f) {
  return qs_smem_layout(f, f.n_codes > kQsMaxNC).end + (size_t)(kQsThreads / 32) * sizeof(Partial);
}

}  // namespace

size_t qs_summary_smem_bytes(const QsForestDev& q) { return qs_summary_smem(q); }

bool qs_summary_available(const ForestDev& f) {
  return f.coded && f.has_trees && f.qs.enabled && qs_summary_smem(f.qs) <= 227 * 1024;
}

// Forest + summary in one kernel (after the posterior kernel wrote a.ei); a.partials receives one
// partial per block (<= SM count).
cudaError_t launch_rf_summary(const SpaceDev& space, const ForestDev& f, const SummaryArgs& a, int sm_count,
                              cudaStream_t s, int* n_partials) {
  const size_t bytes = qs_summary_smem(f.qs);
  auto kern = rf_qs_summary_kernel<0>;
  switch (f.qs.n_codes) {
#define BX_NC(c) \
    case c: kern = rf_qs_summary_kernel<c>; break;
    BX_NC(1) BX_NC(2) BX_NC(3) BX_NC(4) BX_NC(5) BX_NC(6) BX_NC(7) BX_NC(8)
    BX_NC(9) BX_NC(10) BX_NC(11) BX_NC(12) BX_NC(13) BX_NC(14) BX_NC(15) BX_NC(16)
    BX_NC(17) BX_NC(18) BX_NC(19) BX_NC(20) BX_NC(21) BX_NC(22) BX_NC(23) BX_NC(24)
#undef BX_NC
    default: break;
  }
  static_assert(kQsMaxNC == 24, "instantiate rf_qs_summary_kernel<1..kQsMaxNC>");
  cudaError_t e = set_smem(kern, (int)bytes);
  if (e != cudaSuccess) return e;
  int64_t blocks = (a.q + kQsThreads - 1) / kQsThreads;
  if (blocks > sm_count) blocks = sm_count;
  if (blocks < 1) blocks = 1;
  *n_partials = (int)blocks;
  kern<<<(int)blocks, kQsThreads, bytes, s>>>(space, f.qs, a);
  return cudaGetLastError();
}

cudaError_t launch_rf(const SpaceDev& space, const ForestDev& f, const uint32_t* rows, int64_t q,
                      int use_pairwise, double* probs, cudaStream_t s, const uint8_t* pw_rows) {
  if (q <= 0) return cudaSuccess;
  int dev = 0, sms = 148;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  if (f.coded && f.qs.enabled && qs_smem(f.qs) <= 220 * 1024) {
    const size_t bytes = qs_smem(f.qs);
    cudaError_t e = set_smem(rf_qs_kernel, (int)bytes);
    if (e != cudaSuccess) return e;
    int per_sm = 1;
    e = cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, rf_qs_kernel, kQsThreads, bytes);
    if (e != cudaSuccess) return e;
    int64_t blocks = (q + kQsThreads - 1) / kQsThreads;
    const int64_t cap = (int64_t)sms * (per_sm > 0 ? per_sm : 1);
    if (blocks > cap) blocks = cap;
    rf_qs_kernel<<<(int)blocks, kQsThreads, bytes, s>>>(space, f.qs, rows, q, use_pairwise, probs, pw_rows);
    return cudaGetLastError();
  }
  if (f.coded) {
    const bool in_smem = coded_smem(f.cf, true) <= 220 * 1024;
    const size_t bytes = coded_smem(f.cf, in_smem);
    auto kern = in_smem ? pick_real<true>(f.cf.has_real) : pick_real<false>(f.cf.has_real);
    cudaError_t e = set_smem(kern, (int)bytes);
    if (e != cudaSuccess) return e;
    int64_t blocks = (q + kRfThreads - 1) / kRfThreads;
    if (blocks > sms) blocks = sms;
    kern<<<(int)blocks, kRfThreads, bytes, s>>>(space, f.cf, rows, q, use_pairwise, probs, pw_rows);
    return cudaGetLastError();
  }
  int64_t blocks = (q + 255) / 256;
  if (blocks > (int64_t)sms * 16) blocks = (int64_t)sms * 16;
  rf_kernel<<<(int)blocks, 256, 0, s>>>(space, f, rows, q, use_pairwise, probs, pw_rows);
  return cudaGetLastError();
}

}  // namespace bx
