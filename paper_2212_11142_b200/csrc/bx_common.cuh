// bx_common.cuh — internal types and device helpers shared by the sm_100a kernels.
//
// Encoded rows, parameter descriptors and the handle's device-resident model state.  Every
// helper cites the reference expression (file:line under /root/reference/pkg/src/boxtune) whose
// value it reproduces.
#pragma once

#include <cstdint>
#include <cstring>
#include <cuda_runtime.h>

#include "../../include/bx_sm100.h"

namespace bx {

// cudaFuncSetAttribute(MaxDynamicSharedMemorySize) once per kernel and size (host side): the call
// costs microseconds, and the chunked scoring paths launch the same kernels many times
cudaError_t set_smem_once(const void* fn, int bytes);
template <typename K>
inline cudaError_t set_smem(K* fn, int bytes) {
  return set_smem_once(reinterpret_cast<const void*>(fn), bytes);
}

constexpr int kRealGrid = 64;          // space.py:23 REAL_NEIGHBOR_GRID
constexpr double kSqrt5 = 2.23606797749978969640917366873128;  // surrogate.py:35 math.sqrt(5.0)
constexpr double kInvSqrt2Pi = 0.398942280401432702863218082712;  // acquisition.py:27

// expected_improvement_vec (acquisition.py:40-51) for one candidate; the one definition every
// kernel uses, so the value does not depend on which kernel evaluates it
__device__ __forceinline__ double ei_value(double mean, double var, double f_model) {
  const double sd = sqrt(fmax(var, 0.0));
  const double delta = f_model - mean;
  double ei = fmax(delta, 0.0);
  if (sd > 0.0) {
    const double z = delta / sd;
    ei = delta * normcdf(z) + sd * (kInvSqrt2Pi * exp(-0.5 * z * z));
  }
  return fmax(ei, 0.0);
}

// ---- device-resident state owned by a handle -------------------------------------------------

struct SpaceDev {
  const bx_param_desc* params;  // [n_params]
  const double* coord_lut;      // coordinates per domain index / real grid point
  const int32_t* rank_lut;      // categorical label rank (Python sort order)
  const int32_t* feat_param;    // [n_features] parameter of each feature column
  const int32_t* feat_sub;      // [n_features] sub-column (one-hot label / permutation element)
  const int32_t* slot_param;    // [n_slots] neighbour slot -> parameter
  const int32_t* slot_move;     // [n_slots] neighbour slot -> move id inside the parameter
  int32_t n_params;
  int32_t row_words;
  int32_t n_features;
  int32_t n_slots;
};

// Per-parameter training plane for the cross-covariance.  For numeric kinds plane[j] holds the
// training coordinate divided by the lengthscale (double); categorical: domain index (as int64
// in the same 8 bytes); permutation: packed u64.  Kendall additionally keeps the pair-order
// masks (two u64 words for m <= 16).
struct GpDev {
  int32_t n;             // training points
  int32_t ncols_pad;     // n rounded up to 4 (DMMA k-step)
  int32_t rows_pad;      // (n + 1) rounded up to 16 (augmented rows: L^-1 then alpha)
  int32_t lda;           // row stride of A (doubles)
  const double* A;       // [rows_pad x lda]: rows 0..n-1 = L^-1 (lower), row n = alpha
  const uint64_t* planes;   // [n_params x n] 8-byte training planes
  const uint64_t* kmask;    // [n_params x n x 2] Kendall pair masks (only for Kendall params)
  const double* inv_l;      // [n_params] 1 / lengthscale
  const double* inv_l2;     // [n_params] 1 / lengthscale^2 (surrogate.py:222)
  const double* disc_tab;   // discrete contribution tables: (raw / mx) / l^2 per raw value
  const int32_t* disc_off;  // [n_params] offset of the parameter's table in disc_tab
  double outputscale;
  double y_mean, y_std;
};

// Forest nodes repacked breadth-first so that the two children of a node are adjacent.
struct RfNode {
  double thr;     // split threshold (internal) -- feasibility.py:86 `x <= threshold`
  double val;     // feasible fraction stored at every node (feasibility.py:105)
  int32_t feat;   // feature column, -1 for a leaf
  int32_t child;  // index of the left child; right child = child + 1
};

// Integer-coded forest (the fast path).  Every encode_configs column gets a per-candidate integer
// code (domain index of a finite numeric parameter, 0/1 for a one-hot label column, element
// position for a permutation column) and every split `x <= threshold` on it becomes the exact
// test `code < cut` with cut = #{code values whose feature value <= threshold} (coordinates are
// monotone in the domain index).  Real columns keep the f64 comparison against a side table.
// One 64-bit word per node:
//   [23:0] argument (cut / real-threshold index / leaf-value index)   [29:24] code slot
//   [31:30] type (0 integer cut, 1 real, 2 leaf)   [63:32] left child (right = left + 1; a leaf
//   points at itself, so a finished walk stays put)
struct CodedForestDev {
  const uint64_t* nodes;     // [n_nodes]
  const uint32_t* leaf_idx;  // [n_nodes] leaf-value index of leaf nodes
  const double* leaf_val;    // [n_leaves]
  const double* real_thr;    // thresholds of real splits
  const int32_t* roots;      // [n_trees]
  const int32_t* code_param; // [n_codes] parameter of each code slot
  const int32_t* code_sub;   // [n_codes] label / permutation element (or 0)
  int32_t n_nodes;
  int32_t n_leaves;
  int32_t n_codes;
  int32_t n_trees;
  int32_t max_depth;
  int32_t has_real;
  int32_t nodes_in_smem;     // node table + leaf values copied to shared memory
};

// QuickScorer-style tables (Lucchese et al., SIGIR 2015) over the integer codes: leaves of every
// tree are numbered left to right; a node whose test goes right (code >= cut) rules out its left
// subtree's leaves, and the exit leaf is the leftmost leaf no such node rules out.  mask[t][s][v]
// is the AND of those eliminations over tree t's nodes on code slot s for code value v, so a tree
// is n_codes table loads and ANDs plus a find-first-set — no dependent descent.  Needs at most 64
// leaves per tree and integer-coded splits only.
struct QsForestDev {
  const uint64_t* mask;      // [stride][tpad] (slot s, code v at row soff[s] + v; trees contiguous)
  const uint16_t* vid;       // [n_trees][64] leaf value id of leaf l (left-to-right order)
  const double* uval;        // [n_uvals] distinct leaf values
  const int32_t* soff;       // [n_codes] offset of slot s inside a tree's stride
  const int32_t* code_param; // [n_codes] (the coded forest's slots)
  const int32_t* code_sub;
  // a paired slot: code = code(code_param, code_sub) * code_mul + code(code_param2, code_sub2);
  // code_param2 < 0 for a single slot (code_mul 1)
  const int32_t* code_param2;
  const int32_t* code_sub2;
  const int32_t* code_mul;
  int32_t n_trees, n_codes, stride, n_uvals;
  int32_t tpad;              // row length: n_trees rounded up to 8, plus 1 (odd: bank spread)
  int32_t enabled;
  // real features: sorted distinct split thresholds per real parameter; a real code's code_sub is
  // offset | count << 16 into rthr and its value is the number of thresholds below the coordinate
  const double* rthr;
  int32_t has_real;
  // indirect slots: per tree only the few distinct masks are stored (imask) and a [code][tree] table
  // of u16 indices into imask replaces the [code][tree] u64 mask rows (4x smaller).  Real parameters
  // with many distinct thresholds across the forest (code as a real code, ind_sub = its threshold
  // run), and permutations of <= 5 elements as one slot coded by the permutation's rank (ind_sub =
  // -1; m! codes, each the AND of the element-position masks: one table walk instead of m)
  int32_t n_ind;
  int32_t ind_param[4], ind_sub[4], ind_off[4];  // ind_off: first row of the slot in iidx
  const uint16_t* iidx;      // [rows][itpad] index into imask
  const uint64_t* imask;     // [n_imask]
  int32_t itpad, n_iidx_rows, n_imask;
};

struct ForestDev {
  const RfNode* nodes;
  const int32_t* roots;
  int32_t n_trees;
  int32_t max_depth;
  int32_t has_trees;     // 0 -> constant model
  int32_t coded;         // 1 -> use `cf` (integer-coded fast path)
  double constant;       // single-class shortcut (feasibility.py:73-74)
  CodedForestDev cf;
  QsForestDev qs;
};

struct EvalSetDev {
  const uint32_t* rows;       // [count x row_words]
  const int32_t* table;       // open-addressing hash table of row ids, -1 = empty
  int32_t count;
  int32_t table_mask;         // size - 1 (power of two)
};

struct CotDev {
  int32_t n_groups;
  const int32_t* group_kind;        // 0 tree, 1 real singleton, 2 permutation singleton
  const int32_t* group_param_begin;
  const int32_t* group_params;
  const int32_t* group_root;
  const int32_t* child_begin;   // first child node id
  const int32_t* child_count;
  const int32_t* node_value;    // domain index of the node's value
};

struct ConstraintDev {
  int32_t n_constraints;
  const int32_t* prog_begin;
  const int32_t* code;
  const double* consts;
  const int32_t* vtag;      // per (param, domain index): 0 int, 1 float (ordinal value types)
  const int64_t* vint;      // per (param, domain index) integer value
  const double* vflt;       // per (param, domain index) float value
  const int32_t* voff;      // [n_params] offset into the value tables
  const int32_t* str_id;    // per (param, domain index) string id of categorical labels
  int32_t* fault;           // set to 1 when a value leaves the exactly-representable envelope
};

// ---- row accessors ---------------------------------------------------------------------------

__device__ __forceinline__ uint32_t row_word(const uint32_t* row, int w) { return row[w]; }

__device__ __forceinline__ double row_f64(const uint32_t* row, int w) {
  uint64_t bits = (uint64_t)row[w] | ((uint64_t)row[w + 1] << 32);
  return __longlong_as_double((long long)bits);
}

__device__ __forceinline__ uint64_t row_u64(const uint32_t* row, int w) {
  return (uint64_t)row[w] | ((uint64_t)row[w + 1] << 32);
}

__device__ __forceinline__ void put_u64(uint32_t* row, int w, uint64_t v) {
  row[w] = (uint32_t)v;
  row[w + 1] = (uint32_t)(v >> 32);
}

__device__ __forceinline__ void put_f64(uint32_t* row, int w, double v) {
  put_u64(row, w, (uint64_t)__double_as_longlong(v));
}

// element (minus one) at position i of a packed permutation of size m
__device__ __forceinline__ int perm_at(uint64_t p, int m, int i) {
  return (int)((p >> (4 * (m - 1 - i))) & 0xFull);
}

// position of element e (0-based, i.e. value e+1) -- feasibility.py:48 argsort of the values
__device__ __forceinline__ int perm_pos(uint64_t p, int m, int e) {
  uint64_t mask = (m >= 16) ? ~0ull : ((1ull << (4 * m)) - 1ull);
  uint64_t y = (p ^ (0x1111111111111111ull * (uint64_t)e)) & mask;
  uint64_t z = ~(y | (y >> 1) | (y >> 2) | (y >> 3)) & 0x1111111111111111ull & mask;
  int bit = __ffsll((long long)z) - 1;
  return m - 1 - (bit >> 2);
}

// Kendall pair-order masks: bit (i,j), i<j, set iff a_i < a_j (surrogate.py:213)
__device__ __forceinline__ void kendall_mask(uint64_t p, int m, uint64_t& lo, uint64_t& hi) {
  lo = 0; hi = 0;
  int b = 0;
  for (int i = 0; i < m; ++i) {
    int ai = perm_at(p, m, i);
    for (int j = i + 1; j < m; ++j, ++b) {
      if (ai < perm_at(p, m, j)) {
        if (b < 64) lo |= 1ull << b; else hi |= 1ull << (b - 64);
      }
    }
  }
}

// raw (un-normalised) permutation semimetric between two packed permutations.
// surrogate.py:201-218 (_perm_sq_distances) / 54-72 (scalar definitions)
__device__ __forceinline__ int perm_raw(int metric, int m, uint64_t a, uint64_t b, uint64_t alo,
                                        uint64_t ahi, uint64_t blo, uint64_t bhi) {
  if (metric == BX_KENDALL) return __popcll(alo ^ blo) + __popcll(ahi ^ bhi);
  if (metric == BX_NAIVE) return a != b ? 1 : 0;
  if (metric == BX_HAMMING) {
    uint64_t x = a ^ b;
    uint64_t t = (x | (x >> 1) | (x >> 2) | (x >> 3)) & 0x1111111111111111ull;
    return __popcll(t);
  }
  int s = 0;  // spearman: sum of squared element differences
  for (int i = 0; i < m; ++i) {
    int d = perm_at(a, m, i) - perm_at(b, m, i);
    s += d * d;
  }
  return s;
}

// numeric coordinate of parameter p in a row (surrogate.py:163-170 via host LUT)
__device__ __forceinline__ double row_coord(const bx_param_desc& p, const double* coord_lut,
                                            const uint32_t* row) {
  if (p.kind == BX_REAL) return row_f64(row, p.word + 2);
  return coord_lut[p.coord + (int)row[p.word]];
}

// Python tuple order of two encoded configurations (acquisition.py:91, :109-110):
// returns -1, 0, 1.
__device__ __forceinline__ int key_cmp(const bx_param_desc* params, int n_params,
                                       const int32_t* rank_lut, const uint32_t* a,
                                       const uint32_t* b) {
  for (int k = 0; k < n_params; ++k) {
    const bx_param_desc& p = params[k];
    if (p.kind == BX_REAL) {
      double x = row_f64(a, p.word), y = row_f64(b, p.word);
      if (x < y) return -1;
      if (x > y) return 1;
    } else if (p.kind == BX_PERMUTATION) {
      uint64_t x = row_u64(a, p.word), y = row_u64(b, p.word);
      if (x < y) return -1;
      if (x > y) return 1;
    } else if (p.kind == BX_CATEGORICAL) {
      int x = rank_lut[p.rank + (int)a[p.word]], y = rank_lut[p.rank + (int)b[p.word]];
      if (x < y) return -1;
      if (x > y) return 1;
    } else {
      uint32_t x = a[p.word], y = b[p.word];
      if (x < y) return -1;
      if (x > y) return 1;
    }
  }
  return 0;
}

__device__ __forceinline__ uint64_t row_hash(const uint32_t* row, int words) {
  uint64_t h = 1469598103934665603ull;
  for (int w = 0; w < words; ++w) {
    h ^= row[w];
    h *= 1099511628211ull;
    h ^= h >> 29;
  }
  return h;
}

__device__ __forceinline__ bool is_evaluated(const EvalSetDev& ev, const uint32_t* row, int words) {
  if (ev.count == 0) return false;
  uint64_t h = row_hash(row, words);
  int slot = (int)(h & (uint64_t)ev.table_mask);
  for (int probe = 0; probe <= ev.table_mask; ++probe) {
    int id = ev.table[slot];
    if (id < 0) return false;
    const uint32_t* r = ev.rows + (size_t)id * words;
    bool eq = true;
    for (int w = 0; w < words; ++w) eq &= (r[w] == row[w]);
    if (eq) return true;
    slot = (slot + 1) & ev.table_mask;
  }
  return false;
}

// ---- per-warp partial summaries of a score launch --------------------------------------------

struct TopRec {
  double value;
  double prob;
  int64_t index;
};

// Compact partial summary written by every warp of bx_score's kernel and merged afterwards.
// Top-k entries carry no row (rows are gathered by index at the end); the two tracker bests keep
// their rows because their tie-break compares configurations.
struct Partial {
  int64_t n_scored;
  int64_t n_finite;
  int32_t n_top;
  int32_t pad;
  TopRec top[BX_MAX_K];
  TopRec best;
  TopRec best_prob;
  uint32_t best_row[BX_MAX_ROW_WORDS];
  uint32_t best_prob_row[BX_MAX_ROW_WORDS];
};

// ---- launch helpers implemented in the .cu files -------------------------------------------

struct ScoreArgs {
  SpaceDev space;
  GpDev gp;
  ForestDev forest;
  EvalSetDev evald;
  const uint32_t* rows;
  int64_t q;
  int64_t index_base;
  double f_model;
  double eps_f;
  int32_t k;
  int32_t flags;
  int32_t use_forest;
  const double* probs_in;   // feasibility p from rf kernel (NULL without a forest)
  double* values_out;       // optional
  double* probs_out;        // optional
  double* mean_out;         // optional (bx_gp_predict)
  double* var_out;          // optional
  Partial* partials;        // [gridDim.x * warps] per-warp summaries (NULL -> no summary)
};

// Register-resident GP kernel (gp_fused.cu): writes EI (or mean/var) per candidate.
struct FusedArgs {
  SpaceDev space;
  GpDev gp;
  const double* panels;   // panel-major padded copy of A (launch_build_panels)
  const uint32_t* rows;
  int64_t q;
  double f_model;
  double* ei_out;
  double* mean_out;
  double* var_out;
  int32_t mt;             // m-tiles held in registers (8 * mt >= n + 1)
  int32_t n_kendall;
  int32_t kendall_param[BX_MAX_PARAMS];
  // parameters grouped by kind so the distance loops carry no per-parameter dispatch
  int32_t n_num, n_cat, n_perm;
  int32_t num_param[BX_MAX_PARAMS];
  int32_t cat_param[BX_MAX_PARAMS];
  int32_t perm_param[BX_MAX_PARAMS];
  double exp2tab[64];     // 2^(j/64), correctly rounded (host long double)
  int32_t precise;        // 1 -> libm sqrt/exp in the Matérn (BX_MATERN_PRECISE=1)
};

// Feasibility weight, eps_f filter and per-warp summaries over precomputed EI (score_summary.cu).
struct SummaryArgs {
  SpaceDev space;
  EvalSetDev evald;
  const uint32_t* rows;
  int64_t q;
  int64_t index_base;
  const double* ei;
  // mean != NULL: the posterior wrote mean / var instead of the EI, computed here with ei_value
  const double* mean;
  const double* var;
  double f_model;
  const double* probs_in;  // NULL -> constant / no forest
  int32_t use_forest;
  int32_t has_trees;
  double constant;
  double eps_f;
  int32_t k;
  int32_t track_prob;      // also run the probability tracker (only needed when all values are -inf)
  double* values_out;
  double* probs_out;
  Partial* partials;
};

// Tensor-core posterior (gp_tc.cu): FusedArgs plus the digit-sliced [L^-1; alpha^T].
// One coordinate of the Euclidean embedding of the weighted distance W (surrogate.py:173-223):
// W(x, y) = sum_k sq_k(x, y) / l_k^2 = |e(x) - e(y)|^2 for every metric except the naive
// permutation indicator.  Numeric: coord / l; categorical (1{a != b}): the L labels as the vertices
// of a unit-edge simplex in L - 1 dimensions (Helmert basis); Spearman: the position vector in the
// m - 1 dimensional sum-zero subspace; Kendall: the m(m-1)/2 pair-order indicators; Hamming: per
// position the simplex of the m values.  Each coordinate is scaled by sqrt(weight) and centred on
// the training mean, and its values come from a table, so host (training points) and device
// (candidates) evaluate the identical expression.
enum { BX_EMB_CODE = 0, BX_EMB_REAL = 1, BX_EMB_PERM_LIN = 2, BX_EMB_KENDALL = 3, BX_EMB_PERM_HOT = 4 };
struct EmbDim {
  int32_t kind;
  int32_t word;   // row word of the parameter
  int32_t a, b;   // KENDALL: positions a < b; PERM_HOT: position a
  int32_t m;      // permutation size
  int32_t off;    // first table entry
};

__host__ __device__ __forceinline__ int emb_elem(uint64_t x, int m, int i) {
  return (int)((x >> (4 * (m - 1 - i))) & 15u);  // element at position i (0-based value)
}
// CODE: tab[off + domain index]; REAL: coord * tab[off] + tab[off + 1]; PERM_LIN: tab[off + m] +
// sum_i elem_i * tab[off + i]; KENDALL: tab[off + (elem_a < elem_b)]; PERM_HOT: tab[off + elem_a]
__host__ __device__ __forceinline__ double emb_value(const EmbDim& e, const uint32_t* row, const double* tab) {
  if (e.kind == BX_EMB_CODE) return tab[e.off + (int)row[e.word]];
  if (e.kind == BX_EMB_REAL) {
    const uint64_t bits = (uint64_t)row[e.word + 2] | ((uint64_t)row[e.word + 3] << 32);
    double x;
    memcpy(&x, &bits, 8);
    return fma(x, tab[e.off], tab[e.off + 1]);
  }
  const uint64_t x = (uint64_t)row[e.word] | ((uint64_t)row[e.word + 1] << 32);
  if (e.kind == BX_EMB_KENDALL) return tab[e.off + (emb_elem(x, e.m, e.a) < emb_elem(x, e.m, e.b) ? 1 : 0)];
  if (e.kind == BX_EMB_PERM_HOT) return tab[e.off + emb_elem(x, e.m, e.a)];
  double acc = tab[e.off + e.m];
  for (int i = 0; i < e.m; ++i) acc = fma((double)emb_elem(x, e.m, i), tab[e.off + i], acc);
  return acc;
}

// Packed wire format (bx_pack_rows): parameter k at bit `bit` of the packed row, `bits` wide;
// reals carry the f64 value (64 bits) and, when the coordinate is host-dependent (log transform),
// the f64 coordinate (64 more bits), else the coordinate is (v - lo) / (hi - lo) (surrogate.py:
// 163-170: IEEE subtract and divide, bit-identical to numpy's).
struct PackParam {
  int32_t kind, word, bit, bits, carry_coord, pad;
  double lo, hi;
};
struct PackSpec {
  int32_t n, pw;  // parameters, packed words per row
  PackParam p[BX_MAX_PARAMS];
};
// bits 1..64 starting at bit `bit`: a 64-bit window over the field's first two words (a third
// only when a wide field straddles it); never reads a word the field does not touch
__host__ __device__ __forceinline__ uint64_t pk_get(const uint32_t* pk, int bit, int bits) {
  const int w = bit >> 5, o = bit & 31;
  if (bits <= 32) {
    uint64_t win = pk[w];
    if (o + bits > 32) win |= (uint64_t)pk[w + 1] << 32;
    return (win >> o) & (bits == 32 ? 0xFFFFFFFFull : ((1ull << bits) - 1));
  }
  uint64_t v = ((uint64_t)pk[w] | ((uint64_t)pk[w + 1] << 32)) >> o;
  if (o > 0 && o + bits > 64) v |= (uint64_t)pk[w + 2] << (64 - o);
  return bits == 64 ? v : (v & ((1ull << bits) - 1));
}
__host__ __device__ __forceinline__ void pk_put(uint32_t* pk, int bit, int bits, uint64_t v) {
  for (int put = 0; put < bits;) {
    const int w = (bit + put) >> 5, o = (bit + put) & 31, take = (32 - o < bits - put) ? 32 - o : bits - put;
    const uint32_t m = (take == 32 ? 0xFFFFFFFFu : ((1u << take) - 1u));
    pk[w] = (pk[w] & ~(m << o)) | ((uint32_t)(v >> put) & m) << o;
    put += take;
  }
}
__host__ __device__ inline void pack_row(const PackSpec& s, const uint32_t* row, uint32_t* pk) {
  for (int w = 0; w < s.pw; ++w) pk[w] = 0;
  for (int k = 0; k < s.n; ++k) {
    const PackParam& p = s.p[k];
    if (p.kind == BX_REAL) {
      pk_put(pk, p.bit, 64, (uint64_t)row[p.word] | ((uint64_t)row[p.word + 1] << 32));
      if (p.carry_coord) pk_put(pk, p.bit + 64, 64, (uint64_t)row[p.word + 2] | ((uint64_t)row[p.word + 3] << 32));
    } else if (p.kind == BX_PERMUTATION) {
      pk_put(pk, p.bit, p.bits, (uint64_t)row[p.word] | ((uint64_t)row[p.word + 1] << 32));
    } else {
      pk_put(pk, p.bit, p.bits, row[p.word]);
    }
  }
}
// words of the full row not covered by a parameter are zero (as SpaceLayout.encode leaves them)
__host__ __device__ inline void unpack_row(const PackSpec& s, const uint32_t* pk, uint32_t* row, int words) {
  for (int w = 0; w < words; ++w) row[w] = 0;
  for (int k = 0; k < s.n; ++k) {
    const PackParam& p = s.p[k];
    if (p.kind == BX_REAL) {
      const uint64_t v = pk_get(pk, p.bit, 64);
      uint64_t c;
      if (p.carry_coord) {
        c = pk_get(pk, p.bit + 64, 64);
      } else {
        double x;
        memcpy(&x, &v, 8);
        const double cx = (p.hi == p.lo) ? 0.0 : (x - p.lo) / (p.hi - p.lo);
        memcpy(&c, &cx, 8);
      }
      row[p.word] = (uint32_t)v;
      row[p.word + 1] = (uint32_t)(v >> 32);
      row[p.word + 2] = (uint32_t)c;
      row[p.word + 3] = (uint32_t)(c >> 32);
    } else if (p.kind == BX_PERMUTATION) {
      const uint64_t v = pk_get(pk, p.bit, p.bits);
      row[p.word] = (uint32_t)v;
      row[p.word + 1] = (uint32_t)(v >> 32);
    } else {
      row[p.word] = (uint32_t)pk_get(pk, p.bit, p.bits);
    }
  }
}

struct TcArgs {
  FusedArgs f;
  const unsigned char* mdig;  // [chunk][slice] blocks of 6 digit planes x 16 rows x 32 columns
  const double* rowscale;     // [16 * n_chunks] 2^(e_i - 56) * sc (0 beyond row n), then the same
                              // with the alpha / padding rows zeroed, then (tc_row_scale) digit scales
  int32_t n_slices;           // ceil(n / 32) column slices of K*
  int32_t n_chunks;           // floor(n / 16) + 1 row chunks of [L^-1; alpha^T]
  double kscale;              // 2^40 / sc: K* -> 40-bit fixed point
  int32_t n_coord;            // coord_lut entries
  double exp2tab256[256];     // 2^(j/256), correctly rounded (host long double)
  int32_t debug;              // BX_TC_DEBUG bits (timing experiments only): 1 no epilogue, 2 no MMAs,
                              // 4 epilogue TMEM reads without the arithmetic, 8 matrix ring (not resident),
                              // 16 per-pass planes (n > 255); bx_score_host: 64 the copy path for
                              // packed pinned pools instead of zero-copy, 128 the zero-copy path
                              // over a device copy of the pool (isolates the bus reads); 32 packed
                              // rows staged in the row buffer (no separate buffer)
  long long* trace;           // optional role timeline of CTA 0 (BX_TC_TRACE=file), else null
  // streaming host pools: rows arrive by chunks of 2^ready_shift rows; ready[c] != 0 once chunk c
  // is in device memory (written by the copy stream after the chunk), null = all rows present
  const uint32_t* ready;
  int32_t ready_shift;
  // mat_resident != 0: every (chunk, slice) digit block is loaded into shared memory once per CTA
  // and stays there for all tiles (set by launch_gp_tc when it fits; else the 8-stage ring)
  int32_t mat_resident;
  // n > 255 (several passes per tile): [grid][16 n_chunks - 256 rows][128 candidates] partial sums
  // of the rows >= 256, written and read back by the same epilogue thread; null otherwise
  double* part;
  int32_t planes_pp;          // set by launch_gp_tc: planes per pass (tc_layout)
  int32_t mat_stages;         // set by launch_gp_tc: matrix ring stages (not resident)
  // ks > 0: distances on the FP64 tensor cores, W = |x'|^2 + |y'|^2 - 2 x'.y' over the embedding
  // (EmbDim) as one product of ks k-steps of DMMA m8n8k4; the matrix digits carry the C-fragment
  // column permutation (launch_build_mdig perm).  ks == 0: FMA distances per parameter kind.
  int32_t ks;
  int32_t n_emb;              // E embedding coordinates (4 ks >= E)
  int32_t aug;                // E + 2 <= 4 ks: k-rows E, E + 1 carry |y'|^2 . 1 and 1 . |x'|^2
  const EmbDim* emb;          // [E]
  const double* emb_tab;
  int32_t emb_tab_len;
  const double* emb_planes;   // [4 ks][32 n_slices] the B operand: -2 y', (aug: |y'|^2, 1), zeros
  const double* emb_yy;       // [32 n_slices] |y'|^2 (added explicitly when !aug)
  // packed != null: the pool arrives in the packed wire format (streamed host pools); the
  // prefetcher stages packed rows, the decoders unpack them into the staging buffer and write the
  // full rows to f.rows (read by the forest / summary kernels after this one)
  const uint32_t* packed;
  PackSpec pack;
  int32_t pk_sep;             // set by launch_gp_tc: packed rows in their own staging buffer
};


int fused_max_rows();
size_t fused_smem_bytes(int n, int n_params, int n_kendall, int rows8);
size_t panels_doubles(int ncols_pad, int rows8);
cudaError_t launch_build_panels(const double* A, int lda, int rows_src, int ncols_pad, int rows8,
                                double* panels, cudaStream_t s);
cudaError_t launch_gp_fused(const FusedArgs& a, int sm_count, cudaStream_t s);
// tensor-core posterior: n <= kTcMaxRows - 1 training points ([L^-1; alpha^T] has n + 1 rows)
constexpr int kTcMaxRows = 4096;
size_t tc_smem_bytes(int n, int n_params, int n_kendall, int row_words, int ks, int n_emb, int emb_tab_len,
                     bool aug, bool resident);
// partial-sum scratch of the multi-pass posterior (n > 255), in doubles, for `grid` CTAs
size_t tc_part_doubles(int n, int grid);
size_t tc_mdig_bytes(int n);
cudaError_t launch_build_mdig(const double* A, int lda, int n, double sc, unsigned char* mdig,
                              double* rowscale, int perm, cudaStream_t s);
cudaError_t launch_gp_tc(const TcArgs& a, int sm_count, cudaStream_t s);
cudaError_t launch_summary(const SummaryArgs& a, int sm_count, cudaStream_t s, int* n_partials);
int summary_max_partials(int sm_count);

// launch_score returns the number of partials it wrote in *n_partials.
cudaError_t launch_score(const ScoreArgs& a, int sm_count, cudaStream_t s, int* n_partials);
int score_smem_bytes(int cpw, int ncols, int n_params);  // the generic kernel's shared memory
// Merge partials into *out.  When pool_rows is non-NULL the rows of the top-k entries are
// gathered from it (index - index_base); otherwise the caller fills them.
cudaError_t launch_partial_merge(const Partial* partials, int n_partials, const SpaceDev& space, int k,
                                 Partial* acc_out, cudaStream_t s);
cudaError_t launch_summary_merge(const Partial* partials, int n_partials, const SpaceDev& space,
                                 int k, const uint32_t* pool_rows, int64_t index_base,
                                 bx_score_summary* out, cudaStream_t s);
size_t qs_summary_smem_bytes(const QsForestDev& q);
bool qs_summary_available(const ForestDev& f);
cudaError_t launch_rf_summary(const SpaceDev& space, const ForestDev& f, const SummaryArgs& a, int sm_count,
                              cudaStream_t s, int* n_partials);
// pw_rows (device, q flags, nullable): per-row numpy summation order (1: the q == 1 pairwise sum)
cudaError_t launch_rf(const SpaceDev& space, const ForestDev& f, const uint32_t* rows, int64_t q,
                      int pairwise, double* probs, cudaStream_t s, const uint8_t* pw_rows = nullptr);
cudaError_t launch_neighbors(const SpaceDev& space, const CotDev* cot, const uint32_t* rows,
                             int count, uint32_t* out_rows, uint8_t* out_valid, cudaStream_t s);
cudaError_t launch_cot_contains(const SpaceDev& space, const CotDev& cot, const uint32_t* rows,
                                int64_t q, uint8_t* mask, cudaStream_t s);
cudaError_t launch_constraints(const SpaceDev& space, const ConstraintDev& c, const uint32_t* rows,
                               int64_t q, uint8_t* mask, cudaStream_t s);
cudaError_t launch_lml(const double* sq, int n, int D, const double* z, const double* thetas,
                       int c, double* out, double* scratch, cudaStream_t s);
cudaError_t launch_generate(const SpaceDev& space, const CotDev& cot, const int64_t* leaf_count,
                            int mode, uint64_t seed, int64_t index_base, int64_t q, uint32_t* rows,
                            cudaStream_t s);
cudaError_t launch_generate_indexed(const SpaceDev& space, const CotDev& cot,
                                    const int64_t* leaf_count, int mode, uint64_t seed,
                                    const int64_t* host_indices, int count, uint32_t* rows,
                                    cudaStream_t s);
cudaError_t launch_lml_grad(const double* sq, int n, int D, const double* z, const double* prm,
                            int c, double prior_k, double prior_rate, int use_prior, int want_grad,
                            double* out_value, double* out_grad, int* out_ok, double* scratch,
                            cudaStream_t s);
size_t lml_grad_scratch_doubles(int n, int c);
// _lml_core (+ gradient) with everything in one CTA's shared memory, one CTA per setting (small n)
bool lml_small_supported(int n);
cudaError_t launch_lml_small(const double* sq, int n, int D, const double* z, const double* prm, int c,
                             double prior_k, double prior_rate, int use_prior, int want_grad, double* out_value,
                             double* out_grad, int* out_ok, cudaStream_t s);
// _lml_core for c settings, each over the whole GPU, side by side on grid.y (lml_wide.cu), n <= 512
size_t lml_wide_scratch_doubles(int n, int D, int c);
bool lml_wide_supported(int n);
cudaError_t launch_gp_factor(const double* sq, int n, int D, const double* z, const double* prm, double* scratch,
                             const double** L_out, const double** al_out, const int** fail_out,
                             const double** X_out, cudaStream_t s);
size_t lml_coarse_wide_scratch_doubles(int n, int c);
cudaError_t launch_lml_coarse_wide(const double* sq, int n, int D, const double* z, const double* thetas, int c,
                                   double* out, double* scratch, cudaStream_t s);
cudaError_t launch_lml_wide(const double* sq, int n, int D, const double* z, const double* prm, int c, double prior_k,
                            double prior_rate, int use_prior, int want_grad, double* out_value, double* out_grad,
                            int* out_ok, double* scratch, cudaStream_t s);
cudaError_t launch_pairwise_sq(const SpaceDev& space, const uint32_t* a, int qa, const uint32_t* b,
                               int qb, double* out, cudaStream_t s);
cudaError_t launch_gp_planes(const SpaceDev& space, const uint32_t* train_rows, int n,
                             const double* inv_l, uint64_t* planes, uint64_t* kmask,
                             cudaStream_t s);
cudaError_t launch_tri_inverse(const double* L, int n, double* A, int lda, cudaStream_t s);
// rf_fit tree building (forest_fit.cu): one CTA per tree, outputs [T][max_nodes] in local preorder ids
size_t rf_fit_smem_bytes(int n);
size_t rf_fit_stack_bytes(int T, int max_nodes);
cudaError_t launch_rf_fit(const double* X, const double* y, int n, int F, int T, const int32_t* boot,
                          const int32_t* feats, const int32_t* n_drawn, int max_draws, int k, int max_depth,
                          int max_nodes, int32_t* feature, double* threshold, int32_t* left, int32_t* right,
                          double* value, int32_t* n_nodes, int32_t* status, void* stack, cudaStream_t s);

}  // namespace bx
