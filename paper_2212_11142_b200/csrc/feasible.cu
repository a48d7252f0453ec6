// feasible.cu — integer/bit-exact kernels of the known-constraint side of the hot path:
//   neighbours of a configuration      (space.py:258-309, neighbors/_param_neighbors)
//   chain-of-trees membership          (constraints.py:413-430, ChainOfTrees.contains)
//   constraint bytecode interpreter    (constraints.py:309-368, _eval_node/eval_constraint)
#include <climits>

#include "bx_common.cuh"

namespace bx {

namespace {

__device__ __forceinline__ void load_params(const SpaceDev& sp, bx_param_desc* params) {
  for (int i = threadIdx.x; i < sp.n_params * (int)sizeof(bx_param_desc) / 4; i += blockDim.x)
    reinterpret_cast<int32_t*>(params)[i] = reinterpret_cast<const int32_t*>(sp.params)[i];
  __syncthreads();
}

// ChainOfTrees.contains (constraints.py:413-430).  Tree groups walk the children whose value
// equals the configuration's value (domain indices: distinct domain values <-> distinct indices);
// real singletons check lo <= v <= hi (Parameter.contains, space.py:109-110); permutation
// singletons check the bijection (space.py:115-117).
__device__ bool cot_contains_row(const CotDev& cot, const bx_param_desc* params, const uint32_t* row) {
  for (int g = 0; g < cot.n_groups; ++g) {
    const int kind = cot.group_kind[g];
    const int pb = cot.group_param_begin[g], pe = cot.group_param_begin[g + 1];
    if (kind == 1) {
      const bx_param_desc& p = params[cot.group_params[pb]];
      const double v = row_f64(row, p.word);
      if (!(p.lo <= v && v <= p.hi)) return false;
      continue;
    }
    if (kind == 2) {
      const bx_param_desc& p = params[cot.group_params[pb]];
      const uint64_t x = row_u64(row, p.word);
      uint32_t seen = 0;
      for (int i = 0; i < p.size; ++i) seen |= 1u << perm_at(x, p.size, i);
      if (seen != ((p.size >= 32) ? 0xffffffffu : ((1u << p.size) - 1u))) return false;
      if (p.size < 16 && (x >> (4 * p.size)) != 0) return false;
      continue;
    }
    int node = cot.group_root[g];
    for (int li = pb; li < pe; ++li) {
      const bx_param_desc& p = params[cot.group_params[li]];
      const int x = (int)row[p.word];
      int lo = cot.child_begin[node], hi = lo + cot.child_count[node] - 1, found = -1;
      while (lo <= hi) {
        const int mid = (lo + hi) >> 1;
        const int v = cot.node_value[mid];
        if (v == x) { found = mid; break; }
        if (v < x) lo = mid + 1; else hi = mid - 1;
      }
      if (found < 0) return false;
      node = found;
    }
  }
  return true;
}

// One thread per (start row, neighbour slot).
__global__ void neighbors_kernel(SpaceDev sp, CotDev cot, int use_cot, const uint32_t* rows,
                                 int count, uint32_t* out_rows, uint8_t* out_valid) {
  __shared__ bx_param_desc params[BX_MAX_PARAMS];
  load_params(sp, params);
  const int W = sp.row_words;
  const int64_t total = (int64_t)count * sp.n_slots;
  for (int64_t t = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; t < total;
       t += (int64_t)gridDim.x * blockDim.x) {
    const int r = (int)(t / sp.n_slots), s = (int)(t % sp.n_slots);
    const uint32_t* src = rows + (size_t)r * W;
    uint32_t* dst = out_rows + (size_t)t * W;
    for (int w = 0; w < W; ++w) dst[w] = src[w];
    const int k = sp.slot_param[s], mv = sp.slot_move[s];
    const bx_param_desc& p = params[k];
    bool ok = true;
    if (p.kind == BX_INTEGER || p.kind == BX_ORDINAL) {
      // space.py:260-265: value -/+ 1 (integer) or index -/+ 1 (ordinal), in order (-1, +1)
      const int x = (int)src[p.word] + (mv == 0 ? -1 : 1);
      ok = x >= 0 && x < p.size;
      dst[p.word] = (uint32_t)(ok ? x : 0);
    } else if (p.kind == BX_CATEGORICAL) {
      // space.py:266-267: every other label in declaration order
      const int cur = (int)src[p.word];
      dst[p.word] = (uint32_t)(mv < cur ? mv : mv + 1);
    } else if (p.kind == BX_REAL) {
      // space.py:268-277: one step on the 64-point grid, banker's rounding, no FMA
      const double value = row_f64(src, p.word);
      const double i = rint(__ddiv_rn(__dsub_rn(value, p.lo), p.step));
      const double j = i + (mv == 0 ? -1.0 : 1.0);
      ok = j >= 0.0 && j < (double)kRealGrid;
      if (ok) {
        const double v = __dadd_rn(p.lo, __dmul_rn(j, p.step));
        ok = v != value;
        put_f64(dst, p.word, v);
        put_f64(dst, p.word + 2, sp.coord_lut[p.coord + (int)j]);
      }
    } else {
      // space.py:278-286: transposition (a, b), a < b, enumerated a-major
      const int m = p.size;
      int a = 0, rem = mv;
      while (rem >= m - 1 - a) { rem -= m - 1 - a; ++a; }
      const int b = a + 1 + rem;
      uint64_t x = row_u64(src, p.word);
      const int sa = 4 * (m - 1 - a), sb = 4 * (m - 1 - b);
      const uint64_t ea = (x >> sa) & 0xFull, eb = (x >> sb) & 0xFull;
      x &= ~((0xFull << sa) | (0xFull << sb));
      x |= (eb << sa) | (ea << sb);
      put_u64(dst, p.word, x);
    }
    if (ok && use_cot) ok = cot_contains_row(cot, params, dst);
    out_valid[t] = ok ? 1 : 0;
  }
}

__global__ void cot_kernel(SpaceDev sp, CotDev cot, const uint32_t* rows, int64_t q, uint8_t* mask) {
  __shared__ bx_param_desc params[BX_MAX_PARAMS];
  load_params(sp, params);
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < q;
       i += (int64_t)gridDim.x * blockDim.x)
    mask[i] = cot_contains_row(cot, params, rows + (size_t)i * sp.row_words) ? 1 : 0;
}

// ---- constraint bytecode ---------------------------------------------------------------------
// Opcodes (paper_2212_11142_b200/constraints.py emits them):
enum Op {
  OP_NUM = 0,     // push float literal consts[arg]
  OP_VAR = 1,     // push numeric parameter arg (int or float per the Python value type)
  OP_CAT = 2,     // push string id of categorical parameter arg
  OP_STR = 3,     // push string id arg (literal)
  OP_NEG = 4, OP_NOT = 5,
  OP_ADD = 6, OP_SUB = 7, OP_MUL = 8, OP_DIV = 9, OP_MOD = 10,
  OP_LT = 11, OP_LE = 12, OP_GT = 13, OP_GE = 14, OP_EQ = 15, OP_NE = 16,
  OP_AND = 17, OP_OR = 18
};

enum Tag { T_INT = 0, T_FLT = 1, T_BOOL = 2, T_STR = 3 };

struct Val {
  int tag;
  long long i;  // int / bool / string id
  double f;
};

constexpr int kStack = 32;
constexpr long long kExact = 1ll << 53;

// Python int -> float conversion is exact below 2^53; outside we flag the envelope.
__device__ __forceinline__ double as_float(const Val& v, bool& env) {
  if (v.tag == T_FLT) return v.f;
  if (v.i > kExact || v.i < -kExact) env = false;
  return (double)v.i;
}

// Python comparison semantics for int/float mixes: exact for |int| <= 2^53.
__device__ __forceinline__ int cmp_num(const Val& a, const Val& b, bool& env, bool& unordered) {
  unordered = false;
  if (a.tag == T_INT && b.tag == T_INT) return (a.i < b.i) ? -1 : (a.i > b.i ? 1 : 0);
  const double x = as_float(a, env), y = as_float(b, env);
  if (isnan(x) || isnan(y)) { unordered = true; return 0; }
  return (x < y) ? -1 : (x > y ? 1 : 0);
}

// Python float % float (Objects/floatobject.c float_rem)
__device__ __forceinline__ double py_fmod(double vx, double wx) {
  double mod = fmod(vx, wx);
  if (mod != 0.0) {
    if ((wx < 0.0) != (mod < 0.0)) mod += wx;
  } else {
    mod = copysign(0.0, wx);
  }
  return mod;
}

// returns 1 true, 0 false (including ZeroDivision/Overflow faults), -1 outside the envelope
__device__ int eval_program(const ConstraintDev& c, const bx_param_desc* params, const int32_t* code,
                            int len, const uint32_t* row) {
  Val st[kStack];
  int sp = 0;
  bool env = true;
  for (int pc = 0; pc < len; pc += 2) {
    const int op = code[pc], arg = code[pc + 1];
    switch (op) {
      case OP_NUM: st[sp].tag = T_FLT; st[sp].f = c.consts[arg]; st[sp].i = 0; ++sp; break;
      case OP_VAR: {
        const bx_param_desc& p = params[arg];
        if (p.kind == BX_REAL) {
          st[sp].tag = T_FLT; st[sp].f = row_f64(row, p.word); st[sp].i = 0;
        } else {
          const int o = c.voff[arg] + (int)row[p.word];
          st[sp].tag = c.vtag[o] ? T_FLT : T_INT;
          st[sp].i = c.vint[o];
          st[sp].f = c.vflt[o];
        }
        ++sp;
        break;
      }
      case OP_CAT: {
        const bx_param_desc& p = params[arg];
        st[sp].tag = T_STR; st[sp].i = c.str_id[c.voff[arg] + (int)row[p.word]]; ++sp;
        break;
      }
      case OP_STR: st[sp].tag = T_STR; st[sp].i = arg; ++sp; break;
      case OP_NEG: {
        Val& v = st[sp - 1];
        if (v.tag == T_INT) {
          if (v.i == LLONG_MIN) env = false;
          v.i = -v.i;
        } else {
          v.f = -v.f;
        }
        break;
      }
      case OP_NOT: st[sp - 1].i = st[sp - 1].i ? 0 : 1; st[sp - 1].tag = T_BOOL; break;
      case OP_AND: case OP_OR: {
        // `left and right` / `left or right` on bools (constraints.py:346-348), both evaluated
        const Val r = st[--sp];
        Val& l = st[sp - 1];
        l.i = (op == OP_AND) ? (l.i && r.i) : (l.i || r.i);
        l.tag = T_BOOL;
        break;
      }
      case OP_ADD: case OP_SUB: case OP_MUL: case OP_DIV: case OP_MOD: {
        const Val r = st[--sp];
        Val& l = st[sp - 1];
        if (op == OP_DIV) {  // true division: always float; ZeroDivisionError -> False
          const double x = as_float(l, env), y = as_float(r, env);
          if (y == 0.0) return 0;
          l.f = x / y; l.tag = T_FLT;
        } else if (l.tag == T_INT && r.tag == T_INT) {
          long long out;
          bool ovf = false;
          if (op == OP_ADD) {
            out = (long long)((unsigned long long)l.i + (unsigned long long)r.i);
            ovf = ((l.i ^ out) & (r.i ^ out)) < 0;
          } else if (op == OP_SUB) {
            out = (long long)((unsigned long long)l.i - (unsigned long long)r.i);
            ovf = ((l.i ^ r.i) & (l.i ^ out)) < 0;
          } else if (op == OP_MUL) {
            out = (long long)((unsigned long long)l.i * (unsigned long long)r.i);
            ovf = __mul64hi(l.i, r.i) != (out >> 63);
          }
          else {
            if (r.i == 0) return 0;  // ZeroDivisionError
            if (l.i == LLONG_MIN && r.i == -1) { ovf = true; out = 0; }
            else {
              out = l.i % r.i;  // Python floor modulo: sign of the divisor
              if (out != 0 && ((out < 0) != (r.i < 0))) out += r.i;
            }
          }
          if (ovf) env = false;
          l.i = out;
        } else {
          const double x = as_float(l, env), y = as_float(r, env);
          double out;
          if (op == OP_ADD) out = __dadd_rn(x, y);
          else if (op == OP_SUB) out = __dsub_rn(x, y);
          else if (op == OP_MUL) out = __dmul_rn(x, y);
          else {
            if (y == 0.0) return 0;  // ZeroDivisionError: float modulo
            out = py_fmod(x, y);
          }
          l.f = out; l.tag = T_FLT;
        }
        break;
      }
      default: {  // comparisons
        const Val r = st[--sp];
        Val& l = st[sp - 1];
        bool res;
        if (l.tag == T_STR || r.tag == T_STR) {
          const bool eq = l.tag == r.tag && l.i == r.i;
          res = (op == OP_EQ) ? eq : !eq;
        } else {
          bool unordered;
          const int cr = cmp_num(l, r, env, unordered);
          if (unordered) res = (op == OP_NE);
          else if (op == OP_LT) res = cr < 0;
          else if (op == OP_LE) res = cr <= 0;
          else if (op == OP_GT) res = cr > 0;
          else if (op == OP_GE) res = cr >= 0;
          else if (op == OP_EQ) res = cr == 0;
          else res = cr != 0;
        }
        l.tag = T_BOOL; l.i = res ? 1 : 0;
        break;
      }
    }
  }
  if (!env) return -1;
  const Val& top = st[sp - 1];
  if (top.tag == T_BOOL || top.tag == T_INT) return top.i != 0;
  if (top.tag == T_FLT) return top.f != 0.0;
  return 1;
}

__global__ void constraints_kernel(SpaceDev sp, ConstraintDev c, const uint32_t* rows, int64_t q,
                                   uint8_t* mask) {
  __shared__ bx_param_desc params[BX_MAX_PARAMS];
  load_params(sp, params);
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < q;
       i += (int64_t)gridDim.x * blockDim.x) {
    const uint32_t* row = rows + (size_t)i * sp.row_words;
    bool all = true;
    for (int k = 0; k < c.n_constraints && all; ++k) {
      const int b = c.prog_begin[k], e = c.prog_begin[k + 1];
      const int r = eval_program(c, params, c.code + b, e - b, row);
      if (r < 0) { atomicExch(c.fault, 1); all = false; }
      else all = r == 1;
    }
    mask[i] = all ? 1 : 0;
  }
}

int grid_for(int64_t work, int threads) {
  int64_t b = (work + threads - 1) / threads;
  if (b > 148 * 16) b = 148 * 16;
  if (b < 1) b = 1;
  return (int)b;
}

}  // namespace

cudaError_t launch_neighbors(const SpaceDev& space, const CotDev* cot, const uint32_t* rows,
                             int count, uint32_t* out_rows, uint8_t* out_valid, cudaStream_t s) {
  if (count <= 0 || space.n_slots <= 0) return cudaSuccess;
  CotDev empty{};
  neighbors_kernel<<<grid_for((int64_t)count * space.n_slots, 128), 128, 0, s>>>(
      space, cot ? *cot : empty, cot != nullptr, rows, count, out_rows, out_valid);
  return cudaGetLastError();
}

cudaError_t launch_cot_contains(const SpaceDev& space, const CotDev& cot, const uint32_t* rows,
                                int64_t q, uint8_t* mask, cudaStream_t s) {
  if (q <= 0) return cudaSuccess;
  cot_kernel<<<grid_for(q, 256), 256, 0, s>>>(space, cot, rows, q, mask);
  return cudaGetLastError();
}

cudaError_t launch_constraints(const SpaceDev& space, const ConstraintDev& c, const uint32_t* rows,
                               int64_t q, uint8_t* mask, cudaStream_t s) {
  if (q <= 0) return cudaSuccess;
  constraints_kernel<<<grid_for(q, 128), 128, 0, s>>>(space, c, rows, q, mask);
  return cudaGetLastError();
}

}  // namespace bx
