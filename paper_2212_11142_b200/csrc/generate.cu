// generate.cu — device-side candidate generation.
//
// Candidates are produced directly in row form from a counter-based RNG (Philox4x32-10) keyed by
// (seed, global candidate index), so any slice of a pool of up to 2^63 candidates can be
// regenerated independently on any rank:
//   mode 0  uniform over the dense space: the distribution of sample_uniform (space.py:312-332)
//   mode 1  leaf-uniform over the chain of trees: the distribution of
//           ChainOfTrees.sample_leaf_uniform (constraints.py:471-523), realised by a weighted
//           descent on per-node leaf counts (uniform over leaves without materialising them);
//           real and permutation singleton groups are drawn as in mode 0.
//   mode 2  path-biased over the chain of trees: the distribution of sample_path_biased
//           (constraints.py:478-501, 522-523; engine.py:216-217 with cot_sampling == "path"): every
//           level picks one of the node's children uniformly.
// Parity with the reference here is statistical (the reference draws from numpy's PCG64 stream);
// membership is exact.
#include "bx_common.cuh"

namespace bx {

namespace {

struct Philox {
  uint32_t c[4];
  uint32_t k[2];
};

__device__ __forceinline__ void philox_round(uint32_t (&c)[4], const uint32_t (&k)[2]) {
  const uint32_t M0 = 0xD2511F53u, M1 = 0xCD9E8D57u;
  const uint32_t hi0 = __umulhi(M0, c[0]), lo0 = M0 * c[0];
  const uint32_t hi1 = __umulhi(M1, c[2]), lo1 = M1 * c[2];
  const uint32_t n0 = hi1 ^ c[1] ^ k[0], n1 = lo1, n2 = hi0 ^ c[3] ^ k[1], n3 = lo0;
  c[0] = n0; c[1] = n1; c[2] = n2; c[3] = n3;
}

// Philox4x32-10 of counter (index lo, index hi, stream, draw) under key (seed lo, seed hi)
__device__ __forceinline__ void philox(uint64_t seed, uint64_t index, uint32_t stream, uint32_t draw,
                                       uint32_t (&out)[4]) {
  uint32_t c[4] = {(uint32_t)index, (uint32_t)(index >> 32), stream, draw};
  uint32_t k[2] = {(uint32_t)seed, (uint32_t)(seed >> 32)};
#pragma unroll
  for (int r = 0; r < 10; ++r) {
    philox_round(c, k);
    k[0] += 0x9E3779B9u;
    k[1] += 0xBB67AE85u;
  }
  out[0] = c[0]; out[1] = c[1]; out[2] = c[2]; out[3] = c[3];
}

// uniform doubles in [0, 1) with 53 random bits
struct Uniforms {
  uint64_t seed, index;
  uint32_t stream, draw;
  uint32_t buf[4];
  int avail;
  __device__ Uniforms(uint64_t s, uint64_t i, uint32_t st) : seed(s), index(i), stream(st), draw(0), avail(0) {}
  __device__ __forceinline__ double next() {
    if (avail < 2) {
      philox(seed, index, stream, draw++, buf);
      avail = 4;
    }
    const uint32_t a = buf[4 - avail], b = buf[5 - avail];
    avail -= 2;
    return ((double)(a >> 5) * 67108864.0 + (double)(b >> 6)) * (1.0 / 9007199254740992.0);
  }
};

__device__ void draw_param(const bx_param_desc& p, const double* coord_lut, Uniforms& u, uint32_t* row) {
  if (p.kind == BX_REAL) {
    const double v = fma(u.next(), p.hi - p.lo, p.lo);
    double c;
    if (p.is_log) c = (log(v) - log(p.lo)) / (log(p.hi) - log(p.lo));
    else c = (v - p.lo) / (p.hi - p.lo);
    put_f64(row, p.word, v);
    put_f64(row, p.word + 2, c);
  } else if (p.kind == BX_PERMUTATION) {
    int e[BX_MAX_PERM];
    for (int i = 0; i < p.size; ++i) e[i] = i;
    for (int i = p.size - 1; i > 0; --i) {  // Fisher-Yates
      const int j = (int)(u.next() * (double)(i + 1));
      const int t = e[i];
      e[i] = e[j];
      e[j] = t;
    }
    uint64_t x = 0;
    for (int i = 0; i < p.size; ++i) x = (x << 4) | (uint64_t)e[i];
    put_u64(row, p.word, x);
  } else {
    row[p.word] = (uint32_t)(u.next() * (double)p.size);
  }
  (void)coord_lut;
}

__global__ void generate_kernel(SpaceDev sp, CotDev cot, const int64_t* leaf_count, int mode,
                                uint64_t seed, int64_t index_base, int64_t q, uint32_t* rows) {
  __shared__ bx_param_desc params[BX_MAX_PARAMS];
  for (int i = threadIdx.x; i < sp.n_params * (int)sizeof(bx_param_desc) / 4; i += blockDim.x)
    reinterpret_cast<int32_t*>(params)[i] = reinterpret_cast<const int32_t*>(sp.params)[i];
  __syncthreads();
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < q;
       i += (int64_t)gridDim.x * blockDim.x) {
    uint32_t* row = rows + (size_t)i * sp.row_words;
    for (int w = 0; w < sp.row_words; ++w) row[w] = 0;
    const uint64_t gi = (uint64_t)(index_base + i);
    if (mode == 0) {
      for (int k = 0; k < sp.n_params; ++k) {
        Uniforms u(seed, gi, (uint32_t)k);
        draw_param(params[k], sp.coord_lut, u, row);
      }
      continue;
    }
    for (int g = 0; g < cot.n_groups; ++g) {
      Uniforms u(seed, gi, 0x10000u + (uint32_t)g);
      const int pb = cot.group_param_begin[g], pe = cot.group_param_begin[g + 1];
      if (cot.group_kind[g] != 0) {
        draw_param(params[cot.group_params[pb]], sp.coord_lut, u, row);
        continue;
      }
      int node = cot.group_root[g];
      for (int li = pb; li < pe; ++li) {
        const int first = cot.child_begin[node], cnt = cot.child_count[node];
        int pick = first + cnt - 1;
        if (mode == 2) {  // path-biased: a uniform child at every level
          pick = first + min(cnt - 1, (int)(u.next() * (double)cnt));
        } else {  // leaf-uniform: child with probability leaf_count(child) / leaf_count(node)
          const double r = u.next() * (double)leaf_count[node];
          double acc = 0.0;
          for (int c = first; c < first + cnt; ++c) {
            acc += (double)leaf_count[c];
            if (r < acc) { pick = c; break; }
          }
        }
        row[params[cot.group_params[li]].word] = (uint32_t)cot.node_value[pick];
        node = pick;
      }
    }
  }
}

}  // namespace

cudaError_t launch_generate(const SpaceDev& space, const CotDev& cot, const int64_t* leaf_count,
                            int mode, uint64_t seed, int64_t index_base, int64_t q, uint32_t* rows,
                            cudaStream_t s) {
  if (q <= 0) return cudaSuccess;
  int64_t blocks = (q + 255) / 256;
  if (blocks > 148 * 8) blocks = 148 * 8;
  generate_kernel<<<(int)blocks, 256, 0, s>>>(space, cot, leaf_count, mode, seed, index_base, q, rows);
  return cudaGetLastError();
}

// regenerate the rows of given global indices (the top-k of a generated pool)
cudaError_t launch_generate_indexed(const SpaceDev& space, const CotDev& cot,
                                    const int64_t* leaf_count, int mode, uint64_t seed,
                                    const int64_t* host_indices, int count, uint32_t* rows,
                                    cudaStream_t s) {
  for (int i = 0; i < count; ++i) {
    cudaError_t e = launch_generate(space, cot, leaf_count, mode, seed, host_indices[i], 1,
                                    rows + (size_t)i * space.row_words, s);
    if (e != cudaSuccess) return e;
  }
  return cudaSuccess;
}

}  // namespace bx
