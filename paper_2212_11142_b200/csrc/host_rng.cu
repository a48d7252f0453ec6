// host_rng.cu — the candidate pool's permutation draws without a Python loop (host code).
//
// The reference's uniform sampler (space.py:312-332) draws each permutation parameter as n calls of
// numpy's Generator.permutation(m): arange(m) shuffled in place by Fisher-Yates from the top,
// j = random_interval(i) for i = m-1 .. 1 (numpy/random/_generator.pyx shuffle -> _shuffle_raw,
// distributions.c random_interval: the smallest all-ones mask >= i, 32-bit draws rejected above i).
// The 32-bit draws come from PCG64 (XSL-RR 128/64: step the 128-bit LCG, output rotr64(hi ^ lo,
// hi >> 58)), each 64-bit output serving two draws, low half first, the high half buffered in the
// generator's has_uint32 / uinteger state.  Replaying that stream here from the generator's state
// gives the same permutations and the same final state as the Python loop, so the pool - and the
// RNG stream the BO loop continues with - is the reference's.
#include <cstdint>

#include "bx_sm100.h"

namespace {

using u128 = unsigned __int128;

struct Pcg64 {
  u128 state, inc;
  int has32;
  uint32_t buf;

  uint64_t next64() {
    const u128 mult = ((u128)0x2360ED051FC65DA4ull << 64) | 0x4385DF649FCCF645ull;
    state = state * mult + inc;
    const uint64_t hi = (uint64_t)(state >> 64), lo = (uint64_t)state;
    const unsigned rot = (unsigned)(hi >> 58);
    const uint64_t x = hi ^ lo;
    return (x >> rot) | (x << ((64 - rot) & 63));
  }
  uint32_t next32() {
    if (has32) {
      has32 = 0;
      return buf;
    }
    const uint64_t v = next64();
    has32 = 1;
    buf = (uint32_t)(v >> 32);
    return (uint32_t)v;
  }
  // bounded_lemire_uint32: uniform on [0, rng] (numpy's random_bounded_uint64 for rng < 2^32)
  uint32_t lemire(uint32_t rng) {
    if (rng == 0) return 0;  // no draw
    if (rng == 0xFFFFFFFFu) return next32();
    const uint32_t excl = rng + 1;
    uint64_t m = (uint64_t)next32() * excl;
    uint32_t left = (uint32_t)m;
    if (left < excl) {
      const uint32_t threshold = (0xFFFFFFFFu - rng) % excl;
      while (left < threshold) {
        m = (uint64_t)next32() * excl;
        left = (uint32_t)m;
      }
    }
    return (uint32_t)(m >> 32);
  }
  // random_interval(max) for max < 2^32
  uint32_t interval(uint32_t max) {
    if (max == 0) return 0;
    uint32_t mask = max;
    mask |= mask >> 1;
    mask |= mask >> 2;
    mask |= mask >> 4;
    mask |= mask >> 8;
    mask |= mask >> 16;
    uint32_t v;
    while ((v = next32() & mask) > max) {
    }
    return v;
  }
};

Pcg64 load(const uint64_t* state, const int32_t* has_uint32, const uint32_t* uinteger) {
  return Pcg64{((u128)state[0] << 64) | state[1], ((u128)state[2] << 64) | state[3], *has_uint32 != 0, *uinteger};
}
void store(const Pcg64& g, uint64_t* state, int32_t* has_uint32, uint32_t* uinteger) {
  state[0] = (uint64_t)(g.state >> 64);
  state[1] = (uint64_t)g.state;
  *has_uint32 = g.has32;
  *uinteger = g.buf;
}

// np.random.default_rng(seed) for 0 <= seed < 2^64: SeedSequence(seed) (numpy/random/bit_generator.pyx:
// the entropy as little-endian 32-bit words mixed into a 4-word pool by hashmix / mix, then
// generate_state(4, uint64) hashed out of the pool) seeds PCG64 (pcg64_set_seed: state = 0,
// inc = 2 initseq + 1, step, state += initstate, step) with an empty 32-bit buffer.
Pcg64 seeded(uint64_t seed) {
  uint32_t ent[2] = {(uint32_t)seed, (uint32_t)(seed >> 32)};
  const int nent = (seed >> 32) ? 2 : 1;
  uint32_t hc = 0x43b0d7e5u;
  auto hashmix = [&hc](uint32_t v) {
    v ^= hc;
    hc *= 0x931e8875u;
    v *= hc;
    return v ^ (v >> 16);
  };
  auto mix = [](uint32_t x, uint32_t y) {
    const uint32_t r = 0xca01f9ddu * x - 0x4973f715u * y;
    return r ^ (r >> 16);
  };
  uint32_t pool[4];
  for (int i = 0; i < 4; ++i) pool[i] = hashmix(i < nent ? ent[i] : 0u);
  for (int a = 0; a < 4; ++a)
    for (int b = 0; b < 4; ++b)
      if (a != b) pool[b] = mix(pool[b], hashmix(pool[a]));
  uint32_t hb = 0x8b51f9ddu, w[8];
  for (int i = 0; i < 8; ++i) {
    uint32_t v = pool[i & 3] ^ hb;
    hb *= 0x58f38dedu;
    v *= hb;
    w[i] = v ^ (v >> 16);
  }
  uint64_t u[4];
  for (int i = 0; i < 4; ++i) u[i] = (uint64_t)w[2 * i] | ((uint64_t)w[2 * i + 1] << 32);
  Pcg64 g{0, ((((u128)u[2] << 64) | u[3]) << 1) | 1u, 0, 0u};
  g.next64();
  g.state += ((u128)u[0] << 64) | u[1];
  g.next64();
  return g;
}

// Generator.choice(pop, size=k, replace=False) for pop <= 10000 into idx[k]
void choice(Pcg64& g, int32_t pop, int32_t k, int32_t* idx) {
  for (int32_t j = pop - k; j < pop; ++j) {
    const int32_t v = (int32_t)g.lemire((uint32_t)j);
    bool seen = false;
    for (int32_t t = 0; t < j - (pop - k); ++t) seen |= idx[t] == v;
    idx[j - (pop - k)] = seen ? j : v;
  }
  for (int32_t i = k - 1; i >= 1; --i) {  // _shuffle_int: bounded Lemire draws, not random_interval
    const uint32_t s = g.lemire((uint32_t)i);
    const int32_t t = idx[i];
    idx[i] = idx[s];
    idx[s] = t;
  }
}

}  // namespace

// n draws of Generator.choice(pop, size=k, replace=False) for pop <= 10000 (the rf_fit feature
// subsets, feasibility.py:119): Floyd's algorithm (j = pop-k .. pop-1: v uniform on [0, j], taken
// unless already chosen, else j) followed by _shuffle_int of the k chosen (Fisher-Yates from the top
// with v uniform on [0, i] by Lemire's method) (numpy/random/_generator.pyx choice, non-tail branch).
extern "C" int bx_pcg64_choice(uint64_t* state, int32_t* has_uint32, uint32_t* uinteger, int64_t n, int32_t pop,
                               int32_t k, int32_t* out) {
  if (!state || !has_uint32 || !uinteger || n < 0 || pop < 1 || pop > 10000 || k < 0 || k > pop ||
      (n > 0 && k > 0 && !out))
    return BX_ERR_ARG;
  Pcg64 g = load(state, has_uint32, uinteger);
  for (int64_t r = 0; r < n; ++r) choice(g, pop, k, out + r * k);
  store(g, state, has_uint32, uinteger);
  return BX_OK;
}

// The random-forest fit's per-tree draws (feasibility.py:119-190): for each seed t, the tree's
// generator np.random.default_rng(seeds[t]), its bootstrap rows g.integers(0, n, size=n) (Lemire
// draws on [0, n-1], numpy's random_bounded_uint64_fill) and then ndraws feature subsets
// g.choice(pop, size=k, replace=False); the generator's state afterwards goes to state[4t..4t+3] /
// has_uint32[t] / uinteger[t] so that bx_pcg64_choice can continue it.
extern "C" int bx_pcg64_forest_draws(const uint64_t* seeds, int32_t n_trees, int64_t n, int32_t pop, int32_t k,
                                     int32_t ndraws, int32_t* boot, int32_t* subsets, uint64_t* state,
                                     int32_t* has_uint32, uint32_t* uinteger) {
  if (n_trees < 0 || n < 1 || n > 0x7FFFFFFF || pop < 1 || pop > 10000 || k < 0 || k > pop || ndraws < 0 ||
      (n_trees > 0 && (!seeds || !boot || !state || !has_uint32 || !uinteger || (ndraws > 0 && k > 0 && !subsets))))
    return BX_ERR_ARG;
  for (int32_t t = 0; t < n_trees; ++t) {
    Pcg64 g = seeded(seeds[t]);
    int32_t* b = boot + (int64_t)t * n;
    for (int64_t i = 0; i < n; ++i) b[i] = (int32_t)g.lemire((uint32_t)(n - 1));
    for (int32_t r = 0; r < ndraws; ++r) choice(g, pop, k, subsets + ((int64_t)t * ndraws + r) * k);
    store(g, state + 4 * (int64_t)t, has_uint32 + t, uinteger + t);
    state[4 * (int64_t)t + 2] = (uint64_t)(g.inc >> 64);
    state[4 * (int64_t)t + 3] = (uint64_t)g.inc;
  }
  return BX_OK;
}

extern "C" int bx_pcg64_permutations(uint64_t* state, int32_t* has_uint32, uint32_t* uinteger, int64_t n,
                                     int32_t m, uint64_t* packed) {
  if (!state || !has_uint32 || !uinteger || n < 0 || m < 1 || m > 16 || (n > 0 && !packed)) return BX_ERR_ARG;
  Pcg64 g = load(state, has_uint32, uinteger);
  for (int64_t r = 0; r < n; ++r) {
    uint8_t a[16];
    for (int i = 0; i < m; ++i) a[i] = (uint8_t)i;
    for (int i = m - 1; i >= 1; --i) {
      const uint32_t j = g.interval((uint32_t)i);
      const uint8_t t = a[i];
      a[i] = a[j];
      a[j] = t;
    }
    uint64_t x = 0;  // layout.pack_perm: element at position i (0-based value) in nibble m-1-i
    for (int i = 0; i < m; ++i) x = (x << 4) | a[i];
    packed[r] = x;
  }
  store(g, state, has_uint32, uinteger);
  return BX_OK;
}
