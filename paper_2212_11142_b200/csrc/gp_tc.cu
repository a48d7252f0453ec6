// gp_tc.cu — posterior + EI with the n^2 contraction on the 5th-generation tensor cores.
//
// [v ; mean] = [L^-1 ; alpha^T] K*^T (surrogate.py:322-325) is evaluated as an Ozaki-style split
// product in exact integer arithmetic.  Row i of A = [L^-1; alpha^T] is scaled by 2^-e_i and
// written as six balanced base-256 digits (int8), K* is scaled by 1/sc (sc = 2^ceil(log2 sigma))
// and written as five unsigned base-256 digits (uint8):
//     A_ij = 2^e_i sum_a d_a[i][j] 256^-(a+1),    K*_cj = sc sum_b f_b[c][j] 256^-(b+1).
// The 20 digit pairs with a + b <= 5 are u8 x s8 -> s32 GEMMs on tcgen05.mma kind::i8; pairs with
// equal a + b share one TMEM accumulator (6 groups G_t), every sum is exact in int32, and the
// epilogue recombines the groups exactly in int64 before a single conversion to double:
//     v_i = 2^(e_i - 56) sc sum_t G_t 256^(5 - t).
// The dropped pairs and the digit truncation leave ~2^-46 of |A_i| |K*| per row; simulated on the
// golden fixtures the variance moves by <= 1e-7 relative (C1, the worst case), far inside the
// 1e-5 parity bar.  The Matérn evaluation itself stays FP64.
//
// Tile = 128 candidates (the MMA M dimension, one TMEM lane each).  The candidate digits are the
// MMA A operand and live in tensor memory (written by the producers with tcgen05.st), so the
// tensor core reads only the small matrix operand from shared memory.  The matrix is consumed in
// row chunks of 16: chunk c needs column slices 0..c/2 only (lower triangle + alpha).  Chunks run
// from the last to the first, so column slice k is dead after chunk 2k and the producers refill
// it for the next tile while the MMAs finish the smaller chunks.
// CTA = 16 warps (128 registers each), one per SM, persistent over tiles:
//   warp 0         : MMA issuer (5 UTCIMMA 128 x (6-b)*16 x 32 per chunk and slice, b = K* digit)
//   warp 1  lane 0 : TMA producer: the whole digit-sliced matrix once per CTA when it fits in shared
//                    memory (resident for every tile), else one 3 KB bulk copy per (chunk, slice)
//                    block through an 8-stage ring
//   warp 1  lane 1 : row prefetcher: the next tiles' encoded rows, one bulk copy per tile
//   warps 2-3      : decoders: candidate values / masks / forest offsets of the next tile
//   warps 4-7      : epilogue, thread = candidate = TMEM lane: tcgen05.ld of the 6 groups,
//                    int64 recombination, sum of squares, mean, EI — no cross-thread reduction;
//                    between chunks, the candidate's forest probability from QuickScorer tables
//   warps 8-15     : K* producers: 16 Matérn values (FP64) per thread and slice, sliced into
//                    digits and stored into the candidate's TMEM lane (tcgen05.st)
// TMEM (512 columns): two 96-column accumulators (6 groups x 16 rows) so the epilogue of one chunk
// overlaps the MMAs of the next, then 40 columns (5 digits x 32 bytes) per column slice.
#include <algorithm>
#include <type_traits>
#include <cstdio>
#include <cstdlib>

#include "bx_common.cuh"
#include "matern.cuh"
#include "summary.cuh"

namespace bx {

namespace {

constexpr int kM = 128;          // candidates per tile
constexpr int kN = 16;           // matrix rows per chunk
constexpr int kDA = 6;           // matrix digits (signed)
constexpr int kDB = 5;           // K* digits (unsigned)
constexpr int kGroups = 6;       // a + b in 0..5
constexpr int kStages = 8;       // matrix block ring: minimum stages
constexpr int kMaxStages = 32;   // ... and maximum (launch_gp_tc fills the spare shared memory)
constexpr int kMaxChunks = kTcMaxRows / 16;  // n <= 4095
constexpr int kSlots = 8;        // K* column slices held in tensor memory at a time
// n > 255 (more than kSlots column slices): each tile runs one pass per 8 slices.  Pass p holds
// slices 8p..8p+7 (columns 256p..256p+255) in the slots and runs the row chunks of rows >= 256p
// (the lower triangle has no other blocks in those columns).  A row finishes in its last pass,
// min(npass - 1, row / 256); before that its partial sum (exact int64, converted to double - an
// exact integer below 2^53) is parked in global scratch by the epilogue thread that owns the
// candidate and added back in the next pass.
__host__ __device__ __forceinline__ int tc_passes(int nsl) { return (nsl + kSlots - 1) / kSlots; }
// K* producer warps (a multiple of 4: kProdWarps / 4 per TMEM lane quarter).  The DMMA producers
// (KS > 0) are written for two per quarter at 128 registers; the FMA producers (integer-heavy
// distance code, latency bound) run four per quarter at 80 registers.
template <int KS>
constexpr int tc_prod_warps() { return KS == 0 ? 16 : 8; }
template <int KS>
constexpr int tc_threads() { return (8 + tc_prod_warps<KS>()) * 32; }
constexpr int kMatBlock = kDA * kN * 32;  // 3 KB per (chunk, slice)
constexpr int kAccCols = kGroups * kN;    // 96 TMEM columns per accumulator
constexpr int kDigCol0 = 2 * kAccCols;    // first TMEM column of the candidate digits
constexpr int kSliceCols = kDB * 8;       // 40 TMEM columns (5 digits x 32 bytes) per slice
constexpr int kMaxCoord = 1024;           // scaled coordinate table entries kept in shared memory

__device__ __forceinline__ uint32_t su32(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }

__device__ __forceinline__ void mb_init(uint64_t* b, uint32_t n) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(su32(b)), "r"(n));
}
__device__ __forceinline__ void mb_arrive(uint64_t* b) {
  asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(su32(b)) : "memory");
}
__device__ __forceinline__ void mb_expect(uint64_t* b, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(su32(b)), "r"(bytes) : "memory");
}
__device__ __forceinline__ void mb_wait(uint64_t* b, uint32_t phase) {
  uint32_t done = 0;
  while (!done)
    asm volatile("{\n\t.reg .pred p;\n\tmbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\n\t"
                 "selp.u32 %0, 1, 0, p;\n\t}\n"
                 : "=r"(done) : "r"(su32(b)), "r"(phase) : "memory");
}
// For the roles that wait on the producers (MMA issuer, epilogue, decoders, copy threads): the
// suspend-time hint parks the warp until the phase completes instead of re-polling after the
// short default window — when the producers are the bottleneck (mixed spaces) those polling loops
// took ~30 % of the issue slots.
__device__ __forceinline__ void mb_wait_sleep(uint64_t* b, uint32_t phase) {
  uint32_t done = 0;
  while (!done)
    asm volatile("{\n\t.reg .pred p;\n\tmbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2, %3;\n\t"
                 "selp.u32 %0, 1, 0, p;\n\t}\n"
                 : "=r"(done) : "r"(su32(b)), "r"(phase), "n"(1000000) : "memory");
}
__device__ __forceinline__ void bulk_g2s(void* dst, const void* src, uint32_t bytes, uint64_t* bar) {
  asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];"
               ::"r"(su32(dst)), "l"(src), "r"(bytes), "r"(su32(bar)) : "memory");
}
__device__ __forceinline__ void tc_fence_before() { asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory"); }
__device__ __forceinline__ void tc_fence_after() { asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory"); }

// K-major, no swizzle: 8-row x 16-byte core matrices laid out [row group][k half][8 rows][16 B]
__host__ __device__ __forceinline__ int kmaj(int r, int kb) {
  return (r >> 3) * 256 + (kb >> 4) * 128 + (r & 7) * 16 + (kb & 15);
}

// shared-memory matrix descriptor: LBO (k-half stride) 128 B, SBO (row-group stride) 256 B,
// descriptor version 1, no swizzle
__device__ __forceinline__ uint64_t sdesc(const void* p) {
  return (uint64_t)((su32(p) >> 4) & 0x3FFF) | ((uint64_t)(128 >> 4) << 16) |
         ((uint64_t)(256 >> 4) << 32) | ((uint64_t)1 << 46);
}

// Issued by a whole convergent warp; elect.sync picks the one thread that issues, which keeps the
// compiler from wrapping every MMA in a per-thread serialisation loop.
template <uint32_t kIdesc>
__device__ __forceinline__ void mma_i8(uint32_t d, uint32_t a_tmem, uint64_t b, uint32_t acc) {
  asm volatile("{\n\t.reg .pred p, e;\n\telect.sync _|e, 0xffffffff;\n\tsetp.ne.b32 p, %3, 0;\n\t"
               "@e tcgen05.mma.cta_group::1.kind::i8 [%0], [%1], %2, %4, p;\n\t}\n"
               ::"r"(d), "r"(a_tmem), "l"(b), "r"(acc), "n"(kIdesc));
}
__device__ __forceinline__ void tc_commit_warp(uint64_t* bar) {
  asm volatile("{\n\t.reg .pred e;\n\telect.sync _|e, 0xffffffff;\n\t"
               "@e tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];\n\t}\n"
               ::"r"(su32(bar)) : "memory");
}
// s32 accumulate, A (candidate digits) unsigned, B (matrix digits) signed, both K-major, M = 128
template <int N>
constexpr uint32_t idesc_i8() {
  return (2u << 4) | (0u << 7) | (1u << 10) | ((uint32_t)(N >> 3) << 17) | ((uint32_t)(128 >> 4) << 24);
}

__device__ __forceinline__ void tmem_ld8(uint32_t addr, uint32_t (&v)[8]) {
  asm volatile("tcgen05.ld.sync.aligned.32x32b.x8.b32 {%0,%1,%2,%3,%4,%5,%6,%7}, [%8];"
               : "=r"(v[0]), "=r"(v[1]), "=r"(v[2]), "=r"(v[3]), "=r"(v[4]), "=r"(v[5]), "=r"(v[6]),
                 "=r"(v[7])
               : "r"(addr));
}

// role timeline of CTA 0 for BX_TC_TRACE: [role][4096][clock, code << 16 | sub]
#define TC_TRACE(role, code, sub)                                                          \
  do {                                                                                     \
    if (ta.trace && blockIdx.x == 0 && tr_n < 4096) {                                      \
      ta.trace[((role) * 4096 + tr_n) * 2] = clock64();                                    \
      ta.trace[((role) * 4096 + tr_n) * 2 + 1] = ((long long)(code) << 16) | (long long)(sub); \
      ++tr_n;                                                                              \
    }                                                                                      \
  } while (0)

// sigma * matern52(sqrt(W)) * kscale rounded to a 40-bit integer (the producers' hot path), in 14
// FP64 operations: d = sqrt(W) from rsqrt.approx + one Newton step on d (the 1/2 folded into the
// exponent of the approximation, an integer op); e^(-sqrt5 d) as 2^(k/256) (256-entry table, k
// clamped so the exponent stays normal; such K* round to 0) times a degree-3 Taylor polynomial.
// The range reduction runs in units of d (r = d + k ln2 / (256 sqrt5), |sqrt5 r| <= ln2/512), so
// -sqrt5 is folded into the polynomial coefficients instead of a multiply.  Accuracy is sized to the
// 2^-40 fixed point, not to FP64: the one-constant reduction leaves <= 5e-15 and the dropped r^4
// term <= 1.4e-13 of K* (0.15 of the fixed-point quantum; the round-to-nearest is 0.5 of it).
__device__ __forceinline__ unsigned long long kstar_fixed(double W, const MaternConst& m, const double* tab256) {
  const double w = W + 1e-300;                      // W = 0 -> d = 1e-150, K* = sigma
  const double y0 = rsqrt_approx(w);
  const double y0h = __hiloint2double(__double2hiint(y0) - (1 << 20), __double2loint(y0));  // y0 / 2
  const double d0 = w * y0;
  const double e0h = fma(-d0, y0h, 0.5);            // (1 - w y0^2) / 2
  const double d = fma(d0, e0h, d0);                // d0 (1 + e0 / 2)
  const double t = fma(d, -825.8468306507675, 6755399441055744.0);  // -d sqrt5 256 / ln2 + 1.5 * 2^52
  const int k = max(__double2loint(t), -256 * 900);
  const double kf = t - 6755399441055744.0;
  const double r = fma(kf, 0.00121087829230028, d);  // ln2 / (256 sqrt5)
  double p = fma(r, -1.8633899812498247, 2.5);       // e^(-sqrt5 r): -5 sqrt5/6, 5/2, -sqrt5, 1
  p = fma(r, p, -2.23606797749979);
  p = fma(r, p, 1.0);
  const double tj = tab256[k & 255];
  const double scale = __hiloint2double(__double2hiint(tj) + ((k >> 8) << 20), __double2loint(tj));
  // + 2^52: the 40-bit fixed-point value (rounded to nearest) lands in the low mantissa bits, so the
  // last multiply is an FMA and no FP64 -> integer conversion is needed
  const double X = fma(fma(m.s2, W, fma(m.s1, d, m.s0)), p * scale, 4503599627370496.0);
  return (unsigned long long)__double_as_longlong(X) & 0xFFFFFFFFFFull;
}

// FP64 tensor-core MMA m8n8k4: lane holds A[lane/4][lane%4], B[lane%4][lane/4], C[lane/4][2(lane%4)+{0,1}]
__device__ __forceinline__ void dmma884(double& d0, double& d1, double a, double b) {
  asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};"
               : "+d"(d0), "+d"(d1) : "d"(a), "d"(b));
}
// 16 TMEM lanes x 8 columns, the mma C-fragment layout: thread t writes lanes t/4 and t/4 + 8,
// columns 2 (t%4) and 2 (t%4) + 1 (v = {lane t/4: col, col+1; lane t/4+8: col, col+1})
__device__ __forceinline__ void tmem_st_16x256(uint32_t addr, uint32_t v0, uint32_t v1, uint32_t v2, uint32_t v3) {
  asm volatile("tcgen05.st.sync.aligned.16x256b.x1.b32 [%0], {%1,%2,%3,%4};" ::"r"(addr), "r"(v0), "r"(v1),
               "r"(v2), "r"(v3) : "memory");
}
__device__ __forceinline__ void tmem_st1(uint32_t addr, uint32_t v0) {
  asm volatile("tcgen05.st.sync.aligned.32x32b.x1.b32 [%0], {%1};" ::"r"(addr), "r"(v0) : "memory");
}
__device__ __forceinline__ void tmem_st4(uint32_t addr, const uint32_t* v) {
  asm volatile("tcgen05.st.sync.aligned.32x32b.x4.b32 [%0], {%1,%2,%3,%4};" ::"r"(addr), "r"(v[0]), "r"(v[1]),
               "r"(v[2]), "r"(v[3]) : "memory");
}
__device__ __forceinline__ void tmem_st2(uint32_t addr, uint32_t v0, uint32_t v1) {
  asm volatile("tcgen05.st.sync.aligned.32x32b.x2.b32 [%0], {%1,%2};" ::"r"(addr), "r"(v0), "r"(v1) : "memory");
}

struct TcLayout {
  int par, planes, kmask, cval, cmask, exp2, cw, rowscale, yy, rows, pk, stab, emb, emb_tab, mat, bars, total;
};

// (chunk c, slice ks <= min(c / 2, nsl - 1)) blocks of the lower triangle, chunk-major: index of
// chunk c's first block, and the total for nch chunks
__host__ __device__ __forceinline__ int tc_block0(int c, int nsl) {
  int o = 0;
  for (int i = 0; i < c; ++i) o += min(i >> 1, nsl - 1) + 1;
  return o;
}

// ks > 0 (tensor-core distances): the planes hold the B operand (4 ks rows), the candidate buffer
// the tile's E embedding coordinates plus |x'|^2 (one buffer: the producers copy their A fragments
// into registers at the start of a tile and release it).  ks == 0: per-parameter planes and
// candidate values, double-buffered (the FMA producers read them for every slice).
// pp (per-pass planes, n > 255 when the whole-width planes do not fit): the planes / Kendall masks /
// |y'|^2 hold only the current pass's 256 columns and the producers reload them every pass.
__host__ __device__ inline TcLayout tc_layout(int n, int n_params, int n_kendall, int words, int ks, int n_emb,
                                              int emb_tab_len, bool aug, bool resident, bool pp,
                                              int stages = kStages, int pk_bytes = 0) {
  const int nsl = (n + 31) / 32, nch = n / kN + 1;
  const int npad = pp ? 32 * kSlots : 32 * nsl;  // columns held in shared memory
  TcLayout L;
  int off = 0;
  L.par = off;
  off += n_params * (int)sizeof(bx_param_desc);
  off = (off + 15) & ~15;
  L.planes = off;  // ks > 0: row stride npad + 4 doubles (the B-fragment loads are conflict-free)
  off += (ks > 0 ? 4 * ks * (npad + 4) : n_params * npad) * 8;
  off = (off + 15) & ~15;
  L.kmask = off;   // [n_kendall][npad][2]
  off += ks > 0 ? 0 : n_kendall * npad * 16;
  L.cval = off;    // ks > 0: [E][kM + 1] (odd row stride: conflict-free decoder stores)
  off += ks > 0 ? n_emb * (kM + 1) * 8 : 2 * n_params * kM * 8;
  off = (off + 15) & ~15;
  L.cmask = off;   // [2][n_kendall][128][2] candidate Kendall masks
  off += ks > 0 ? 0 : 2 * n_kendall * kM * 16;
  L.exp2 = off;    // 2^(j/256), j < 256
  off += 256 * 8;
  L.cw = off;      // [n_params] permutation weight per raw unit: 1 / l^2 / raw_mx
  off += ks > 0 ? 0 : ((n_params + 1) & ~1) * 8;
  L.rowscale = off;  // [2][16 nch]: row factors, then the same with the alpha / padding rows zeroed
  off += 2 * nch * kN * 8;
  L.yy = off;        // [npad] |y'|^2 (ks > 0 without the augmented rows)
  off += (ks > 0 && !aug) ? npad * 8 : 0;
  L.rows = off;      // [128 x row_words] encoded rows of the next tile (bulk-copy staging)
  off += ((kM * words * 4) + 15) & ~15;
  L.pk = off;        // pk_bytes > 0: [128 x packed words] a tile's packed rows (TcArgs.pk_sep)
  off += (pk_bytes + 15) & ~15;
  L.stab = off;      // coord_lut / lengthscale of the finite numeric domains (FMA producers)
  off += ks > 0 ? 0 : kMaxCoord * 8;
  L.emb = off;
  off += ks > 0 ? ((n_emb * (int)sizeof(EmbDim) + 15) & ~15) : 0;
  L.emb_tab = off;
  off += ks > 0 ? emb_tab_len * 8 : 0;
  off = (off + 1023) & ~1023;
  L.mat = off;     // [stage][digit][16 x 32 B], or every block of the triangle when resident
  off += (resident ? tc_block0(nch, nsl) : stages) * kMatBlock;
  L.bars = off;    // cand_full, slice_empty[8], mat_full/empty[8], acc_full/empty[2], rows_full/empty, cval_full/free[2], tmem
  off += (1 + kSlots + 2 * kMaxStages + 4 + 2 + 4 + 1) * 8;
  L.total = off;
  return L;
}

// KS > 0: tensor-core (DMMA) distances over the embedding with KS k-steps; KS == 0: FMA distances.
// kMulti: n > 255, several column passes per tile (a separate instance: the one-pass kernel carries
// none of the parking / per-pass planes code).
template <bool kPrecise, int KS, bool kMulti>
__global__ void __launch_bounds__((tc_threads<KS>()), 1) gp_tc_kernel(TcArgs ta) {
  constexpr bool kDmma = KS > 0;
  constexpr int kProdWarps = tc_prod_warps<KS>();
  constexpr int kColsPerItem = 32 / (kProdWarps / 4);  // columns of a slice per FMA producer thread
  extern __shared__ __align__(1024) unsigned char smem[];
  const FusedArgs& a = ta.f;
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  const int n = a.gp.n, n_params = a.space.n_params, words = a.space.row_words;
  const int nsl = ta.n_slices, nch = ta.n_chunks, npad = 32 * nsl;
  const int npass = kMulti ? tc_passes(nsl) : 1;
  const bool pp = kMulti && ta.planes_pp != 0;  // per-pass planes (tc_layout)
  const int nst = ta.mat_stages;                 // matrix ring stages (not resident)
  const int ppad = pp ? 32 * kSlots : npad;  // columns of the planes in shared memory
  const int E = ta.n_emb;
  constexpr int kCvs = kM + 1;        // DMMA mode: candidate-buffer row stride (doubles)
  const int pls = ppad + 4;           // DMMA mode: planes row stride (doubles)
  const bool resident = ta.mat_resident != 0;
  const TcLayout L = tc_layout(n, n_params, a.n_kendall, words, KS, E, ta.emb_tab_len, ta.aug != 0, resident, pp, nst,
                               ta.pk_sep ? kM * ta.pack.pw * 4 : 0);
  bx_param_desc* params = reinterpret_cast<bx_param_desc*>(smem + L.par);
  uint64_t* planes = reinterpret_cast<uint64_t*>(smem + L.planes);
  uint64_t* kmask = reinterpret_cast<uint64_t*>(smem + L.kmask);
  uint64_t* cval = reinterpret_cast<uint64_t*>(smem + L.cval);
  uint64_t* cmask = reinterpret_cast<uint64_t*>(smem + L.cmask);
  double* s_exp2 = reinterpret_cast<double*>(smem + L.exp2);
  double* s_cw = reinterpret_cast<double*>(smem + L.cw);
  double* rowscale = reinterpret_cast<double*>(smem + L.rowscale);
  double* rowscale_ss = rowscale + nch * kN;
  double* s_yy = reinterpret_cast<double*>(smem + L.yy);
  EmbDim* s_emb = reinterpret_cast<EmbDim*>(smem + L.emb);
  double* s_etab = reinterpret_cast<double*>(smem + L.emb_tab);
  unsigned char* mat = smem + L.mat;
  uint64_t* bars = reinterpret_cast<uint64_t*>(smem + L.bars);
  uint64_t* cand_full = bars;
  uint64_t* slice_empty = bars + 1;
  uint64_t* mat_full = slice_empty + kSlots;
  uint64_t* mat_empty = mat_full + kMaxStages;
  uint64_t* acc_full = mat_empty + kMaxStages;
  uint64_t* acc_empty = acc_full + 2;
  uint64_t* rows_full = acc_empty + 2;   // the staging buffer holds the next tile's rows
  uint64_t* rows_empty = rows_full + 1;  // the decoders are done with them
  uint64_t* cval_full = rows_empty + 1;  // [2] the decoders filled a tile's candidate values
  uint64_t* cval_free = cval_full + 2;   // [2] every producer is done with them
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(cval_free + 2);
  uint32_t* rowsbuf = reinterpret_cast<uint32_t*>(smem + L.rows);
  // pk_sep: packed rows land in their own buffer, released as soon as the decoders hold them in
  // registers, so the prefetcher fetches the next tile (over the bus, for a zero-copy host pool)
  // while this one is being decoded; else they land at the end of the staging buffer
  uint32_t* pkbuf = reinterpret_cast<uint32_t*>(smem + L.pk);
  const bool pk_sep = ta.pk_sep != 0;
  // rows are staged by 16-byte bulk copies when the pool pointer allows it
  const bool stage_rows = (reinterpret_cast<uintptr_t>(a.rows) & 15) == 0;

  for (int i = tid; i < n_params * (int)sizeof(bx_param_desc) / 4; i += blockDim.x)
    reinterpret_cast<int32_t*>(params)[i] = reinterpret_cast<const int32_t*>(a.space.params)[i];
  // the planes (DMMA: B operand and |y'|^2; FMA: per-parameter training values and Kendall masks)
  // of columns c0 .. c0 + ppad - 1
  auto load_planes = [&](int c0, int i0, int step) {
    if constexpr (kDmma) {
      for (int i = i0; i < 4 * KS * ppad; i += step) {
        const int k = i / ppad, j = c0 + i % ppad;
        planes[k * pls + i % ppad] = j < npad ? (uint64_t)__double_as_longlong(ta.emb_planes[(size_t)k * npad + j]) : 0;
      }
      if (!ta.aug)
        for (int i = i0; i < ppad; i += step) s_yy[i] = c0 + i < npad ? ta.emb_yy[c0 + i] : 0.0;
    } else {
      for (int i = i0; i < n_params * ppad; i += step) {
        const int k = i / ppad, j = c0 + i % ppad;
        planes[i] = j < n ? a.gp.planes[(size_t)k * n + j] : 0;
      }
      for (int i = i0; i < a.n_kendall * ppad; i += step) {
        const int kk = i / ppad, j = c0 + i % ppad;
        const size_t src = ((size_t)a.kendall_param[kk] * n + j) * 2;
        kmask[2 * i] = j < n ? a.gp.kmask[src] : 0;
        kmask[2 * i + 1] = j < n ? a.gp.kmask[src + 1] : 0;
      }
    }
  };
  if (!pp) load_planes(0, tid, blockDim.x);  // pp: the producers load each pass's columns
  if constexpr (kDmma) {
    for (int i = tid; i < E * (int)sizeof(EmbDim) / 4; i += blockDim.x)
      reinterpret_cast<int32_t*>(s_emb)[i] = reinterpret_cast<const int32_t*>(ta.emb)[i];
    for (int i = tid; i < ta.emb_tab_len; i += blockDim.x) s_etab[i] = ta.emb_tab[i];
  } else {
    for (int k = tid; k < n_params; k += blockDim.x)
      s_cw[k] = a.space.params[k].kind == BX_PERMUTATION ? a.gp.inv_l2[k] / a.space.params[k].raw_mx : 0.0;
  }
  for (int i = tid; i < 256; i += blockDim.x) s_exp2[i] = ta.exp2tab256[i];
  // finite numeric coordinates pre-divided by the lengthscale: decode = two shared loads
  double* stab = reinterpret_cast<double*>(smem + L.stab);
  const bool use_stab = !kDmma && ta.n_coord <= kMaxCoord;
  if (use_stab)
    for (int k = 0; k < n_params; ++k) {
      const bx_param_desc& p = a.space.params[k];
      if (p.kind == BX_REAL || p.kind == BX_CATEGORICAL || p.kind == BX_PERMUTATION) continue;
      for (int d = tid; d < p.size; d += blockDim.x) stab[p.coord + d] = a.space.coord_lut[p.coord + d] * a.gp.inv_l[k];
    }
  for (int i = tid; i < nch * kN; i += blockDim.x) {
    rowscale[i] = ta.rowscale[i];
    rowscale_ss[i] = i < n ? ta.rowscale[i] : 0.0;  // sum-of-squares rows: L^-1 only
  }
  if (tid == 0) {
    mb_init(cand_full, kProdWarps);
    for (int i = 0; i < kSlots; ++i) mb_init(&slice_empty[i], 1);
    for (int i = 0; i < nst; ++i) {
      mb_init(&mat_full[i], 1);
      mb_init(&mat_empty[i], 1);
    }
    for (int i = 0; i < 2; ++i) {
      mb_init(&acc_full[i], 1);
      mb_init(&acc_empty[i], 4);
      mb_init(&cval_full[i], 1);
      mb_init(&cval_free[i], kProdWarps);
    }
    mb_init(rows_full, 1);
    mb_init(rows_empty, 1);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  if (warp == 0) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(su32(tmem_slot)), "r"(512));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
  }
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = *tmem_slot;
  int tr_n = 0;
  const int64_t n_tiles = (a.q + kM - 1) / kM;
  const int my_tiles = (int)((n_tiles - blockIdx.x + gridDim.x - 1) / gridDim.x);

  // words of tile t's rows held in the staging buffer (the rest, if any, is read from global)
  auto staged_words = [&](int64_t tile) -> int {
    if (!stage_rows) return 0;
    const int64_t count = min((int64_t)kM, a.q - tile * kM);
    return (int)(((count * words * 4) & ~(int64_t)15) / 4);
  };
  // packed pools: the tile's packed rows are bulk-copied to the END of the staging buffer and the
  // decoders unpack them in place (every thread reads its packed rows before any full row is
  // written; full row c never overlaps a packed row c' > c)
  const int pw = ta.pack.pw;
  const int pk_off = (words - pw) * kM;  // words; a multiple of 4 (16-byte aligned)
  auto staged_packed = [&](int64_t tile) -> int {
    const int64_t count = min((int64_t)kM, a.q - tile * kM);
    return (int)(((count * pw * 4) & ~(int64_t)15) / 4);
  };

  if (warp == 2 || warp == 3) {
    // ---- decoders: the next tile's candidates into the candidate buffer --------------------------
    const int dt = tid - 64;  // 0..63
    for (int t = 0; t < my_tiles; ++t) {
      const int64_t tile = blockIdx.x + (int64_t)t * gridDim.x;
      const int buf = kDmma ? 0 : (t & 1);
      // the buffer's previous contents are released by every producer warp: at the start of tile
      // t - 1 (ks > 0: A fragments copied to registers), or at the end of tile t - 2 (FMA)
      if (kDmma ? t >= 1 : t >= 2)
        mb_wait_sleep(&cval_free[buf], (uint32_t)((kDmma ? (t - 1) : ((t - 2) >> 1)) & 1));
      mb_wait_sleep(rows_full, (uint32_t)(t & 1));
      int sw = staged_words(tile);
      if (ta.packed) {
        // unpack: packed rows (staged or, for a ragged tail, global) into full rows in the staging
        // buffer and to HBM (the forest / summary kernels read them)
        const int spw = staged_packed(tile);
        auto write_back = [&](const uint32_t* dstr, int64_t gi) {
          uint32_t* g = const_cast<uint32_t*>(a.rows) + (size_t)gi * words;
          if ((words & 3) == 0 && stage_rows) {  // 16-byte stores (16-byte aligned pool and rows)
            for (int w = 0; w < words; w += 4)
              *reinterpret_cast<uint4*>(g + w) = *reinterpret_cast<const uint4*>(dstr + w);
          } else {
            for (int w = 0; w < words; ++w) g[w] = dstr[w];
          }
        };
        if (pk_sep) {
          // packed rows in their own buffer: unpacked straight from it (or, for a ragged tail,
          // from global), then the buffer goes back to the prefetcher for the next tile
#pragma unroll
          for (int h2 = 0; h2 < 2; ++h2) {
            const int cc = dt + 64 * h2;
            const int64_t gi = tile * kM + cc;
            if (gi < a.q) {
              const uint32_t* src = (cc + 1) * pw <= spw ? pkbuf + cc * pw : ta.packed + (size_t)gi * pw;
              uint32_t* dstr = rowsbuf + cc * words;
              unpack_row(ta.pack, src, dstr, words);
              write_back(dstr, gi);
            }
          }
          asm volatile("bar.sync 3, 64;" ::: "memory");
          if (dt == 0) mb_arrive(rows_empty);  // the prefetcher may fetch the next tile now
        } else {
          // packed rows at the end of the staging buffer: every thread takes its packed rows into
          // registers before any full row overwrites them
          uint32_t pk[2][16];
#pragma unroll
          for (int h2 = 0; h2 < 2; ++h2) {
            const int cc = dt + 64 * h2;
            const int64_t gi = tile * kM + cc;
#pragma unroll
            for (int w = 0; w < 16; ++w) {
              const int o = cc * pw + w;
              pk[h2][w] = (w < pw && gi < a.q) ? (o < spw ? rowsbuf[pk_off + o] : ta.packed[(size_t)gi * pw + w]) : 0u;
            }
          }
          asm volatile("bar.sync 3, 64;" ::: "memory");
#pragma unroll
          for (int h2 = 0; h2 < 2; ++h2) {
            const int cc = dt + 64 * h2;
            const int64_t gi = tile * kM + cc;
            if (gi < a.q) {
              uint32_t* dstr = rowsbuf + cc * words;
              unpack_row(ta.pack, pk[h2], dstr, words);
              write_back(dstr, gi);
            }
          }
          asm volatile("bar.sync 3, 64;" ::: "memory");
        }
        sw = (int)(min((int64_t)kM, a.q - tile * kM) * words);  // every row is now staged
      }
      if constexpr (kDmma) {
        // thread = candidate (two per thread, every lane doing the same coordinate at a time: the
        // FP64 work of the permutation coordinates stays dense); the producers form |x'|^2
        for (int cc = dt; cc < kM; cc += 64) {
          const int64_t gi = tile * kM + cc;
          const uint32_t* rw = (cc + 1) * words <= sw ? rowsbuf + cc * words : a.rows + (size_t)gi * words;
          for (int e = 0; e < E; ++e)
            cval[e * kCvs + cc] = (uint64_t)__double_as_longlong(gi < a.q ? emb_value(s_emb[e], rw, s_etab) : 0.0);
        }
        asm volatile("bar.sync 3, 64;" ::: "memory");
        if (dt == 0) {
          if (!(ta.packed && pk_sep)) mb_arrive(rows_empty);
          mb_arrive(&cval_full[0]);
        }
        continue;
      }
      uint64_t* cv = cval + (size_t)buf * n_params * kM;
      for (int idx = dt; idx < n_params * kM; idx += 64) {
        const int k = idx / kM, cc = idx % kM;
        const int64_t gi = tile * kM + cc;
        const bx_param_desc& p = params[k];
        auto word = [&](int w) -> uint32_t {
          const int o = cc * words + w;
          return o < sw ? rowsbuf[o] : a.rows[(size_t)gi * words + w];
        };
        uint64_t v = 0;
        if (gi < a.q) {
          if (p.kind == BX_PERMUTATION) {
            v = (uint64_t)word(p.word) | ((uint64_t)word(p.word + 1) << 32);
          } else if (p.kind == BX_CATEGORICAL) {
            v = word(p.word);
          } else {
            double x;
            if (p.kind == BX_REAL)
              x = __longlong_as_double((long long)((uint64_t)word(p.word + 2) | ((uint64_t)word(p.word + 3) << 32))) *
                  a.gp.inv_l[k];
            else if (use_stab)
              x = stab[p.coord + (int)word(p.word)];
            else
              x = a.space.coord_lut[p.coord + (int)word(p.word)] * a.gp.inv_l[k];
            v = (uint64_t)__double_as_longlong(x);
          }
        }
        cv[idx] = v;
      }
      asm volatile("bar.sync 3, 64;" ::: "memory");
      if (dt == 0 && !(ta.packed && pk_sep)) mb_arrive(rows_empty);
      uint64_t* cm = cmask + (size_t)buf * a.n_kendall * kM * 2;
      for (int idx = dt; idx < a.n_kendall * kM; idx += 64) {
        const int kk = idx / kM, cc = idx % kM;
        const bx_param_desc& p = params[a.kendall_param[kk]];
        uint64_t lo = 0, hi = 0;
        kendall_mask(cv[a.kendall_param[kk] * kM + cc], p.size, lo, hi);
        cm[2 * idx] = lo;
        cm[2 * idx + 1] = hi;
      }
      asm volatile("bar.sync 3, 64;" ::: "memory");
      if (dt == 0) mb_arrive(&cval_full[buf]);
    }
  } else if (warp == 1 && lane == 1) {
    // ---- row prefetcher: the encoded rows of each tile, one bulk copy ahead ----------------
    for (int t = 0; t < my_tiles; ++t) {
      const int64_t tile = blockIdx.x + (int64_t)t * gridDim.x;
      if (t >= 1) mb_wait_sleep(rows_empty, (uint32_t)((t - 1) & 1));
      if (ta.ready) {  // streaming pool: wait until the copy stream has landed this tile's chunk
        const int64_t last = min(a.q, (tile + 1) * kM) - 1;
        const uint32_t* flag = ta.ready + (last >> ta.ready_shift);
        uint32_t ok = 0;
        for (long long spins = 0;; ++spins) {
          asm volatile("ld.acquire.gpu.global.u32 %0, [%1];" : "=r"(ok) : "l"(flag) : "memory");
          if (ok) break;
          if (spins > (1ll << 26)) asm volatile("trap;");  // ~20 s without the chunk: fail loudly
          __nanosleep(256);
        }
        asm volatile("fence.proxy.async.global;" ::: "memory");  // make the data visible to TMA
      }
      const int sw = ta.packed ? staged_packed(tile) : staged_words(tile);
      if (sw > 0) {
        mb_expect(rows_full, (uint32_t)sw * 4);
        if (ta.packed)
          bulk_g2s(pk_sep ? pkbuf : rowsbuf + pk_off, ta.packed + (size_t)tile * kM * pw, (uint32_t)sw * 4, rows_full);
        else
          bulk_g2s(rowsbuf, a.rows + (size_t)tile * kM * words, (uint32_t)sw * 4, rows_full);
      } else {
        mb_arrive(rows_full);
      }
    }
  } else if (warp == 1 && lane == 0) {
    // ---- TMA producer: matrix digit blocks in MMA consumption order ------------------------
    if (resident) {  // the whole triangle once, on one barrier
      const int nb = tc_block0(nch, nsl);
      if (my_tiles > 0) {
        mb_expect(&mat_full[0], (uint32_t)(nb * kMatBlock));
        for (int c = 0; c < nch; ++c)
          for (int ks = 0; ks <= min(c >> 1, nsl - 1); ++ks)
            bulk_g2s(mat + (size_t)(tc_block0(c, nsl) + ks) * kMatBlock, ta.mdig + ((size_t)c * nsl + ks) * kMatBlock,
                     kMatBlock, &mat_full[0]);
      }
    } else {
      uint32_t ph = 0;  // parity bit per stage
      int s = 0, issued = 0;
      for (int t = 0; t < my_tiles; ++t)
        for (int p = 0; p < npass; ++p)
        for (int c = nch - 1; c >= 2 * kSlots * p; --c)
          for (int ks = kSlots * p; ks <= min(c >> 1, min(nsl, kSlots * (p + 1)) - 1); ++ks) {
            if (issued >= nst) {
              mb_wait_sleep(&mat_empty[s], (ph >> s) & 1u);
              ph ^= 1u << s;
            }
            TC_TRACE(3, 1, c * 16 + ks);
            mb_expect(&mat_full[s], kMatBlock);
            bulk_g2s(mat + (size_t)s * kMatBlock, ta.mdig + ((size_t)c * nsl + ks) * kMatBlock, kMatBlock,
                     &mat_full[s]);
            ++issued;
            s = (s + 1 == nst) ? 0 : s + 1;
          }
    }
  } else if (warp == 0) {
    // ---- MMA issuer (whole warp, one elected thread issues) ---------------------------------
    // The B tile of a (chunk, slice) block stacks the six matrix digits (6 x 16 rows), so one MMA
    // per candidate digit b covers every group t = a + b <= 5 at once: N = (6 - b) * 16 rows
    // starting at matrix digit 0, accumulated at TMEM column b * 16 (group-major accumulator).
    const uint64_t bdesc0 = sdesc(mat);
    uint32_t ph_m = 0, ph_e = 0, ph_c = 0;  // parity bits per stage / accumulator
    int s = 0, chunk_no = 0;
    for (int t = 0; t < my_tiles; ++t)
    for (int p = 0; p < npass; ++p) {
      const int lo = kSlots * p, hi = min(nsl, kSlots * (p + 1));  // this pass's column slices
      const int soff = p == 0 ? 0 : kSlots - (hi - lo);  // pass 1 takes the slots pass 0 frees first
      if (lane == 0) TC_TRACE(1, 1, t);
      mb_wait_sleep(cand_full, ph_c);
      ph_c ^= 1u;
      tc_fence_after();
      if (lane == 0) TC_TRACE(1, 2, t);
      for (int c = nch - 1; c >= 2 * kSlots * p; --c, ++chunk_no) {
        const int buf = chunk_no & 1;
        if (chunk_no >= 2) {
          mb_wait(&acc_empty[buf], (ph_e >> buf) & 1u);
          ph_e ^= 1u << buf;
          tc_fence_after();
        }
        const uint32_t dbase = tmem + (uint32_t)(buf * kAccCols);
        const int b0 = resident ? tc_block0(c, nsl) : 0;
        for (int ks = lo; ks <= min(c >> 1, hi - 1); ++ks) {
          if (!resident || chunk_no == 0) {  // resident: the one load, before the first chunk
            mb_wait_sleep(&mat_full[resident ? 0 : s], resident ? 0u : (ph_m >> s) & 1u);
            if (!resident) ph_m ^= 1u << s;
            tc_fence_after();
          }
          const uint64_t bd = bdesc0 + (uint64_t)(((resident ? b0 + ks : s) * kMatBlock) >> 4);
          const uint32_t at = tmem + (uint32_t)(kDigCol0 + (ks - lo + soff) * kSliceCols);
          const uint32_t acc = ks > lo ? 1u : 0u;
          if (!(ta.debug & 2)) {
            mma_i8<idesc_i8<6 * kN>()>(dbase, at, bd, acc);
            mma_i8<idesc_i8<5 * kN>()>(dbase + 1 * kN, at + 1 * 8, bd, 1u);
            mma_i8<idesc_i8<4 * kN>()>(dbase + 2 * kN, at + 2 * 8, bd, 1u);
            mma_i8<idesc_i8<3 * kN>()>(dbase + 3 * kN, at + 3 * 8, bd, 1u);
            mma_i8<idesc_i8<2 * kN>()>(dbase + 4 * kN, at + 4 * 8, bd, 1u);
          }
          if (!resident) {
            tc_commit_warp(&mat_empty[s]);  // the stage is free once these MMAs retire
            s = (s + 1 == nst) ? 0 : s + 1;
          }
        }
        tc_commit_warp(&acc_full[buf]);
        // chunk c is the last reader of slice c / 2 (slot c / 2 - lo) when c is even (chunks run
        // downwards)
        if (!(c & 1) && (c >> 1) >= lo && (c >> 1) < hi) tc_commit_warp(&slice_empty[(c >> 1) - lo + soff]);
        if (lane == 0) TC_TRACE(1, 3, c);
      }
    }
  } else if (warp >= 4 && warp < 8) {
    // ---- epilogue: thread = candidate = TMEM lane ------------------------------------------
    const int r = (warp - 4) * 32 + lane;
    const uint32_t lane_base = (uint32_t)((warp - 4) * 32) << 16;
    const double sigma = a.gp.outputscale;
    uint32_t ph_f = 0;
    int chunk_no = 0;
    for (int t = 0; t < my_tiles; ++t) {
      const int64_t tile = blockIdx.x + (int64_t)t * gridDim.x;
      double ss = 0.0, ss1 = 0.0, mean_s = 0.0;
      for (int p = 0; p < npass; ++p)
      for (int c = nch - 1; c >= 2 * kSlots * p; --c, ++chunk_no) {
        // several passes (n > 255): a row >= 256 parks its partial sum in this CTA's scratch
        // ([16 nch - 256 rows][128 candidates], coalesced per row) until its last pass.  mode 0:
        // complete in this pass, 1: park, 3: add to the parked sum, 2: last pass, add it back.
        const int last = min(npass - 1, c / (2 * kSlots));
        const int mode = last == 0 ? 0 : (p == 0 ? 1 : (p < last ? 3 : 2));
        double* park = mode ? ta.part + (size_t)blockIdx.x * (kN * nch - kSlots * 32) * kM + r : nullptr;  // + (row - 256) * kM
        const int buf = chunk_no & 1;
        // parked, not spinning: measured the same at M200 / C3 and leaves the issue slots to the
        // producers sharing the sub-partition
        mb_wait_sleep(&acc_full[buf], (ph_f >> buf) & 1u);
        ph_f ^= 1u << buf;
        tc_fence_after();
        if (lane == 0 && warp == 4) TC_TRACE(2, 1, c);
        const uint32_t base = tmem + lane_base + (uint32_t)(buf * kAccCols);
        // exact int64 recombination of the six digit groups of row kN c + r0 + j
        auto recombine = [&](const uint32_t (&g)[kGroups][8], int j) -> double {
          long long Z = (long long)(int32_t)g[0][j] << 40;
          Z += (long long)(int32_t)g[1][j] << 32;
          Z += (long long)(int32_t)g[2][j] << 24;
          Z += (long long)(int32_t)g[3][j] << 16;
          Z += (long long)(int32_t)g[4][j] << 8;
          Z += (long long)(int32_t)g[5][j];
          return (double)Z;
        };
        // one loop per parking mode (uniform per chunk): the parked sums of a group of 8 rows are
        // loaded together with its TMEM reads
        auto drain = [&](auto mode_c) {
          constexpr int kMode = decltype(mode_c)::value;
          for (int r0 = 0; r0 < kN && kN * c + r0 <= n && !(ta.debug & 1); r0 += 8) {
            uint32_t g[kGroups][8];
#pragma unroll
            for (int q = 0; q < kGroups; ++q) tmem_ld8(base + (uint32_t)(q * kN + r0), g[q]);
            double prev[8];
            if constexpr (kMode >= 2) {
#pragma unroll
              for (int j = 0; j < 8; ++j) prev[j] = park[(size_t)(kN * c + r0 + j - kSlots * 32) * kM];
            }
            asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
#pragma unroll
            for (int j = 0; j < 8; ++j) {
              if (ta.debug & 4) break;  // timing experiment: TMEM reads only
              const int row = kN * c + r0 + j;
              double zd = recombine(g, j);
              if constexpr (kMode == 1 || kMode == 3) {  // park: first pass / running sum of the passes
                park[(size_t)(row - kSlots * 32) * kM] = kMode == 3 ? prev[j] + zd : zd;
              } else {
                if constexpr (kMode == 2) zd += prev[j];  // last pass: add the parked sum back
                const double v = zd * rowscale_ss[row];  // 0 for the alpha row and the padding rows
                // (several passes: two independent FMA chains measure faster, one pass: one chain)
                if (kMulti && (j & 1)) ss1 = fma(v, v, ss1); else ss = fma(v, v, ss);
                if (row == n) mean_s = zd * rowscale[row];  // only in the alpha row's chunk
              }
            }
          }
        };
        if constexpr (kMulti) {
          switch (mode) {
            case 1: drain(std::integral_constant<int, 1>{}); break;
            case 2: drain(std::integral_constant<int, 2>{}); break;
            case 3: drain(std::integral_constant<int, 3>{}); break;
            default: drain(std::integral_constant<int, 0>{}); break;
          }
        } else {
          drain(std::integral_constant<int, 0>{});  // every row completes in its one pass
        }
        tc_fence_before();
        __syncwarp();
        if (lane == 0) mb_arrive(&acc_empty[buf]);
        if (lane == 0 && warp == 4) TC_TRACE(2, 2, c);
      }
      const int64_t gi = tile * kM + r;
      if constexpr (kMulti) ss += ss1;
      if (gi < a.q) {
        const double var_s = fmax(sigma - ss, 0.0);                 // surrogate.py:324-325
        const double mean = a.gp.y_mean + a.gp.y_std * mean_s;      // :328
        const double var = (a.gp.y_std * a.gp.y_std) * var_s;
        if (a.mean_out) a.mean_out[gi] = mean;
        if (a.var_out) a.var_out[gi] = var;
        if (a.ei_out) a.ei_out[gi] = ei_value(mean, var, a.f_model);  // acquisition.py:40-51
      }
    }
  } else if (kDmma && warp >= 8) {
    // ---- K* producers, FP64 tensor-core distances over the embedding -----------------------------
    // Warp (quarter q, half h) owns candidates 32 q + 16 h + 0..15 (TMEM lanes of its quarter) and
    // every column of a slice.  W = |x'|^2 + |y'|^2 + x'.(-2 y') is one product of the candidate
    // embedding [x', 1, |x'|^2] and the training operand [-2 y'; |y'|^2; 1] on DMMA m8n8k4 (2 row
    // blocks x 4 column blocks x KS k-steps per slice; without room for the two augmented k-rows
    // |x'|^2 + |y'|^2 is added to the fragments); the Matérn runs on the C fragments and the digits
    // go to TMEM with the matching 16x256b store.  Within a slice the K order is permuted so that
    // each thread's C columns are 8 consecutive K bytes: K byte 8 t0 + 4 hh + 2 jj + e <- column
    // 8 (2 hh + jj) + 2 t0 + e (mdig_kernel builds the matrix digits with the same permutation).
    const int pt = tid - 8 * 32;
    const int quarter = warp & 3, half = (warp - 8) >> 2;
    const int t0 = lane & 3, t1 = lane >> 2;
    const uint32_t lane_base = (uint32_t)(quarter * 32 + half * 16) << 16;
    const double sigma = a.gp.outputscale;
    const MaternConst mc{sigma * ta.kscale, sigma * kSqrt5 * ta.kscale, sigma * (5.0 / 3.0) * ta.kscale};
    const bool aug = ta.aug != 0;
    uint32_t slot_used = 0, slot_par = 0;
    for (int t = 0; t < my_tiles; ++t) {
      if (pt == 0) TC_TRACE(0, 1, t);
      mb_wait_sleep(&cval_full[0], (uint32_t)(t & 1));  // parked: the decoders need the issue slots
      if (pt == 0) TC_TRACE(0, 2, t);
      // A fragments: row = candidate 32 q + 16 h + 8 rb + t1, k = t0 + 4 kk of [x', 1, |x'|^2, 0..];
      // |x'|^2 summed over the four lanes t0 that hold the candidate's coordinates
      double afr[2][KS > 0 ? KS : 1], xx[2];
#pragma unroll
      for (int rb = 0; rb < 2; ++rb) {
        const int c = quarter * 32 + half * 16 + 8 * rb + t1;
        xx[rb] = 0.0;
#pragma unroll
        for (int kk = 0; kk < KS; ++kk) {
          const int k = t0 + 4 * kk;
          afr[rb][kk] = k < E ? __longlong_as_double((long long)cval[k * kCvs + c]) : 0.0;
          xx[rb] = fma(afr[rb][kk], afr[rb][kk], xx[rb]);
        }
        xx[rb] += __shfl_xor_sync(0xffffffffu, xx[rb], 1);
        xx[rb] += __shfl_xor_sync(0xffffffffu, xx[rb], 2);
        if (aug)
#pragma unroll
          for (int kk = 0; kk < KS; ++kk) {
            const int k = t0 + 4 * kk;
            if (k == E) afr[rb][kk] = 1.0;
            if (k == E + 1) afr[rb][kk] = xx[rb];
          }
      }
      __syncwarp();
      if (lane == 0) mb_arrive(&cval_free[0]);  // the decoders may write the next tile
      for (int p = 0; p < npass; ++p) {
      const int lo = kSlots * p, hi = min(nsl, kSlots * (p + 1));
      const int soff = p == 0 ? 0 : kSlots - (hi - lo);
      if (pp) {  // every producer is done with the previous pass's columns; load this pass's
        asm volatile("bar.sync 4, %0;" ::"r"(kProdWarps * 32) : "memory");
        load_planes(32 * lo, pt, kProdWarps * 32);
        asm volatile("bar.sync 4, %0;" ::"r"(kProdWarps * 32) : "memory");
      }
      for (int ks = hi - 1; ks >= lo; --ks) {
        const int slot = ks - lo + soff;
        const int j0 = 32 * (pp ? ks - lo : ks);  // column of the slice in the planes
        double acc[2][4][2];
#pragma unroll
        for (int rb = 0; rb < 2; ++rb)
#pragma unroll
          for (int j = 0; j < 4; ++j) acc[rb][j][0] = acc[rb][j][1] = 0.0;
#pragma unroll
        for (int kk = 0; kk < KS; ++kk) {
          const double* brow = reinterpret_cast<const double*>(planes) + (size_t)(t0 + 4 * kk) * pls + j0 + t1;
#pragma unroll
          for (int j = 0; j < 4; ++j) {
            const double b = brow[8 * j];  // B[k = t0 + 4 kk][column 8 j + t1]
            dmma884(acc[0][j][0], acc[0][j][1], afr[0][kk], b);
            dmma884(acc[1][j][0], acc[1][j][1], afr[1][kk], b);
          }
        }
        if (!aug) {  // uniform branch: |x'|^2 + |y'|^2 added to the C fragments
#pragma unroll
          for (int j = 0; j < 4; ++j) {
            const double2 y = *reinterpret_cast<const double2*>(s_yy + j0 + 8 * j + 2 * t0);
#pragma unroll
            for (int rb = 0; rb < 2; ++rb) {
              acc[rb][j][0] += xx[rb] + y.x;
              acc[rb][j][1] += xx[rb] + y.y;
            }
          }
        }
        // acc[rb][j][e] = W(candidate row rb, column 8 j + 2 t0 + e) -> K byte 8 t0 + 4 (j / 2) + 2 (j % 2) + e
        uint32_t dw[kDB][4];  // [digit][rb * 2 + hh]
#pragma unroll
        for (int rb = 0; rb < 2; ++rb)
#pragma unroll
          for (int hh = 0; hh < 2; ++hh) {
            uint32_t lo4[4], hi4[4];
#pragma unroll
            for (int v = 0; v < 4; ++v) {
              const unsigned long long X = kstar_fixed(fabs(acc[rb][2 * hh + (v >> 1)][v & 1]), mc, s_exp2);
              lo4[v] = (uint32_t)X;
              hi4[v] = (uint32_t)(X >> 32);
            }
            const uint32_t p01 = __byte_perm(lo4[0], lo4[1], 0x5140), p23 = __byte_perm(lo4[2], lo4[3], 0x5140);
            const uint32_t q01 = __byte_perm(lo4[0], lo4[1], 0x7362), q23 = __byte_perm(lo4[2], lo4[3], 0x7362);
            const uint32_t h01 = __byte_perm(hi4[0], hi4[1], 0x5140), h23 = __byte_perm(hi4[2], hi4[3], 0x5140);
            dw[0][rb * 2 + hh] = __byte_perm(h01, h23, 0x5410);
            dw[1][rb * 2 + hh] = __byte_perm(q01, q23, 0x7632);
            dw[2][rb * 2 + hh] = __byte_perm(q01, q23, 0x5410);
            dw[3][rb * 2 + hh] = __byte_perm(p01, p23, 0x7632);
            dw[4][rb * 2 + hh] = __byte_perm(p01, p23, 0x5410);
          }
        if (pt == 0) TC_TRACE(0, 3, ks);
        if ((slot_used >> slot) & 1u) {
          mb_wait(&slice_empty[slot], (slot_par >> slot) & 1u);
          slot_par ^= 1u << slot;
          tc_fence_after();
        }
        slot_used |= 1u << slot;
        if (pt == 0) TC_TRACE(0, 4, ks);
#pragma unroll
        for (int b = 0; b < kDB; ++b)
          tmem_st_16x256(tmem + lane_base + (uint32_t)(kDigCol0 + slot * kSliceCols + b * 8), dw[b][0], dw[b][1],
                         dw[b][2], dw[b][3]);
      }
      asm volatile("tcgen05.wait::st.sync.aligned;" ::: "memory");
      tc_fence_before();
      __syncwarp();
      if (lane == 0) mb_arrive(cand_full);
      }
      if (pt == 0) TC_TRACE(0, 6, t);
    }
  } else if (warp >= 8) {
    // ---- K* producers, FMA distances per parameter kind -----------------------------------------
    const int pt = tid - 8 * 32;  // 0..kProdThreads-1
    // warp w may only access TMEM lanes 32 (w % 4) .. +31: candidate = that lane, and the four
    // warps sharing a lane quarter split each 32-column slice into 8-column parts
    const int quarter = warp & 3, part = (warp - 8) >> 2;
    const int c = quarter * 32 + lane;
    const uint32_t lane_base = (uint32_t)(quarter * 32) << 16;
    const double sigma = a.gp.outputscale;
    // K* * kscale: the fixed-point scale is folded into the Matérn polynomial
    const MaternConst mc{sigma * ta.kscale, sigma * kSqrt5 * ta.kscale, sigma * (5.0 / 3.0) * ta.kscale};
    const double kscale = ta.kscale;
    uint32_t slot_used = 0, slot_par = 0;  // per TMEM slot: filled before / parity of its next wait
    for (int t = 0; t < my_tiles; ++t) {
      if (pt == 0) TC_TRACE(0, 1, t);
      const int cb = t & 1;
      mb_wait(&cval_full[cb], (uint32_t)((t >> 1) & 1));
      const uint64_t* cv = cval + (size_t)cb * n_params * kM;
      const uint64_t* cmk = cmask + (size_t)cb * a.n_kendall * kM * 2;
      if (pt == 0) TC_TRACE(0, 2, t);
      for (int p = 0; p < npass; ++p) {
      const int lo = kSlots * p, hi = min(nsl, kSlots * (p + 1));  // this pass's column slices
      const int soff = p == 0 ? 0 : kSlots - (hi - lo);  // a partial last pass takes the slots freed first
      if (pp) {  // every producer is done with the previous pass's columns; load this pass's
        asm volatile("bar.sync 4, %0;" ::"r"(kProdWarps * 32) : "memory");
        load_planes(32 * lo, pt, kProdWarps * 32);
        asm volatile("bar.sync 4, %0;" ::"r"(kProdWarps * 32) : "memory");
      }
      for (int ks = hi - 1; ks >= lo; --ks) {
        const int slot = ks - lo + soff;
        const int j0 = 32 * (pp ? ks - lo : ks) + kColsPerItem * part;  // planes column; warp-uniform
        double W[kColsPerItem];
#pragma unroll
        for (int u = 0; u < kColsPerItem; ++u) W[u] = 0.0;
        for (int i = 0; i < a.n_num; ++i) {
          const int k = a.num_param[i];
          const double x = __longlong_as_double((long long)cv[k * kM + c]);
          // 16-byte broadcast loads: half the shared-memory wavefronts of scalar loads
          const double2* pl = reinterpret_cast<const double2*>(planes + (size_t)k * ppad + j0);
#pragma unroll
          for (int u = 0; u < kColsPerItem / 2; ++u) {
            const double2 y = pl[u];
            const double d0 = x - y.x, d1 = x - y.y;
            W[2 * u] = fma(d0, d0, W[2 * u]);
            W[2 * u + 1] = fma(d1, d1, W[2 * u + 1]);
          }
        }
        for (int i = 0; i < a.n_cat; ++i) {
          const int k = a.cat_param[i];
          const uint64_t x = cv[k * kM + c];
          const double wl = a.gp.inv_l2[k];
          const uint64_t* pl = planes + (size_t)k * ppad + j0;
#pragma unroll
          for (int u = 0; u < kColsPerItem; ++u) W[u] += (x != pl[u]) ? wl : 0.0;
        }
        for (int i = 0, kend = 0; i < a.n_perm; ++i) {
          const int k = a.perm_param[i];
          const bx_param_desc& p = params[k];
          const uint64_t x = cv[k * kM + c];
          const uint64_t* pl = planes + (size_t)k * ppad + j0;
          // the reference's (raw / raw_mx) / l^2 (surrogate.py:222-223) as raw * (1 / l^2 / raw_mx):
          // one FMA per pair instead of a table load
          const double cw = s_cw[k];
          if (p.metric == BX_KENDALL) {  // discordant pairs: popcount of the pair-order masks
            const uint64_t xl = cmk[2 * (kend * kM + c)], xh = cmk[2 * (kend * kM + c) + 1];
            const uint64_t* km = kmask + ((size_t)kend * ppad + j0) * 2;
#pragma unroll
            for (int u = 0; u < kColsPerItem; ++u) {
              const int raw = __popcll(xl ^ km[2 * u]) + __popcll(xh ^ km[2 * u + 1]);
              W[u] = fma((double)raw, cw, W[u]);
            }
            ++kend;
          } else if (p.metric == BX_SPEARMAN) {
            // sum (a_i - b_i)^2 = 2 (sum_{v<m} v^2 - sum a_i b_i) for permutations of 0..m-1; the
            // dot product of the packed nibbles as byte dot products (even / odd nibbles)
            const int m = p.size;
            const int c2 = (m - 1) * m * (2 * m - 1) / 3;
            const uint64_t xe = x & 0x0F0F0F0F0F0F0F0Full, xo = (x >> 4) & 0x0F0F0F0F0F0F0F0Full;
#pragma unroll
            for (int u = 0; u < kColsPerItem; ++u) {
              const uint64_t y = pl[u];
              const uint64_t ye = y & 0x0F0F0F0F0F0F0F0Full, yo = (y >> 4) & 0x0F0F0F0F0F0F0F0Full;
              int dot = __dp4a((unsigned)xe, (unsigned)ye, 0u);
              dot = __dp4a((unsigned)xo, (unsigned)yo, (unsigned)dot);
              if (m > 8) {
                dot = __dp4a((unsigned)(xe >> 32), (unsigned)(ye >> 32), (unsigned)dot);
                dot = __dp4a((unsigned)(xo >> 32), (unsigned)(yo >> 32), (unsigned)dot);
              }
              W[u] = fma((double)(c2 - 2 * dot), cw, W[u]);
            }
          } else {
#pragma unroll
            for (int u = 0; u < kColsPerItem; ++u)
              W[u] = fma((double)perm_raw(p.metric, p.size, x, pl[u], 0, 0, 0, 0), cw, W[u]);
          }
        }
        // K* -> 40-bit fixed point -> five base-256 digits, 4 columns per 32-bit word.  Straight-line
        // code (padding columns are evaluated on the zero planes and masked afterwards) so the
        // independent Matérn chains interleave.
        uint32_t dw[kDB][kColsPerItem / 4];
#pragma unroll
        for (int qd = 0; qd < kColsPerItem / 4; ++qd) {
          uint32_t lo[4], hi[4];
#pragma unroll
          for (int v = 0; v < 4; ++v) {
            const int u = 4 * qd + v;
            // columns j >= n meet zero matrix digits and candidates beyond q are never stored, so
            // neither needs masking; sc leaves >= 2^-20 headroom, so X < 2^40 without a clamp
            const unsigned long long X =
                kPrecise ? __double2ull_rz(kstar(fabs(W[u]), sigma) * kscale) : kstar_fixed(fabs(W[u]), mc, s_exp2);
            lo[v] = (uint32_t)X;
            hi[v] = (uint32_t)(X >> 32);
          }
          const uint32_t p01 = __byte_perm(lo[0], lo[1], 0x5140), p23 = __byte_perm(lo[2], lo[3], 0x5140);
          const uint32_t q01 = __byte_perm(lo[0], lo[1], 0x7362), q23 = __byte_perm(lo[2], lo[3], 0x7362);
          const uint32_t h01 = __byte_perm(hi[0], hi[1], 0x5140), h23 = __byte_perm(hi[2], hi[3], 0x5140);
          dw[0][qd] = __byte_perm(h01, h23, 0x5410);  // bits 32..39
          dw[1][qd] = __byte_perm(q01, q23, 0x7632);  // bits 24..31
          dw[2][qd] = __byte_perm(q01, q23, 0x5410);  // bits 16..23
          dw[3][qd] = __byte_perm(p01, p23, 0x7632);  // bits 8..15
          dw[4][qd] = __byte_perm(p01, p23, 0x5410);  // bits 0..7
        }
        if (pt == 0) TC_TRACE(0, 3, ks);
        if ((slot_used >> slot) & 1u) {  // every producer waits for the MMAs to release the slot
          mb_wait(&slice_empty[slot], (slot_par >> slot) & 1u);
          slot_par ^= 1u << slot;
          tc_fence_after();
        }
        slot_used |= 1u << slot;
        if (pt == 0) TC_TRACE(0, 4, ks);
#pragma unroll
        for (int b = 0; b < kDB; ++b)
        {
          const uint32_t col = tmem + lane_base + (uint32_t)(kDigCol0 + slot * kSliceCols + b * 8 + part * (kColsPerItem / 4));
          if constexpr (kColsPerItem == 8) tmem_st2(col, dw[b][0], dw[b][1]);
          else if constexpr (kColsPerItem == 16) tmem_st4(col, dw[b]);
          else tmem_st1(col, dw[b][0]);
        }
      }
      asm volatile("tcgen05.wait::st.sync.aligned;" ::: "memory");
      tc_fence_before();
      __syncwarp();
      if (lane == 0) {
        mb_arrive(cand_full);        // one arrival per producer warp and pass
        if (p == npass - 1) mb_arrive(&cval_free[cb]);  // the decoders may refill this parity's buffers
      }
      }
      if (pt == 0) TC_TRACE(0, 6, t);
    }
  }
  // the copy / decoder warps (1-3) never touch tensor memory: they leave as soon as their work is
  // done; the TMEM users meet on a named barrier before warp 0 frees it
  if (warp >= 1 && warp <= 3) return;
  tc_fence_before();
  asm volatile("bar.sync 5, %0;" ::"r"((int)blockDim.x - 96) : "memory");
  if (warp == 0) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem), "r"(512));
}

// per-row scale: e_i = exponent of max_j |A_ij| + 2, so |A_ij| 2^-e_i < 1/4 and the top digit of
// rint(A_ij 2^(48 - e_i)) stays within +-65
__global__ void row_scale_kernel(const double* A, int lda, int n, double sc, double* rowscale) {
  const int row = blockIdx.x, lane = threadIdx.x;
  double m = 0.0;
  if (row <= n)
    for (int j = lane; j < n; j += 32) m = fmax(m, fabs(A[(size_t)row * lda + j]));
  for (int off = 16; off; off >>= 1) m = fmax(m, __shfl_xor_sync(0xffffffffu, m, off));
  if (lane == 0) {
    int E = 0;
    if (m > 0.0) frexp(m, &E);
    const bool live = row <= n && m > 0.0;
    rowscale[row] = live ? ldexp(sc, E + 2 - 56) : 0.0;                      // epilogue factor
    rowscale[kTcMaxRows + row] = live ? ldexp(1.0, 48 - (E + 2)) : 0.0;  // digit scale
  }
}

// [chunk][slice][digit][32 rows x 32 columns, K-major] balanced base-256 digits of A
// perm: K byte kb of a slice holds column 8 (2 hh + jj) + 2 t0 + e, kb = 8 t0 + 4 hh + 2 jj + e (the
// C-fragment order of the DMMA producers)
__global__ void mdig_kernel(const double* A, int lda, int n, int nsl, int nch, const double* rowscale,
                            unsigned char* mdig, int perm) {
  const int64_t total = (int64_t)nch * nsl * kN * 32;
  for (int64_t t = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; t < total;
       t += (int64_t)gridDim.x * blockDim.x) {
    const int kb = (int)(t & 31), r = (int)((t >> 5) & (kN - 1));
    const int blk = (int)(t / (kN * 32));
    const int ks = blk % nsl, c = blk / nsl;
    const int kc = perm ? 8 * (2 * ((kb >> 2) & 1) + ((kb >> 1) & 1)) + 2 * (kb >> 3) + (kb & 1) : kb;
    const int row = c * kN + r, col = ks * 32 + kc;
    const double x = (row <= n && col < n) ? A[(size_t)row * lda + col] : 0.0;
    long long X = __double2ll_rn(x * rowscale[kTcMaxRows + row]);
    unsigned char* out = mdig + (size_t)blk * kMatBlock + kmaj(r, kb);
#pragma unroll
    for (int d = kDA - 1; d >= 0; --d) {
      int v = (int)(X & 255);
      if (v >= 128) v -= 256;
      out[d * kN * 32] = (unsigned char)(v & 255);
      X = (X - v) >> 8;
    }
  }
}

}  // namespace

size_t tc_smem_bytes(int n, int n_params, int n_kendall, int row_words, int ks, int n_emb, int emb_tab_len,
                     bool aug, bool resident) {
  // the smallest layout the kernel can run with (per-pass planes when there are several passes)
  return tc_layout(n, n_params, n_kendall, row_words, ks, n_emb, emb_tab_len, aug, resident,
                   tc_passes((n + 31) / 32) > 1).total;
}

size_t tc_part_doubles(int n, int grid) {
  const int nch = n / kN + 1;
  return tc_passes((n + 31) / 32) > 1 ? (size_t)grid * (kN * nch - kSlots * 32) * kM : 0;
}

size_t tc_mdig_bytes(int n) {
  const int nsl = (n + 31) / 32, nch = n / kN + 1;
  return (size_t)nsl * nch * kMatBlock;
}

// rowscale must hold 2 * kTcMaxRows doubles (epilogue factors, then digit scales)
cudaError_t launch_build_mdig(const double* A, int lda, int n, double sc, unsigned char* mdig,
                              double* rowscale, int perm, cudaStream_t s) {
  const int nsl = (n + 31) / 32, nch = n / kN + 1;
  if (nch > kMaxChunks) return cudaErrorInvalidValue;
  row_scale_kernel<<<kTcMaxRows, 32, 0, s>>>(A, lda, n, sc, rowscale);
  cudaError_t e = cudaGetLastError();
  if (e != cudaSuccess) return e;
  mdig_kernel<<<148, 256, 0, s>>>(A, lda, n, nsl, nch, rowscale, mdig, perm);
  return cudaGetLastError();
}

cudaError_t launch_gp_tc(const TcArgs& a0, int sm_count, cudaStream_t s) {
  TcArgs a = a0;
  const int n = a.f.gp.n, P = a.f.space.n_params, K = a.f.n_kendall, W = a.f.space.row_words;
  const bool multi = tc_passes(a.n_slices) > 1;
  // the whole-width planes when they fit, else per pass (BX_TC_DEBUG bit 16: per pass whenever
  // there are several passes)
  a.planes_pp = multi && ((a.debug & 16) || tc_layout(n, P, K, W, a.ks, a.n_emb, a.emb_tab_len, a.aug != 0, false,
                                                      false).total > 227 * 1024);
  // matrix digits resident in shared memory when they fit (BX_TC_DEBUG bit 8: always the ring)
  a.mat_resident = !(a.debug & 8) && tc_layout(n, P, K, W, a.ks, a.n_emb, a.emb_tab_len, a.aug != 0, true,
                                               a.planes_pp != 0).total <= 227 * 1024;
  // the ring takes the shared memory left over, up to kMaxStages (L2 latency x MMA block rate)
  a.mat_stages = kStages;
  if (!a.mat_resident) {
    const int base = tc_layout(n, P, K, W, a.ks, a.n_emb, a.emb_tab_len, a.aug != 0, false, a.planes_pp != 0, 0).total;
    a.mat_stages = std::max(kStages, std::min(kMaxStages, (227 * 1024 - base) / kMatBlock));
    if (const char* st = getenv("BX_TC_STAGES")) a.mat_stages = std::max(2, std::min(a.mat_stages, atoi(st)));
  }
  TcLayout L = tc_layout(n, P, K, W, a.ks, a.n_emb, a.emb_tab_len, a.aug != 0, a.mat_resident != 0,
                         a.planes_pp != 0, a.mat_stages);
  // packed pools: their own staging buffer when it fits next to everything else (BX_TC_DEBUG bit
  // 32: never), the static shared memory counted
  a.pk_sep = 0;
  if (a.packed && !(a.debug & 32)) {
    const TcLayout L2 = tc_layout(n, P, K, W, a.ks, a.n_emb, a.emb_tab_len, a.aug != 0, a.mat_resident != 0,
                                  a.planes_pp != 0, a.mat_stages, kM * a.pack.pw * 4);
    if (L2.total + 1024 <= 227 * 1024) {
      a.pk_sep = 1;
      L = L2;
    }
  }
  if (L.total > 227 * 1024 || a.n_chunks > kMaxChunks || a.ks > 8 || (a.ks > 0 && a.f.precise) ||
      (multi && !a.part))
    return cudaErrorInvalidValue;
  if (getenv("BX_TC_INFO"))  // development aid: kernel geometry
    fprintf(stderr, "gp_tc: n %d ks %d E %d aug %d smem %d resident %d planes_pp %d stages %d words %d pk_sep %d\n", n,
            a.ks, a.n_emb, a.aug, L.total, a.mat_resident, a.planes_pp, a.mat_stages, W, a.pk_sep);
  auto kernel = a.f.precise ? (multi ? gp_tc_kernel<true, 0, true> : gp_tc_kernel<true, 0, false>)
                            : (multi ? gp_tc_kernel<false, 0, true> : gp_tc_kernel<false, 0, false>);
  int threads = tc_threads<0>();
  switch (a.ks) {
#define BX_KS(k)                                                                   \
    case k:                                                                        \
      kernel = multi ? gp_tc_kernel<false, k, true> : gp_tc_kernel<false, k, false>; \
      threads = tc_threads<k>();                                                   \
      break;
    BX_KS(1) BX_KS(2) BX_KS(3) BX_KS(4) BX_KS(5) BX_KS(6) BX_KS(7) BX_KS(8)
#undef BX_KS
    default: break;
  }
  cudaError_t e = set_smem(kernel, L.total);
  if (e != cudaSuccess) return e;
  const int64_t tiles = (a.f.q + kM - 1) / kM;
  int64_t grid = sm_count;
  if (tiles < grid) grid = tiles;
  if (grid < 1) grid = 1;
  kernel<<<(int)grid, threads, L.total, s>>>(a);
  return cudaGetLastError();
}

}  // namespace bx
