/*
 * bx_sm100.h — C ABI of libbx_sm100.so, the B200 (sm_100a) candidate-acquisition scorer.
 *
 * The reference ("boxtune", a pure NumPy/SciPy re-implementation of BaCO, arXiv 2212.11142)
 * has no FFI: its hot path is a set of Python functions.  Each entry point below replaces one
 * of them; the Python package `paper_2212_11142_b200` binds these symbols with ctypes and
 * installs itself at the reference's own call sites.
 *
 *   bx_set_space        model-independent space tables   (surrogate.py:163-170 _numeric_coords,
 *                                                          feasibility.py:33-51 encode_configs,
 *                                                          space.py:258-286 _param_neighbors)
 *   bx_set_gp           GPModel state                    (surrogate.py:274-303 GPModel.__init__)
 *   bx_set_forest       FeasibilityModel flat arrays     (feasibility.py:54-71)
 *   bx_set_evaluated    AcquisitionContext.evaluated     (acquisition.py:63, used at :107)
 *   bx_set_cot          ChainOfTrees groups              (constraints.py:398-430)
 *   bx_set_constraints  parsed ConstraintExpr list       (constraints.py:297-368)
 *   bx_score            _scores + tracker + argsort      (acquisition.py:70-79, :97-111, :186-188)
 *   bx_rf_predict       predict_proba_batch              (feasibility.py:72-89)
 *   bx_gp_predict       GPModel.predict_batch            (surrogate.py:315-328)
 *   bx_neighbors        neighbors(space, cfg, cot)       (space.py:289-309)
 *   bx_cot_contains     ChainOfTrees.contains            (constraints.py:413-430)
 *   bx_constraints_eval eval_constraint over a batch     (constraints.py:351-368)
 *   bx_lml_batched      _batched_coarse_lml              (surrogate.py:420-456)
 *
 * Conventions
 *   - Every function returns BX_OK (0) or a BX_ERR_* code; bx_last_error(h) describes the last
 *     failure on that handle.  No C++ exception crosses this boundary.
 *   - Buffers named dev_* are caller-owned DEVICE pointers (cudaMalloc / torch tensors); buffers
 *     named host_* are caller-owned HOST pointers that are copied during the call.  The library
 *     owns only the per-handle model state uploaded by the bx_set_* calls.
 *   - `stream` is a cudaStream_t passed as void* (NULL = legacy default stream).  All work of a
 *     call is enqueued on it; calls that return host results synchronise that stream.
 *   - A handle is bound to one device and is not thread-safe; use one handle per thread/rank.
 *
 * Encoded configuration rows (the data layout in HBM)
 *   A configuration is a row of `row_words` uint32 words.  Parameter k occupies words
 *   [word, word+nwords) given by its bx_param_desc:
 *     integer      1 word : value - lo
 *     ordinal      1 word : index into the declared values
 *     categorical  1 word : index into the declared labels (declaration order)
 *     real         4 words: f64 raw value, then f64 coordinate (min-max / log-min-max, host-made)
 *     permutation  2 words: u64, element at position i stored minus one in nibble (m-1-i), so
 *                           the integer order of the u64 equals Python's tuple order (m <= 16)
 */
#ifndef BX_SM100_H
#define BX_SM100_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#if defined(__GNUC__)
#pragma GCC visibility push(default)
#endif

#define BX_ABI_VERSION 1

enum bx_status {
  BX_OK = 0,
  BX_ERR_ARG = 1,          /* bad argument (maps to ValueError)                          */
  BX_ERR_CUDA = 2,         /* CUDA runtime failure (RuntimeError)                          */
  BX_ERR_NOT_PD = 3,       /* Cholesky failed: Gram not positive definite (SurrogateError) */
  BX_ERR_STATE = 4,        /* required bx_set_* call missing (RuntimeError)                */
  BX_ERR_UNSUPPORTED = 5,  /* outside the supported envelope, e.g. m > 16 (ValueError)     */
  BX_ERR_NO_TREES = 6      /* forest without trees (FeasibilityError, feasibility.py:75)   */
};

enum bx_kind { BX_REAL = 0, BX_INTEGER = 1, BX_ORDINAL = 2, BX_CATEGORICAL = 3, BX_PERMUTATION = 4 };
enum bx_perm_metric { BX_KENDALL = 0, BX_SPEARMAN = 1, BX_HAMMING = 2, BX_NAIVE = 3 };

#define BX_MAX_PARAMS 64
#define BX_MAX_ROW_WORDS 64
#define BX_MAX_K 32
#define BX_MAX_PERM 16

/* One parameter of the space.  Tables are indexed through the offsets. */
typedef struct {
  int32_t kind;      /* bx_kind                                                               */
  int32_t word;      /* first uint32 word of the parameter in a row                            */
  int32_t size;      /* finite kinds: domain size; permutation: m; real: 64 (neighbour grid)    */
  int32_t metric;    /* bx_perm_metric (permutations only)                                      */
  int32_t coord;     /* offset into coord_lut: finite numeric -> coordinate of each domain index;
                        real -> coordinate of each of the 64 neighbour-grid points (space.py:23) */
  int32_t rank;      /* offset into rank_lut: categorical label -> rank under Python str order  */
  int32_t feat;      /* first feature column of this parameter in encode_configs order          */
  int32_t is_log;    /* transform == "log" and transforms enabled                               */
  double lo, hi;     /* real: bounds (contains / neighbour grid); integer: lo, hi as doubles   */
  double step;       /* real: (hi - lo) / (REAL_NEIGHBOR_GRID - 1), computed by the host        */
  double raw_mx;     /* permutation: permutation_metric_max(metric, m) (surrogate.py:75-85)    */
} bx_param_desc;

/* One scored candidate. */
typedef struct {
  double value;                     /* acquisition value (EI * p, or -inf)                     */
  double prob;                      /* feasibility probability p (1.0 without a forest)        */
  int64_t index;                    /* global pool index (index_base + local index); -1 = none */
  uint32_t row[BX_MAX_ROW_WORDS];   /* the encoded configuration                               */
} bx_cand;

/* Result of one bx_score call over a pool. */
typedef struct {
  int64_t n_scored;                 /* q                                                       */
  int64_t n_finite;                 /* #values != -inf       (acquisition.py:179)               */
  int32_t k;                        /* requested top-k (n_starts)                              */
  int32_t n_top;                    /* valid entries in top[] (<= k; -inf never listed)         */
  bx_cand top[BX_MAX_K];            /* stable argsort(-values)[:k]      (acquisition.py:188)    */
  bx_cand best;                     /* _Tracker over values: max value, ties -> smallest config,
                                       evaluated and -inf skipped      (acquisition.py:97-111) */
  bx_cand best_prob;                /* _Tracker over probs (fallback)   (acquisition.py:181)    */
} bx_score_summary;

typedef struct bx_handle bx_handle;

/* ---- lifetime --------------------------------------------------------------------------- */
bx_handle* bx_create(int device);
void bx_destroy(bx_handle* h);
const char* bx_last_error(bx_handle* h);
int bx_abi_version(void);
int bx_device_sm_count(bx_handle* h);
/* Which posterior kernel the current model state runs (valid after bx_set_gp):
   BX_GP_TENSOR (tcgen05 int8 split product), BX_GP_DMMA (register-resident FP64 DMMA) or
   BX_GP_GENERIC (shared-memory FP64 kernel for n + 1 > 256). */
enum { BX_GP_GENERIC = 0, BX_GP_DMMA = 1, BX_GP_TENSOR = 2 };
/* Handle options.  BX_OPT_LML_NARROW = 1: bx_lml_core / bx_lml_batched run one CTA per setting
   instead of the whole-GPU kernels (A/B measurements).  Either way a setting's value and gradient
   do not depend on the batch it came in. */
enum bx_option { BX_OPT_LML_NARROW = 1 };
int bx_set_option(bx_handle* h, int32_t option, int32_t value);
int bx_gp_kernel(bx_handle* h);
/* GPModel.__init__ (surrogate.py:286-303) on the device: the Gram of the n training rows
   (dev_train_rows, encoded) under (outputscale, noise_variance, lengthscales[n_params]) with the
   noise floor and jitter on its diagonal, its Cholesky factor and alpha = K^-1 z for the
   standardised targets host_z[n].  Writes host_L (n x n, row-major, lower, zeros above) and
   host_alpha (n); BX_ERR_NOT_PD when the factorisation fails (numpy's LinAlgError).  n <= 512.
   Values are FP64, not bit-identical to LAPACK's. */
int bx_gp_factor(bx_handle* h, const uint32_t* dev_train_rows, int32_t n, const double* host_z, double outputscale,
                 double noise_variance, const double* lengthscales, double* host_L, double* host_alpha, void* stream);

/* Tensor-core posterior only: the DMMA k-steps of its distance product over the Euclidean
   embedding of W (0: FMA distances per parameter kind, or not the tensor-core kernel). */
int bx_gp_distance_ksteps(bx_handle* h);
/* ... and the embedding's coordinate count E (|x'|^2 + |y'|^2 rides in two extra k-rows when
   E + 2 <= 4 k-steps, else it is added to the products). */
int bx_gp_embedding_dims(bx_handle* h);

/* ---- model state (once per BO iteration) ------------------------------------------------ */
/* Space tables.  coord_lut / rank_lut are host arrays indexed by bx_param_desc offsets;
   n_features = encode_configs width (feasibility.py:33-51).  Setting a space clears every other
   piece of model state (GP, forest, evaluated set, chain of trees, constraints): each must be set
   again for the new space before the calls that need it (they return BX_ERR_STATE until then). */
int bx_set_space(bx_handle* h, const bx_param_desc* host_params, int32_t n_params, int32_t row_words,
                 const double* host_coord_lut, int32_t coord_len,
                 const int32_t* host_rank_lut, int32_t rank_len, int32_t n_features);

/* GP posterior state.  host_train_rows: n encoded training configurations; host_L: the
   lower Cholesky factor of K + (noise + 1e-9) I, n x n row-major (only the lower triangle is
   read, cho_factor leaves stale K above it: surrogate.py:300); host_alpha = K^-1 z.  The
   library forms L^-1 on the device.  lengthscales has n_params entries. */
int bx_set_gp(bx_handle* h, const uint32_t* host_train_rows, int32_t n, const double* host_L,
              const double* host_alpha, double outputscale, const double* host_lengthscales,
              double y_mean, double y_std, void* stream);

/* rf_fit's tree building (feasibility.py:95-197) on the device, bit-exact: host_X / host_y = the
   canonically sorted encode_configs matrix [n][F] and labels; per tree its bootstrap rows [n] and
   the feature subsets its generator drew in order [max_draws][k] (host_n_drawn of them); outputs
   [n_trees][max_nodes] in the tree's own preorder ids (-1 = none), the node counts and a status per
   tree (0 ok, 1 needs more feature subsets: draw more from the same generator and call again,
   2 max_nodes exceeded). */
int bx_rf_fit(bx_handle* h, const double* host_X, const double* host_y, int32_t n, int32_t F, int32_t n_trees,
              const int32_t* host_boot, const int32_t* host_feats, const int32_t* host_n_drawn, int32_t max_draws,
              int32_t k, int32_t max_depth, int32_t max_nodes, int32_t* host_feature, double* host_threshold,
              int32_t* host_left, int32_t* host_right, double* host_value, int32_t* host_n_nodes,
              int32_t* host_status, void* stream);

/* Random forest in the reference's flat layout (feasibility.py:54-71).  `constant` is the
   single-class shortcut value, or NaN when the forest has trees. */
int bx_set_forest(bx_handle* h, const int32_t* host_feature, const double* host_threshold,
                  const int32_t* host_left, const int32_t* host_right, const double* host_value,
                  int32_t n_nodes, const int32_t* host_roots, int32_t n_trees, int32_t max_depth,
                  double constant);
int bx_clear_forest(bx_handle* h);

/* Evaluated configurations (exact row match excludes them from the trackers). */
int bx_set_evaluated(bx_handle* h, const uint32_t* host_rows, int32_t count);

/* Chain of trees, flattened.  Groups are listed in the reference's order.  For group g:
   group_kind[g] (0 tree, 1 real singleton, 2 permutation singleton), group_param_begin[g] ..
   group_param_begin[g+1] index into group_params (parameter indices, declaration order);
   group_root[g] is a node id.  Node u has child_count[u] children with consecutive ids starting
   at child_begin[u]; node_value[c] is the domain index of node c's value, ascending among
   siblings. */
int bx_set_cot(bx_handle* h, int32_t n_groups, const int32_t* host_group_kind,
               const int32_t* host_group_param_begin, const int32_t* host_group_params,
               const int32_t* host_group_root, int32_t n_nodes, const int32_t* host_child_begin,
               const int32_t* host_child_count, const int32_t* host_node_value,
               const int64_t* host_node_leaf_count /* nullable: needed by bx_generate mode 1 */);
int bx_clear_cot(bx_handle* h);

/* Known constraints as stack bytecode (opcode table in paper_2212_11142_b200/constraints.py).
   Program c is code[prog_begin[c] .. prog_begin[c+1]) as (opcode, argument) int pairs; consts
   holds the float literals.  The value tables give, for every finite parameter (in parameter
   order, domain index inner), the Python value the expression sees: value_tag 0 = int (value_int)
   or 1 = float (value_float); value_str = string id of categorical labels (literals are interned
   into the same id space by the host, so `==` on strings is id equality). */
int bx_set_constraints(bx_handle* h, int32_t n_constraints, const int32_t* host_prog_begin,
                       const int32_t* host_code, int32_t code_len, const double* host_consts,
                       int32_t n_consts, const int32_t* host_value_tag,
                       const int64_t* host_value_int, const double* host_value_float,
                       const int32_t* host_value_str, int32_t n_values);

/* ---- hot path --------------------------------------------------------------------------- */
enum bx_score_flags {
  BX_SCORE_RF_PAIRWISE = 1,   /* numpy pairwise-8 tree sum (what predict_proba does at q == 1) */
  BX_SCORE_NO_SUMMARY = 2,    /* skip the top-k / tracker reduction                             */
  BX_SCORE_TIMING = 4,        /* record per-kernel CUDA-event durations (bx_last_timing)        */
  BX_SCORE_TIMING_POSTERIOR = 8, /* time the posterior kernel only (two events; rf / merge = -1) */
  BX_SCORE_PACKED = 16           /* bx_score_host: the host pool is in the packed wire format      */
};

/* Durations (ms, CUDA events on the call's stream) of the forest, fused-score and merge kernels
   of the last bx_score call made with BX_SCORE_TIMING. */
int bx_last_timing(bx_handle* h, float* rf_ms, float* score_ms, float* merge_ms);

/* Diagnostic (no reference counterpart): measured FP64 peaks of the DFMA pipe and of the DMMA
   m8n8k4 tensor path on `device`, in TFLOP/s - the roofline denominator of the contraction. */
int bx_probe_fp64(int device, double* dfma_tflops, double* dmma_tflops);
/* Live int8 tcgen05.mma rates: dense_mac_s = MACs/s of the peak shape (M128 N256 K32, operands in
   shared memory) over every SM; block_ns = one (chunk, slice) block of the posterior's split
   product (five MMAs, A from TMEM, N = 96..32) on one SM.  The roofline denominators of bench.py. */
int bx_probe_int8(int device, double* dense_mac_s, double* block_ns);

/* Score dev_rows[0..q) (encoded, device).  f_model = objective_to_model(best feasible value);
   eps_f = feasibility limit.  Writes values/probs when non-NULL (device, q doubles each) and,
   unless BX_SCORE_NO_SUMMARY, the summary to host_summary (host; the call synchronises). */
int bx_score(bx_handle* h, const uint32_t* dev_rows, int64_t q, int64_t index_base, double f_model,
             double eps_f, int32_t k, int32_t flags, double* dev_values, double* dev_probs,
             bx_score_summary* host_summary, void* stream);

/* Same as bx_score but the pool is a HOST buffer (pinned or pageable).  This is the end-to-end
   entry point.  With BX_SCORE_PACKED the host rows are in the packed wire format (bx_pack_rows),
   which the tensor-core posterior unpacks on the fly (2-4x fewer bytes over PCIe for typical
   spaces); a packed pool in pinned memory is read by the posterior straight from host memory
   (zero-copy), otherwise the call copies the pool in chunks that the posterior consumes as they
   land. */
int bx_score_host(bx_handle* h, const uint32_t* host_rows, int64_t q, int64_t index_base,
                  double f_model, double eps_f, int32_t k, int32_t flags,
                  bx_score_summary* host_summary, void* stream);

/* Packed wire format of the current space: each parameter at its bit width (finite kinds: domain
   index; permutation: 4 bits per element; real: the f64 value, plus the f64 coordinate only when a
   log transform makes it host-dependent - otherwise the device recomputes (v - lo) / (hi - lo)
   bit-exactly, surrogate.py:163-170), rows padded to whole 32-bit words.  Host-side conversions
   (CPU loops, no device work). */
int bx_packed_row_words(bx_handle* h);
int bx_pack_rows(bx_handle* h, const uint32_t* host_rows, int64_t q, uint32_t* host_packed);
int bx_unpack_rows(bx_handle* h, const uint32_t* host_packed, int64_t q, uint32_t* host_rows);

/* Host-side: n draws of numpy's Generator.permutation(m) (m <= 16) replayed from a PCG64 state -
   state = {state_hi, state_lo, inc_hi, inc_lo}, has_uint32 / uinteger = the generator's 32-bit
   buffer - written as packed rows (element at position i in nibble m-1-i, 0-based values); the
   state is advanced exactly as the n Python calls advance it (space.py:330-331).  No device work. */
int bx_pcg64_permutations(uint64_t* state, int32_t* has_uint32, uint32_t* uinteger, int64_t n, int32_t m,
                          uint64_t* packed);
/* ... and n draws of Generator.choice(pop, size=k, replace=False) (pop <= 10000: Floyd's algorithm
   and a shuffle), k indices per draw into out[n][k] - the rf_fit feature subsets
   (feasibility.py:119). */
int bx_pcg64_choice(uint64_t* state, int32_t* has_uint32, uint32_t* uinteger, int64_t n, int32_t pop, int32_t k,
                    int32_t* out);
/* ... and the random-forest fit's per-tree draws (feasibility.py:119-190, replacing the n_trees
   np.random.default_rng(seed) generators): tree t's generator is seeded from seeds[t] (< 2^64) as
   SeedSequence + PCG64 seed it, draws its bootstrap rows integers(0, n, size=n) into boot[t][n]
   and then ndraws feature subsets choice(pop, size=k, replace=False) into subsets[t][ndraws][k];
   its state afterwards goes to state[t][4] / has_uint32[t] / uinteger[t] (bx_pcg64_choice
   continues it). */
int bx_pcg64_forest_draws(const uint64_t* seeds, int32_t n_trees, int64_t n, int32_t pop, int32_t k, int32_t ndraws,
                          int32_t* boot, int32_t* subsets, uint64_t* state, int32_t* has_uint32, uint32_t* uinteger);

/* Host-side: first-occurrence de-duplication of q encoded rows (list(dict.fromkeys(raw)),
   acquisition.py:173): writes the indices of the first occurrences, in order, to first_idx[q] and
   returns their count (negative: -bx_status).  No device work. */
int64_t bx_unique_rows(const uint32_t* rows, int64_t q, int32_t words, int64_t* first_idx);

/* Device-side candidate generation: q rows for global indices
   index_base .. index_base+q-1 from Philox4x32-10 keyed by (seed, index); mode 0 = uniform over the
   dense space (sample_uniform's distribution, space.py:312-332), mode 1 = leaf-uniform over the
   chain of trees (sample_leaf_uniform's, constraints.py:471-523; needs bx_set_cot leaf counts). mode 2 = path-biased over the chain of trees
   (sample_path_biased's, constraints.py:478-501, 522-523: a uniform child at every level). */
int bx_generate(bx_handle* h, uint64_t seed, int64_t index_base, int64_t q, int32_t mode,
                uint32_t* dev_rows, void* stream);

/* Score a device-generated pool of q candidates chunk by chunk without materialising it (pools of
   10^9 and beyond); the summary's top-k rows are regenerated from their indices. */
int bx_score_generated(bx_handle* h, uint64_t seed, int64_t index_base, int64_t q, int32_t mode,
                       double f_model, double eps_f, int32_t k, bx_score_summary* host_summary,
                       void* stream);

/* Posterior mean / latent variance, de-standardised (predict_batch, include_noise=False). */
int bx_gp_predict(bx_handle* h, const uint32_t* dev_rows, int64_t q, double* dev_mean,
                  double* dev_var, void* stream);

/* Feasibility probability (predict_proba_batch).  flags: BX_SCORE_RF_PAIRWISE. */
int bx_rf_predict(bx_handle* h, const uint32_t* dev_rows, int64_t q, int32_t flags,
                  double* dev_probs, void* stream);

/* The hill climb of optimize_acquisition (acquisition.py:186-202) on the device.  n_starts starts
   (<= BX_MAX_K): rows host_start_index[i] of the device pool, with their values (host); per step the neighbours of every start still
   climbing (CoT-filtered when use_cot, space.py:289-309), scored like _scores (a start with exactly
   one neighbour gets the forest's q == 1 summation order, feasibility.py:89), each start moved to
   its argbest under (value desc, configuration asc) iff strictly better (:87-94, :200), every
   scored neighbour folded into the best-unevaluated tracker (:105-111).  host_best is the tracker
   in / out (index < 0: empty; value, row).  Steps are issued four at a time with one 4-byte
   device -> host read per four (a step after every start stopped changes nothing); *host_steps =
   the steps that had a climbing start, the reference's loop count. */
int bx_climb(bx_handle* h, const uint32_t* dev_pool_rows, const int64_t* host_start_index,
             const double* host_start_values, int32_t n_starts, int32_t use_cot, double f_model, double eps_f,
             int32_t max_steps, bx_cand* host_best, int32_t* host_steps, void* stream);

/* All single-parameter moves of `count` rows.  Slot s of row r goes to
   dev_out_rows[(r * n_slots + s) * row_words]; dev_out_valid[r * n_slots + s] is 1 when the
   move exists and (with use_cot) lies in the chain of trees.  Slot order = the reference's
   neighbour order.  n_slots is returned by bx_neighbor_slots. */
int bx_neighbor_slots(bx_handle* h);
int bx_neighbors(bx_handle* h, const uint32_t* dev_rows, int32_t count, int32_t use_cot,
                 uint32_t* dev_out_rows, uint8_t* dev_out_valid, void* stream);

/* Membership masks over a batch (bit-exact). */
int bx_cot_contains(bx_handle* h, const uint32_t* dev_rows, int64_t q, uint8_t* dev_mask,
                    void* stream);
/* mask = all constraints evaluate True (constraints.py:351-368; faults -> False). */
int bx_constraints_eval(bx_handle* h, const uint32_t* dev_rows, int64_t q, uint8_t* dev_mask,
                        void* stream);

/* Batched coarse log marginal likelihood (surrogate.py:420-456).  dev_sq: D x n x n f64
   per-parameter squared distances, dev_z: n, dev_thetas: c x (2 + D) rows
   (log sigma, log noise, log l_1..l_D).  dev_out: c values, -inf where Cholesky fails. */
int bx_lml_batched(bx_handle* h, const double* dev_sq, int32_t n, int32_t D, const double* dev_z,
                   const double* dev_thetas, int32_t c, double* dev_out, void* stream);

/* Log marginal posterior and its gradient (_lml_core, surrogate.py:356-400) for c hyperparameter
   settings at once, one CTA each.  dev_params: c rows of (sigma, noise, l_1..l_D) in natural
   units (noise floored at 1e-6 as the reference does).  use_prior adds the Gamma(prior_shape,
   prior_rate) lengthscale log-density.  Writes dev_value[c], dev_grad[c x (2+D)] (d/dlog sigma,
   d/dlog noise, d/dlog l_i) when want_grad, and dev_ok[c] = 0 where the Cholesky factorisation
   fails (the reference raises LinAlgError there; value -inf, gradient 0). */
int bx_lml_core(bx_handle* h, const double* dev_sq, int32_t n, int32_t D, const double* dev_z,
                const double* dev_params, int32_t c, double prior_shape, double prior_rate,
                int32_t use_prior, int32_t want_grad, double* dev_value, double* dev_grad,
                int32_t* dev_ok, void* stream);
/* ... the same with host parameters and host results (gradient always): host_params[c][2+D] in,
   host_value[c], host_grad[c][2+D], host_ok[c] out through one pinned staging buffer; returns
   after the results are in host memory (hyperfit's L-BFGS-B objective, surrogate.py:510-516). */
int bx_lml_core_host(bx_handle* h, const double* dev_sq, int32_t n, int32_t D, const double* dev_z,
                     const double* host_params, int32_t c, double prior_shape, double prior_rate, int32_t use_prior,
                     double* host_value, double* host_grad, int32_t* host_ok, void* stream);

/* Per-parameter squared distances between rows (pairwise_sq_distances, surrogate.py:173-198),
   dev_out: D x qa x qb f64. */
int bx_pairwise_sq(bx_handle* h, const uint32_t* dev_a, int32_t qa, const uint32_t* dev_b,
                   int32_t qb, double* dev_out, void* stream);

#if defined(__GNUC__)
#pragma GCC visibility pop
#endif

#ifdef __cplusplus
}
#endif
#endif /* BX_SM100_H */
