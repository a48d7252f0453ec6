// bx_model.cu — per-iteration model uploads behind the C ABI: bx_set_gp (L^-1, the digit planes
// of the tensor-core contraction, the Euclidean embedding of W and its DMMA operand) and
// bx_set_forest (breadth-first nodes, the integer-coded forest and the QuickScorer tables with
// their indirect slots).
#include "bx_handle.cuh"

static int build_coded_forest(bx_handle* h, const std::vector<RfNode>& nodes,
                              const std::vector<int32_t>& roots, int max_depth);


// Helmert basis: (L - 1) x L orthonormal rows spanning the sum-zero subspace of R^L
static std::vector<double> helmert(int L) {
  std::vector<double> Q((size_t)(L - 1) * L, 0.0);
  for (int j = 1; j < L; ++j) {
    const double nrm = std::sqrt((double)j * (j + 1));
    for (int i = 0; i < j; ++i) Q[(size_t)(j - 1) * L + i] = 1.0 / nrm;
    Q[(size_t)(j - 1) * L + j] = -(double)j / nrm;
  }
  return Q;
}

// The Euclidean embedding of W = sum_k sq_k / l_k^2 (surrogate.py:173-223; EmbDim in bx_common.cuh),
// centred on the training mean; planes = the DMMA B operand [4 ks][npad] (-2 y', then |y'|^2 and 1
// when they fit the padding: *aug), yy[npad] = |y'|^2.  False when a metric does not embed (naive
// permutation indicator) or the centred coordinates are too large for the |x|^2 + |y|^2 - 2 x.y
// form (bound 256: the cancellation error stays near the 2^-40 fixed point of K*).
static bool build_embedding(const bx_handle* h, const uint32_t* train_rows, int n, const double* inv_l,
                            const double* inv_l2, int npad, std::vector<EmbDim>& emb, std::vector<double>& tab,
                            std::vector<double>& planes, std::vector<double>& yy, bool* aug) {
  std::vector<int> seg;  // table entries per coordinate that carry the centring
  for (int k = 0; k < h->n_params; ++k) {
    const bx_param_desc& p = h->params[k];
    if (p.kind == BX_INTEGER || p.kind == BX_ORDINAL) {
      emb.push_back(EmbDim{BX_EMB_CODE, p.word, 0, 0, 0, (int)tab.size()});
      for (int i = 0; i < p.size; ++i) tab.push_back(h->coord_host[p.coord + i] * inv_l[k]);
      seg.push_back(p.size);
    } else if (p.kind == BX_REAL) {
      emb.push_back(EmbDim{BX_EMB_REAL, p.word, 0, 0, 0, (int)tab.size()});
      tab.push_back(inv_l[k]);
      tab.push_back(0.0);
      seg.push_back(0);
    } else if (p.kind == BX_CATEGORICAL) {
      const int L = p.size;
      const std::vector<double> Q = helmert(L);
      const double sw = std::sqrt(inv_l2[k] / 2.0);  // unit-edge simplex: |V_a - V_b|^2 = 1
      for (int j = 0; j + 1 < L; ++j) {
        emb.push_back(EmbDim{BX_EMB_CODE, p.word, 0, 0, 0, (int)tab.size()});
        for (int a = 0; a < L; ++a) tab.push_back(Q[(size_t)j * L + a] * sw);
        seg.push_back(L);
      }
    } else {  // permutation
      const int m = p.size;
      const double wm = inv_l2[k] / p.raw_mx;
      if (p.metric == BX_SPEARMAN) {
        const std::vector<double> Q = helmert(m);
        for (int j = 0; j + 1 < m; ++j) {
          emb.push_back(EmbDim{BX_EMB_PERM_LIN, p.word, 0, 0, m, (int)tab.size()});
          for (int i = 0; i < m; ++i) tab.push_back(Q[(size_t)j * m + i] * std::sqrt(wm));
          tab.push_back(0.0);
          seg.push_back(-1);
        }
      } else if (p.metric == BX_KENDALL) {
        for (int a = 0; a < m; ++a)
          for (int b = a + 1; b < m; ++b) {
            emb.push_back(EmbDim{BX_EMB_KENDALL, p.word, a, b, m, (int)tab.size()});
            tab.push_back(0.0);
            tab.push_back(std::sqrt(wm));
            seg.push_back(2);
          }
      } else if (p.metric == BX_HAMMING) {
        const std::vector<double> Q = helmert(m);
        for (int pos = 0; pos < m; ++pos)
          for (int j = 0; j + 1 < m; ++j) {
            emb.push_back(EmbDim{BX_EMB_PERM_HOT, p.word, pos, 0, m, (int)tab.size()});
            for (int v = 0; v < m; ++v) tab.push_back(Q[(size_t)j * m + v] * std::sqrt(wm / 2.0));
            seg.push_back(m);
          }
      } else {
        return false;  // the naive indicator 1{a != b} over m! permutations does not embed cheaply
      }
    }
    if (emb.size() > 32) return false;
  }
  const int E = (int)emb.size();
  if (E == 0) return false;
  // centre on the training mean (translation leaves every distance unchanged)
  for (int e = 0; e < E; ++e) {
    double mu = 0.0;
    for (int j = 0; j < n; ++j) mu += emb_value(emb[e], train_rows + (size_t)j * h->row_words, tab.data());
    mu /= n;
    const EmbDim& d = emb[e];
    if (seg[e] > 0) {
      for (int i = 0; i < seg[e]; ++i) tab[d.off + i] -= mu;
    } else if (d.kind == BX_EMB_REAL) {
      tab[d.off + 1] = -mu;
    } else {
      tab[d.off + d.m] = -mu;
    }
  }
  // magnitude bound over the whole domain
  double bound = 0.0;
  for (int e = 0; e < E; ++e) {
    const EmbDim& d = emb[e];
    double mx = 0.0;
    if (seg[e] > 0) {
      for (int i = 0; i < seg[e]; ++i) mx = std::max(mx, std::fabs(tab[d.off + i]));
    } else if (d.kind == BX_EMB_REAL) {
      int kp = 0;
      while (kp + 1 < h->n_params && h->params[kp].word != d.word) ++kp;
      const bx_param_desc& p = h->params[kp];
      for (int i : {0, p.size - 1}) mx = std::max(mx, std::fabs(h->coord_host[p.coord + i] * tab[d.off] + tab[d.off + 1]));
    } else {
      mx = std::fabs(tab[d.off + d.m]);
      for (int i = 0; i < d.m; ++i) mx += std::fabs(tab[d.off + i]) * (d.m - 1);
    }
    bound += mx * mx;
  }
  if (!(bound <= 256.0)) return false;
  const int ks = (E + 3) / 4;
  *aug = E + 2 <= 4 * ks;
  planes.assign((size_t)4 * ks * npad, 0.0);
  yy.assign((size_t)npad, 0.0);
  for (int j = 0; j < n; ++j) {
    const uint32_t* row = train_rows + (size_t)j * h->row_words;
    double s2 = 0.0;
    for (int e = 0; e < E; ++e) {
      const double y = emb_value(emb[e], row, tab.data());
      planes[(size_t)e * npad + j] = -2.0 * y;
      s2 = std::fma(y, y, s2);
    }
    yy[j] = s2;
    if (*aug) {
      planes[(size_t)E * npad + j] = s2;
      planes[(size_t)(E + 1) * npad + j] = 1.0;
    }
  }
  return true;
}



extern "C" {
int bx_set_gp(bx_handle* h, const uint32_t* train_rows, int32_t n, const double* L,
              const double* alpha, double outputscale, const double* lengthscales, double y_mean,
              double y_std, void* stream) {
  int r = check_space(h);
  if (r) return r;
  if (n < 1) return fail(h, BX_ERR_ARG, "need at least one training point");
  if (!(outputscale > 0)) return fail(h, BX_ERR_ARG, "outputscale must be positive");
  cudaSetDevice(h->device);
  h->has_gp = false;  // until this call succeeds
  cudaStream_t s = (cudaStream_t)stream;
  const int D = h->n_params;
  std::vector<double> inv_l(D), inv_l2(D);
  std::vector<int32_t> disc_off(D, 0);
  std::vector<double> disc;
  for (int k = 0; k < D; ++k) {
    const double l = lengthscales[k];
    if (!(l > 0)) return fail(h, BX_ERR_ARG, "lengthscale %d must be positive", k);
    inv_l[k] = 1.0 / l;
    inv_l2[k] = 1.0 / (l * l);  // surrogate.py:222 1.0 / l ** 2
    const bx_param_desc& p = h->params[k];
    disc_off[k] = (int)disc.size();
    if (p.kind == BX_PERMUTATION) {
      const int m = p.size;
      int raw_max = m * m * m;  // >= every semimetric maximum
      for (int raw = 0; raw <= raw_max; ++raw) disc.push_back(((double)raw / p.raw_mx) * inv_l2[k]);
    } else if (p.kind == BX_CATEGORICAL) {
      disc.push_back(0.0);
      disc.push_back(inv_l2[k]);
    }
  }
  disc.push_back(0.0);
  h->gp_n = n;
  h->gp_ncols = ((n + 15) / 16) * 16;
  h->gp_rows = ((n + 1 + 15) / 16) * 16;
  h->gp_lda = h->gp_ncols;
  const size_t a_elems = (size_t)h->gp_rows * h->gp_lda;
  BX_CUDA(h, h->d_A.ensure(a_elems * 8));
  BX_CUDA(h, cudaMemsetAsync(h->d_A.p, 0, a_elems * 8, s));
  BX_CUDA(h, h->d_L.ensure((size_t)n * n * 8));
  BX_CUDA(h, cudaMemcpyAsync(h->d_L.p, L, (size_t)n * n * 8, cudaMemcpyHostToDevice, s));
  BX_CUDA(h, cudaMemcpyAsync(h->d_A.as<double>() + (size_t)n * h->gp_lda, alpha, (size_t)n * 8,
                             cudaMemcpyHostToDevice, s));
  BX_CUDA(h, h->d_train.ensure((size_t)n * h->row_words * 4));
  BX_CUDA(h, cudaMemcpyAsync(h->d_train.p, train_rows, (size_t)n * h->row_words * 4,
                             cudaMemcpyHostToDevice, s));
  BX_CUDA(h, h->d_inv_l.ensure(D * 8));
  BX_CUDA(h, cudaMemcpyAsync(h->d_inv_l.p, inv_l.data(), D * 8, cudaMemcpyHostToDevice, s));
  BX_CUDA(h, h->d_inv_l2.ensure(D * 8));
  BX_CUDA(h, cudaMemcpyAsync(h->d_inv_l2.p, inv_l2.data(), D * 8, cudaMemcpyHostToDevice, s));
  BX_CUDA(h, h->d_disc_tab.ensure(disc.size() * 8));
  BX_CUDA(h, cudaMemcpyAsync(h->d_disc_tab.p, disc.data(), disc.size() * 8, cudaMemcpyHostToDevice, s));
  BX_CUDA(h, h->d_disc_off.ensure(D * 4));
  BX_CUDA(h, cudaMemcpyAsync(h->d_disc_off.p, disc_off.data(), D * 4, cudaMemcpyHostToDevice, s));
  BX_CUDA(h, h->d_planes.ensure((size_t)D * n * 8));
  BX_CUDA(h, h->d_kmask.ensure((size_t)D * n * 16));
  BX_CUDA(h, launch_tri_inverse(h->d_L.as<double>(), n, h->d_A.as<double>(), h->gp_lda, s));
  BX_CUDA(h, launch_gp_planes(space_dev(h), h->d_train.as<uint32_t>(), n, h->d_inv_l.as<double>(),
                              h->d_planes.as<uint64_t>(), h->d_kmask.as<uint64_t>(), s));
  // register-resident path: n + 1 rows must fit 8 * 32 register rows and the smem budget
  h->use_fused = false;
  h->n_kendall = 0;
  for (int k = 0; k < D; ++k)
    if (h->params[k].kind == BX_PERMUTATION && h->params[k].metric == BX_KENDALL)
      h->kendall_param[h->n_kendall++] = k;
  const int mt = ((n + 1 + 15) / 16) * 2;  // m-tiles of 8 rows covering rows 0..n, even count
  if (!h->no_fused && 8 * mt <= fused_max_rows()) {
    const size_t smem = fused_smem_bytes(n, D, h->n_kendall, 8 * mt);
    if (smem <= 200 * 1024) {
      h->mt = mt;
      h->rows8 = 8 * mt;
      BX_CUDA(h, h->d_panels.ensure(panels_doubles(h->gp_ncols, h->rows8) * 8));
      BX_CUDA(h, launch_build_panels(h->d_A.as<double>(), h->gp_lda, h->gp_rows, h->gp_ncols,
                                     h->rows8, h->d_panels.as<double>(), s));
      h->use_fused = true;
    }
  }
  // tensor-core path: n < kTcMaxRows (n > 255 runs one column pass per 256 columns per tile) and
  // the shared-memory budget.  Distances on the FP64 tensor cores over the Euclidean embedding of W
  // (EmbDim) when every metric embeds and the centred coordinates stay small, else FMA distances.
  h->use_tc = false;
  h->tc_ks = 0;
  if (!h->no_tc && n < kTcMaxRows) {
    h->tc_emb.clear();
    h->tc_tab.clear();
    std::vector<double> planes, yy;
    const int nsl = (n + 31) / 32;
    bool dmma = !h->tc_no_dmma && !h->matern_precise &&
                build_embedding(h, train_rows, n, inv_l.data(), inv_l2.data(), 32 * nsl, h->tc_emb, h->tc_tab,
                                planes, yy, &h->tc_aug);
    const int E = (int)h->tc_emb.size();
    const int ks = dmma ? (E + 3) / 4 : 0;
    dmma = dmma && ks >= 1 && ks <= 8 &&
           tc_smem_bytes(n, D, h->n_kendall, h->row_words, ks, E, (int)h->tc_tab.size(), h->tc_aug, false) <= 227 * 1024;
    if (dmma || tc_smem_bytes(n, D, h->n_kendall, h->row_words, 0, 0, 0, false, false) <= 227 * 1024) {
      int Ex = 0;
      const double m = frexp(outputscale, &Ex);  // sigma < 2^Ex = sc
      if (m > 1.0 - ldexp(1.0, -20)) ++Ex;        // headroom: K* * 2^40 / sc < 2^40 - 2^20
      h->tc_nsl = nsl;
      h->tc_nch = n / 16 + 1;
      h->tc_kscale = ldexp(1.0, 40 - Ex);
      BX_CUDA(h, h->d_mdig.ensure(tc_mdig_bytes(n)));
      BX_CUDA(h, h->d_rowscale.ensure(2 * kTcMaxRows * 8));
      if (h->tc_nsl > 8)  // partial sums of rows >= 256: [CTA][16 nch - 256 rows][128 candidates]
        BX_CUDA(h, h->d_tc_part.ensure(tc_part_doubles(n, h->sm_count) * 8));
      if (dmma) {
        h->tc_ks = ks;
        BX_CUDA(h, upload(h->d_emb, h->tc_emb.data(), h->tc_emb.size()));
        BX_CUDA(h, upload(h->d_emb_tab, h->tc_tab.data(), h->tc_tab.size()));
        planes.resize((size_t)4 * ks * 32 * nsl, 0.0);  // k-rows beyond E (+2) are zero
        BX_CUDA(h, upload(h->d_emb_planes, planes.data(), planes.size()));
        BX_CUDA(h, upload(h->d_emb_yy, yy.data(), yy.size()));
      }
      h->use_tc = true;
      BX_CUDA(h, launch_build_mdig(h->d_A.as<double>(), h->gp_lda, n, ldexp(1.0, Ex),
                                   h->d_mdig.as<unsigned char>(), h->d_rowscale.as<double>(), dmma ? 1 : 0, s));
    }
  }
  BX_CUDA(h, cudaStreamSynchronize(s));  // host vectors above go out of scope
  if (!h->use_tc && !h->use_fused && score_smem_bytes(8, h->gp_ncols, D) > 227 * 1024)
    return fail(h, BX_ERR_UNSUPPORTED, "n = %d training points is beyond the posterior kernels (tensor-core path: n < %d)",
                n, kTcMaxRows);
  h->outputscale = outputscale;
  h->y_mean = y_mean;
  h->y_std = y_std;
  h->has_gp = true;
  return BX_OK;
}

int bx_set_forest(bx_handle* h, const int32_t* feature, const double* threshold, const int32_t* left,
                  const int32_t* right, const double* value, int32_t n_nodes, const int32_t* roots,
                  int32_t n_trees, int32_t max_depth, double constant) {
  int r = check_space(h);
  if (r) return r;
  cudaSetDevice(h->device);
  h->forest = ForestDev{};
  if (!std::isnan(constant)) {
    h->forest.has_trees = 0;
    h->forest.constant = constant;
    h->forest.n_trees = 0;
    h->has_forest = true;
    return BX_OK;
  }
  if (n_trees < 1 || !roots)
    return fail(h, BX_ERR_NO_TREES, "feasibility model has no trees");
  // Re-pack breadth-first per tree so that children are adjacent; keep values of every node.
  std::vector<RfNode> nodes;
  nodes.reserve(n_nodes);
  std::vector<int32_t> new_roots(n_trees);
  std::vector<int32_t> queue;
  for (int t = 0; t < n_trees; ++t) {
    const int root = roots[t];
    if (root < 0 || root >= n_nodes) return fail(h, BX_ERR_ARG, "root %d out of range", root);
    new_roots[t] = (int)nodes.size();
    nodes.push_back(RfNode{threshold[root], value[root], feature[root], -1});
    queue.assign(1, root);
    std::vector<int32_t> slot(1, new_roots[t]);
    for (size_t qi = 0; qi < queue.size(); ++qi) {
      const int old = queue[qi];
      const int me = slot[qi];
      if (feature[old] < 0) continue;
      if (feature[old] >= h->n_features)
        return fail(h, BX_ERR_ARG, "node %d splits on feature %d >= %d", old, feature[old], h->n_features);
      const int l = left[old], rr = right[old];
      if (l < 0 || l >= n_nodes || rr < 0 || rr >= n_nodes)
        return fail(h, BX_ERR_ARG, "node %d has a child out of range", old);
      nodes[me].child = (int)nodes.size();
      nodes.push_back(RfNode{threshold[l], value[l], feature[l], -1});
      nodes.push_back(RfNode{threshold[rr], value[rr], feature[rr], -1});
      queue.push_back(l);
      slot.push_back(nodes[me].child);
      queue.push_back(rr);
      slot.push_back(nodes[me].child + 1);
    }
  }
  BX_CUDA(h, upload(h->d_nodes, nodes.data(), nodes.size()));
  BX_CUDA(h, upload(h->d_roots, new_roots.data(), new_roots.size()));
  h->forest.nodes = h->d_nodes.as<RfNode>();
  h->forest.roots = h->d_roots.as<int32_t>();
  h->forest.n_trees = n_trees;
  h->forest.max_depth = max_depth;
  h->forest.has_trees = 1;
  h->forest.constant = 0.0;
  h->forest.coded = 0;
  h->has_forest = true;
  if (!h->no_coded_forest) {
    r = build_coded_forest(h, nodes, new_roots, max_depth);
    if (r) return r;
  }
  return BX_OK;
}

// Integer-coded node table for rf_coded_kernel (see CodedForestDev).  Falls back to the generic
// kernel (coded = 0) whenever an assumption does not hold: a leaf deeper than max_depth, a
// non-monotone coordinate table, or a field overflow.
int bx_clear_forest(bx_handle* h) {
  if (!h) return BX_ERR_ARG;
  h->has_forest = false;
  return BX_OK;
}

int bx_rf_fit(bx_handle* h, const double* X, const double* y, int32_t n, int32_t F, int32_t n_trees,
              const int32_t* boot, const int32_t* feats, const int32_t* n_drawn, int32_t max_draws, int32_t k,
              int32_t max_depth, int32_t max_nodes, int32_t* feature, double* threshold, int32_t* left,
              int32_t* right, double* value, int32_t* n_nodes, int32_t* status, void* stream) {
  if (!h) return BX_ERR_ARG;
  if (n < 1 || F < 1 || n_trees < 1 || k < 1 || k > F || max_draws < 1 || max_nodes < 1)
    return fail(h, BX_ERR_ARG, "bad rf_fit shape n=%d F=%d T=%d k=%d", n, F, n_trees, k);
  if (rf_fit_smem_bytes(n) > 200 * 1024) return fail(h, BX_ERR_UNSUPPORTED, "rf_fit: %d rows exceed the tile", n);
  cudaSetDevice(h->device);
  cudaStream_t s = (cudaStream_t)stream;
  const size_t nt = (size_t)n_trees * max_nodes;
  size_t off = 0;
  auto take = [&](size_t bytes) { const size_t o = off; off += (bytes + 255) & ~(size_t)255; return o; };
  const size_t oX = take((size_t)n * F * 8), oy = take((size_t)n * 8), ob = take((size_t)n_trees * n * 4),
               of = take((size_t)n_trees * max_draws * k * 4), od = take((size_t)n_trees * 4),
               oF = take(nt * 4), oT = take(nt * 8), oL = take(nt * 4), oR = take(nt * 4), oV = take(nt * 8),
               oN = take((size_t)n_trees * 4), oS = take((size_t)n_trees * 4),
               oK = take(rf_fit_stack_bytes(n_trees, max_nodes));
  BX_CUDA(h, h->d_fit.ensure(off));
  unsigned char* b = h->d_fit.as<unsigned char>();
  BX_CUDA(h, cudaMemcpyAsync(b + oX, X, (size_t)n * F * 8, cudaMemcpyHostToDevice, s));
  BX_CUDA(h, cudaMemcpyAsync(b + oy, y, (size_t)n * 8, cudaMemcpyHostToDevice, s));
  BX_CUDA(h, cudaMemcpyAsync(b + ob, boot, (size_t)n_trees * n * 4, cudaMemcpyHostToDevice, s));
  BX_CUDA(h, cudaMemcpyAsync(b + of, feats, (size_t)n_trees * max_draws * k * 4, cudaMemcpyHostToDevice, s));
  BX_CUDA(h, cudaMemcpyAsync(b + od, n_drawn, (size_t)n_trees * 4, cudaMemcpyHostToDevice, s));
  BX_CUDA(h, launch_rf_fit(reinterpret_cast<double*>(b + oX), reinterpret_cast<double*>(b + oy), n, F, n_trees,
                           reinterpret_cast<int32_t*>(b + ob), reinterpret_cast<int32_t*>(b + of),
                           reinterpret_cast<int32_t*>(b + od), max_draws, k, max_depth, max_nodes,
                           reinterpret_cast<int32_t*>(b + oF), reinterpret_cast<double*>(b + oT),
                           reinterpret_cast<int32_t*>(b + oL), reinterpret_cast<int32_t*>(b + oR),
                           reinterpret_cast<double*>(b + oV), reinterpret_cast<int32_t*>(b + oN),
                           reinterpret_cast<int32_t*>(b + oS), b + oK, s));
  BX_CUDA(h, cudaMemcpyAsync(feature, b + oF, nt * 4, cudaMemcpyDeviceToHost, s));
  BX_CUDA(h, cudaMemcpyAsync(threshold, b + oT, nt * 8, cudaMemcpyDeviceToHost, s));
  BX_CUDA(h, cudaMemcpyAsync(left, b + oL, nt * 4, cudaMemcpyDeviceToHost, s));
  BX_CUDA(h, cudaMemcpyAsync(right, b + oR, nt * 4, cudaMemcpyDeviceToHost, s));
  BX_CUDA(h, cudaMemcpyAsync(value, b + oV, nt * 8, cudaMemcpyDeviceToHost, s));
  BX_CUDA(h, cudaMemcpyAsync(n_nodes, b + oN, (size_t)n_trees * 4, cudaMemcpyDeviceToHost, s));
  BX_CUDA(h, cudaMemcpyAsync(status, b + oS, (size_t)n_trees * 4, cudaMemcpyDeviceToHost, s));
  BX_CUDA(h, cudaStreamSynchronize(s));
  return BX_OK;
}

}  // extern "C"

static int build_coded_forest(bx_handle* h, const std::vector<RfNode>& nodes,
                              const std::vector<int32_t>& roots, int max_depth) {
  const int D = h->n_params;
  std::vector<int32_t> slot_base(D), code_param, code_sub;
  for (int k = 0; k < D; ++k) {
    const bx_param_desc& p = h->params[k];
    slot_base[k] = (int)code_param.size();
    // one code per encode_configs column: a one-hot label and a permutation position each get
    // their own slot, so every non-real split is `code < cut`
    const int cnt = (p.kind == BX_PERMUTATION || p.kind == BX_CATEGORICAL) ? p.size : 1;
    for (int e = 0; e < cnt; ++e) {
      code_param.push_back(k);
      code_sub.push_back(e);
    }
    if (p.kind == BX_INTEGER || p.kind == BX_ORDINAL)
      for (int i = 1; i < p.size; ++i)
        if (!(h->coord_host[p.coord + i - 1] <= h->coord_host[p.coord + i])) return BX_OK;
  }
  if ((int)code_param.size() > 64) return BX_OK;
  // depth of every node (breadth-first layout: children after parents)
  std::vector<int> depth(nodes.size(), -1);
  for (int32_t r : roots) depth[r] = 0;
  for (size_t u = 0; u < nodes.size(); ++u) {
    if (depth[u] < 0) return BX_OK;
    if (nodes[u].feat >= 0) {
      if (depth[u] + 1 > max_depth) return BX_OK;  // traversal would stop on an internal node
      depth[nodes[u].child] = depth[nodes[u].child + 1] = depth[u] + 1;
    }
  }
  std::vector<uint64_t> coded(nodes.size());
  std::vector<uint32_t> leaf_idx(nodes.size(), 0);
  std::vector<double> leaf_val, real_thr;
  bool has_real = false;
  for (size_t u = 0; u < nodes.size(); ++u) {
    const RfNode& nd = nodes[u];
    uint64_t type, slot = 0, arg, child;
    if (nd.feat < 0) {
      // leaf: `code[0] >= 0xFFFFFF` never holds and the left child is the leaf itself, so a walk
      // that reached it stays; its value index lives in leaf_idx
      type = 2;
      arg = 0xFFFFFF;
      leaf_idx[u] = (uint32_t)leaf_val.size();
      leaf_val.push_back(nd.val);
      child = (uint64_t)u;
      coded[u] = arg | (type << 30) | (child << 32);
      continue;
    } else {
      const int k = h->feat_param_host[nd.feat], sub = h->feat_sub_host[nd.feat];
      const bx_param_desc& p = h->params[k];
      const double t = nd.thr;
      child = (uint64_t)(uint32_t)nd.child;
      if (p.kind == BX_REAL) {
        type = 1;
        slot = slot_base[k];
        arg = real_thr.size();
        real_thr.push_back(t);
        has_real = true;
      } else {
        type = 0;
        int cut1 = 0;  // number of code values whose feature value is <= t
        slot = slot_base[k] + ((p.kind == BX_PERMUTATION || p.kind == BX_CATEGORICAL) ? sub : 0);
        if (p.kind == BX_PERMUTATION) {
          for (int i = 0; i < p.size; ++i) cut1 += ((double)i <= t) ? 1 : 0;
        } else if (p.kind == BX_CATEGORICAL) {
          cut1 = (0.0 <= t ? 1 : 0) + (1.0 <= t ? 1 : 0);  // one-hot code in {0, 1}
        } else {
          for (int i = 0; i < p.size; ++i) cut1 += (h->coord_host[p.coord + i] <= t) ? 1 : 0;
        }
        arg = (uint64_t)cut1;
      }
    }
    if (arg >= (1u << 24) || slot >= 64) return BX_OK;
    coded[u] = arg | (slot << 24) | (type << 30) | (child << 32);
  }
  h->forest.cf.has_real = has_real ? 1 : 0;
  if (leaf_val.empty()) leaf_val.push_back(0.0);
  if (real_thr.empty()) real_thr.push_back(0.0);
  BX_CUDA(h, upload(h->d_cnodes, coded.data(), coded.size()));
  BX_CUDA(h, upload(h->d_leaf_val, leaf_val.data(), leaf_val.size()));
  BX_CUDA(h, upload(h->d_leaf_idx, leaf_idx.data(), leaf_idx.size()));
  h->forest.cf.leaf_idx = h->d_leaf_idx.as<uint32_t>();
  BX_CUDA(h, upload(h->d_real_thr, real_thr.data(), real_thr.size()));
  BX_CUDA(h, upload(h->d_code_param, code_param.data(), code_param.size()));
  BX_CUDA(h, upload(h->d_code_sub, code_sub.data(), code_sub.size()));
  CodedForestDev& cf = h->forest.cf;
  cf.nodes = h->d_cnodes.as<uint64_t>();
  cf.leaf_val = h->d_leaf_val.as<double>();
  cf.real_thr = h->d_real_thr.as<double>();
  cf.roots = h->forest.roots;
  cf.code_param = h->d_code_param.as<int32_t>();
  cf.code_sub = h->d_code_sub.as<int32_t>();
  cf.n_nodes = (int)coded.size();
  cf.n_codes = (int)code_param.size();
  cf.n_trees = h->forest.n_trees;
  cf.max_depth = max_depth;
  cf.n_leaves = (int)leaf_val.size();
  cf.nodes_in_smem = 0;  // decided at launch from the smem budget
  h->forest.coded = 1;

  // QuickScorer tables (QsForestDev): integer splits only, <= 64 leaves per tree
  QsForestDev& qs = h->forest.qs;
  qs = QsForestDev{};
  // real features: the code of a real parameter is the number of its distinct split thresholds
  // below the candidate's coordinate, so `x <= thr_j` (go left) is `code < j + 1` like every other
  // split (thresholds sorted per parameter; the device finds the code by binary search)
  std::vector<std::vector<double>> rthr(D);
  std::vector<int32_t> qcut(nodes.size(), 0);
  bool rthr_ok = true;
  if (has_real) {
    for (size_t u = 0; u < nodes.size(); ++u)
      if (nodes[u].feat >= 0 && h->params[h->feat_param_host[nodes[u].feat]].kind == BX_REAL)
        rthr[h->feat_param_host[nodes[u].feat]].push_back(nodes[u].thr);
    for (int k = 0; k < D; ++k) {
      std::sort(rthr[k].begin(), rthr[k].end());
      rthr[k].erase(std::unique(rthr[k].begin(), rthr[k].end()), rthr[k].end());
      if (rthr[k].size() >= 32768) rthr_ok = false;
    }
    for (size_t u = 0; u < nodes.size(); ++u)
      if (nodes[u].feat >= 0 && h->params[h->feat_param_host[nodes[u].feat]].kind == BX_REAL) {
        const std::vector<double>& tv = rthr[h->feat_param_host[nodes[u].feat]];
        qcut[u] = (int32_t)(std::lower_bound(tv.begin(), tv.end(), nodes[u].thr) - tv.begin()) + 1;
      }
  }
  std::vector<int32_t> roff(D, 0);
  std::vector<double> rflat;
  for (int k = 0; k < D; ++k) {
    roff[k] = (int32_t)rflat.size();
    rflat.insert(rflat.end(), rthr[k].begin(), rthr[k].end());
  }
  if (rflat.size() >= 65536) rthr_ok = false;
  if (rflat.empty()) rflat.push_back(0.0);
  if (rthr_ok) {
    const int S = (int)code_param.size();
    std::vector<int32_t> soff(S), range(S);
    int stride = 0;
    for (int c = 0; c < S; ++c) {
      const bx_param_desc& p = h->params[code_param[c]];
      range[c] = p.kind == BX_CATEGORICAL ? 2 : (p.kind == BX_REAL ? (int)rthr[code_param[c]].size() + 1 : p.size);
      soff[c] = stride;
      stride += range[c];
    }
    const int T = h->forest.n_trees;
    std::vector<uint64_t> mask((size_t)T * stride, ~0ull);
    std::vector<uint16_t> vid((size_t)T * 64, 0);
    std::vector<double> uval;
    bool ok = (size_t)T * stride <= ((size_t)1 << 24);  // host tables; the shared-memory budget is checked below
    std::vector<int32_t> lo(nodes.size()), mid(nodes.size()), hi(nodes.size());
    for (int t = 0; ok && t < T; ++t) {
      // left-to-right leaf numbering and subtree leaf ranges by an explicit post-order walk
      int leaves = 0;
      std::vector<std::pair<int, int>> stack{{roots[t], 0}};  // (node, phase)
      while (!stack.empty() && ok) {
        const int u = stack.back().first;
        const int phase = stack.back().second;
        const RfNode& nd = nodes[u];
        if (nd.feat < 0) {
          if (leaves >= 64) { ok = false; break; }
          const double v = nd.val;
          size_t id = 0;
          while (id < uval.size() && std::memcmp(&uval[id], &v, 8) != 0) ++id;
          if (id == uval.size()) uval.push_back(v);
          if (id > 65535) { ok = false; break; }
          vid[(size_t)t * 64 + leaves] = (uint16_t)id;
          lo[u] = leaves;
          hi[u] = ++leaves;
          stack.pop_back();
        } else if (phase == 0) {
          stack.back().second = 1;
          lo[u] = leaves;
          stack.push_back({nd.child, 0});
        } else if (phase == 1) {
          stack.back().second = 2;
          mid[u] = leaves;
          stack.push_back({nd.child + 1, 0});
        } else {
          hi[u] = leaves;
          // going right (code >= cut) rules out the left subtree's leaves [lo, mid)
          const uint32_t lo32 = (uint32_t)coded[u];
          const bool real_split = ((coded[u] >> 30) & 3u) == 1u;
          const int slot = (int)((lo32 >> 24) & 63u), cut = real_split ? qcut[u] : (int)(lo32 & 0xFFFFFFu);
          const uint64_t left = ((mid[u] - lo[u]) >= 64 ? ~0ull : ((1ull << (mid[u] - lo[u])) - 1)) << lo[u];
          for (int v = cut; v < range[slot]; ++v) mask[(size_t)t * stride + soff[slot] + v] &= ~left;
          stack.pop_back();
        }
      }
    }
    // one code per categorical parameter instead of one per one-hot feature: the mask of label L
    // is the AND over the parameter's one-hot codes of their masks at [L == sub] (fewer table
    // loads per candidate: one per parameter and tree)
    std::vector<int32_t> qparam, qsub, qsoff, qrange;
    if (ok) {
      std::vector<int> merged(h->n_params, -1), newidx(S, -1);
      for (int c = 0; c < S; ++c) {
        const bx_param_desc& p = h->params[code_param[c]];
        if (p.kind == BX_CATEGORICAL) {
          if (merged[code_param[c]] >= 0) continue;
          merged[code_param[c]] = (int)qparam.size();
          qparam.push_back(code_param[c]);
          qsub.push_back(-1);
          qrange.push_back(p.size);
        } else {
          newidx[c] = (int)qparam.size();
          qparam.push_back(code_param[c]);
          // a real code carries its threshold run: offset | count << 16 into qs.rthr
          qsub.push_back(p.kind == BX_REAL ? (int32_t)(roff[code_param[c]] | (rthr[code_param[c]].size() << 16))
                                           : code_sub[c]);
          qrange.push_back(range[c]);
        }
      }
      int stride2 = 0;
      for (size_t c = 0; c < qparam.size(); ++c) {
        qsoff.push_back(stride2);
        stride2 += qrange[c];
      }
      {
        std::vector<uint64_t> m2((size_t)T * stride2, ~0ull);
        for (int t = 0; t < T; ++t) {
          for (int c = 0; c < S; ++c) {
            const bx_param_desc& p = h->params[code_param[c]];
            if (p.kind == BX_CATEGORICAL) {
              const int mc = merged[code_param[c]];
              for (int L = 0; L < p.size; ++L)
                m2[(size_t)t * stride2 + qsoff[mc] + L] &=
                    mask[(size_t)t * stride + soff[c] + (L == code_sub[c] ? 1 : 0)];
            } else {
              const int c2 = newidx[c];
              for (int v = 0; v < range[c]; ++v)
                m2[(size_t)t * stride2 + qsoff[c2] + v] = mask[(size_t)t * stride + soff[c] + v];
            }
          }
        }
        mask.swap(m2);
        stride = stride2;
      }
    }
    // indirect slots: real parameters whose codes span many thresholds keep, per tree, only the few
    // distinct masks its own splits produce (runs of equal masks along the code) and a [code][tree]
    // u16 index into them
    // indirect slots (QsForestDev): a real parameter whose codes span many thresholds, and a
    // permutation of <= 5 elements as ONE slot coded by its rank (m! codes, the AND of its element
    // positions' masks) instead of m position slots
    struct Ind {
      int param, sub, range;
      std::vector<int> slots;  // the q-slots it replaces
    };
    std::vector<Ind> ind;
    std::vector<char> taken(qparam.size(), 0);
    std::vector<int32_t> dparam, dsub, dsoff, dparam2, dsub2, dmul;
    std::vector<std::pair<int, int>> dslots;
    int dstride = 0;
    if (ok) {
      for (size_t c = 0; c < qparam.size() && ind.size() < 4; ++c)
        if (h->params[qparam[c]].kind == BX_REAL && qrange[c] > 32) {
          ind.push_back(Ind{qparam[c], qsub[c], qrange[c], {(int)c}});
          taken[c] = 1;
        }
      for (int k = 0; k < h->n_params && ind.size() < 4; ++k) {
        const bx_param_desc& p = h->params[k];
        if (p.kind != BX_PERMUTATION || p.size > 5) continue;
        Ind d{k, -1, 1, std::vector<int>(p.size, -1)};
        for (int i = 2; i <= p.size; ++i) d.range *= i;
        for (size_t c = 0; c < qparam.size(); ++c)
          if (qparam[c] == k) d.slots[qsub[c]] = (int)c;  // slot of element e (code = its position)
        if (std::find(d.slots.begin(), d.slots.end(), -1) != d.slots.end()) continue;
        for (int c : d.slots) taken[c] = 1;
        ind.push_back(d);
      }
    }
    if (ok) {
      // indirect tables: rows (slot, code) x itpad u16 indices (itpad = 8 * odd: 16-byte rows)
      int itpad = (T + 7) / 8 * 8;
      if ((itpad / 8) % 2 == 0) itpad += 8;
      int irows = 0;
      for (const Ind& d : ind) irows += d.range;
      ok = (size_t)irows * itpad * 2 <= 96 * 1024;
      std::vector<uint16_t> iidx((size_t)std::max(irows, 1) * itpad, 0);
      std::vector<uint64_t> imask;
      qs.n_ind = (int)ind.size();
      int ioff = 0;
      for (size_t i = 0; i < ind.size() && ok; ++i) {
        const Ind& d = ind[i];
        qs.ind_param[i] = d.param;
        qs.ind_sub[i] = d.sub;
        qs.ind_off[i] = ioff;
        const bx_param_desc& p = h->params[d.param];
        for (int t = 0; t < T && ok; ++t) {
          int cur = -1;
          for (int v = 0; v < d.range; ++v) {
            uint64_t mv;
            if (p.kind == BX_REAL) {
              mv = mask[(size_t)t * stride + qsoff[d.slots[0]] + v];
            } else {  // permutation of rank v (Lehmer code): AND of the element-position masks
              int a[16], used = 0, r = v;
              for (int i = 0; i < p.size; ++i) {
                int f = 1;
                for (int j = 2; j <= p.size - 1 - i; ++j) f *= j;
                int c = r / f;
                r %= f;
                for (int e = 0; e < p.size; ++e)
                  if (!((used >> e) & 1) && c-- == 0) {
                    a[i] = e;
                    used |= 1 << e;
                    break;
                  }
              }
              mv = ~0ull;
              for (int i = 0; i < p.size; ++i) mv &= mask[(size_t)t * stride + qsoff[d.slots[a[i]]] + i];
            }
            if (cur < 0 || imask[cur] != mv) {
              cur = -1;
              for (size_t u = imask.size() > 64 ? imask.size() - 64 : 0; u < imask.size(); ++u)
                if (imask[u] == mv) cur = (int)u;  // reuse a recent equal mask (same tree)
              if (cur < 0) {
                cur = (int)imask.size();
                imask.push_back(mv);
              }
            }
            if (cur > 65535) { ok = false; break; }
            iidx[(size_t)(ioff + v) * itpad + t] = (uint16_t)cur;
          }
        }
        ioff += d.range;
      }
      if (imask.empty()) imask.push_back(~0ull);
      int tpad = (T + 7) / 8 * 8 + 1;
      // shared memory left for the direct table next to everything else rf_qs_summary_kernel holds
      const size_t other = ((size_t)std::max<size_t>(uval.size(), 1) * 8) + (((size_t)T * 64 * 2 + 15) & ~(size_t)15) +
                           (((size_t)std::max(irows, 1) * itpad * 2 + 15) & ~(size_t)15) + imask.size() * 8 +
                           32 * sizeof(Partial) + 2048;
      const size_t budget = std::min<size_t>(160 * 1024, other < 227 * 1024 ? 227 * 1024 - other : 0);
      // direct slots, small ones paired: a pair (a, b) is one slot with code = code_a * range_b +
      // code_b whose rows are the ANDs of the two slots' rows (one table walk instead of two);
      // greedily the two smallest while the product stays <= 64 rows and the summary kernel's
      // shared memory (tables + indirect tables + partials) stays within 227 KB
      std::vector<int> single;  // dslots: (q-slot a, q-slot b or -1)
      for (size_t c = 0; c < qparam.size(); ++c)
        if (!taken[c]) single.push_back((int)c);
      std::sort(single.begin(), single.end(), [&](int x, int y) { return qrange[x] < qrange[y]; });
      int rows_total = 0;
      for (int c : single) rows_total += qrange[c];
      size_t i0 = 0;
      while (i0 + 1 < single.size()) {
        const int a = single[i0], b = single[i0 + 1];
        const int grown = rows_total - qrange[a] - qrange[b] + qrange[a] * qrange[b];
        if (qrange[a] * qrange[b] > 64 || (size_t)tpad * grown * 8 > budget) break;
        dslots.push_back({a, b});
        rows_total = grown;
        i0 += 2;
      }
      for (; i0 < single.size(); ++i0) dslots.push_back({single[i0], -1});
      std::sort(dslots.begin(), dslots.end());
      for (const auto& ds : dslots) {
        dparam.push_back(qparam[ds.first]);
        dsub.push_back(qsub[ds.first]);
        dparam2.push_back(ds.second >= 0 ? qparam[ds.second] : -1);
        dsub2.push_back(ds.second >= 0 ? qsub[ds.second] : 0);
        dmul.push_back(ds.second >= 0 ? qrange[ds.second] : 1);
        dsoff.push_back(dstride);
        dstride += qrange[ds.first] * (ds.second >= 0 ? qrange[ds.second] : 1);
      }
      ok = ok && (size_t)tpad * dstride * 8 <= 160 * 1024;
      if (uval.empty()) uval.push_back(0.0);
      // direct slots transposed to [slot value][tree] so a group of 8 trees is one 64-byte run per
      // slot; odd row length (in 8-byte words): the <= 16 distinct code-value rows a half-warp reads
      // with 8-byte loads fall in 16 distinct bank pairs (groups of 8 trees read t .. t+7)
      std::vector<uint64_t> mt((size_t)std::max(dstride, 1) * tpad, ~0ull);
      for (size_t d = 0; d < dslots.size(); ++d) {
        const int a = dslots[d].first, b = dslots[d].second;
        const int rb = b >= 0 ? qrange[b] : 1;
        for (int va = 0; va < qrange[a]; ++va)
          for (int vb = 0; vb < rb; ++vb)
            for (int t = 0; t < T; ++t)
              mt[(size_t)(dsoff[d] + va * rb + vb) * tpad + t] =
                  mask[(size_t)t * stride + qsoff[a] + va] & (b >= 0 ? mask[(size_t)t * stride + qsoff[b] + vb] : ~0ull);
      }
      if (ok) {
        qs.tpad = tpad;
        BX_CUDA(h, upload(h->d_qmask, mt.data(), mt.size()));
        BX_CUDA(h, upload(h->d_qvid, vid.data(), vid.size()));
        BX_CUDA(h, upload(h->d_quval, uval.data(), uval.size()));
        if (dsoff.empty()) {
          dsoff.push_back(0); dparam.push_back(0); dsub.push_back(0);
          dparam2.push_back(-1); dsub2.push_back(0); dmul.push_back(1);
        }
        BX_CUDA(h, upload(h->d_qsoff, dsoff.data(), dsoff.size()));
        BX_CUDA(h, upload(h->d_qcode_param, dparam.data(), dparam.size()));
        BX_CUDA(h, upload(h->d_qcode_sub, dsub.data(), dsub.size()));
        BX_CUDA(h, upload(h->d_qcode_param2, dparam2.data(), dparam2.size()));
        BX_CUDA(h, upload(h->d_qcode_sub2, dsub2.data(), dsub2.size()));
        BX_CUDA(h, upload(h->d_qcode_mul, dmul.data(), dmul.size()));
        qs.code_param2 = h->d_qcode_param2.as<int32_t>();
        qs.code_sub2 = h->d_qcode_sub2.as<int32_t>();
        qs.code_mul = h->d_qcode_mul.as<int32_t>();
        BX_CUDA(h, upload(h->d_qrthr, rflat.data(), rflat.size()));
        BX_CUDA(h, upload(h->d_qiidx, iidx.data(), iidx.size()));
        BX_CUDA(h, upload(h->d_qimask, imask.data(), imask.size()));
        qs.rthr = h->d_qrthr.as<double>();
        qs.has_real = has_real ? 1 : 0;
        qs.mask = h->d_qmask.as<uint64_t>();
        qs.vid = h->d_qvid.as<uint16_t>();
        qs.uval = h->d_quval.as<double>();
        qs.soff = h->d_qsoff.as<int32_t>();
        qs.code_param = h->d_qcode_param.as<int32_t>();
        qs.code_sub = h->d_qcode_sub.as<int32_t>();
        qs.iidx = h->d_qiidx.as<uint16_t>();
        qs.imask = h->d_qimask.as<uint64_t>();
        qs.itpad = itpad;
        qs.n_iidx_rows = irows;
        qs.n_imask = (int)imask.size();
        qs.n_trees = T;
        qs.n_codes = dstride > 0 ? (int)dparam.size() : 0;
        qs.stride = dstride;
        qs.n_uvals = (int)uval.size();
        qs.enabled = h->no_qs_forest ? 0 : 1;
        if (getenv("BX_QS_INFO"))  // development aid: table geometry
          fprintf(stderr, "qs: trees %d codes %d (+%d indirect: %d rows, %d masks) stride %d tpad %d uvals %d masks %zu B summary smem %zu B\n",
                  T, qs.n_codes, qs.n_ind, irows, qs.n_imask, dstride, tpad, qs.n_uvals, (size_t)dstride * tpad * 8,
                  (size_t)qs_summary_smem_bytes(qs));
      }
    }
  }
  return BX_OK;
}

