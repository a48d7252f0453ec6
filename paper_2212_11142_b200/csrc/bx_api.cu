// bx_api.cu — the C ABI (include/bx_sm100.h): handle lifecycle and options, the space tables,
// the evaluated set, chain-of-trees and constraint uploads, the packed wire format and the
// integer entry points (neighbours, chain-of-trees / constraint masks).  Model uploads are in
// bx_model.cu, scoring in bx_score.cu, the marginal likelihood in bx_lml.cu.
#include "bx_handle.cuh"

cudaError_t bx::set_smem_once(const void* fn, int bytes) {
  static std::mutex mu;
  static std::unordered_map<const void*, int> done;
  std::lock_guard<std::mutex> lock(mu);
  int& have = done[fn];
  if (bytes <= have) return cudaSuccess;
  const cudaError_t e = cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize, bytes);
  if (e == cudaSuccess) have = bytes;
  return e;
}


extern "C" {

int bx_abi_version(void) { return BX_ABI_VERSION; }

bx_handle* bx_create(int device) {
  if (cudaSetDevice(device) != cudaSuccess) return nullptr;
  bx_handle* h = new (std::nothrow) bx_handle();
  if (!h) return nullptr;
  h->device = device;
  const char* generic = getenv("BX_FOREST_GENERIC");
  h->no_coded_forest = generic && generic[0] == '1';
  cudaDeviceGetAttribute(&h->sm_count, cudaDevAttrMultiProcessorCount, device);
  cudaStreamCreateWithFlags(&h->copy_stream, cudaStreamNonBlocking);
  cudaEventCreateWithFlags(&h->ev_copy, cudaEventDisableTiming);
  cudaEventCreateWithFlags(&h->ev_done, cudaEventDisableTiming);
  for (int i = 0; i < 5; ++i) cudaEventCreate(&h->ev_t[i]);
  const char* gpg = getenv("BX_GP_GENERIC");
  h->no_fused = gpg && gpg[0] == '1';
  if (const char* dbg = getenv("BX_TC_DEBUG")) h->tc_debug = atoi(dbg);
  h->tc_trace = getenv("BX_TC_TRACE") != nullptr;
  if (const char* ln = getenv("BX_LML_NARROW")) h->lml_narrow = ln[0] == '1';
  if (const char* sm = getenv("BX_LML_SMALL_MAX")) h->lml_small_max = atoi(sm);
  if (const char* nd = getenv("BX_TC_NO_DMMA")) h->tc_no_dmma = nd[0] == '1';
  const char* fw = getenv("BX_FOREST_WALK");
  h->no_qs_forest = fw && fw[0] == '1';
  const char* dm = getenv("BX_GP_DMMA");
  h->no_tc = h->no_fused || (dm && dm[0] == '1');
  const char* mp = getenv("BX_MATERN_PRECISE");
  h->matern_precise = mp && mp[0] == '1';
  cudaStreamCreateWithFlags(&h->rf_stream, cudaStreamNonBlocking);
  cudaEventCreateWithFlags(&h->ev_fork, cudaEventDisableTiming);
  cudaEventCreateWithFlags(&h->ev_rf, cudaEventDisableTiming);
  return h;
}

void bx_destroy(bx_handle* h) {
  if (!h) return;
  cudaSetDevice(h->device);
  DevBuf* bufs[] = {&h->d_params, &h->d_coord, &h->d_rank, &h->d_feat_param, &h->d_feat_sub,
                    &h->d_slot_param, &h->d_slot_move, &h->d_A, &h->d_L, &h->d_planes,
                    &h->d_kmask, &h->d_inv_l, &h->d_inv_l2, &h->d_disc_tab, &h->d_disc_off,
                    &h->d_train, &h->d_nodes, &h->d_roots, &h->d_ev_rows, &h->d_ev_table,
                    &h->d_g_kind, &h->d_g_pbeg, &h->d_g_params, &h->d_g_root,
                    &h->d_child_begin, &h->d_child_count, &h->d_child_value, &h->d_prog_begin, &h->d_code,
                    &h->d_consts, &h->d_vtag, &h->d_vint, &h->d_vflt, &h->d_voff, &h->d_str_id,
                    &h->d_fault, &h->d_probs, &h->d_partials, &h->d_summary, &h->d_lml_scratch,
                    &h->d_cnodes, &h->d_leaf_val,
                    &h->d_real_thr, &h->d_code_param, &h->d_code_sub, &h->d_leaf_idx,
                    &h->d_qmask, &h->d_qvid, &h->d_quval, &h->d_qsoff, &h->d_qcode_param,
                    &h->d_qcode_sub, &h->d_qrthr, &h->d_qiidx, &h->d_qimask,
                    &h->d_qcode_param2, &h->d_qcode_sub2, &h->d_qcode_mul};
  for (DevBuf* b : bufs) b->release();
  if (h->copy_stream) cudaStreamDestroy(h->copy_stream);
  if (h->ev_copy) cudaEventDestroy(h->ev_copy);
  if (h->ev_done) cudaEventDestroy(h->ev_done);
  for (int i = 0; i < 5; ++i)
    if (h->ev_t[i]) cudaEventDestroy(h->ev_t[i]);
  h->d_panels.release();
  h->d_pool.release();
  h->d_ready.release();
  h->d_emb.release();
  h->d_packed.release();
  h->d_climb.release();
  h->d_fit.release();
  h->d_emb_tab.release();
  h->d_emb_planes.release();
  h->d_emb_yy.release();
  if (h->h_ones) cudaFreeHost(h->h_ones);
  if (h->h_climb_flag) cudaFreeHost(h->h_climb_flag);
  if (h->h_lml_stage) cudaFreeHost(h->h_lml_stage);
  h->d_lml_stage.release();
  h->d_mdig.release();
  h->d_rowscale.release();
  h->d_tc_part.release();
  h->d_factor.release();
  h->d_ei.release();
  h->d_grad_scratch.release();
  h->d_leaf_count.release();
  h->d_gen_rows.release();
  if (h->rf_stream) cudaStreamDestroy(h->rf_stream);
  if (h->ev_fork) cudaEventDestroy(h->ev_fork);
  if (h->ev_rf) cudaEventDestroy(h->ev_rf);
  delete h;
}

const char* bx_last_error(bx_handle* h) { return h ? h->err.c_str() : "null handle"; }

int bx_device_sm_count(bx_handle* h) { return h ? h->sm_count : 0; }

int bx_gp_kernel(bx_handle* h) {
  if (!h) return BX_GP_GENERIC;
  return h->use_tc ? BX_GP_TENSOR : h->use_fused ? BX_GP_DMMA : BX_GP_GENERIC;
}

int bx_gp_distance_ksteps(bx_handle* h) { return h && h->use_tc ? h->tc_ks : 0; }
int bx_gp_embedding_dims(bx_handle* h) { return h && h->use_tc && h->tc_ks ? (int)h->tc_emb.size() : 0; }

int bx_set_option(bx_handle* h, int32_t option, int32_t value) {
  if (!h) return BX_ERR_ARG;
  if (option == BX_OPT_LML_NARROW) {
    h->lml_narrow = value != 0;
    return BX_OK;
  }
  return fail(h, BX_ERR_ARG, "unknown option %d", option);
}

int bx_packed_row_words(bx_handle* h) { return h && h->has_space ? h->pack.pw : 0; }

int bx_pack_rows(bx_handle* h, const uint32_t* rows, int64_t q, uint32_t* packed) {
  int r = check_space(h);
  if (r) return r;
  if (q < 0 || (q > 0 && (!rows || !packed))) return fail(h, BX_ERR_ARG, "bad buffers");
  for (int64_t i = 0; i < q; ++i) pack_row(h->pack, rows + (size_t)i * h->row_words, packed + (size_t)i * h->pack.pw);
  return BX_OK;
}

int bx_unpack_rows(bx_handle* h, const uint32_t* packed, int64_t q, uint32_t* rows) {
  int r = check_space(h);
  if (r) return r;
  if (q < 0 || (q > 0 && (!rows || !packed))) return fail(h, BX_ERR_ARG, "bad buffers");
  for (int64_t i = 0; i < q; ++i)
    unpack_row(h->pack, packed + (size_t)i * h->pack.pw, rows + (size_t)i * h->row_words, h->row_words);
  return BX_OK;
}

int bx_set_space(bx_handle* h, const bx_param_desc* params, int32_t n_params, int32_t row_words,
                 const double* coord_lut, int32_t coord_len, const int32_t* rank_lut,
                 int32_t rank_len, int32_t n_features) {
  if (!h) return BX_ERR_ARG;
  if (n_params < 1 || n_params > BX_MAX_PARAMS)
    return fail(h, BX_ERR_UNSUPPORTED, "n_params=%d outside [1, %d]", n_params, BX_MAX_PARAMS);
  if (row_words < 1 || row_words > BX_MAX_ROW_WORDS)
    return fail(h, BX_ERR_UNSUPPORTED, "row_words=%d outside [1, %d]", row_words, BX_MAX_ROW_WORDS);
  cudaSetDevice(h->device);
  std::vector<int32_t> fparam, fsub, sparam, smove;
  for (int k = 0; k < n_params; ++k) {
    const bx_param_desc& p = params[k];
    int nw = p.kind == BX_REAL ? 4 : (p.kind == BX_PERMUTATION ? 2 : 1);
    if (p.word < 0 || p.word + nw > row_words)
      return fail(h, BX_ERR_ARG, "parameter %d overflows the row (%d words)", k, row_words);
    if (p.kind == BX_PERMUTATION) {
      if (p.size < 2 || p.size > BX_MAX_PERM)
        return fail(h, BX_ERR_UNSUPPORTED, "permutation size %d outside [2, 16]", p.size);
      if ((p.word & 1) != 0) return fail(h, BX_ERR_ARG, "permutation %d not 8-byte aligned", k);
      for (int e = 0; e < p.size; ++e) { fparam.push_back(k); fsub.push_back(e); }
      for (int m = 0; m < p.size * (p.size - 1) / 2; ++m) { sparam.push_back(k); smove.push_back(m); }
    } else if (p.kind == BX_CATEGORICAL) {
      for (int e = 0; e < p.size; ++e) { fparam.push_back(k); fsub.push_back(e); }
      for (int m = 0; m < p.size - 1; ++m) { sparam.push_back(k); smove.push_back(m); }
    } else {
      if (p.kind == BX_REAL && (p.word & 1) != 0)
        return fail(h, BX_ERR_ARG, "real parameter %d not 8-byte aligned", k);
      fparam.push_back(k);
      fsub.push_back(0);
      sparam.push_back(k); smove.push_back(0);
      sparam.push_back(k); smove.push_back(1);
    }
  }
  if ((int)fparam.size() != n_features)
    return fail(h, BX_ERR_ARG, "n_features=%d but the parameters imply %d", n_features,
                (int)fparam.size());
  BX_CUDA(h, upload(h->d_params, params, n_params));
  BX_CUDA(h, upload(h->d_coord, coord_lut, (size_t)coord_len));
  BX_CUDA(h, upload(h->d_rank, rank_lut, (size_t)rank_len));
  BX_CUDA(h, upload(h->d_feat_param, fparam.data(), fparam.size()));
  BX_CUDA(h, upload(h->d_feat_sub, fsub.data(), fsub.size()));
  BX_CUDA(h, upload(h->d_slot_param, sparam.data(), sparam.size()));
  BX_CUDA(h, upload(h->d_slot_move, smove.data(), smove.size()));
  h->params.assign(params, params + n_params);
  h->feat_param_host = fparam;
  h->feat_sub_host = fsub;
  h->coord_host.assign(coord_lut, coord_lut + coord_len);
  h->rank_host.assign(rank_lut, rank_lut + rank_len);
  h->n_params = n_params;
  h->row_words = row_words;
  h->n_features = n_features;
  h->n_slots = (int)sparam.size();
  // packed wire format: parameters in order at their bit widths
  {
    PackSpec& ps = h->pack;
    ps = PackSpec{};
    ps.n = n_params;
    int bit = 0;
    for (int k = 0; k < n_params; ++k) {
      const bx_param_desc& p = params[k];
      PackParam& q = ps.p[k];
      q.kind = p.kind;
      q.word = p.word;
      q.bit = bit;
      q.lo = p.lo;
      q.hi = p.hi;
      if (p.kind == BX_REAL) {
        q.carry_coord = p.is_log ? 1 : 0;
        q.bits = q.carry_coord ? 128 : 64;
      } else if (p.kind == BX_PERMUTATION) {
        q.bits = 4 * p.size;
      } else {
        int b = 1;
        while ((1 << b) < p.size) ++b;
        q.bits = b;
      }
      bit += q.bits;
    }
    ps.pw = (bit + 31) / 32;
  }
  h->has_space = true;
  // every other piece of model state is expressed in the old space's rows / features / domain
  // indices: drop it, so a caller that forgets to re-set it gets BX_ERR_STATE, not stale reads
  h->has_gp = false;
  h->has_forest = false;
  h->has_cot = false;
  h->has_leaf_count = false;
  h->has_constraints = false;
  h->ev_count = 0;
  return BX_OK;
}

int bx_set_evaluated(bx_handle* h, const uint32_t* rows, int32_t count) {
  int r = check_space(h);
  if (r) return r;
  cudaSetDevice(h->device);
  const int W = h->row_words;
  h->ev_count = count > 0 ? count : 0;
  if (h->ev_count == 0) return BX_OK;
  int size = 16;
  while (size < 2 * count) size <<= 1;
  std::vector<int32_t> table(size, -1);
  for (int i = 0; i < count; ++i) {
    const uint32_t* row = rows + (size_t)i * W;
    int slot = (int)(host_row_hash(row, W) & (uint64_t)(size - 1));
    while (table[slot] >= 0) {
      if (std::memcmp(rows + (size_t)table[slot] * W, row, W * 4) == 0) break;  // duplicate
      slot = (slot + 1) & (size - 1);
    }
    if (table[slot] < 0) table[slot] = i;
  }
  BX_CUDA(h, upload(h->d_ev_rows, rows, (size_t)count * W));
  BX_CUDA(h, upload(h->d_ev_table, table.data(), table.size()));
  h->ev_mask = size - 1;
  return BX_OK;
}

int bx_set_cot(bx_handle* h, int32_t n_groups, const int32_t* group_kind,
               const int32_t* group_param_begin, const int32_t* group_params,
               const int32_t* group_root, int32_t n_nodes, const int32_t* child_begin,
               const int32_t* child_count, const int32_t* node_value,
               const int64_t* node_leaf_count) {
  int r = check_space(h);
  if (r) return r;
  if (n_groups < 0 || n_nodes < 0) return fail(h, BX_ERR_ARG, "bad chain-of-trees sizes");
  cudaSetDevice(h->device);
  const int np = group_param_begin[n_groups];
  for (int g = 0; g < n_groups; ++g) {
    if (group_kind[g] == 0 && (group_root[g] < 0 || group_root[g] >= n_nodes))
      return fail(h, BX_ERR_ARG, "group %d root out of range", g);
  }
  for (int u = 0; u < n_nodes; ++u)
    if (child_count[u] < 0 || child_begin[u] < 0 || child_begin[u] + child_count[u] > n_nodes)
      return fail(h, BX_ERR_ARG, "node %d children out of range", u);
  BX_CUDA(h, upload(h->d_g_kind, group_kind, n_groups));
  BX_CUDA(h, upload(h->d_g_pbeg, group_param_begin, n_groups + 1));
  BX_CUDA(h, upload(h->d_g_params, group_params, np));
  BX_CUDA(h, upload(h->d_g_root, group_root, n_groups));
  BX_CUDA(h, upload(h->d_child_begin, child_begin, n_nodes));
  BX_CUDA(h, upload(h->d_child_count, child_count, n_nodes));
  BX_CUDA(h, upload(h->d_child_value, node_value, n_nodes));
  h->cot.n_groups = n_groups;
  h->cot.group_kind = h->d_g_kind.as<int32_t>();
  h->cot.group_param_begin = h->d_g_pbeg.as<int32_t>();
  h->cot.group_params = h->d_g_params.as<int32_t>();
  h->cot.group_root = h->d_g_root.as<int32_t>();
  h->cot.child_begin = h->d_child_begin.as<int32_t>();
  h->cot.child_count = h->d_child_count.as<int32_t>();
  h->cot.node_value = h->d_child_value.as<int32_t>();
  h->has_leaf_count = node_leaf_count != nullptr;
  if (node_leaf_count) BX_CUDA(h, upload(h->d_leaf_count, node_leaf_count, n_nodes));
  h->has_cot = true;
  return BX_OK;
}

int bx_clear_cot(bx_handle* h) {
  if (!h) return BX_ERR_ARG;
  h->has_cot = false;
  return BX_OK;
}

int bx_set_constraints(bx_handle* h, int32_t n_constraints, const int32_t* prog_begin,
                       const int32_t* code, int32_t code_len, const double* consts,
                       int32_t n_consts, const int32_t* value_tag, const int64_t* value_int,
                       const double* value_float, const int32_t* value_str, int32_t n_values) {
  int r = check_space(h);
  if (r) return r;
  if (n_constraints < 0 || code_len < 0 || n_consts < 0)
    return fail(h, BX_ERR_ARG, "bad constraint program sizes");
  cudaSetDevice(h->device);
  const int D = h->n_params;
  std::vector<int32_t> voff(D);
  int total = 0;
  for (int k = 0; k < D; ++k) {
    voff[k] = total;
    const bx_param_desc& p = h->params[k];
    total += (p.kind == BX_REAL || p.kind == BX_PERMUTATION) ? 0 : p.size;
  }
  if (total != n_values)
    return fail(h, BX_ERR_ARG, "constraint value tables: expected %d entries, got %d", total, n_values);
  if (n_constraints > 0 && prog_begin[n_constraints] != code_len)
    return fail(h, BX_ERR_ARG, "prog_begin[n] != code_len");
  const int lit = n_consts;
  std::vector<int32_t> vtag(value_tag, value_tag + total), sid(value_str, value_str + total);
  std::vector<int64_t> vint(value_int, value_int + total);
  std::vector<double> vflt(value_float, value_float + total);
  vtag.push_back(0); sid.push_back(0); vint.push_back(0); vflt.push_back(0.0);
  BX_CUDA(h, upload(h->d_prog_begin, prog_begin, n_constraints + 1));
  BX_CUDA(h, upload(h->d_code, code, code_len));
  BX_CUDA(h, upload(h->d_consts, consts, lit));
  BX_CUDA(h, upload(h->d_vtag, vtag.data(), vtag.size()));
  BX_CUDA(h, upload(h->d_vint, vint.data(), vint.size()));
  BX_CUDA(h, upload(h->d_vflt, vflt.data(), vflt.size()));
  BX_CUDA(h, upload(h->d_voff, voff.data(), voff.size()));
  BX_CUDA(h, upload(h->d_str_id, sid.data(), sid.size()));
  BX_CUDA(h, h->d_fault.ensure(16));
  BX_CUDA(h, cudaMemset(h->d_fault.p, 0, 16));
  h->cons.n_constraints = n_constraints;
  h->cons.prog_begin = h->d_prog_begin.as<int32_t>();
  h->cons.code = h->d_code.as<int32_t>();
  h->cons.consts = h->d_consts.as<double>();
  h->cons.vtag = h->d_vtag.as<int32_t>();
  h->cons.vint = h->d_vint.as<int64_t>();
  h->cons.vflt = h->d_vflt.as<double>();
  h->cons.voff = h->d_voff.as<int32_t>();
  h->cons.str_id = h->d_str_id.as<int32_t>();
  h->cons.fault = h->d_fault.as<int32_t>();
  h->has_constraints = true;
  return BX_OK;
}

// ---- scoring --------------------------------------------------------------------------------

// Summary pass over the EI / probability buffers of the last fused scoring launch.
int bx_neighbor_slots(bx_handle* h) { return (h && h->has_space) ? h->n_slots : -1; }

int bx_neighbors(bx_handle* h, const uint32_t* rows, int32_t count, int32_t use_cot,
                 uint32_t* out_rows, uint8_t* out_valid, void* stream) {
  int r = check_space(h);
  if (r) return r;
  if (use_cot && !h->has_cot) return fail(h, BX_ERR_STATE, "bx_set_cot has not been called");
  cudaSetDevice(h->device);
  BX_CUDA(h, launch_neighbors(space_dev(h), use_cot ? &h->cot : nullptr, rows, count, out_rows,
                              out_valid, (cudaStream_t)stream));
  return BX_OK;
}

int bx_cot_contains(bx_handle* h, const uint32_t* rows, int64_t q, uint8_t* mask, void* stream) {
  int r = check_space(h);
  if (r) return r;
  if (!h->has_cot) return fail(h, BX_ERR_STATE, "bx_set_cot has not been called");
  cudaSetDevice(h->device);
  BX_CUDA(h, launch_cot_contains(space_dev(h), h->cot, rows, q, mask, (cudaStream_t)stream));
  return BX_OK;
}

int bx_constraints_eval(bx_handle* h, const uint32_t* rows, int64_t q, uint8_t* mask, void* stream) {
  int r = check_space(h);
  if (r) return r;
  if (!h->has_constraints) return fail(h, BX_ERR_STATE, "bx_set_constraints has not been called");
  cudaSetDevice(h->device);
  cudaStream_t s = (cudaStream_t)stream;
  BX_CUDA(h, cudaMemsetAsync(h->d_fault.p, 0, 4, s));
  BX_CUDA(h, launch_constraints(space_dev(h), h->cons, rows, q, mask, s));
  int fault = 0;
  BX_CUDA(h, cudaMemcpyAsync(&fault, h->d_fault.p, 4, cudaMemcpyDeviceToHost, s));
  BX_CUDA(h, cudaStreamSynchronize(s));
  if (fault)
    return fail(h, BX_ERR_UNSUPPORTED,
                "constraint arithmetic left the exact int64/2^53 envelope of the device evaluator");
  return BX_OK;
}

}  // extern "C"
