"""Device-resident acquisition state and typed wrappers around every libbx_sm100 entry point.

`Scorer` owns one native handle on one CUDA device.  It uploads the per-iteration model state
(space tables, GP posterior, forest, evaluated set, chain of trees, constraint bytecode) and runs
the hot-path kernels on torch-allocated device buffers, on torch's current stream.  All model
objects are read through the attributes the reference defines, so the reference's own `GPModel`,
`FeasibilityModel`, `ChainOfTrees` and `SearchSpace` are accepted as they are.
"""
from __future__ import annotations

import ctypes as C
import math
from dataclasses import dataclass

import numpy as np
import torch

from . import _native as N
from .constraints import CotTables, Program, flatten_cot
from .layout import SpaceLayout


def _ptr(a) -> C.c_void_p:
    if isinstance(a, torch.Tensor):
        return C.c_void_p(a.data_ptr())
    if isinstance(a, np.ndarray):
        return a.ctypes.data_as(C.c_void_p)
    if a is None:
        return C.c_void_p(0)
    return C.c_void_p(a)


def _host(a, dtype) -> np.ndarray:
    return np.ascontiguousarray(np.asarray(a, dtype=dtype))


@dataclass(slots=True)
class Candidate:
    value: float
    prob: float
    index: int
    row: np.ndarray  # uint32 [row_words]


@dataclass
class Summary:
    n_scored: int
    n_finite: int
    top: list          # [Candidate], stable argsort(-values)[:k] with -inf excluded
    best: Candidate | None       # tracker over values (unevaluated, finite)
    best_prob: Candidate | None  # tracker over probabilities (unevaluated)


_CAND_SIZE, _TOP_OFF, _ROW_OFF = C.sizeof(N.Cand), N.ScoreSummary.top.offset, N.Cand.row.offset


def _cand(c: N.Cand, words: int) -> Candidate | None:
    if c.index < 0:
        return None
    return Candidate(c.value, c.prob, c.index, np.frombuffer(c.row, dtype=np.uint32, count=words).copy())


class Scorer:
    """One device's worth of acquisition state."""

    def __init__(self, device: int | None = None):
        if not torch.cuda.is_available():
            raise RuntimeError("paper_2212_11142_b200 needs a CUDA device (there is no CPU path)")
        self.device = torch.cuda.current_device() if device is None else int(device)
        self._lib = N.lib()
        with torch.cuda.device(self.device):
            h = self._lib.bx_create(self.device)
        if not h:
            raise RuntimeError(f"bx_create({self.device}) failed")
        self.h = C.c_void_p(h)
        self.layout: SpaceLayout | None = None
        self._space_key = None
        self.has_forest = False
        self.n_slots = 0
        self.space_gen = 0  # bumped whenever the space tables (and so every model upload) change

    def close(self):
        if getattr(self, "h", None):
            self._lib.bx_destroy(self.h)
            self.h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    # -- helpers --------------------------------------------------------------------------------
    def _check(self, code):
        N.check(self.h, code)

    @property
    def stream(self) -> C.c_void_p:
        return C.c_void_p(torch.cuda.current_stream(self.device).cuda_stream)

    def to_device(self, rows: np.ndarray) -> torch.Tensor:
        rows = np.ascontiguousarray(rows, dtype=np.uint32)
        t = torch.from_numpy(rows.view(np.int32))
        return t.to(f"cuda:{self.device}", non_blocking=False)

    # -- model state ----------------------------------------------------------------------------
    def layout_for(self, space) -> SpaceLayout:
        """The resident layout when it already describes `space`, else a fresh upload."""
        if self.layout is not None and self.layout.space is space:
            return self.layout
        return self.set_space(space, True)

    def set_space(self, space, use_transforms: bool = True) -> SpaceLayout:
        key = (id(space), bool(use_transforms))
        if self._space_key == key and self.layout is not None and self.layout.space is space:
            return self.layout
        lay = SpaceLayout(space, use_transforms)
        self._check(self._lib.bx_set_space(self.h, C.cast(lay.params, C.c_void_p), lay.n_params,
                                           lay.row_words, _ptr(lay.coord_lut), len(lay.coord_lut),
                                           _ptr(lay.rank_lut), len(lay.rank_lut), lay.n_features))
        self.layout = lay
        self._space_key = key
        self.space_gen += 1
        self.n_slots = self._lib.bx_neighbor_slots(self.h)
        self._cot_key = None  # bx_set_space cleared every other piece of model state
        self._cons_key = None
        self.has_forest = False
        return lay

    def set_gp(self, gp):
        """Upload a GPModel (reference surrogate.py:264-332, or GPState) - L, alpha, encodings."""
        lay = self.set_space(gp.space, getattr(gp, "use_transforms", True))
        rows = lay.encode(gp.configs)
        L = np.tril(np.asarray(gp._cho[0], dtype=np.float64))  # upper triangle is stale K (:300)
        L = np.ascontiguousarray(L)
        alpha = _host(gp.alpha, np.float64)
        h = gp.hyperparameters
        ls = _host(h.lengthscales, np.float64)
        self._check(self._lib.bx_set_gp(self.h, _ptr(rows), len(rows), _ptr(L), _ptr(alpha),
                                        float(h.outputscale), _ptr(ls), float(gp.y_mean),
                                        float(gp.y_std), self.stream))
        self.gp = gp

    def set_forest(self, feas):
        """Upload a FeasibilityModel (feasibility.py:54-71) or clear it (None)."""
        if feas is None:
            self._check(self._lib.bx_clear_forest(self.h))
            self.has_forest = False
            return
        if feas.constant is not None:
            self._check(self._lib.bx_set_forest(self.h, None, None, None, None, None, 0, None, 0,
                                                int(feas.max_depth), float(feas.constant)))
            self.has_forest = True
            return
        if feas.roots is None or len(feas.roots) == 0:
            raise N.NativeError(N.BX_ERR_NO_TREES, "feasibility model has no trees")
        f = _host(feas.feature, np.int32)
        t = _host(feas.threshold, np.float64)
        lft = _host(feas.left, np.int32)
        rgt = _host(feas.right, np.int32)
        v = _host(feas.value, np.float64)
        roots = _host(feas.roots, np.int32)
        self._check(self._lib.bx_set_forest(self.h, _ptr(f), _ptr(t), _ptr(lft), _ptr(rgt), _ptr(v),
                                            len(f), _ptr(roots), len(roots), int(feas.max_depth),
                                            float("nan")))
        self.has_forest = True

    def set_evaluated(self, configs):
        configs = list(configs)
        rows = self.layout.encode(configs) if configs else np.zeros((0, self.layout.row_words), np.uint32)
        self._check(self._lib.bx_set_evaluated(self.h, _ptr(rows), len(rows)))

    def set_evaluated_rows(self, rows: np.ndarray):
        rows = np.ascontiguousarray(rows, np.uint32)
        self._check(self._lib.bx_set_evaluated(self.h, _ptr(rows), len(rows)))

    def set_cot(self, cot):
        """Upload the reference's ChainOfTrees (constraints.py:398-410), or pre-flattened
        `CotTables` (workloads loaded without the reference)."""
        key = id(cot)
        if getattr(self, "_cot_key", None) == key:
            return
        t = cot if isinstance(cot, CotTables) else flatten_cot(cot, self.layout)
        self._check(self._lib.bx_set_cot(self.h, t.n_groups, _ptr(t.group_kind),
                                         _ptr(t.group_param_begin), _ptr(t.group_params),
                                         _ptr(t.group_root), t.n_nodes, _ptr(t.child_begin),
                                         _ptr(t.child_count), _ptr(t.node_value), _ptr(t.leaf_count)))
        self._cot_tables = t
        self._cot_key = key

    def set_constraints(self, space):
        key = id(space)
        if getattr(self, "_cons_key", None) == key:
            return
        p = Program(space, self.layout)
        self._check(self._lib.bx_set_constraints(
            self.h, p.n, _ptr(p.prog_begin), _ptr(p.code), p.code_len, _ptr(p.consts_arr),
            len(p.consts), _ptr(p.value_tag), _ptr(p.value_int), _ptr(p.value_float),
            _ptr(p.value_str), p.n_values))
        self._program = p
        self._cons_key = key

    # -- hot path -------------------------------------------------------------------------------
    def _summary(self, s: N.ScoreSummary) -> Summary:
        w, n = self.layout.row_words, s.n_top
        # the top-k rows in one copy out of the struct (rows[i] are views of it)
        raw = np.frombuffer(s, dtype=np.uint8)
        rows = raw[_TOP_OFF:_TOP_OFF + n * _CAND_SIZE].reshape(n, _CAND_SIZE)[:, _ROW_OFF:_ROW_OFF + 4 * w]
        rows = rows.copy().view(np.uint32)
        top = [Candidate(c.value, c.prob, c.index, rows[i]) for i, c in enumerate(s.top[:n])]
        return Summary(s.n_scored, s.n_finite, top, _cand(s.best, w), _cand(s.best_prob, w))

    def score(self, rows: torch.Tensor, f_model: float, eps_f: float = 0.0, k: int = 10,
              want_values: bool = False, summary: bool = True, rf_pairwise: bool | None = None,
              index_base: int = 0, timing: bool | str = False):
        """bx_score over device rows.  Returns (Summary | None, values | None, probs | None).
        timing=True records every kernel's duration, timing="posterior" only the posterior's."""
        q = rows.shape[0]
        flags = N.BX_SCORE_TIMING_POSTERIOR if timing == "posterior" else (N.BX_SCORE_TIMING if timing else 0)
        if rf_pairwise if rf_pairwise is not None else q == 1:
            flags |= N.BX_SCORE_RF_PAIRWISE
        if not summary:
            flags |= N.BX_SCORE_NO_SUMMARY
        values = probs = None
        if want_values:
            values = torch.empty(q, dtype=torch.float64, device=rows.device)
            probs = torch.empty(q, dtype=torch.float64, device=rows.device)
        s = N.ScoreSummary()
        self._check(self._lib.bx_score(self.h, _ptr(rows), q, index_base, float(f_model), float(eps_f),
                                       int(k), flags, _ptr(values), _ptr(probs),
                                       C.byref(s) if summary else None, self.stream))
        return (self._summary(s) if summary else None), values, probs

    def gp_kernel(self) -> str:
        """Posterior kernel the current model state runs: "tensor", "dmma" or "generic"."""
        return {0: "generic", 1: "dmma", 2: "tensor"}[self._lib.bx_gp_kernel(self.h)]

    def distance_ksteps(self) -> int:
        """DMMA k-steps of the tensor-core posterior's embedding distance product (0: FMA)."""
        return int(self._lib.bx_gp_distance_ksteps(self.h))

    def embedding_dims(self) -> int:
        """Coordinates E of the Euclidean embedding the DMMA distances run over (0: FMA)."""
        return int(self._lib.bx_gp_embedding_dims(self.h))

    def last_timing(self) -> dict:
        """CUDA-event durations (ms) of the forest / fused-score / merge kernels of the last
        score(..., timing=True) call."""
        t = [C.c_float(), C.c_float(), C.c_float()]
        self._check(self._lib.bx_last_timing(self.h, *(C.byref(x) for x in t)))
        return {"rf_ms": t[0].value, "score_ms": t[1].value, "merge_ms": t[2].value}

    def score_host(self, rows: np.ndarray | torch.Tensor, f_model: float, eps_f: float = 0.0,
                   k: int = 10, index_base: int = 0, packed: bool = False) -> Summary:
        """bx_score_host: the pool stays in host memory.  packed=True: the rows are in the packed
        wire format (pack()); from pinned memory the posterior reads them zero-copy, otherwise
        chunked copies overlap the scoring."""
        q = rows.shape[0]
        s = N.ScoreSummary()
        self._check(self._lib.bx_score_host(self.h, _ptr(rows), q, index_base, float(f_model),
                                            float(eps_f), int(k), N.BX_SCORE_PACKED if packed else 0,
                                            C.byref(s), self.stream))
        return self._summary(s)

    def packed_words(self) -> int:
        return int(self._lib.bx_packed_row_words(self.h))

    def pack(self, rows: np.ndarray, out: np.ndarray | None = None) -> np.ndarray:
        """Encoded rows -> the packed wire format of the current space (host, bx_pack_rows)."""
        rows = np.ascontiguousarray(rows, dtype=np.uint32)
        q = rows.shape[0]
        if out is None:
            out = np.empty((q, self.packed_words()), dtype=np.uint32)
        self._check(self._lib.bx_pack_rows(self.h, _ptr(rows), q, _ptr(out)))
        return out

    def unpack(self, packed: np.ndarray) -> np.ndarray:
        packed = np.ascontiguousarray(packed, dtype=np.uint32)
        q = packed.shape[0]
        out = np.empty((q, self.layout.row_words), dtype=np.uint32)
        self._check(self._lib.bx_unpack_rows(self.h, _ptr(packed), q, _ptr(out)))
        return out

    def generate(self, q: int, seed: int, mode: int = 0, index_base: int = 0) -> torch.Tensor:
        """bx_generate: q device-generated rows (mode 0 uniform, 1 chain-of-trees leaf-uniform)."""
        out = torch.empty((q, self.layout.row_words), dtype=torch.int32, device=f"cuda:{self.device}")
        self._check(self._lib.bx_generate(self.h, C.c_uint64(seed), index_base, q, mode, _ptr(out),
                                          self.stream))
        return out

    def score_generated(self, q: int, seed: int, f_model: float, eps_f: float = 0.0, k: int = 10,
                        mode: int = 0, index_base: int = 0) -> Summary:
        """bx_score_generated: score a device-generated pool of q candidates chunk by chunk."""
        s = N.ScoreSummary()
        self._check(self._lib.bx_score_generated(self.h, C.c_uint64(seed), index_base, q, mode,
                                                 float(f_model), float(eps_f), int(k), C.byref(s),
                                                 self.stream))
        return self._summary(s)

    def predict(self, rows: torch.Tensor):
        q = rows.shape[0]
        mean = torch.empty(q, dtype=torch.float64, device=rows.device)
        var = torch.empty(q, dtype=torch.float64, device=rows.device)
        self._check(self._lib.bx_gp_predict(self.h, _ptr(rows), q, _ptr(mean), _ptr(var), self.stream))
        return mean, var

    def rf_predict(self, rows: torch.Tensor, pairwise: bool | None = None):
        q = rows.shape[0]
        probs = torch.empty(q, dtype=torch.float64, device=rows.device)
        pw = (q == 1) if pairwise is None else pairwise
        self._check(self._lib.bx_rf_predict(self.h, _ptr(rows), q, N.BX_SCORE_RF_PAIRWISE if pw else 0,
                                            _ptr(probs), self.stream))
        return probs

    def neighbors(self, rows: torch.Tensor, use_cot: bool):
        count = rows.shape[0]
        w = self.layout.row_words
        out = torch.empty((count * self.n_slots, w), dtype=torch.int32, device=rows.device)
        valid = torch.empty(count * self.n_slots, dtype=torch.uint8, device=rows.device)
        self._check(self._lib.bx_neighbors(self.h, _ptr(rows), count, int(bool(use_cot)), _ptr(out),
                                           _ptr(valid), self.stream))
        return out, valid

    def climb(self, pool_rows: torch.Tensor, start_index, start_values, use_cot: bool, f_model: float,
              eps_f: float, best: Candidate | None, max_steps: int = 50):
        """bx_climb: the hill climb from pool rows start_index on the device.  Returns (best, steps):
        the best-unevaluated tracker folded over every scored neighbour (None if still empty)."""
        idx = np.ascontiguousarray(start_index, dtype=np.int64)
        n = len(idx)
        vals = np.ascontiguousarray(start_values, dtype=np.float64)
        c = N.Cand()
        if best is None:
            c.value, c.prob, c.index = -math.inf, -math.inf, -1
        else:
            c.value, c.prob, c.index = best.value, best.prob, max(best.index, 0)
            np.ctypeslib.as_array(c.row)[:len(best.row)] = best.row
        steps = C.c_int32(0)
        self._check(self._lib.bx_climb(self.h, _ptr(pool_rows), _ptr(idx), _ptr(vals), n, int(bool(use_cot)),
                                       float(f_model), float(eps_f), int(max_steps), C.byref(c), C.byref(steps),
                                       self.stream))
        return _cand(c, self.layout.row_words), int(steps.value)

    def cot_contains(self, rows: torch.Tensor) -> torch.Tensor:
        mask = torch.empty(rows.shape[0], dtype=torch.uint8, device=rows.device)
        self._check(self._lib.bx_cot_contains(self.h, _ptr(rows), rows.shape[0], _ptr(mask), self.stream))
        return mask

    def constraints_eval(self, rows: torch.Tensor) -> torch.Tensor:
        mask = torch.empty(rows.shape[0], dtype=torch.uint8, device=rows.device)
        self._check(self._lib.bx_constraints_eval(self.h, _ptr(rows), rows.shape[0], _ptr(mask),
                                                  self.stream))
        return mask

    def pairwise_sq(self, a: torch.Tensor, b: torch.Tensor) -> torch.Tensor:
        out = torch.empty((self.layout.n_params, a.shape[0], b.shape[0]), dtype=torch.float64,
                          device=a.device)
        self._check(self._lib.bx_pairwise_sq(self.h, _ptr(a), a.shape[0], _ptr(b), b.shape[0],
                                             _ptr(out), self.stream))
        return out

    def gp_factor(self, rows: torch.Tensor, z: np.ndarray, outputscale: float, noise_variance: float,
                  lengthscales) -> tuple:
        """bx_gp_factor: (L (n, n) lower, alpha (n,)) of GPModel.__init__ computed on the device."""
        n = rows.shape[0]
        z = np.ascontiguousarray(z, dtype=np.float64)
        ls = np.ascontiguousarray(lengthscales, dtype=np.float64)
        L = np.empty((n, n), dtype=np.float64)
        alpha = np.empty(n, dtype=np.float64)
        self._check(self._lib.bx_gp_factor(self.h, _ptr(rows), n, _ptr(z), float(outputscale), float(noise_variance),
                                           _ptr(ls), _ptr(L), _ptr(alpha), self.stream))
        return L, alpha

    def lml_core(self, sq: torch.Tensor, z: torch.Tensor, params: torch.Tensor, want_grad: bool,
                 prior=None):
        """bx_lml_core: (values[c], grads[c, 2+D] | None, ok[c]) for rows (sigma, noise, l...)."""
        D, n, _ = sq.shape
        c = params.shape[0]
        dev = sq.device
        value = torch.empty(c, dtype=torch.float64, device=dev)
        grad = torch.empty((c, 2 + D), dtype=torch.float64, device=dev) if want_grad else None
        ok = torch.empty(c, dtype=torch.int32, device=dev)
        k, rate = (float(prior.shape), float(prior.rate)) if prior is not None else (0.0, 0.0)
        self._check(self._lib.bx_lml_core(self.h, _ptr(sq.contiguous()), n, D, _ptr(z.contiguous()),
                                          _ptr(params.contiguous()), c, k, rate, int(prior is not None),
                                          int(want_grad), _ptr(value), _ptr(grad), _ptr(ok), self.stream))
        return value, grad, ok

    def lml_core_host(self, sq: torch.Tensor, z: torch.Tensor, params: np.ndarray, prior=None):
        """bx_lml_core_host: lml_core with host parameters and host results (values, grads, ok) - one
        staged copy each way inside the library (the L-BFGS-B driver's per-iteration call,
        hyperfit.py)."""
        D, n, _ = sq.shape
        params = np.ascontiguousarray(params, dtype=np.float64)
        c = params.shape[0]
        value = np.empty(c, dtype=np.float64)
        grad = np.empty((c, 2 + D), dtype=np.float64)
        ok = np.empty(c, dtype=np.int32)
        k, rate = (float(prior.shape), float(prior.rate)) if prior is not None else (0.0, 0.0)
        self._check(self._lib.bx_lml_core_host(self.h, _ptr(sq), n, D, _ptr(z), _ptr(params), c, k, rate,
                                               int(prior is not None), _ptr(value), _ptr(grad), _ptr(ok),
                                               self.stream))
        return value, grad, ok

    def lml_batched(self, sq: torch.Tensor, z: torch.Tensor, thetas: torch.Tensor) -> torch.Tensor:
        D, n, _ = sq.shape
        c = thetas.shape[0]
        out = torch.empty(c, dtype=torch.float64, device=sq.device)
        self._check(self._lib.bx_lml_batched(self.h, _ptr(sq.contiguous()), n, D, _ptr(z.contiguous()),
                                             _ptr(thetas.contiguous()), c, _ptr(out), self.stream))
        return out


_SCORERS: dict = {}


def scorer(device: int | None = None) -> Scorer:
    """Process-wide Scorer per device (one handle per device, reused across iterations)."""
    dev = torch.cuda.current_device() if device is None else int(device)
    s = _SCORERS.get(dev)
    if s is None:
        s = _SCORERS[dev] = Scorer(dev)
    return s
