"""Multi-rank pool sharding on CPU (gloo, world_size 2): the all-gathered, merged summary equals the
single-process summary of the whole pool (the result is independent of the number of ranks)."""
import os
import socket

import numpy as np
import pytest
import torch.distributed as dist
import torch.multiprocessing as mp

import oracle
from golden_io import load, oracle_model, to_cfg
from paper_2212_11142_b200.device import Candidate, Summary
from paper_2212_11142_b200.distributed import allgather_summary, merge, pack, shard_range, unpack
from paper_2212_11142_b200.layout import SpaceLayout

K = 10


def host_summary(values, probs, rows, cfgs, base, evaluated, k=K) -> Summary:
    """The reductions of acquisition.py:97-111,179-188 written out on the host (test reference)."""
    order = [i for i in np.argsort(-values, kind="stable")[:k] if values[i] != -np.inf]
    top = [Candidate(float(values[i]), float(probs[i]), base + int(i), rows[i]) for i in order]

    def track(score, finite_only):
        best = None
        for i, c in enumerate(cfgs):
            if c in evaluated or (finite_only and values[i] == -np.inf):
                continue
            if best is None or score[i] > score[best] or (score[i] == score[best] and c < cfgs[best]):
                best = i
        return None if best is None else Candidate(float(values[best]), float(probs[best]),
                                                   base + best, rows[best])

    return Summary(len(values), int(np.sum(values != -np.inf)), top, track(values, True), track(probs, False))


def shard_data(rank, world):
    meta, arr, space = load("mixed_metrics")
    og, of = oracle_model(meta, arr, space)
    cands = [to_cfg(space, c) for c in meta["cands"]]
    lay = SpaceLayout(space, meta["use_transforms"])
    rows = lay.encode(cands)
    ev = {to_cfg(space, c) for c in meta["evaluated"]} | set(cands[::37])
    lo, hi = shard_range(len(cands), rank, world)
    v, p = oracle.scores(og, of, cands[lo:hi], meta["f_best"], meta["eps_f"])
    return host_summary(v, p, rows[lo:hi], cands[lo:hi], lo, ev), lay, (cands, rows, og, of, meta, ev)


def _worker(rank, world, port, out):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        summ, lay, _ = shard_data(rank, world)
        merged = allgather_summary(summ, K, lay)
        out[rank] = (merged.n_scored, merged.n_finite, [c.index for c in merged.top],
                     merged.best.index if merged.best else None,
                     merged.best_prob.index if merged.best_prob else None,
                     [list(map(int, c.row)) for c in merged.top])
    finally:
        dist.destroy_process_group()


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def test_pack_unpack_round_trip():
    summ, lay, _ = shard_data(0, 1)
    back = unpack(pack(summ, K, lay.row_words), K, lay.row_words)
    assert [c.index for c in back.top] == [c.index for c in summ.top]
    assert back.best.index == summ.best.index and back.best_prob.index == summ.best_prob.index
    assert all(np.array_equal(a.row, b.row) for a, b in zip(back.top, summ.top))


@pytest.mark.parametrize("world", [2, 3])
def test_merge_is_rank_count_independent(world):
    full, lay, (cands, rows, og, of, meta, ev) = shard_data(0, 1)
    parts = [shard_data(r, world)[0] for r in range(world)]
    m = merge(parts, K, key=lambda row: lay.decode(row)[0])
    assert [c.index for c in m.top] == [c.index for c in full.top]
    assert m.best.index == full.best.index and m.best_prob.index == full.best_prob.index
    assert (m.n_scored, m.n_finite) == (full.n_scored, full.n_finite)


def test_gloo_allgather_two_ranks():
    full, _, _ = shard_data(0, 1)
    out = mp.Manager().dict()
    mp.spawn(_worker, args=(2, _free_port(), out), nprocs=2, join=True)
    want = (full.n_scored, full.n_finite, [c.index for c in full.top], full.best.index,
            full.best_prob.index, [list(map(int, c.row)) for c in full.top])
    assert out[0] == want and out[1] == want
