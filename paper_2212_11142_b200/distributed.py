"""Pool sharding across GPUs: contiguous index ranges per rank, one all-gather of top-k records.

SURVEY.md §8e: candidates are independent, so each rank scores its own contiguous slice of the pool
with the fused kernel and keeps only its summary (stable top-k, the two tracker bests, the finite
count).  The single collective is an all-gather of those fixed-size records (a few KB) over NCCL;
every rank then merges them with the reductions' own total orders, so the result does not depend
on the number of ranks:

    top-k     : (value desc, global index asc)            acquisition.py:188
    best      : (value desc, configuration asc)           acquisition.py:97-111
    best_prob : (probability desc, configuration asc)     acquisition.py:181
"""
from __future__ import annotations

import numpy as np
import torch
import torch.distributed as dist

from .device import Candidate, Summary

# record layout (float64 words): value, prob, index, valid, row words (as float64 of uint32)
_HDR = 4


def shard_range(q: int, rank: int, world: int) -> tuple[int, int]:
    """Contiguous [lo, hi) slice of a q-candidate pool for `rank` (sizes differ by at most one)."""
    base, extra = divmod(q, world)
    lo = rank * base + min(rank, extra)
    return lo, lo + base + (1 if rank < extra else 0)


def _rec_width(row_words: int) -> int:
    return _HDR + row_words


def pack(summary: Summary, k: int, row_words: int) -> torch.Tensor:
    """Summary -> float64 tensor [(k + 2) records + 2 counters] (fixed size for all-gather)."""
    w = _rec_width(row_words)
    out = np.zeros((k + 2) * w + 2, dtype=np.float64)

    def put(slot, c: Candidate | None):
        if c is None:
            return
        base = slot * w
        out[base:base + 4] = (c.value, c.prob, float(c.index), 1.0)
        out[base + 4:base + w] = c.row.astype(np.float64)

    for i, c in enumerate(summary.top[:k]):
        put(i, c)
    put(k, summary.best)
    put(k + 1, summary.best_prob)
    out[-2:] = (summary.n_scored, summary.n_finite)
    return torch.from_numpy(out)


def unpack(t: torch.Tensor, k: int, row_words: int) -> Summary:
    a = t.detach().cpu().numpy()
    w = _rec_width(row_words)

    def get(slot):
        base = slot * w
        if a[base + 3] != 1.0:
            return None
        return Candidate(float(a[base]), float(a[base + 1]), int(a[base + 2]),
                         a[base + 4:base + w].astype(np.uint32))

    top = [c for c in (get(i) for i in range(k)) if c is not None]
    return Summary(int(a[-2]), int(a[-1]), top, get(k), get(k + 1))


def merge(parts: list[Summary], k: int, key) -> Summary:
    """Merge per-rank summaries.  `key(row) -> comparable` gives the configuration order
    (decoded Python tuples, i.e. the reference's own comparison)."""
    tops = sorted((c for p in parts for c in p.top), key=lambda c: (-c.value, c.index))[:k]

    def pick(cands, score):
        best = None
        for c in cands:
            if c is None:
                continue
            if best is None or score(c) > score(best) or (score(c) == score(best)
                                                             and key(c.row) < key(best.row)):
                best = c
        return best

    return Summary(sum(p.n_scored for p in parts), sum(p.n_finite for p in parts), tops,
                   pick([p.best for p in parts], lambda c: c.value),
                   pick([p.best_prob for p in parts], lambda c: c.prob))


def allgather_summary(summary: Summary, k: int, layout, group=None, device=None) -> Summary:
    """One all-gather of the fixed-size record block; identical merged result on every rank."""
    world = dist.get_world_size(group)
    local = pack(summary, k, layout.row_words)
    if device is not None:
        local = local.to(device)
    if dist.get_backend(group) == "nccl":
        gathered = torch.empty(world * local.numel(), dtype=local.dtype, device=local.device)
        dist.all_gather_into_tensor(gathered, local, group=group)
        chunks = gathered.view(world, -1)
    else:
        chunks = [torch.empty_like(local) for _ in range(world)]
        dist.all_gather(chunks, local, group=group)
    parts = [unpack(c, k, layout.row_words) for c in chunks]
    return merge(parts, k, key=lambda row: layout.decode(row)[0])
