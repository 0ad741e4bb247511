"""Pair-grid sharding of ONE collection across ranks.

The pair evaluations are independent, so the (base, appended) grid is cut into 2-D tiles, one per rank:
with a G_r x G_c rank grid (G_r * G_c = world size, as square as the factorisation allows), the pair
(i, j) belongs to rank (i mod G_r) * G_c + (j mod G_c).  The cyclic assignment keeps the tiles balanced for
the triangular pair sets of the all-pairs harness, and a rank only ever touches the bases of its row group
and the operands of its column group.  Each rank evaluates its tile through its own libcmsvd context (the
per-block states are computed by every rank here: "replicated spectra"; exchanging them instead is the
all-gather of §8(e)), then ONE collective gathers the fixed-size result rows (torch.distributed
``all_gather`` on padded tiles: NCCL on CUDA tensors, gloo on CPU tensors) and every rank reassembles
the outputs in the caller's pair order.

Plumbing only: no arithmetic of the method lives here (the evaluator is ``Context.pair_errors``).
Hardware status: this pod has one GPU per call, so the N > 1 path is covered by world-size-2 gloo tests
on CPU (partition, padding, gather, reassembly) and by a single-GPU test that evaluates the shards of a
world of 4 one after the other and compares their union bitwise with the unsharded call.
"""
from __future__ import annotations

import numpy as np


def rank_grid(world_size: int) -> tuple[int, int]:
    """G_r x G_c = world_size with G_r <= G_c as close as possible."""
    if world_size < 1:
        raise ValueError("world_size must be >= 1")
    gr = int(np.floor(np.sqrt(world_size)))
    while world_size % gr:
        gr -= 1
    return gr, world_size // gr


def owner(pairs: np.ndarray, world_size: int) -> np.ndarray:
    """Rank owning each (base, appended) pair."""
    pairs = np.asarray(pairs).reshape(-1, 2)
    gr, gc = rank_grid(world_size)
    return (pairs[:, 0] % gr) * gc + (pairs[:, 1] % gc)


def partition_pairs(pairs: np.ndarray, world_size: int) -> list[np.ndarray]:
    """Indices (into ``pairs``, ascending) of every rank's tile; a partition of range(P)."""
    own = owner(pairs, world_size)
    return [np.flatnonzero(own == r) for r in range(world_size)]


def _gather_rows(local: np.ndarray, counts: list[int], group, device):
    """all_gather of per-rank (count_r, C) float64 row blocks, padded to the largest count."""
    import torch
    import torch.distributed as dist
    ws = dist.get_world_size(group)
    cmax = max(max(counts), 1)
    C = local.shape[1]
    buf = torch.zeros((cmax, C), dtype=torch.float64, device=device)
    if local.shape[0]:
        buf[:local.shape[0]] = torch.from_numpy(np.ascontiguousarray(local, dtype=np.float64)).to(device)
    out = [torch.empty_like(buf) for _ in range(ws)]
    dist.all_gather(out, buf, group=group)
    return [o[:counts[r]].cpu().numpy() for r, o in enumerate(out)]


def sharded_pair_errors(evaluate, pairs, group=None, device="cpu"):
    """Evaluate ``pairs`` (P, 2) across the ranks of ``group`` and return the full result on every rank.

    ``evaluate(local_pairs) -> {"err2": (p, 3), "total": (p,)}`` is the rank's evaluator, e.g.
    ``lambda p: ctx.pair_errors(p, kinds=..., operand=..., want_sigma=False, want_mu=False)``.
    ``device``: where the gather buffers live ("cuda" for the NCCL backend, "cpu" for gloo).
    Without an initialised process group this is the single-rank call.
    """
    import torch.distributed as dist
    pairs = np.ascontiguousarray(pairs, dtype=np.int32).reshape(-1, 2)
    P = pairs.shape[0]
    if not (dist.is_available() and dist.is_initialized()):
        res = evaluate(pairs)
        return {"err2": np.asarray(res["err2"], np.float64), "total": np.asarray(res["total"], np.float64)}
    ws, rank = dist.get_world_size(group), dist.get_rank(group)
    parts = partition_pairs(pairs, ws)
    mine = parts[rank]
    if mine.size:
        res = evaluate(pairs[mine])
        local = np.concatenate([np.asarray(res["err2"], np.float64).reshape(-1, 3),
                                np.asarray(res["total"], np.float64).reshape(-1, 1)], axis=1)
    else:
        local = np.zeros((0, 4))
    rows = _gather_rows(local, [int(p.size) for p in parts], group, device)
    err2 = np.empty((P, 3))
    total = np.empty(P)
    for r in range(ws):
        err2[parts[r]] = rows[r][:, :3]
        total[parts[r]] = rows[r][:, 3]
    return {"err2": err2, "total": total}
