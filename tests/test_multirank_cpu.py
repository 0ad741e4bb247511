"""N > 1 host logic on CPU with the gloo backend (world_size 2): bench.py's
replica launch (torchrun, 127.0.0.1 rendezvous), the per-rank workload
seeding, the max-over-ranks timing reduction, and the --impl reference arm
(rank 0 alone runs the oracle and prints one JSON line; the other rank exits
0 without work).  The GPU arm's data path has no collective ("replicas
only")."""
import json
import os
import socket
import subprocess
import sys

import numpy as np
import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    return port


def _worker(rank, ws, port, q):
    import torch.distributed as dist
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port), RANK=str(rank), WORLD_SIZE=str(ws))
    import bench
    r, w, local, d = bench.dist_init()
    assert (r, w) == (rank, ws) and d is not None and d.get_backend() == "gloo"
    mx = bench.max_over_ranks(d, float(10 * rank + 1))
    col = bench.workload("config1", rank)
    q.put((rank, mx, float(col.blocks[0, 0, 0]), col.blocks.shape))
    d.barrier()
    d.destroy_process_group()


def test_max_over_ranks_and_per_rank_workloads():
    import torch.multiprocessing as mp
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = free_port()
    procs = [ctx.Process(target=_worker, args=(r, 2, port, q)) for r in range(2)]
    for p in procs:
        p.start()
    for p in procs:
        p.join(120)
        assert p.exitcode == 0
    res = sorted(q.get() for _ in range(2))
    assert res[0][1] == res[1][1] == 11.0                 # max over ranks, seen by every rank
    assert res[0][3] == res[1][3]                          # same shapes (weak scaling)
    assert res[0][2] != res[1][2]                          # distinct seeded collections per rank


def test_max_over_ranks_single_process():
    import bench
    assert bench.max_over_ranks(None, 3.5) == 3.5


def test_torchrun_reference_arm_two_ranks():
    port = free_port()
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", "--nproc-per-node", "2",
           "--master-addr", "127.0.0.1", "--master-port", str(port), os.path.join(ROOT, "bench.py"),
           "--impl", "reference", "--gpus", "2", "--steps", "1", "--warmup", "0", "--config", "config1",
           "--ref-sample", "8"]
    env = dict(os.environ, OMP_NUM_THREADS="2")
    r = subprocess.run(cmd, capture_output=True, text=True, timeout=600, cwd=ROOT, env=env)
    assert r.returncode == 0, r.stderr[-2000:]
    lines = [l for l in r.stdout.splitlines() if l.startswith("{")]
    assert len(lines) == 1, r.stdout                       # rank 0 alone prints
    d = json.loads(lines[0])
    assert d["impl"] == "reference" and d["n_gpus"] == 2 and d["value"] > 0
    assert d["cpu_baseline"]["kind"] == "oracle" and d["e2e"]["h2d_bytes_per_step"] == 0


# ---------------------------------------------------------------------------
# N4: pair-grid sharding of one collection (paper_2601_11626_b200/shard.py), host logic on gloo
# ---------------------------------------------------------------------------
def _fake_eval(pairs):
    """Stand-in evaluator (no GPU here): a deterministic function of the pair ids, so that the gathered
    result can be checked exactly."""
    p = np.asarray(pairs, np.float64)
    err2 = np.stack([p[:, 0] * 1000 + p[:, 1], p[:, 0] - p[:, 1], p[:, 0] * p[:, 1]], axis=1)
    return {"err2": err2, "total": p.sum(axis=1)}


def test_partition_is_exact_and_balanced():
    from paper_2601_11626_b200 import shard
    import synth
    order = np.arange(64)
    pairs = synth.all_pairs_by_norm_order(order)          # 2016 ordered pairs (config 4's pair set)
    for ws in (1, 2, 3, 4, 6, 8):
        parts = shard.partition_pairs(pairs, ws)
        allidx = np.sort(np.concatenate(parts))
        assert np.array_equal(allidx, np.arange(len(pairs)))          # every pair exactly once
        sizes = np.array([len(p) for p in parts])
        assert sizes.max() <= 1.15 * len(pairs) / ws + 8             # balanced tiles
        gr, gc = shard.rank_grid(ws)
        assert gr * gc == ws and gr <= gc
        for r, idx in enumerate(parts):                               # 2-D tile: base row group x operand column group
            assert np.all(pairs[idx, 0] % gr == r // gc) and np.all(pairs[idx, 1] % gc == r % gc)


def _shard_worker(rank, ws, port, q):
    import torch.distributed as dist
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port), RANK=str(rank), WORLD_SIZE=str(ws))
    dist.init_process_group("gloo", rank=rank, world_size=ws)
    from paper_2601_11626_b200 import shard
    import synth
    pairs = synth.all_pairs_by_norm_order(np.arange(16)[::-1].copy())
    calls = []

    def ev(p):
        calls.append(len(p))
        return _fake_eval(p)
    out = shard.sharded_pair_errors(ev, pairs, device="cpu")
    empty = shard.sharded_pair_errors(ev, pairs[:0], device="cpu")      # empty pair list: no evaluator call
    one = shard.sharded_pair_errors(ev, pairs[:1], device="cpu")        # fewer pairs than ranks
    q.put((rank, out["err2"], out["total"], calls, empty["err2"].shape, one["err2"]))
    dist.barrier()
    dist.destroy_process_group()


def test_sharded_pair_errors_gloo_world2():
    import torch.multiprocessing as mp
    import synth
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = free_port()
    procs = [ctx.Process(target=_shard_worker, args=(r, 2, port, q)) for r in range(2)]
    for p in procs:
        p.start()
    res = sorted((q.get(timeout=120) for _ in range(2)), key=lambda t: t[0])
    for p in procs:
        p.join(120)
        assert p.exitcode == 0
    pairs = synth.all_pairs_by_norm_order(np.arange(16)[::-1].copy())
    ref = _fake_eval(pairs)
    for rank, err2, total, calls, eshape, one in res:
        assert np.array_equal(err2, ref["err2"]) and np.array_equal(total, ref["total"])   # caller's order, every rank
        assert eshape == (0, 3)
        assert np.array_equal(one, ref["err2"][:1])
    assert res[0][3][0] + res[1][3][0] == len(pairs)        # each rank evaluated only its tile
    assert abs(res[0][3][0] - res[1][3][0]) <= 0.15 * len(pairs)
