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
