"""Config 5 scaling sweep (BASELINE.json configs[4]): evaluations/s vs N in {512, 2048} and r in {16, 64}
on N*k candidate pairs (k = 16 partners per block, seeded and drawn uniformly: the cost of an evaluation
does not depend on which partner it is), all three estimators, RAW operand, device-resident pairs and
outputs, CUDA-event timing (median of 5 after a warm-up).  The one-time register + spectra time is
reported separately.  Usage: python tools/c5_sweep.py [k]"""
import os
import statistics
import sys
import time

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import synth  # noqa: E402
import paper_2601_11626_b200 as cm  # noqa: E402

k = int(sys.argv[1]) if len(sys.argv) > 1 else 16
cm.load()
for N in (512, 2048):
    for r in (16, 64):
        col = synth.config5(N=N, r=r)
        rng = np.random.default_rng(100 + N + r)
        nbr = np.stack([rng.choice(np.delete(np.arange(N), i), k, replace=False) for i in range(N)])
        pairs = synth.knn_pairs(nbr)
        P = pairs.shape[0]
        stream = torch.cuda.Stream()
        with torch.cuda.stream(stream), cm.Context(0, stream.cuda_stream) as ctx:
            blocks = torch.from_numpy(col.blocks).cuda()
            t0 = time.perf_counter()
            ctx.register(blocks)
            ctx.block_spectra(r)
            torch.cuda.synchronize()
            t_spec = time.perf_counter() - t0
            dp = torch.from_numpy(pairs).cuda()
            out = {"err2": torch.empty((P, 3), dtype=torch.float64, device="cuda"),
                   "total": torch.empty(P, dtype=torch.float64, device="cuda"),
                   "sigma_tilde": torch.empty((P, r), dtype=torch.float32, device="cuda"),
                   "mu": torch.empty((P, r), dtype=torch.float32, device="cuda")}
            ctx.pair_errors(dp, out=out)
            ts = []
            for _ in range(5):
                a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
                a.record(stream)
                ctx.pair_errors(dp, out=out)
                b.record(stream)
                torch.cuda.synchronize()
                ts.append(a.elapsed_time(b))
            ms = statistics.median(ts)
        print(f"config5 N={N:5d} r={r:3d}: {P:6d} pairs (k={k}) {ms:8.3f} ms = {P / ms * 1e3:10.0f} evals/s; "
              f"register+spectra {t_spec * 1e3:7.1f} ms (one-time)", flush=True)
