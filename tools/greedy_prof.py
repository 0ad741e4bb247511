"""Greedy-driver probe: wall time of Alg. 3 (residual sort) on config 2 and the per-category
kernel time of its tentative evaluations (cluster-internal kernels are not categorised)."""
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import synth  # noqa: E402
import paper_2601_11626_b200 as cm  # noqa: E402

alg = {"approx": cm.ALG_APPROX, "residual": cm.ALG_RESIDUAL}[sys.argv[1] if len(sys.argv) > 1 else "approx"]
srt = cm.SORT_RESIDUAL if (len(sys.argv) <= 2 or sys.argv[2] == "residual") else cm.SORT_FROBENIUS
col = synth.config2()
with cm.Context(0) as ctx:
    ctx.register(col.blocks)
    ctx.block_spectra(col.r)
    ctx.cluster(alg, 0.05, sort=srt)
    ctx.profile(True)
    l0 = ctx.launches
    t = time.time()
    g = ctx.cluster(alg, 0.05, sort=srt)
    dt = time.time() - t
    p = ctx.profile_read()
    print(f"greedy {dt*1e3:.1f} ms, {len(g['clusters'])} clusters, {g['n_evals']} evals, {ctx.launches - l0} launches")
    for k, (ms, n) in sorted(p.items(), key=lambda kv: -kv[1][0]):
        if n:
            print(f"  {k:14s} {ms:8.2f} ms  {n}")
