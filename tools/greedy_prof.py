import sys, time, torch, numpy as np
sys.path.insert(0, '/root/repo')
import synth, paper_2601_11626_b200 as cm
col = synth.config2()
with cm.Context(0) as ctx:
    ctx.register(col.blocks); ctx.block_spectra(col.r)
    ctx.cluster(cm.ALG_APPROX, 0.05, sort=cm.SORT_RESIDUAL)
    ctx.profile(True)
    t = time.time(); g = ctx.cluster(cm.ALG_APPROX, 0.05, sort=cm.SORT_RESIDUAL); dt = time.time() - t
    p = ctx.profile_read()
    print(f"greedy {dt*1e3:.1f} ms, {len(g['clusters'])} clusters, {g['n_evals']} evals")
    for k, (ms, n) in sorted(p.items(), key=lambda kv: -kv[1][0]):
        if n: print(f"  {k:14s} {ms:8.2f} ms  {n}")
