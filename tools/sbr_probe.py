"""Timing probe of the batched eigensolver (cmsvd_sym_eigvals) on n x n Gram matrices: per-category CUDA-event
times (sbr_panel / sbr_symm / sbr_syr2k / sbr_chase / bisect) and max error vs LAPACK on the unique matrices.
Usage: python tools/sbr_probe.py [n] [count] [kw]"""
import os
import sys
import time

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2601_11626_b200 as cm  # noqa: E402

n = int(sys.argv[1]) if len(sys.argv) > 1 else 512
count = int(sys.argv[2]) if len(sys.argv) > 2 else 1184
kw = int(sys.argv[3]) if len(sys.argv) > 3 else n // 2
R = np.random.default_rng(0)
uniq = []
for u in range(8):
    X = R.standard_normal((n, n + 3)) * (np.arange(1, n + 4) ** -0.3)
    uniq.append(X @ X.T)
mats = [uniq[p % 8] for p in range(count)]
cm.load()
with cm.Context(0) as ctx:
    ev, _ = ctx.sym_eigvals(mats, kw)
    for rep in range(2):
        ctx.profile(True)
        t0 = time.perf_counter()
        ev, _ = ctx.sym_eigvals(mats, kw)
        wall = time.perf_counter() - t0
        prof = ctx.profile_read()
        ctx.profile(False)
        print(f"n={n} count={count} kw={kw} wall {wall * 1e3:.1f} ms (incl. H2D of {count * n * n * 8 / 1e9:.2f} GB):",
              {k: round(v[0], 3) for k, v in prof.items() if v[1]}, flush=True)
err = 0.0
for u in range(min(8, count)):
    ref = np.linalg.eigvalsh(uniq[u])[::-1][:kw]
    err = max(err, float(np.max(np.abs(ev[u] - ref)) / ref[0]))
print(f"max |ev - eigvalsh| / lambda_1 = {err:.3e}")
