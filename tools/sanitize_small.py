"""Small end-to-end workload for compute-sanitizer (one --tool per gpurun call): every kernel family on
small inputs -- S1/S2 on tall-thin and A22 (square, guarded subspace iteration) blocks, the pair path on
both operands (tcgen05 pair kernel, tcgen05 GEMM tiles, SIMT), the eigensolvers of every size class
(register / shared-memory kernels, the two-stage band reduction), the greedy drivers and N1 verify."""
import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import synth  # noqa: E402
import paper_2601_11626_b200 as cm  # noqa: E402

cm.load()
R = np.random.default_rng(0)
with cm.Context(0) as ctx:
    mats = []
    for n in (40, 128, 160, 200, 512):
        X = R.standard_normal((n, n + 3))
        mats.append(X @ X.T)
    ev, _ = ctx.sym_eigvals(mats, 32)
    col = synth.config1()
    ctx.register(col.blocks)
    E, sig, rank = ctx.block_spectra(col.r)
    order = np.argsort(-E, kind="stable")
    pairs = synth.all_pairs_by_norm_order(order)
    out = ctx.pair_errors(pairs)
    g = ctx.cluster(cm.ALG_APPROX, 0.05, sort=cm.SORT_RESIDUAL)
    v = ctx.cluster_verify(np.asarray(g["assign"], np.int32))
    g2 = ctx.cluster(cm.ALG_RESIDUAL, 0.05, sort=cm.SORT_RESIDUAL, knn=2)
    col4 = synth.config4(N=3, m=640, rank=64)
    ctx.register(col4.blocks)
    ctx.block_spectra(192)
    out4 = ctx.pair_errors(np.array([[0, 1], [1, 2], [2, 0]], np.int32), operand=cm.TRUNC)
    g4 = ctx.cluster(cm.ALG_APPROX, 0.15, sort=cm.SORT_RESIDUAL, operand=cm.TRUNC)
print("sanitize workload done", float(out["err2"].sum()), float(out4["err2"].sum()), len(g["clusters"]),
      len(g4["clusters"]))
