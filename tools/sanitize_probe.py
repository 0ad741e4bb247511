"""Small end-to-end run of every kernel family (synchronous launches: CUDA_LAUNCH_BLOCKING=1 surfaces the
first faulting kernel; compute-sanitizer is not available on the GPU pool): config 1 pairs (all kinds, RAW and
TRUNC), ragged random collection, tight variants, greedy Algs 1-3 (knn 1 and 3), sequence errors, cluster
verification, a small wide-block (A22) collection with r > 128 (tcgen05 GEMM tiles, subspace iteration)."""
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import synth  # noqa: E402
import paper_2601_11626_b200 as cm  # noqa: E402

cm.load()
col = synth.config1()
with cm.Context(0) as ctx:
    ctx.register(torch.from_numpy(col.blocks).cuda())
    E, sig, rank = ctx.block_spectra(col.r)
    order = np.array(sorted(range(col.N), key=lambda i: (-E[i], i)))
    pairs = synth.all_pairs_by_norm_order(order)
    ctx.pair_errors(pairs)
    ctx.pair_errors(pairs, operand=cm.TRUNC)
    ctx.pair_errors_tight(pairs)
    for alg in (cm.ALG_MAX_NORM, cm.ALG_RESIDUAL, cm.ALG_APPROX):
        for knn in (1, 3):
            g = ctx.cluster(alg, 0.05, sort=cm.SORT_RESIDUAL, knn=knn)
    ctx.sequence_errors([[0, 4, 8], [1, 2]])
    ctx.cluster_verify(np.asarray(g["assign"], np.int32))
rng = np.random.default_rng(7)
blocks = [np.asfortranarray(rng.standard_normal((80, int(rng.integers(3, 40)))).astype(np.float32)) for _ in range(7)]
with cm.Context(0) as ctx:
    ctx.register(blocks)
    ctx.block_spectra(5)
    pr = np.array([(i, j) for i in range(7) for j in range(7) if i != j], np.int32)
    ctx.pair_errors(pr)
    ctx.cluster(cm.ALG_APPROX, 0.2, sort=cm.SORT_RESIDUAL)
big = synth.config4(N=3, m=1024, rank=64)
with cm.Context(0) as ctx:
    ctx.register(big.blocks)
    ctx.block_spectra(160)
    ctx.pair_errors(np.array([[0, 1], [1, 2], [2, 0]], np.int32), operand=cm.TRUNC)
c2 = synth.config2()
with cm.Context(0) as ctx:
    ctx.register(c2.blocks[:12])
    ctx.block_spectra(c2.r)
    ctx.pair_errors(np.array([[0, 1], [2, 3], [4, 5], [6, 7]], np.int32))
    ctx.cluster(cm.ALG_APPROX, 0.05, sort=cm.SORT_RESIDUAL, knn=2)
print("sanitize probe done")
