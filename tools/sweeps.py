"""Compression-vs-error and compression-vs-rank sweeps and the random-clustering baseline
(Figure 2 / Table 3 protocols on synthetic data).

For each (eps, r): Alg. 3 (approximate incremental, residual sort) on the collection, then
cmsvd_cluster_verify for the exact per-cluster errors and the compression ratio (reading A23).
Random baseline: K uniformly random clusters, same accounting.

  python tools/sweeps.py [config2] [out.json]
"""
import json
import os
import sys
import time

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import synth  # noqa: E402
import paper_2601_11626_b200 as cm  # noqa: E402


def main():
    name = sys.argv[1] if len(sys.argv) > 1 else "config2"
    out_path = sys.argv[2] if len(sys.argv) > 2 else None
    col = synth.make_config(name)
    res = {"config": name, "eps_sweep": [], "rank_sweep": [], "random": []}
    with cm.Context(0) as ctx:
        ctx.register(col.blocks)

        def run(eps, r):
            ctx.block_spectra(r)
            t = time.time()
            g = ctx.cluster(cm.ALG_APPROX, eps, sort=cm.SORT_RESIDUAL)
            dt = time.time() - t
            v = ctx.cluster_verify(np.asarray(g["assign"], np.int32), r)
            return {"eps": eps, "r": r, "clusters": len(g["clusters"]), "n_evals": int(g["n_evals"]),
                    "ratio": float(v["ratio"]), "rel_max": float(np.max(v["rel"])),
                    "rel_mean": float(np.mean(v["rel"])), "violations": int(np.sum(v["rel"] > eps)),
                    "wall_ms": 1e3 * dt}

        for eps in (0.02, 0.05, 0.1, 0.2, 0.3):
            res["eps_sweep"].append(run(eps, col.r))
        for r in (8, 16, 24, 32, 48, 64):
            res["rank_sweep"].append(run(0.05, r))
        ctx.block_spectra(col.r)
        R = np.random.default_rng(7)
        for K in (8, 32, 128):
            assign = R.integers(0, K, col.N).astype(np.int32)
            # relabel to 0..K'-1 (every cluster non-empty)
            _, assign = np.unique(assign, return_inverse=True)
            v = ctx.cluster_verify(assign.astype(np.int32), col.r)
            res["random"].append({"K": int(assign.max() + 1), "ratio": float(v["ratio"]),
                                  "rel_mean": float(np.mean(v["rel"])), "rel_std": float(np.std(v["rel"]))})
    print(f"{name}: Alg. 3 (residual sort) sweeps; exact errors from cmsvd_cluster_verify")
    print("(viol = clusters whose exact rel error exceeds eps: singletons whose own rank-r error already does)")
    print(f"{'eps':>5} {'r':>3} {'clusters':>8} {'ratio':>8} {'rel max':>8} {'viol':>4} {'evals':>6} {'ms':>8}")
    for row in res["eps_sweep"] + res["rank_sweep"]:
        print(f"{row['eps']:5.2f} {row['r']:3d} {row['clusters']:8d} {row['ratio']:8.3f} {row['rel_max']:8.4f} "
              f"{row['violations']:4d} {row['n_evals']:6d} {row['wall_ms']:8.1f}")
    print("random clustering baseline:")
    for row in res["random"]:
        print(f"  K={row['K']:4d}: ratio {row['ratio']:8.3f}, rel error {row['rel_mean']:.3f} +- {row['rel_std']:.3f}")
    if out_path:
        json.dump(res, open(out_path, "w"), indent=1)


if __name__ == "__main__":
    main()
