"""Estimator conservativeness diagnostic (Figure 1):
for a fixed target rank r, uniformly sample subsets of K blocks, compute the predicted
rank-r errors of each estimator for the subset (cmsvd_sequence_errors: Weyl, residual,
incremental in sampled append order) and the exact error of the explicit concatenation
(cmsvd_cluster_verify), and report the slack Delta = E~_r - E_r (Frobenius error norms,
absolute and relative to ||M||_F; reading A18: both units) over 10 trials per size.

  python tools/slack.py [config2] [out.json]
"""
import json
import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import synth  # noqa: E402
import paper_2601_11626_b200 as cm  # noqa: E402


def main():
    name = sys.argv[1] if len(sys.argv) > 1 else "config2"
    out_path = sys.argv[2] if len(sys.argv) > 2 else None
    col = synth.make_config(name)
    sizes = [2, 4, 8, 16] if col.N >= 16 else [2, 4, 8]
    trials = 10
    R = np.random.default_rng(2601)
    seqs = []
    for K in sizes:
        for _ in range(trials):
            seqs.append(list(map(int, R.choice(col.N, size=K, replace=False))))
    kinds = cm.ALL
    with cm.Context(0) as ctx:
        ctx.register(col.blocks)
        ctx.block_spectra(col.r)
        pred = ctx.sequence_errors(seqs, kinds=kinds)
        exact = []
        for q in seqs:
            assign = np.ones(col.N, np.int32)
            assign[q] = 0
            exact.append(ctx.cluster_verify(assign)["exact_err2"][0])
    exact = np.asarray(exact)
    tot = pred["total"]
    rows = []
    names = ["weyl", "residual", "incremental"]
    for i, K in enumerate(sizes):
        sl = slice(i * trials, (i + 1) * trials)
        row = {"K": K, "exact_rel_mean": float(np.mean(np.sqrt(exact[sl] / tot[sl])))}
        for k, nm in enumerate(names):
            d_abs = np.sqrt(pred["err2"][sl, k]) - np.sqrt(exact[sl])
            d_rel = d_abs / np.sqrt(tot[sl])
            row[nm] = {"slack_abs_mean": float(np.mean(d_abs)), "slack_abs_min": float(np.min(d_abs)),
                       "slack_abs_max": float(np.max(d_abs)), "slack_rel_mean": float(np.mean(d_rel)),
                       "slack_rel_min": float(np.min(d_rel)), "slack_rel_max": float(np.max(d_rel))}
        rows.append(row)
    res = {"config": name, "r": col.r, "trials": trials, "sizes": sizes, "rows": rows,
           "note": "Delta = predicted - exact rank-r error (Frobenius norms); rel = Delta / ||M||_F"}
    print(f"{name}: r={col.r}, {trials} trials per cluster size (uniform block samples)")
    print(f"{'K':>3} {'exact rel':>10} " + " ".join(f"{nm + ' dRel mean [min,max]':>34}" for nm in names))
    for row in rows:
        cells = [f"{row[nm]['slack_rel_mean']:10.2e} [{row[nm]['slack_rel_min']:9.2e},{row[nm]['slack_rel_max']:9.2e}]"
                 for nm in names]
        print(f"{row['K']:>3} {row['exact_rel_mean']:10.4f} " + " ".join(f"{c:>34}" for c in cells))
    if out_path:
        json.dump(res, open(out_path, "w"), indent=1)


if __name__ == "__main__":
    main()
