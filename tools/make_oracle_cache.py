"""Full-size oracle results for the GPU parity tests (tests/test_gpu_fullsize.py).

Calls ONLY oracle/ (the float64 CPU oracle) and synth/ (seeded input
generators): no value here comes from the CUDA path.  The generators are
deterministic (numpy PCG64, same image on the dev host and the GPU box), so
the cached expected values apply to the collections the GPU tests rebuild.

Writes tests/oracle_cache/<name>.npz (compressed):
  config2_pairs     all 8128 norm-ordered pairs, RAW, all three estimators
  config4_pairs     all 2016 norm-ordered pairs, TRUNC (A6), all three estimators,
                    + the block spectra (top-r sigma) and energies
  config5_N{N}_r{r} the N*16 seeded candidate pairs of tools/c5_sweep.py, RAW
  greedy_<...>      oracle greedy runs (assign / order / n_evals / err2 / total)
err2 / total are float64; sigma_tilde / mu are stored as float32 (the parity
tolerance on singular values is 1e-4 relative, float32 rounding is 6e-8).

Usage: python tools/make_oracle_cache.py config2|config4|config5|greedy3|greedy5|greedy5big [...]
"""
from __future__ import annotations

import os
import sys
import time

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import oracle  # noqa: E402
from oracle import cluster as oc  # noqa: E402
import synth  # noqa: E402

OUT = os.path.join(ROOT, "tests", "oracle_cache")


def norm_order(E):
    return np.array(sorted(range(len(E)), key=lambda i: (-E[i], i)))


def save(name, **kw):
    os.makedirs(OUT, exist_ok=True)
    kw["numpy_version"] = np.array(np.__version__)
    np.savez_compressed(os.path.join(OUT, name + ".npz"), **kw)
    print(f"wrote {name}.npz", flush=True)


def pairs_cache(name, col, operand, pairs=None, nvec=None):
    t0 = time.time()
    sp = oracle.block_spectra(col.blocks, nvec=nvec)
    t_spec = time.time() - t0
    if pairs is None:
        pairs = synth.all_pairs_by_norm_order(norm_order(sp.E))
    t0 = time.time()
    res = oracle.pair_errors(sp, pairs, col.r, 7, operand)
    print(f"{name}: spectra {t_spec:.1f}s, {len(pairs)} pairs {time.time() - t0:.1f}s", flush=True)
    save(name, pairs=pairs, err2=res.err2, total=res.total, sigma_tilde=res.sigma_tilde.astype(np.float32),
         mu=res.mu.astype(np.float32), E=sp.E, sig=np.stack([s[:col.r] for s in sp.sig]).astype(np.float64),
         r=np.array(col.r), operand=np.array(operand))
    return sp


def c5_pairs(N, r, k=16):
    """tools/c5_sweep.py's seeded candidate list: k partners per block drawn uniformly."""
    rng = np.random.default_rng(100 + N + r)
    nbr = np.stack([rng.choice(np.delete(np.arange(N), i), k, replace=False) for i in range(N)])
    return synth.knn_pairs(nbr)


def greedy_cache(name, sp, r, runs, operand):
    out = {}
    for alg, srt, eps, knn in runs:
        t0 = time.time()
        g = oc.cluster(sp, alg, r, eps, srt, knn=knn, operand=operand)
        key = f"a{alg}_s{srt}_e{eps}_k{knn}"
        out[key + "_assign"] = g.assign
        out[key + "_order"] = g.order
        out[key + "_err2"] = np.asarray(g.err2)
        out[key + "_total"] = np.asarray(g.total)
        out[key + "_nevals"] = np.array(g.n_evals)
        print(f"{name} {key}: {len(g.clusters)} clusters, {g.n_evals} evals, {time.time() - t0:.1f}s", flush=True)
    save(name, **out)


def main():
    for what in sys.argv[1:]:
        if what == "config2":
            pairs_cache("config2_pairs", synth.config2(), oracle.RAW)
        elif what == "config4":
            col = synth.config4()
            sp = pairs_cache("config4_pairs", col, oracle.TRUNC, nvec=col.r)
            greedy_cache("greedy_config4", sp, col.r, [(oc.APPROX, oc.SORT_RESIDUAL, 0.15, 1)], oracle.TRUNC)
        elif what == "config5":
            for N in (512, 2048):
                for r in (16, 64):
                    col = synth.config5(N=N, r=r)
                    pairs_cache(f"config5_N{N}_r{r}", col, oracle.RAW, pairs=c5_pairs(N, r))
        elif what == "greedy3":
            col = synth.config3()
            sp = oracle.block_spectra(col.blocks, nvec=col.r)
            greedy_cache("greedy_config3", sp, col.r,
                         [(oc.APPROX, oc.SORT_RESIDUAL, 0.1, 1), (oc.APPROX, oc.SORT_RESIDUAL, 0.3, 1),
                          (oc.APPROX, oc.SORT_FROBENIUS, 0.3, 1)], oracle.TRUNC)
        elif what in ("greedy5", "greedy5big"):
            for N, r in (((512, 16), (512, 64)) if what == "greedy5" else ((2048, 16),)):
                col = synth.config5(N=N, r=r)
                sp = oracle.block_spectra(col.blocks)
                greedy_cache(f"greedy_config5_N{N}_r{r}", sp, r, [(oc.APPROX, oc.SORT_RESIDUAL, 0.1, 16)], oracle.RAW)
        else:
            raise SystemExit(f"unknown cache {what}")


if __name__ == "__main__":
    main()
