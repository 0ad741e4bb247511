"""Pins of the oracle's greedy drivers (Appendix E):
certified clustering (P12: Algs 1-2 clusters have exact relative error
<= eps), Alg. 3 never violates eps (P13,
provable by F3), cover/determinism, and the paper's regimes on config 1."""
import numpy as np
import pytest

import oracle
from oracle import cluster as oc
import synth


def random_collection(seed, N=10, m=16, n=3, G=3, noise=0.02):
    R = np.random.default_rng(seed)
    U = [np.linalg.qr(R.standard_normal((m, 2)))[0] for _ in range(G)]
    blocks = []
    for i in range(N):
        a = U[i % G] @ R.standard_normal((2, n)) * R.uniform(0.5, 2) + noise * R.standard_normal((m, n))
        blocks.append(a)
    return oracle.block_spectra(blocks)


def check_cover(res, N):
    assert sorted(np.concatenate([np.array(c) for c in res.clusters]).tolist()) == list(range(N))
    for cid, c in enumerate(res.clusters):
        for pos, b in enumerate(c):
            assert res.assign[b] == cid and res.order[b] == pos


def exact_rel(sp, members, r):
    e2 = oracle.exact_groups(sp, [members], r)[0]
    return np.sqrt(e2 / sum(sp.E[b] for b in members))


@pytest.mark.parametrize("seed", range(6))
@pytest.mark.parametrize("eps", [0.05, 0.2])
@pytest.mark.parametrize("r", [2, 4])
def test_certified_algorithms(seed, eps, r):
    sp = random_collection(seed)
    N = len(sp.A)
    runs = [oc.cluster(sp, oc.MAX_NORM, r, eps)]
    for srt in (oc.SORT_FROBENIUS, oc.SORT_RESIDUAL):
        runs.append(oc.cluster(sp, oc.RESIDUAL_ALG, r, eps, srt))
        runs.append(oc.cluster(sp, oc.APPROX, r, eps, srt))
    for k, res in enumerate(runs):
        check_cover(res, N)
        for c, e2, tot in zip(res.clusters, res.err2, res.total):
            if len(c) == 1:
                continue
            rel = exact_rel(sp, c, r)
            assert rel <= eps + 1e-9, (k, c, rel)
            # the certificate itself upper-bounds the exact error
            assert rel <= np.sqrt(e2 / tot) + 1e-9


def test_deterministic():
    sp = random_collection(3)
    a = oc.cluster(sp, oc.APPROX, 3, 0.1, oc.SORT_RESIDUAL)
    b = oc.cluster(sp, oc.APPROX, 3, 0.1, oc.SORT_RESIDUAL)
    assert a.clusters == b.clusters and a.err2 == b.err2


def test_max_norm_spec_example():
    """anchor energy 100 (4 cols), r = 4, eps = 0.05, two tail
    blocks of energy 0.1 -> both merged (rel = sqrt(0.2/100.2) = 0.0447)."""
    R = np.random.default_rng(0)
    Q = np.linalg.qr(R.standard_normal((12, 6)))[0]
    anchor = Q[:, :4] * 5.0                  # energy 4*25 = 100
    t1 = Q[:, 4:5] * np.sqrt(0.1)
    t2 = Q[:, 5:6] * np.sqrt(0.1) * 0.999
    sp = oracle.block_spectra([anchor, t1, t2])
    res = oc.cluster(sp, oc.MAX_NORM, 4, 0.05)
    # head = anchor (width 4 = r); tail blocks are appended smallest first
    assert res.clusters == [[0, 2, 1]]
    assert abs(np.sqrt(res.err2[0] / res.total[0]) - np.sqrt(0.1999 / 100.1999)) < 1e-4


def test_zero_blocks_merge_unconditionally():
    R = np.random.default_rng(1)
    A = R.standard_normal((8, 4))
    sp = oracle.block_spectra([A, np.zeros((8, 2)), R.standard_normal((8, 4))])
    res = oc.cluster(sp, oc.APPROX, 2, 0.01)
    assert any(1 in c and len(c) > 1 for c in res.clusters)


def test_config1_regimes():
    """Config 1 (BASELINE configs[0]): residual-sort Alg. 3 recovers the 4
    hidden groups at eps = 0.05 (SURVEY §8(d) simulated outcome)."""
    col = synth.config1()
    sp = oracle.block_spectra(col.blocks)
    res = oc.cluster(sp, oc.APPROX, col.r, 0.05, oc.SORT_RESIDUAL)
    assert len(res.clusters) == 4
    for c in res.clusters:
        assert len({int(col.groups[b]) for b in c}) == 1
    for c in res.clusters:
        assert exact_rel(sp, c, col.r) <= 0.05


def test_compression_closed_forms():
    """P14: PDEBench (Table 1: 5000 blocks of 3072 x 67, r = 67) in one cluster gives Table 2's
    45.4341; all-singleton clusterings of BigEarthNet (1440 x 20, r = 20) give
    exactly 1.0 (Table 2's 1.000*, reading A23)."""
    from oracle.cluster import compression
    mem, ratio = compression(3072, np.full(5000, 67), [list(range(5000))], 67)
    assert abs(ratio - 45.43411) < 5e-5
    assert mem[0] == 67 * (3072 + 5000 * 67)
    mem, ratio = compression(1440, np.full(10, 20), [[i] for i in range(10)], 20)
    assert ratio == 1.0 and np.all(mem == 1440 * 20)
    # a compressible pair next to raw singletons
    mem, ratio = compression(12800, np.full(4, 20), [[0, 1], [2], [3]], 20)
    assert list(mem) == [20 * (12800 + 40), 12800 * 20, 12800 * 20]


def test_sequence_errors_pins():
    """N2 estimates of block sequences: a 2-block sequence equals the pair estimators (same
    definitions), every estimate of a K-block sequence is >= the exact error of the explicit
    concatenation (Thm 1, Cor 1, F3), and a single block gives its own tail for every kind."""
    col = synth.config1()
    sp = oracle.block_spectra(col.blocks)
    r = col.r
    R = np.random.default_rng(3)
    e2, tot = oc.sequence_errors(sp, [[3, 7]], r)
    pe = oracle.pair_errors(sp, [[3, 7]], r, 7)
    assert np.allclose(e2[0], pe.err2[0], rtol=1e-12, atol=1e-12 * tot[0])
    seqs = [list(R.choice(col.N, size=int(R.integers(1, 7)), replace=False)) for _ in range(12)]
    e2, tot = oc.sequence_errors(sp, seqs, r)
    ex = oracle.exact_groups(sp, seqs, r)
    for s, seq in enumerate(seqs):
        assert np.all(e2[s] >= ex[s] - 1e-9 * tot[s]), (seq, e2[s], ex[s])
        if len(seq) == 1:
            tail = float(np.sum(sp.sig[seq[0]][r:] ** 2))
            assert np.allclose(e2[s], tail, rtol=1e-9, atol=1e-9 * tot[s])


def _axis_runs():
    import axis_example as ax
    return ax, sorted(ax.RUNS)


@pytest.mark.parametrize("key", _axis_runs()[1])
def test_hand_traced_greedy_run(key):
    """Exact compositions, append orders, certificates and every tentative evaluation of Algs 2-3 on the
    axis-aligned collection of tests/axis_example.py, whose run is traced by hand there (candidate order
    of both sort modes, stop on the first rejection, the kNN window, the commit's truncation, and the
    point where Alg. 2 and Alg. 3 part)."""
    ax, _ = _axis_runs()
    alg, sort, eps, knn = key
    clusters, err2, total, evals = ax.RUNS[key]
    sp = oracle.block_spectra(ax.blocks())
    res = oc.cluster(sp, alg, ax.R, eps, sort, knn)
    assert res.clusters == clusters
    check_cover(res, 5)
    assert np.allclose(res.total, total, rtol=1e-12)
    assert np.allclose(res.err2, err2, rtol=0, atol=1e-10)
    assert res.n_evals == len(evals)
    got = [(c, b, e2, tot, ok) for (c, b, _, e2, tot, ok) in res.decisions]
    for g, e in zip(got, evals):
        assert g[0] == e[0] and g[1] == e[1] and g[4] == e[4], (g, e)
        assert abs(g[2] - e[2]) <= 1e-10 and abs(g[3] - e[3]) <= 1e-10, (g, e)
