"""GPU greedy drivers (cmsvd_cluster, S10) vs the oracle's (-m gpu).

Assignment parity follows DESIGN.md reading A12: Algorithm 1 must match the
oracle exactly; for Algorithms 2-3 the GPU's decisions are *replayed* in the
oracle -- every appended block must be the oracle's optimal candidate (within
1e-5 relative of its sort key) and accepted by the oracle's certificate, and
every cluster close must be an oracle rejection, unless the oracle's relative
error lies within 1e-3 relative of eps (the north_star tie band).  A single
near-tied divergence would otherwise cascade through the rest of a greedy run.
"""
import numpy as np
import pytest

import oracle
from oracle import cluster as oc
import synth

pytestmark = pytest.mark.gpu
torch = pytest.importorskip("torch")


@pytest.fixture(scope="module")
def cm():
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    import paper_2601_11626_b200 as cm
    cm.load()
    return cm


def in_tie_band(e2, tot, eps):
    rel = np.sqrt(max(e2, 0.0) / tot)
    return abs(rel - eps) <= 1e-3 * eps


def replay(sp, gpu, algorithm, r, eps, sort, operand=oracle.RAW):
    """Walk the GPU clusters through the oracle's state machine."""
    N = len(sp.A)
    E = sp.E
    remaining = sorted(range(N), key=lambda i: (-E[i], i))
    State = oc._ResidualState if algorithm == oc.RESIDUAL_ALG else oc._IncrementalState
    for members in gpu["clusters"]:
        anchor = members[0]
        assert anchor == remaining[0], f"anchor {anchor} is not the largest remaining block {remaining[0]}"
        remaining.remove(anchor)
        st = State(sp, anchor, r)
        for b in members[1:]:
            F = oc._operand(sp, b, r, operand)
            if sort == oc.SORT_FROBENIUS:
                best = min(remaining, key=lambda j: (E[j], j))
                assert E[b] <= E[best] * (1 + 1e-12), f"block {b} is not the smallest-norm candidate {best}"
            else:
                keys = {j: st.key(oc._operand(sp, j, r, operand)) for j in remaining}
                kmin = min(keys.values())
                assert keys[b] <= kmin * (1 + 1e-5) + 1e-12 * E[b], \
                    f"block {b} key {keys[b]} is not oracle-optimal ({kmin})"
            e2, tot, data = st.tentative(F, E[b])
            ok = (E[b] == 0.0) or (e2 <= eps * eps * tot)
            assert ok or in_tie_band(e2, tot, eps), f"oracle rejects appended block {b}: rel {np.sqrt(e2 / tot)}"
            st.commit(E[b], data)
            remaining.remove(b)
        if remaining:
            if sort == oc.SORT_FROBENIUS:
                nxt = min(remaining, key=lambda j: (E[j], j))
            else:
                nxt = min(remaining, key=lambda j: (st.key(oc._operand(sp, j, r, operand)), j))
            e2, tot, _ = st.tentative(oc._operand(sp, nxt, r, operand), E[nxt])
            ok = (E[nxt] == 0.0) or (e2 <= eps * eps * tot)
            assert (not ok) or in_tie_band(e2, tot, eps), \
                f"GPU closed a cluster but the oracle accepts {nxt}: rel {np.sqrt(e2 / tot)}"
    assert not remaining


def run_gpu(cm, blocks, r, alg, eps, sort, knn=1, operand=0):
    ctx = cm.Context(0)
    ctx.register(blocks)
    ctx.block_spectra(r)
    res = ctx.cluster(alg, eps, sort=sort, knn=knn, operand=operand)
    ctx.close()
    return res


@pytest.mark.parametrize("eps", [0.05, 0.1, 0.3])
def test_c1_max_norm_exact(cm, eps):
    col = synth.config1()
    sp = oracle.block_spectra(col.blocks)
    g = run_gpu(cm, col.blocks, col.r, cm.ALG_MAX_NORM, eps, 0)
    o = oc.cluster(sp, oc.MAX_NORM, col.r, eps)
    assert g["clusters"] == o.clusters
    assert np.allclose(g["err2"], o.err2, rtol=1e-9, atol=1e-9 * max(o.total))


@pytest.mark.parametrize("alg", [oc.RESIDUAL_ALG, oc.APPROX])
@pytest.mark.parametrize("sort", [oc.SORT_FROBENIUS, oc.SORT_RESIDUAL])
@pytest.mark.parametrize("eps", [0.05, 0.3])
def test_c1_tracked_replay(cm, alg, sort, eps):
    col = synth.config1()
    sp = oracle.block_spectra(col.blocks)
    g = run_gpu(cm, col.blocks, col.r, alg, eps, sort)
    replay(sp, g, alg, col.r, eps, sort)
    o = oc.cluster(sp, alg, col.r, eps, sort)
    # on config 1 the merges lie far from eps and the keys are well separated: identical partitions
    assert g["clusters"] == o.clusters
    assert g["n_evals"] == o.n_evals
    rel_g = np.sqrt(np.asarray(g["err2"]) / np.asarray(g["total"]))
    rel_o = np.sqrt(np.asarray(o.err2) / np.asarray(o.total))
    assert np.allclose(rel_g, rel_o, rtol=1e-3, atol=1e-4)


def test_c1_recovers_groups(cm):
    col = synth.config1()
    g = run_gpu(cm, col.blocks, col.r, cm.ALG_APPROX, 0.05, cm.SORT_RESIDUAL)
    assert len(g["clusters"]) == 4
    for c in g["clusters"]:
        assert len({int(col.groups[b]) for b in c}) == 1


@pytest.mark.parametrize("eps", [0.02, 0.05])
def test_c2_approx_residual_replay(cm, eps):
    """Config 2, Alg. 3 residual sort: 8 group-pure clusters of 16."""
    col = synth.config2()
    sp = oracle.block_spectra(col.blocks)
    g = run_gpu(cm, col.blocks, col.r, cm.ALG_APPROX, eps, cm.SORT_RESIDUAL)
    assert len(g["clusters"]) == 8
    for c in g["clusters"]:
        assert len({int(col.groups[b]) for b in c}) == 1 and len(c) == 16
    replay(sp, g, oc.APPROX, col.r, eps, oc.SORT_RESIDUAL)


def test_c2_frobenius_and_residual_alg(cm):
    col = synth.config2()
    sp = oracle.block_spectra(col.blocks)
    g = run_gpu(cm, col.blocks, col.r, cm.ALG_APPROX, 0.05, cm.SORT_FROBENIUS)
    replay(sp, g, oc.APPROX, col.r, 0.05, oc.SORT_FROBENIUS)
    g2 = run_gpu(cm, col.blocks, col.r, cm.ALG_RESIDUAL, 0.05, cm.SORT_FROBENIUS)
    replay(sp, g2, oc.RESIDUAL_ALG, col.r, 0.05, oc.SORT_FROBENIUS)
    g3 = run_gpu(cm, col.blocks, col.r, cm.ALG_MAX_NORM, 0.05, 0)
    assert g3["clusters"] == oc.cluster(sp, oc.MAX_NORM, col.r, 0.05).clusters


@pytest.mark.parametrize("seed", range(3))
def test_random_collections_replay(cm, seed):
    R = np.random.default_rng(500 + seed)
    N, m, n, G = 14, 40, 6, 3
    U = [np.linalg.qr(R.standard_normal((m, 3)))[0] for _ in range(G)]
    blocks = np.stack([(U[i % G] @ R.standard_normal((3, n)) * R.uniform(0.5, 2)
                        + 0.03 * R.standard_normal((m, n))).T for i in range(N)]).astype(np.float32)
    sp = oracle.block_spectra(blocks)
    for alg in (oc.RESIDUAL_ALG, oc.APPROX):
        for sort in (oc.SORT_FROBENIUS, oc.SORT_RESIDUAL):
            g = run_gpu(cm, blocks, 4, alg, 0.1, sort)
            replay(sp, g, alg, 4, 0.1, sort)
            # certified algorithms: every GPU cluster's exact error is within eps
            for c, e2, tot in zip(g["clusters"], g["err2"], g["total"]):
                if len(c) > 1 and alg == oc.RESIDUAL_ALG:
                    ex = oracle.exact_groups(sp, [c], 4)[0]
                    assert np.sqrt(ex / tot) <= 0.1 + 1e-6


@pytest.mark.parametrize("alg", [oc.RESIDUAL_ALG, oc.APPROX])
@pytest.mark.parametrize("knn", [2, 4])
def test_knn_window_matches_oracle(cm, alg, knn):
    """kNN window (skip-and-continue over the knn best-ranked candidates, A10) on config 1 and a
    reduced config 5 (tall-thin 2048 x 64, 32 hidden groups): identical partitions and
    evaluation counts (keys and merges are well separated on these inputs)."""
    for col, eps in [(synth.config1(), 0.05), (synth.config5(N=48, r=16), 0.1)]:
        sp = oracle.block_spectra(col.blocks)
        g = run_gpu(cm, col.blocks, col.r, alg, eps, oc.SORT_RESIDUAL, knn=knn)
        o = oc.cluster(sp, alg, col.r, eps, oc.SORT_RESIDUAL, knn=knn)
        assert g["clusters"] == o.clusters, (col.name, knn)
        assert g["n_evals"] == o.n_evals


def _clusters_of(assign):
    nc = int(np.max(assign)) + 1
    return [sorted(np.flatnonzero(assign == c).tolist()) for c in range(nc)]


@pytest.mark.parametrize("alg", [oc.MAX_NORM, oc.RESIDUAL_ALG, oc.APPROX])
def test_cluster_verify_c1(cm, alg):
    """N1: exact per-cluster errors of the explicit concatenations (both Gram orientations: singletons
    N_c = 32 < m = 64, merged clusters N_c > m) vs the oracle's brute-force SVD; compression accounting
    identical to the oracle's (reading A23); certified algorithms stay within eps (P12)."""
    from tolerances import assert_err2
    col = synth.config1()
    sp = oracle.block_spectra(col.blocks)
    eps = 0.05
    with cm.Context(0) as ctx:
        ctx.register(col.blocks)
        ctx.block_spectra(col.r)
        g = ctx.cluster(alg, eps, sort=cm.SORT_RESIDUAL if alg else cm.SORT_FROBENIUS)
        assign = np.asarray(g["assign"], np.int32)
        v = ctx.cluster_verify(assign)
    groups = _clusters_of(assign)
    ex = oracle.exact_groups(sp, groups, col.r)
    tot = np.array([sum(sp.E[i] for i in gr) for gr in groups])
    assert np.allclose(v["total"], tot, rtol=1e-12)
    assert_err2(v["exact_err2"], ex, tot, "cluster exact error")
    mem, ratio = oc.compression(col.m, sp.n, groups, col.r)
    assert np.array_equal(v["mem"], mem) and abs(v["ratio"] - ratio) < 1e-12 * ratio
    if alg in (oc.MAX_NORM, oc.RESIDUAL_ALG):      # certified clusterings (P12)
        assert np.all(v["rel"] <= eps * (1 + 1e-3))


def test_cluster_verify_c2_row_gram(cm):
    """Config 2, Alg. 3 residual sort at eps = 0.05: 8 clusters of 16 blocks, N_c = 2048 > m = 512 (row
    Gram, 512 x 512 eigen-solve); two clusters checked against the oracle's explicit SVD, all within eps."""
    from tolerances import assert_err2
    col = synth.config2()
    sp = oracle.block_spectra(col.blocks)
    with cm.Context(0) as ctx:
        ctx.register(col.blocks)
        ctx.block_spectra(col.r)
        g = ctx.cluster(cm.ALG_APPROX, 0.05, sort=cm.SORT_RESIDUAL)
        assign = np.asarray(g["assign"], np.int32)
        v = ctx.cluster_verify(assign)
    groups = _clusters_of(assign)
    assert len(groups) == 8
    ex = oracle.exact_groups(sp, groups[:2], col.r)
    assert_err2(v["exact_err2"][:2], ex, v["total"][:2], "config2 cluster exact error")
    assert np.all(v["rel"] <= 0.05)
    mem, ratio = oc.compression(col.m, sp.n, groups, col.r)
    assert np.array_equal(v["mem"], mem)


@pytest.mark.parametrize("name", ["config1", "config2"])
def test_sequence_errors_vs_oracle(cm, name):
    """N2: Weyl / residual / incremental estimates of random block sequences (K = 1..6, the slack
    diagnostic's inputs) against the oracle's state machines; every estimate >= the exact error of
    the explicit concatenation (GPU cluster_verify)."""
    from tolerances import assert_err2
    col = synth.make_config(name)
    sp = oracle.block_spectra(col.blocks)
    R = np.random.default_rng(11)
    seqs = [list(map(int, R.choice(col.N, size=int(R.integers(1, 7)), replace=False))) for _ in range(10)]
    ref, tot = oc.sequence_errors(sp, seqs, col.r)
    with cm.Context(0) as ctx:
        ctx.register(col.blocks)
        ctx.block_spectra(col.r)
        out = ctx.sequence_errors(seqs)
        ex = []
        for q in seqs:     # exact error of each sequence's concatenation: one cluster of its members
            assign = np.ones(col.N, np.int32)
            assign[q] = 0
            ex.append(ctx.cluster_verify(assign)["exact_err2"][0])
    assert np.allclose(out["total"], tot, rtol=1e-12)
    for k, nm in enumerate(["weyl", "residual", "incremental"]):
        assert_err2(out["err2"][:, k], ref[:, k], tot, f"{name} sequence {nm}")
        assert np.all(out["err2"][:, k] >= np.asarray(ex) * (1 - 2e-3) - 1e-7 * tot)


@pytest.mark.parametrize("name", ["config1", "config2"])
def test_cluster_factors_reconstruction(cm, name):
    """N1 codec: per-cluster factors Ũ_c = U_c S_c and V_c of the rank-r truncated SVD of the
    concatenation; reconstructing every block as Ũ_c V_{c,i}^T gives the exact
    rank-r error of the cluster (Thm EYM) -- checked against cmsvd_cluster_verify and, for config 1,
    the oracle's explicit SVD; V_c has orthonormal columns (both Gram orientations are exercised)."""
    col = synth.make_config(name)
    with cm.Context(0) as ctx:
        ctx.register(col.blocks)
        ctx.block_spectra(col.r)
        g = ctx.cluster(cm.ALG_APPROX, 0.05, sort=cm.SORT_RESIDUAL)
        assign = np.asarray(g["assign"], np.int32)
        fac = ctx.cluster_factors(assign)
        v = ctx.cluster_verify(assign)
    for c, (members, Ut, V) in enumerate(fac):
        X = np.concatenate([col.blocks[i].T.astype(np.float64) for i in members], axis=1)
        Xh = Ut.astype(np.float64) @ V.astype(np.float64).T
        err2 = float(np.sum((X - Xh) ** 2))
        tot = float(np.sum(X * X))
        assert abs(err2 - v["exact_err2"][c]) <= 2e-3 * v["exact_err2"][c] + 1e-6 * tot, (c, err2, v["exact_err2"][c])
        G = V.astype(np.float64).T @ V.astype(np.float64)
        live = np.linalg.norm(Ut, axis=0) > 0
        assert np.allclose(G[np.ix_(live, live)], np.eye(int(live.sum())), atol=1e-5)
    if name == "config1":
        sp = oracle.block_spectra(col.blocks)
        ex = oracle.exact_groups(sp, [list(mb) for mb, _, _ in fac], col.r)
        from tolerances import assert_err2
        assert_err2(v["exact_err2"], ex, v["total"], "config1 cluster exact")


@pytest.mark.parametrize("knn", [1, 4])
def test_c2_commit_reuse_matches_full_commit(cm, knn, monkeypatch):
    """Alg. 3 commits from the evaluation's saved reflectors (default) vs the full QL commit
    (CMSVD_COMMIT_TOPK=0) on config 2 (n = r + w = 160, register-resident kernel; knn = 4 exercises the
    per-pair save stride of the evaluation window): the same clusters, certificates within 1e-6."""
    col = synth.config2()
    res = []
    for flag in ("1", "0"):
        monkeypatch.setenv("CMSVD_COMMIT_TOPK", flag)
        with cm.Context(0, torch.cuda.current_stream().cuda_stream) as ctx:
            ctx.register(torch.from_numpy(col.blocks).cuda())
            ctx.block_spectra(col.r)
            res.append(ctx.cluster(cm.ALG_APPROX, 0.05, sort=cm.SORT_RESIDUAL, knn=knn))
    a, b = res
    assert np.array_equal(np.asarray(a["assign"]), np.asarray(b["assign"]))
    assert np.allclose(a["err2"], b["err2"], rtol=1e-6, atol=1e-9 * float(np.max(b["total"])))


@pytest.mark.parametrize("alg", [oc.RESIDUAL_ALG, oc.APPROX])
@pytest.mark.parametrize("sort", [oc.SORT_FROBENIUS, oc.SORT_RESIDUAL])
@pytest.mark.parametrize("eps", [0.02, 0.05, 0.1])
def test_c2_full_size_greedy_grid(cm, alg, sort, eps):
    """BASELINE.json config 2 at full size, every eps it is quoted with, Algs. 2 and 3 x both sort modes:
    decision replay of the GPU run in the oracle (A12), and Alg. 1 exact."""
    col = synth.config2()
    sp = _c2_spectra()
    g = run_gpu(cm, col.blocks, col.r, alg, eps, sort)
    replay(sp, g, alg, col.r, eps, sort)
    assert sum(len(c) for c in g["clusters"]) == col.N
    g1 = run_gpu(cm, col.blocks, col.r, cm.ALG_MAX_NORM, eps, 0)
    assert g1["clusters"] == oc.cluster(sp, oc.MAX_NORM, col.r, eps).clusters


_C2 = {}


def _c2_spectra():
    if "sp" not in _C2:
        _C2["sp"] = oracle.block_spectra(synth.config2().blocks)
    return _C2["sp"]


def _axis_keys():
    import axis_example as ax
    return sorted(ax.RUNS)


@pytest.mark.parametrize("key", _axis_keys())
def test_hand_traced_greedy_run(cm, key):
    """The hand-traced axis-aligned run of tests/axis_example.py (ragged widths 1-2, m = 6): compositions,
    append orders, number of tentative evaluations and certificates, against values derived by hand
    (not the oracle's output); fp32 inputs, so the integers hold to ~1e-6 of the cluster energy."""
    import axis_example as ax
    alg, sort, eps, knn = key
    clusters, err2, total, evals = ax.RUNS[key]
    g = run_gpu(cm, ax.blocks(np.float32), ax.R, alg, eps, sort, knn=knn)
    assert [list(c) for c in g["clusters"]] == clusters
    assert g["n_evals"] == len(evals)
    assert np.allclose(g["total"], total, rtol=1e-6)
    assert np.allclose(g["err2"], err2, rtol=0, atol=1e-5 * max(total))
