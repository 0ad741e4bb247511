"""GPU parity on collections of blocks wider than 512 columns (configs 3 and 4,
square weight-like blocks), reading A22: spectra by subspace
iteration on the GPU vs the oracle's exact m x m Gram eigendecomposition; the
base range is R^m so the paper-literal residual vanishes.  Reduced sizes keep
the oracle within seconds; the full-size config-4 case checks sampled pairs."""
import numpy as np
import pytest

import oracle
from oracle import cluster as oc
import synth
from tolerances import assert_err2, assert_sigma

pytestmark = pytest.mark.gpu

torch = pytest.importorskip("torch")


@pytest.fixture(scope="module")
def cm():
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    import paper_2601_11626_b200 as cm
    cm.load()
    return cm


def norm_order(E):
    return np.array(sorted(range(len(E)), key=lambda i: (-E[i], i)))


def compare(out, ref, kinds, what):
    for k, name in enumerate(["weyl", "residual", "incremental"]):
        if kinds & (1 << k):
            assert_err2(out["err2"][:, k], ref.err2[:, k], ref.total, f"{what} {name}")
    assert np.allclose(out["total"], ref.total, rtol=1e-12)
    if kinds & 4:
        assert_sigma(out["sigma_tilde"], ref.sigma_tilde, ref.sigma_tilde[:, 0], f"{what} sigma~")
    if kinds & 2:
        assert_sigma(out["mu"], ref.mu, ref.mu[:, 0], f"{what} mu")


def run_pairs(cm, col, r, pairs=None):
    sp = oracle.block_spectra(col.blocks)
    with cm.Context(0) as ctx:
        ctx.register(col.blocks)
        E, sig, rank = ctx.block_spectra(r)
        if pairs is None:
            pairs = synth.all_pairs_by_norm_order(norm_order(sp.E))
        out = ctx.pair_errors(pairs, kinds=7, operand=cm.TRUNC)
    return sp, E, sig, rank, pairs, out


@pytest.fixture(scope="module")
def c3(cm):
    col = synth.config3(N=6)
    return (col,) + run_pairs(cm, col, col.r)


def test_c3_spectra(c3):
    col, sp, E, sig, rank, *_ = c3
    assert np.allclose(E, sp.E, rtol=1e-12)
    ref = np.stack([s[:col.r] for s in sp.sig])
    assert_sigma(sig, ref, ref[:, 0], "config3 block sigma")
    assert np.all(rank == col.m)          # A22: rank = min(m, n)


def test_c3_all_pairs_trunc(c3):
    col, sp, E, sig, rank, pairs, out = c3
    ref = oracle.pair_errors(sp, pairs, col.r, 7, oracle.TRUNC)
    compare(out, ref, 7, "config3")
    # A22: residual = E_i + E_j - sum_{l<=r} sigma_l(A_i)^2 exactly (R = 0)
    tops = np.array([np.sum(s[:col.r] ** 2) for s in sp.sig])
    res = sp.E[pairs[:, 0]] + sp.E[pairs[:, 1]] - tops[pairs[:, 0]]
    assert np.allclose(ref.err2[:, 1], res, rtol=1e-12)
    # soundness ordering of the estimates (P6): incremental <= residual, all >= 0
    assert np.all(out["err2"][:, 2] <= out["err2"][:, 1] * (1 + 1e-6))


def test_c4_reduced(cm):
    col = synth.config4(N=4, m=1024, rank=64)
    r = 64
    sp, E, sig, rank, pairs, out = run_pairs(cm, col, r)
    ref = np.stack([s[:r] for s in sp.sig])
    assert_sigma(sig, ref, ref[:, 0], "config4-reduced block sigma")
    orc = oracle.pair_errors(sp, pairs, r, 7, oracle.TRUNC)
    compare(out, orc, 7, "config4-reduced")


def test_c3_cluster_replay(cm):
    """Alg. 3 (incremental) greedy growth on a reduced config 3 at eps = 0.3,
    residual sort, TRUNC operand: decision replay in the oracle (A12)."""
    from test_gpu_cluster import replay
    col = synth.config3(N=8)
    sp = oracle.block_spectra(col.blocks)
    with cm.Context(0) as ctx:
        ctx.register(col.blocks)
        ctx.block_spectra(col.r)
        g = ctx.cluster(cm.ALG_APPROX, 0.3, sort=cm.SORT_RESIDUAL, operand=cm.TRUNC)
    replay(sp, g, oc.APPROX, col.r, 0.3, oc.SORT_RESIDUAL, operand=oracle.TRUNC)
    assert sum(len(c) for c in g["clusters"]) == col.N


def test_big_edge_cases(cm):
    col = synth.config3(N=3, m=640)
    with cm.Context(0) as ctx:
        ctx.register(col.blocks)
        ctx.block_spectra(32)
        with pytest.raises(cm.CmsvdError):          # RAW operand: core 32 + 640 > 512
            ctx.pair_errors(np.array([[0, 1]]), kinds=7, operand=cm.RAW)
        out = ctx.pair_errors(np.array([[0, 1]]), kinds=1, operand=cm.RAW)   # Weyl needs no core
        assert np.isfinite(out["err2"][0, 0])
        with pytest.raises(cm.CmsvdError):          # Alg. 2 state needs an explicit range basis
            ctx.cluster(cm.ALG_RESIDUAL, 0.3, operand=cm.TRUNC)
    # mixing wide and narrow blocks is rejected
    with cm.Context(0) as ctx:
        ctx.register([np.asfortranarray(np.ones((640, 640), np.float32)), np.asfortranarray(np.ones((640, 8), np.float32))])
        with pytest.raises(cm.CmsvdError):
            ctx.block_spectra(8)
    # tall blocks with more than 512 columns are rejected
    with cm.Context(0) as ctx:
        ctx.register([np.asfortranarray(np.random.default_rng(0).standard_normal((700, 600)).astype(np.float32))] * 2)
        with pytest.raises(cm.CmsvdError):
            ctx.block_spectra(8)


def test_c3_tight_variants(cm):
    """N3 variants on A22 bases (square blocks): the U_r residual is a real projection here
    (the full-range residual vanishes), per-index Weyl from the top-r spectra."""
    col = synth.config3(N=4)
    sp = oracle.block_spectra(col.blocks)
    pairs = synth.all_pairs_by_norm_order(norm_order(sp.E))
    ref, tot = oracle.pair_errors_tight(sp, pairs, col.r, oracle.TRUNC)
    with cm.Context(0) as ctx:
        ctx.register(col.blocks)
        ctx.block_spectra(col.r)
        out = ctx.pair_errors_tight(pairs, operand=cm.TRUNC)
    assert_err2(out["err2x"][:, 0], ref[:, 0], tot, "config3 residual(U_r)")
    assert_err2(out["err2x"][:, 1], ref[:, 1], tot, "config3 per-index Weyl")


def _subset_spectra(col, ids):
    """Oracle spectra of a subset of blocks (the oracle's per-block results do not depend on the rest)."""
    return oracle.block_spectra(np.ascontiguousarray(col.blocks[ids]))


@pytest.mark.parametrize("name", ["config3", "config4"])
def test_full_size_sampled_pairs(cm, name):
    """BASELINE.json's full-size configs 3 (256 x 1024^2, r = 128) and 4 (64 x 4096^2, r = 256) in the
    bench launch configuration (all blocks registered, all-pairs chunking), sampled pairs checked
    against the oracle evaluated on just the blocks they touch."""
    col = synth.make_config(name)
    ids = [0, 1, 2, col.N - 1] if name == "config3" else [0, 5, col.N - 1]
    sp = _subset_spectra(col, ids)
    sub_pairs = np.array([[a, b] for a in range(len(ids)) for b in range(len(ids)) if a != b], np.int32)
    ref = oracle.pair_errors(sp, sub_pairs, col.r, 7, oracle.TRUNC)
    full_pairs = np.array([[ids[a], ids[b]] for a, b in sub_pairs], np.int32)
    with cm.Context(0) as ctx:
        ctx.register(torch.from_numpy(col.blocks).cuda())
        E, sig, rank = ctx.block_spectra(col.r)
        out = ctx.pair_errors(full_pairs, kinds=7, operand=cm.TRUNC)
    refs = np.stack([s[:col.r] for s in sp.sig])
    assert_sigma(sig[ids], refs, refs[:, 0], f"{name} block sigma")
    assert np.allclose(E[ids], sp.E, rtol=1e-12)
    compare(out, ref, 7, f"{name} full size")


@pytest.mark.parametrize("tc_big,tc_ws", [("1", "1"), ("1", "0"), ("0", "1")])
def test_c4_reduced_wide_operands(cm, tc_big, tc_ws, monkeypatch):
    """r = 192 > 128: bases and TRUNC operands wider than one 128-column tile take the warp-specialised
    TMA-fed tcgen05 kernel on pre-split tf32 planes (k_gemm_ws: Z = Q^T F, R' = F - Q Z, W' = R'^T R'; ragged
    here: 192 = 128 + 64 rows of Z, 192 of the 256 tile columns), with CMSVD_TC_WS=0 the staged GEMM tiles
    (k_gemm_tc), with CMSVD_TC_BIG=0 the SIMT path.  All three against the oracle."""
    monkeypatch.setenv("CMSVD_TC_BIG", tc_big)
    monkeypatch.setenv("CMSVD_TC_WS", tc_ws)
    col = synth.config4(N=4, m=1024, rank=64)
    r = 192
    sp, E, sig, rank, pairs, out = run_pairs(cm, col, r)
    orc = oracle.pair_errors(sp, pairs, r, 7, oracle.TRUNC)
    compare(out, orc, 7, f"config4-reduced r=192 tc_big={tc_big} tc_ws={tc_ws}")


def test_core_gram_lower_storage_only(cm, monkeypatch):
    """Core Grams above n = 160 are built in lower storage only (k_build_G leaves the strict upper triangle of
    G unwritten, and reads only the lower triangles of W' and Z^T Z).  Poisoning the upper triangle with NaN
    (CMSVD_G_UPPER=2) or writing it in full (=0) must not change a single output bit: nothing downstream of
    k_build_G reads it.  Checked against the oracle as well."""
    col = synth.config4(N=4, m=1024, rank=64)
    r = 192
    outs = {}
    for mode in ("1", "2", "0"):
        monkeypatch.setenv("CMSVD_G_UPPER", mode)
        sp, E, sig, rank, pairs, outs[mode] = run_pairs(cm, col, r)
    for mode in ("2", "0"):
        for key in ("err2", "total", "sigma_tilde", "mu"):
            a, b = outs["1"][key], outs[mode][key]
            if a is not None:
                assert np.array_equal(np.asarray(a), np.asarray(b), equal_nan=True), (mode, key)
    orc = oracle.pair_errors(sp, pairs, r, 7, oracle.TRUNC)
    compare(outs["1"], orc, 7, "config4-reduced r=192, lower-storage core Grams")


def _flat_block(R, m, decay):
    U = np.linalg.qr(R.standard_normal((m, m)))[0]
    V = np.linalg.qr(R.standard_normal((m, m)))[0]
    s = np.exp(-decay * np.arange(m))
    return ((U * s) @ V.T).astype(np.float32)


def test_a22_guard_catches_unresolved_spectrum(cm, monkeypatch):
    """Reading A22's subspace iteration carries an a-posteriori guard: the Ritz residuals
    ||A A^T u_l - lambda_l u_l|| / lambda_l of the returned l < r must be <= 1e-4 (which bounds the relative
    error of sigma_l by 5e-5), else more power iterations run, and CMSVD_E_NOCONV after
    CMSVD_SUBSPACE_MAX.  A spectrum sigma_l = exp(-0.006 l) around r = 32 (s = 64: convergence factor
    (sigma_65 / sigma_32)^2 = 0.67 per step) cannot be resolved by 2 iterations -> NOCONV, not a silent
    result; with the defaults (12, up to 48) the guard extends the iteration and the result matches the
    oracle's exact spectrum."""
    R = np.random.default_rng(21)
    m, r = 640, 32
    blocks = np.stack([_flat_block(R, m, 0.006).T for _ in range(2)])
    monkeypatch.setenv("CMSVD_SUBSPACE_ITERS", "2")
    monkeypatch.setenv("CMSVD_SUBSPACE_MAX", "2")
    with cm.Context(0) as ctx:
        ctx.register(blocks)
        with pytest.raises(cm.CmsvdError) as ei:
            ctx.block_spectra(r)
        assert ei.value.status == 5   # CMSVD_E_NOCONV
    monkeypatch.delenv("CMSVD_SUBSPACE_ITERS")
    monkeypatch.delenv("CMSVD_SUBSPACE_MAX")
    sp = oracle.block_spectra(blocks, nvec=r)
    with cm.Context(0) as ctx:
        ctx.register(blocks)
        E, sig, rank = ctx.block_spectra(r)
        resid, iters = ctx.spectra_diagnostics()
    assert resid <= 1e-4 and iters > 12, (resid, iters)
    ref = np.stack([s_[:r] for s_ in sp.sig])
    assert_sigma(sig, ref, ref[:, 0], "flat-spectrum block sigma")


@pytest.mark.parametrize("name", ["config3", "config4"])
def test_a22_guard_quiet_on_bench_configs(cm, name):
    """On BASELINE.json's configs 3 and 4 the default 12 power iterations already pass the guard."""
    col = synth.make_config(name, N=4) if name == "config3" else synth.config4(N=4)
    with cm.Context(0) as ctx:
        ctx.register(col.blocks)
        ctx.block_spectra(col.r)
        resid, iters = ctx.spectra_diagnostics()
    assert resid <= 1e-4 and iters == 12, (resid, iters)
