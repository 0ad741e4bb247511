"""GPU parity: the CUDA path (through the C ABI) vs the float64 oracle,
element by element on the same seeded inputs (-m gpu)."""
import numpy as np
import pytest

import oracle
import synth
from tolerances import assert_err2, assert_sigma, err2_ok

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


def gpu_ctx(cm, blocks, r, device_input=True):
    ctx = cm.Context(0, torch.cuda.current_stream().cuda_stream)
    if device_input and isinstance(blocks, np.ndarray):
        ctx.register(torch.from_numpy(np.ascontiguousarray(blocks)).cuda())
    else:
        ctx.register(blocks)
    E, sig, rank = ctx.block_spectra(r)
    return ctx, E, sig, rank


def compare_pairs(out, ref, kinds=7, what=""):
    for k, name in enumerate(["weyl", "residual", "incremental"]):
        if kinds & (1 << k):
            assert_err2(out["err2"][:, k], ref.err2[:, k], ref.total, f"{what} {name}")
        else:
            assert np.all(np.isnan(out["err2"][:, k]))
    assert np.allclose(out["total"], ref.total, rtol=1e-12)
    if kinds & 4:
        s1 = np.maximum(ref.sigma_tilde[:, 0], 1e-300)
        assert_sigma(out["sigma_tilde"], ref.sigma_tilde, s1, f"{what} sigma~")
    if kinds & 2:
        s1 = np.maximum(ref.mu[:, 0], 1e-300)
        assert_sigma(out["mu"], ref.mu, s1, f"{what} mu")


# --------------------------------------------------------------- config 1 --
@pytest.fixture(scope="module")
def c1(cm):
    col = synth.config1()
    sp = oracle.block_spectra(col.blocks)
    ctx, E, sig, rank = gpu_ctx(cm, col.blocks, col.r)
    yield col, sp, ctx, E, sig, rank
    ctx.close()


def test_c1_energies_and_spectra(c1):
    col, sp, ctx, E, sig, rank = c1
    assert np.allclose(E, sp.E, rtol=1e-12, atol=0)
    ref = np.stack([s[:col.r] for s in sp.sig])
    assert_sigma(sig, ref, ref[:, 0], "config1 block sigma")
    assert np.array_equal(rank, sp.rank)


def test_c1_all_pairs_all_kinds(c1):
    col, sp, ctx, *_ = c1
    pairs = synth.all_pairs_by_norm_order(norm_order(sp.E))
    ref = oracle.pair_errors(sp, pairs, col.r, 7, oracle.RAW)
    out = ctx.pair_errors(pairs)
    compare_pairs(out, ref, 7, "config1")


@pytest.mark.parametrize("kinds", [1, 2, 4, 3, 5, 6])
def test_c1_kind_subsets(c1, kinds):
    col, sp, ctx, *_ = c1
    pairs = synth.all_pairs_by_norm_order(norm_order(sp.E))[:37]
    ref = oracle.pair_errors(sp, pairs, col.r, kinds, oracle.RAW)
    out = ctx.pair_errors(pairs, kinds=kinds)
    compare_pairs(out, ref, kinds, f"config1 kinds={kinds}")


def test_c1_trunc_operand(c1, cm):
    col, sp, ctx, *_ = c1
    pairs = synth.all_pairs_by_norm_order(norm_order(sp.E))
    ref = oracle.pair_errors(sp, pairs, col.r, 7, oracle.TRUNC)
    out = ctx.pair_errors(pairs, operand=cm.TRUNC)
    compare_pairs(out, ref, 7, "config1 TRUNC")


def test_c1_reversed_orientation_and_self_pairs(c1):
    """Orientation matters (A7): reversed pairs; base == app is [A, A] (P8)."""
    col, sp, ctx, *_ = c1
    pairs = synth.all_pairs_by_norm_order(norm_order(sp.E))[:, ::-1].copy()
    pairs = np.concatenate([pairs, np.stack([np.arange(col.N)] * 2, 1).astype(np.int32)])
    ref = oracle.pair_errors(sp, pairs, col.r, 7, oracle.RAW)
    out = ctx.pair_errors(pairs)
    compare_pairs(out, ref, 7, "config1 reversed+self")


def test_device_path_equals_host_path(c1):
    col, sp, ctx, *_ = c1
    pairs = synth.all_pairs_by_norm_order(norm_order(sp.E))
    host = ctx.pair_errors(pairs)
    P, r = pairs.shape[0], col.r
    dp = torch.from_numpy(pairs).cuda()
    out = {"err2": torch.zeros((P, 3), dtype=torch.float64, device="cuda"),
           "total": torch.zeros(P, dtype=torch.float64, device="cuda"),
           "sigma_tilde": torch.zeros((P, r), dtype=torch.float32, device="cuda"),
           "mu": torch.zeros((P, r), dtype=torch.float32, device="cuda")}
    ctx.pair_errors(dp, out=out)
    torch.cuda.synchronize()
    assert np.array_equal(out["err2"].cpu().numpy(), host["err2"])
    assert np.array_equal(out["sigma_tilde"].cpu().numpy(), host["sigma_tilde"])
    assert np.array_equal(out["mu"].cpu().numpy(), host["mu"])


def test_deterministic(c1):
    col, sp, ctx, *_ = c1
    pairs = synth.all_pairs_by_norm_order(norm_order(sp.E))
    a = ctx.pair_errors(pairs)
    b = ctx.pair_errors(pairs)
    for k in a:
        assert np.array_equal(a[k], b[k])


def test_errors_and_edges(c1, cm):
    col, sp, ctx, *_ = c1
    out = ctx.pair_errors(np.zeros((0, 2), np.int32))
    assert out["err2"].shape == (0, 3)
    with pytest.raises(cm.CmsvdError) as e:
        ctx.pair_errors(np.array([[0, col.N]], np.int32))
    assert e.value.status == 2
    with pytest.raises(cm.CmsvdError) as e:
        ctx.pair_errors(np.array([[0, 1]], np.int32), r=col.r + 1)
    assert e.value.status == 4
    bad = torch.tensor([[0, 99]], dtype=torch.int32, device="cuda")
    o = {"err2": torch.zeros((1, 3), dtype=torch.float64, device="cuda"),
         "total": torch.zeros(1, dtype=torch.float64, device="cuda")}
    with pytest.raises(cm.CmsvdError):
        ctx.pair_errors(bad, out=o)


def test_nonfinite_and_shape_rejected(cm):
    ctx = cm.Context(0)
    a = np.ones((3, 8, 16), np.float32)
    a[1, 2, 3] = np.nan
    with pytest.raises(cm.CmsvdError) as e:
        ctx.register(a)
    assert e.value.status == 3
    with pytest.raises(cm.CmsvdError) as e:
        ctx.block_spectra(4)
    assert e.value.status == 4
    ctx.close()


# ------------------------------------------------------------ small edges --
@pytest.mark.parametrize("seed", range(4))
def test_random_small_shapes_and_ragged(cm, seed):
    """Random m, widths that do not divide the 64-wide tiles, r above and
    below the ranks, a zero block and an exactly low-rank block."""
    R = np.random.default_rng(1000 + seed)
    m = int(R.integers(5, 150))
    n = int(R.integers(1, min(m, 70) + 1))
    N = int(R.integers(3, 9))
    blocks = R.standard_normal((N, n, m)).astype(np.float32)
    blocks[0] *= 0.0
    if N > 3:
        lr = (R.standard_normal((m, 2)) @ R.standard_normal((2, n))).astype(np.float32)
        blocks[1] = lr.T
    for r in sorted({1, max(1, n // 2), n, n + 3}):
        sp = oracle.block_spectra(blocks)
        ctx, E, sig, rank = gpu_ctx(cm, blocks, r)
        pairs = np.array([(i, j) for i in range(N) for j in range(N)], np.int32)
        ref = oracle.pair_errors(sp, pairs, r, 7, oracle.RAW)
        out = ctx.pair_errors(pairs)
        compare_pairs(out, ref, 7, f"random m={m} n={n} r={r}")
        ctx.close()


def test_orthogonal_blocks_exact(cm):
    """P7: mutually orthogonal column spaces -> residual = incremental = exact."""
    R = np.random.default_rng(7)
    m, n, N = 96, 8, 6
    Q = np.linalg.qr(R.standard_normal((m, n * N)))[0]
    blocks = np.stack([(Q[:, i * n:(i + 1) * n] @ np.diag(np.linspace(3, 1, n)) @
                        np.linalg.qr(R.standard_normal((n, n)))[0]).T for i in range(N)]).astype(np.float32)
    sp = oracle.block_spectra(blocks)
    for r in (4, 8, 12):
        ctx, *_ = gpu_ctx(cm, blocks, r)
        pairs = np.array([(i, j) for i in range(N) for j in range(N) if i != j], np.int32)
        out = ctx.pair_errors(pairs)
        ex = oracle.exact_groups(sp, [list(p) for p in pairs], r)
        assert_err2(out["err2"][:, 1], ex, out["total"], "orth residual")
        assert_err2(out["err2"][:, 2], ex, out["total"], "orth incremental")
        ctx.close()


# --------------------------------------------------------------- config 2 --
@pytest.fixture(scope="module")
def c2(cm):
    col = synth.config2()
    sp = oracle.block_spectra(col.blocks)
    ctx, E, sig, rank = gpu_ctx(cm, col.blocks, col.r)
    yield col, sp, ctx, E, sig, rank
    ctx.close()


def test_c2_spectra(c2):
    col, sp, ctx, E, sig, rank = c2
    assert np.allclose(E, sp.E, rtol=1e-12, atol=0)
    ref = np.stack([s[:col.r] for s in sp.sig])
    assert_sigma(sig, ref, ref[:, 0], "config2 block sigma")
    assert np.array_equal(rank, sp.rank)


def test_c2_sampled_pairs_full_size_launch(c2):
    """All 8128 pairs in the bench's launch configuration; a deterministic
    sample (every 127th pair + same-group pairs) checked against the oracle
    one by one; invariants on all pairs."""
    col, sp, ctx, *_ = c2
    pairs = synth.all_pairs_by_norm_order(norm_order(sp.E))
    out = ctx.pair_errors(pairs)
    e2 = out["err2"]
    assert np.all(np.isfinite(e2)) and np.all(e2 >= 0) and np.all(e2 <= out["total"][:, None])
    # incremental <= weyl (F4 chain, base = larger top-r energy holds up to near-ties)
    assert np.all(e2[:, 2] <= e2[:, 0] * (1 + 1e-6))
    same = col.groups[pairs[:, 0]] == col.groups[pairs[:, 1]]
    idx = np.unique(np.concatenate([np.arange(0, len(pairs), 127), np.flatnonzero(same)[::40]]))
    ref = oracle.pair_errors(sp, pairs[idx], col.r, 7, oracle.RAW)
    sub = {k: (v[idx] if v is not None else None) for k, v in out.items()}
    compare_pairs(sub, ref, 7, "config2 sample")


def test_c2_regimes(c2):
    """Same-group pairs are admissible at eps = 0.02 under the incremental
    estimate, cross-group pairs are not even at eps = 0.1."""
    col, sp, ctx, *_ = c2
    pairs = synth.all_pairs_by_norm_order(norm_order(sp.E))
    out = ctx.pair_errors(pairs, kinds=4)
    rel = np.sqrt(out["err2"][:, 2] / out["total"])
    same = col.groups[pairs[:, 0]] == col.groups[pairs[:, 1]]
    assert rel[same].max() < 0.02 and rel[~same].min() > 0.1


# --------------------------------------------------------------- config 5 --
@pytest.mark.parametrize("N,r", [(512, 16), (512, 64), (2048, 64)])
def test_c5_knn_sample(cm, N, r):
    """Config 5 scaling sweep sizes (N in {512, 2048}, r in {16, 64}): sampled pairs of the full
    registered collection against the oracle."""
    col = synth.config5(N=N, r=r)
    sp = oracle.block_spectra(col.blocks)
    ctx, E, sig, rank = gpu_ctx(cm, col.blocks, r)
    R = np.random.default_rng(5)
    pairs = np.stack([R.integers(0, col.N, 96), R.integers(0, col.N, 96)], 1).astype(np.int32)
    ref = oracle.pair_errors(sp, pairs, r, 7, oracle.RAW)
    out = ctx.pair_errors(pairs)
    compare_pairs(out, ref, 7, f"config5 r={r}")
    if r == 64:
        # r = n: untruncated base, incremental is exact (P5) -> same as oracle exact
        ex = oracle.exact_groups(sp, [list(p) for p in pairs[:24]], r)
        assert_err2(out["err2"][:24, 2], ex, out["total"][:24], "config5 exactness")
    ctx.close()


# ------------------------------------------------- N3 (beyond the paper) --
def test_tight_variants_c1_all_pairs(c1, cm):
    """cmsvd_pair_errors_tight (residual with U_r, per-index Weyl) vs the oracle, all config-1 pairs,
    RAW and TRUNC, plus the ordering against the paper's estimators."""
    col, sp, ctx, *_ = c1
    pairs = synth.all_pairs_by_norm_order(norm_order(sp.E))
    for operand in (cm.RAW, cm.TRUNC):
        ref, tot = oracle.pair_errors_tight(sp, pairs, col.r, operand)
        out = ctx.pair_errors_tight(pairs, operand=operand)
        assert np.allclose(out["total"], tot, rtol=1e-12)
        assert_err2(out["err2x"][:, 0], ref[:, 0], tot, "residual(U_r)")
        assert_err2(out["err2x"][:, 1], ref[:, 1], tot, "per-index Weyl")
        std = ctx.pair_errors(pairs, operand=operand)
        assert np.all(out["err2x"][:, 0] <= std["err2"][:, 1] * (1 + 2e-3) + 1e-7 * tot)
        assert np.all(out["err2x"][:, 1] <= std["err2"][:, 0] * (1 + 1e-9) + 1e-9 * tot)
        assert np.all(std["err2"][:, 2] <= out["err2x"][:, 0] * (1 + 2e-3) + 1e-7 * tot)


def test_tight_variants_c2_sampled(c2):
    col, sp, ctx, E, *_ = c2
    pairs = synth.all_pairs_by_norm_order(norm_order(sp.E))
    sel = pairs[np.random.default_rng(7).choice(pairs.shape[0], 64, replace=False)]
    ref, tot = oracle.pair_errors_tight(sp, sel, col.r)
    out = ctx.pair_errors_tight(sel)
    assert_err2(out["err2x"][:, 0], ref[:, 0], tot, "config2 residual(U_r)")
    assert_err2(out["err2x"][:, 1], ref[:, 1], tot, "config2 per-index Weyl")


@pytest.mark.parametrize("seed", [0, 1])
def test_syrk_zz_bitwise_equals_gemm_path(cm, seed, monkeypatch):
    """k_syrk_zz (default Z^T Z kernel, w <= 128) and the generic fp64-accumulated SIMT GEMM
    (CMSVD_ZZ_SYRK=0) accumulate in the same order: every output must be bitwise equal.  Ragged
    widths and ranks exercise the partial tiles and the q-chunk tail (q not a multiple of 32)."""
    rng = np.random.default_rng(100 + seed)
    m = 96
    blocks = []
    for i in range(10):
        n = int(rng.integers(5, 41))
        k = int(rng.integers(2, n + 1))
        a = rng.standard_normal((m, k)) @ rng.standard_normal((k, n)) + 1e-3 * rng.standard_normal((m, n))
        blocks.append(np.asfortranarray(a.astype(np.float32)))
    r = 7
    pairs = np.array([(i, j) for i in range(10) for j in range(10) if i != j], np.int32)
    outs = []
    for flag in ("0", "1"):
        monkeypatch.setenv("CMSVD_ZZ_SYRK", flag)
        ctx = cm.Context(0, torch.cuda.current_stream().cuda_stream)
        ctx.register(blocks)
        ctx.block_spectra(r)
        outs.append(ctx.pair_errors(pairs))
        ctx.close()
    for key in ("err2", "total", "sigma_tilde", "mu"):
        assert np.array_equal(outs[0][key], outs[1][key], equal_nan=True), key


def test_duo160_ragged_vs_oracle_and_one_problem_kernel(cm, monkeypatch):
    """Incremental Grams of 128 < n <= 160 on the two-problem eigen kernel (k_tridiag_duo<5>, problem 0
    split between registers and shared memory) vs the oracle, ragged n = r' + w in 129..160 mixed with
    n = 2..4 and n = 33..34 in one launch, and an odd problem count (the last CTA carries one problem); the one-problem kernel (CMSVD_EIG_DUO160=0) must
    agree with it to the same tolerance."""
    rng = np.random.default_rng(160)
    m = 256
    widths = [97, 100, 111, 119, 124, 127, 128, 1, 2]   # + tiny blocks: Grams of n = 2..4 in the same launch
    blocks = []
    for n in widths:
        k = int(rng.integers(40, n + 1)) if n > 40 else n
        a = (rng.standard_normal((m, k)) * np.geomspace(1.0, 1e-2 if n > 40 else 0.5, k)) @ rng.standard_normal((k, n))
        blocks.append(np.asfortranarray((a + 1e-3 * rng.standard_normal((m, n))).astype(np.float32)))
    r = 32
    nb = len(widths)
    pairs = np.array([(i, j) for i in range(nb) for j in range(nb) if i != j], np.int32)[1:]  # 71
    sp = oracle.block_spectra(blocks)
    ref = oracle.pair_errors(sp, pairs, r)
    outs = []
    for flag in ("1", "0"):
        monkeypatch.setenv("CMSVD_EIG_DUO160", flag)
        ctx = cm.Context(0, torch.cuda.current_stream().cuda_stream)
        ctx.register(blocks)
        ctx.block_spectra(r)
        outs.append(ctx.pair_errors(pairs))
        ctx.close()
        compare_pairs(outs[-1], ref, what=f"duo160={flag}")
    assert_err2(outs[0]["err2"][:, 2], outs[1]["err2"][:, 2], ref.total, "duo160 vs one-problem kernel")


def test_sharded_union_equals_unsharded(cm):
    """N4 (pair-grid sharding, shard.py): the tiles of a world of 4, evaluated one after the other on this
    GPU, reassemble bitwise to the unsharded call (the evaluations are independent of their batch)."""
    from paper_2601_11626_b200 import shard
    col = synth.config1()
    with cm.Context(0) as ctx:
        ctx.register(col.blocks)
        E, sig, rank = ctx.block_spectra(col.r)
        order = np.array(sorted(range(col.N), key=lambda i: (-E[i], i)))
        pairs = synth.all_pairs_by_norm_order(order)
        full = ctx.pair_errors(pairs)
        err2 = np.full_like(full["err2"], np.nan)
        total = np.full_like(full["total"], np.nan)
        for idx in shard.partition_pairs(pairs, 4):
            part = ctx.pair_errors(pairs[idx])
            err2[idx] = part["err2"]
            total[idx] = part["total"]
    assert np.array_equal(err2, full["err2"]) and np.array_equal(total, full["total"])
