"""Pins of the float64 oracle against what the paper and the mathematics fix
(never against itself).  CPU only (-m "not gpu").

A plausible mistake anywhere in the oracle (a dropped term, a wrong sign or
index, a transposed operand) fails at least one of these:
  * SVD vs LAPACK (numpy) + reconstruction + closed forms  -> or_svd
  * brute-force exact error of the explicit concatenation  -> all estimators
  * Example D.1, Prop. 1 (corrected, A2), [A, A], nested ranges,
    untruncated exactness (Cor. 2), Lemma 1 step-by-step   -> each estimator
  * soundness chain exact <= inc <= res <= weyl (F3, F4)   -> signs / terms
"""
import json
import os

import numpy as np
import pytest

import oracle

GOLD = json.load(open(os.path.join(os.path.dirname(__file__), "golden", "paper_pins.json")))


def rng(seed=0):
    return np.random.default_rng(seed)


def spec_of(blocks, tau=oracle.TAU):
    return oracle.block_spectra([np.asarray(b, dtype=np.float64) for b in blocks], tau)


def eval_pair(blocks, r, operand=oracle.RAW):
    sp = spec_of(blocks)
    res = oracle.pair_errors(sp, np.array([[0, 1]], np.int32), r, 7, operand)
    return sp, res


def exact(blocks, r):
    M = np.concatenate([np.asarray(b, dtype=np.float64) for b in blocks], axis=1)
    return float(np.sum(np.linalg.svd(M, compute_uv=False)[r:] ** 2))


# ----------------------------------------------------------------- SVD -----
@pytest.mark.parametrize("shape", [(8, 5), (5, 8), (64, 32), (40, 40), (97, 13), (1, 7), (7, 1)])
def test_svd_matches_lapack(shape):
    A = rng(1).standard_normal(shape)
    s, U, V = oracle.svd(A, True, True)
    s_ref = np.linalg.svd(A, compute_uv=False)
    assert np.allclose(s, s_ref, rtol=1e-12, atol=1e-13 * s_ref[0])
    assert np.linalg.norm(U @ np.diag(s) @ V.T - A) <= 1e-12 * np.linalg.norm(A)
    k = min(shape)
    assert np.abs(U.T @ U - np.eye(k)).max() < 1e-12
    assert np.abs(V.T @ V - np.eye(k)).max() < 1e-12
    assert np.all(np.diff(s) <= 0)


def test_svd_closed_forms():
    assert np.allclose(oracle.svd(np.eye(3)), [1, 1, 1])
    u = rng(2).standard_normal(6); u /= np.linalg.norm(u)
    v = rng(3).standard_normal(4); v /= np.linalg.norm(v)
    s = oracle.svd(5 * np.outer(u, v))
    assert abs(s[0] - 5) < 1e-13 and np.all(np.abs(s[1:]) < 1e-13)
    g = GOLD["diag_321"]
    assert abs(oracle.exact_err2(np.diag(g["diag"]), g["r"]) - g["exact_err2"]) < 1e-13


def test_svd_rank_deficient_and_zero():
    A = rng(4).standard_normal((30, 3)) @ rng(5).standard_normal((3, 10))
    s = oracle.svd(A)
    assert np.all(s[3:] < 1e-12 * s[0])
    assert np.allclose(s[:3], np.linalg.svd(A, compute_uv=False)[:3], rtol=1e-12)
    assert np.all(oracle.svd(np.zeros((5, 3))) == 0)


def test_energy_closed_form():
    g = GOLD["frobenius_2x2"]
    assert oracle.energy(np.array(g["M"], np.float32)) == g["energy"]
    assert oracle.energy(np.eye(3, dtype=np.float32)) == 3.0


def test_energy_split_identity():
    """P1: sum_{j<=r} sigma_j^2 + E_r^2 = ||M||_F^2."""
    M = rng(6).standard_normal((20, 12))
    s = oracle.svd(M)
    for r in range(0, 13):
        assert abs(np.sum(s[:r] ** 2) + oracle.exact_err2(M, r) - np.sum(M * M)) < 1e-11 * np.sum(M * M)


# -------------------------------------------------------- estimators -------
def test_example_d1_weyl_looseness():
    """Example D.1: rank-one A_j = u s_j v_j^T."""
    g = GOLD["example_d1"]
    R = rng(7)
    u = R.standard_normal(5); u /= np.linalg.norm(u)
    blocks = []
    for sj in g["s"]:
        v = R.standard_normal(3); v /= np.linalg.norm(v)
        blocks.append(sj * np.outer(u, v))
    sp, res = eval_pair(blocks, g["r"])
    w, rr, inc = res.err2[0]
    assert abs(w - g["weyl_err2"]) < 1e-12
    assert abs(rr - g["residual_err2"]) < 1e-12
    assert abs(inc - g["incremental_err2"]) < 1e-12
    assert abs(exact(blocks, g["r"]) - g["exact_err2"]) < 1e-12


def test_weyl_bound_k3_formula():
    """Eq. 5 with K=3 and r >= rank: sum s^2 - max s^2;
    checked through pairwise composition: (A1, A2) then total energy."""
    g = GOLD["example_d1_k3"]
    s = g["s"]
    assert sum(x * x for x in s) - max(x * x for x in s) == g["weyl_err2"]


def test_thm2_per_index_claim_false_partial_sums_hold():
    """A1: Thm 2's per-index claim fails, the partial-sum
    (weak majorisation) form used by Cor. 1 holds."""
    g = GOLD["thm2_counterexample"]
    A1 = np.array(g["A1"], float); A2 = np.array(g["A2"], float)
    sp, res = eval_pair([A1, A2], 2)
    mu = res.mu[0]
    sM = np.linalg.svd(np.concatenate([A1, A2], 1), compute_uv=False)
    assert np.allclose(sM, g["sigma_M"], rtol=1e-14)
    assert np.allclose(mu, g["mu"], rtol=1e-14)
    assert sM[1] < mu[1]
    assert np.all(np.cumsum(mu ** 2) <= np.cumsum(sM ** 2) + 1e-14)


def _orthogonal_blocks(R, m, ns, ranks):
    Q = np.linalg.qr(R.standard_normal((m, sum(ranks))))[0]
    out, c = [], 0
    for n, k in zip(ns, ranks):
        out.append(Q[:, c:c + k] @ (R.standard_normal((k, n)) * R.uniform(0.5, 3)))
        c += k
    return out


@pytest.mark.parametrize("r", [1, 3, 5, 9])
def test_orthogonal_column_spaces_union_spectrum(r):
    """P7 / Prop. 1 (corrected reading A2): mutually
    orthogonal column spaces give sigma(M) = union of the block spectra, and
    the residual and incremental estimates are exact."""
    blocks = _orthogonal_blocks(rng(8), 24, [7, 6], [4, 5])
    sM = np.linalg.svd(np.concatenate(blocks, 1), compute_uv=False)
    union = np.sort(np.concatenate([np.linalg.svd(b, compute_uv=False) for b in blocks]))[::-1]
    assert np.allclose(sM[:union.size], union, atol=1e-12 * sM[0])
    sp, res = eval_pair(blocks, r)
    ex = exact(blocks, r)
    w, rr, inc = res.err2[0]
    tol = 1e-11 * res.total[0]
    assert abs(rr - ex) < tol and abs(inc - ex) < tol and w >= ex - tol


@pytest.mark.parametrize("r", [1, 2, 4, 6])
def test_duplicate_block_closed_forms(r):
    """P8: [A, A] has sigma = sqrt(2) sigma(A); exact = incremental = 2 t,
    Weyl = residual = E_A + t, t = tail_r(A) (derivation)."""
    A = rng(9).standard_normal((12, 6))
    sA = np.linalg.svd(A, compute_uv=False)
    t = float(np.sum(sA[r:] ** 2)); EA = float(np.sum(A * A))
    sM = np.linalg.svd(np.concatenate([A, A], 1), compute_uv=False)
    assert np.allclose(sM[:6], np.sqrt(2) * sA, rtol=1e-13)
    sp, res = eval_pair([A, A], r)
    w, rr, inc = res.err2[0]
    tol = 1e-11 * EA
    assert abs(exact([A, A], r) - 2 * t) < tol
    assert abs(inc - 2 * t) < tol
    assert abs(w - (EA + t)) < tol
    assert abs(rr - (EA + t)) < tol


def test_nested_ranges_residual_degeneracy():
    """P10 / Prop. 1 degeneracy: range(B) in range(A),
    r >= rank(A): residual = ||B||^2 while exact = incremental = 0."""
    R = rng(10)
    A = R.standard_normal((15, 4))
    B = A @ R.standard_normal((4, 3))
    sp, res = eval_pair([A, B], 4)
    w, rr, inc = res.err2[0]
    EB = float(np.sum(B * B))
    assert abs(rr - EB) < 1e-10 * EB
    assert abs(inc) < 1e-10 * EB
    assert exact([A, B], 4) < 1e-10 * EB


@pytest.mark.parametrize("seed", range(6))
def test_untruncated_incremental_is_exact(seed):
    """P5 / Cor. 2: base rank <= r and RAW operand, no
    truncation happens, so the plug-in estimate equals the exact error."""
    R = rng(100 + seed)
    A = R.standard_normal((20, 3)) @ R.standard_normal((3, 9))     # rank 3
    B = R.standard_normal((20, 7))
    for r in (3, 4, 6):
        sp, res = eval_pair([A, B], r)
        ex = exact([A, B], r)
        assert abs(res.err2[0, 2] - ex) < 1e-10 * res.total[0]
        assert np.allclose(res.sigma_tilde[0], np.linalg.svd(np.concatenate([A, B], 1), compute_uv=False)[:r],
                           rtol=1e-10, atol=1e-12)


@pytest.mark.parametrize("seed", range(4))
def test_incremental_equals_lemma1_pipeline(seed):
    """P3: the oracle's plain definition sigma~ = sigma([U_r S_r, F]) equals
    the paper's step-by-step Lemma 1 + Cor. 3 pipeline (Y = Q^T A, R = A - QY,
    R = Q_res B, S = [[S+YY^T, YB^T],[BY^T, BB^T]], eig -> sqrt)
    (PAPER.md:1309-1333, 1399-1436), with truncation to r."""
    R = rng(200 + seed)
    A = R.standard_normal((30, 10)); B = R.standard_normal((30, 8))
    r = 4
    sp, res = eval_pair([A, B], r)
    UA, sA, _ = np.linalg.svd(A, full_matrices=False)
    Q = UA[:, :r]; St = np.diag(sA[:r] ** 2)
    Y = Q.T @ B
    Rr = B - Q @ Y
    Qres, Bf = np.linalg.qr(Rr)
    S1 = np.block([[St + Y @ Y.T, Y @ Bf.T], [Bf @ Y.T, Bf @ Bf.T]])
    lam = np.sort(np.linalg.eigvalsh(S1))[::-1]
    assert np.allclose(res.sigma_tilde[0], np.sqrt(np.maximum(lam[:r], 0)), rtol=1e-11)
    # Lemma 1 itself, untruncated: Q S Q^T = M M^T (P4)
    Qf = UA[:, :10]; Sf = np.diag(sA ** 2)
    Yf = Qf.T @ B; Rf = B - Qf @ Yf
    Qr2, B2 = np.linalg.qr(Rf)
    S2 = np.block([[Sf + Yf @ Yf.T, Yf @ B2.T], [B2 @ Yf.T, B2 @ B2.T]])
    Q2 = np.concatenate([Qf, Qr2], 1)
    M = np.concatenate([A, B], 1)
    assert np.linalg.norm(Q2 @ S2 @ Q2.T - M @ M.T) <= 1e-10 * np.linalg.norm(M) ** 2


def test_residual_mu_equals_svd_of_explicit_concatenation():
    """Proof Step 5: mu = sigma([A_i, R]) = sigma(A_i) u sigma(R)."""
    R = rng(11)
    A = R.standard_normal((25, 6)); B = R.standard_normal((25, 5))
    r = 8
    sp, res = eval_pair([A, B], r)
    Q = np.linalg.svd(A, full_matrices=False)[0]
    Rr = B - Q @ (Q.T @ B)
    mu = np.linalg.svd(np.concatenate([A, Rr], 1), compute_uv=False)[:r]
    assert np.allclose(res.mu[0], mu, rtol=1e-11, atol=1e-12)
    assert abs(res.err2[0, 1] - (res.total[0] - np.sum(mu ** 2))) < 1e-10 * res.total[0]


def test_weyl_is_eq5():
    """Eq. 5 against a direct numpy evaluation."""
    R = rng(12)
    A = R.standard_normal((16, 5)) * 3; B = R.standard_normal((16, 7))
    for r in (1, 2, 5, 7):
        sp, res = eval_pair([A, B], r)
        sA = np.linalg.svd(A, compute_uv=False); sB = np.linalg.svd(B, compute_uv=False)
        ref = np.sum(A * A) + np.sum(B * B) - max(np.sum(sA[:r] ** 2), np.sum(sB[:r] ** 2))
        assert abs(res.err2[0, 0] - ref) < 1e-11 * res.total[0]


@pytest.mark.parametrize("seed", range(30))
def test_soundness_chain(seed):
    """P6 (Thm 1, Cor. 1, F3, F4): exact <= incremental <= residual <= Weyl
    with the base = the block of larger top-r energy; all three >= exact; the
    weak majorisation sum mu^2 <= sum sigma^2 (P11); sigma~_j <= sigma_j (P17)."""
    R = rng(300 + seed)
    m = int(R.integers(6, 20))
    n1, n2 = int(R.integers(1, 7)), int(R.integers(1, 7))
    if seed % 2:
        U = np.linalg.qr(R.standard_normal((m, 3)))[0]
        A = U @ R.standard_normal((3, n1)) + 0.05 * R.standard_normal((m, n1))
        B = U @ R.standard_normal((3, n2)) + 0.05 * R.standard_normal((m, n2))
    else:
        A = R.standard_normal((m, n1)); B = R.standard_normal((m, n2))
    r = int(R.integers(1, min(m, n1 + n2) + 1))
    sA = np.linalg.svd(A, compute_uv=False); sB = np.linalg.svd(B, compute_uv=False)
    if np.sum(sB[:r] ** 2) > np.sum(sA[:r] ** 2):
        A, B = B, A
    sp, res = eval_pair([A, B], r)
    w, rr, inc = res.err2[0]
    ex = exact([A, B], r)
    tol = 1e-10 * res.total[0]
    assert ex <= inc + tol
    assert inc <= rr + tol
    assert rr <= w + tol
    sM = np.linalg.svd(np.concatenate([A, B], 1), compute_uv=False)
    k = min(r, sM.size)
    assert np.all(np.cumsum(res.mu[0, :k] ** 2) <= np.cumsum(sM[:k] ** 2) + tol)
    assert np.all(res.sigma_tilde[0, :k] <= sM[:k] + 1e-10 * sM[0])


def test_trunc_operand_is_still_upper_bound():
    """A6 / F4: F = U_r diag(s_r) of the appended block gives F F^T <= B B^T,
    so the TRUNC estimates stay >= exact; with n <= r it equals RAW."""
    R = rng(13)
    U = np.linalg.qr(R.standard_normal((20, 4)))[0]
    A = U @ R.standard_normal((4, 9)) + 0.1 * R.standard_normal((20, 9))
    B = U @ R.standard_normal((4, 9)) + 0.1 * R.standard_normal((20, 9))
    for r in (2, 4, 6):
        sp, res_t = eval_pair([A, B], r, oracle.TRUNC)
        ex = exact([A, B], r)
        assert np.all(res_t.err2[0] >= ex - 1e-10 * res_t.total[0])
    C = R.standard_normal((20, 3)); D = R.standard_normal((20, 3))
    _, a = eval_pair([C, D], 5, oracle.RAW)
    _, b = eval_pair([C, D], 5, oracle.TRUNC)
    assert np.allclose(a.err2, b.err2, rtol=1e-10, atol=1e-10)


def test_energy_matches_sum():
    A = rng(14).standard_normal((33, 7)).astype(np.float32)
    assert abs(oracle.energy(A) - float(np.sum(A.astype(np.float64) ** 2))) <= 1e-12 * oracle.energy(A)


def test_clamp_and_single_block_weyl():
    """Weyl with r >= rank of both blocks reduces to the smaller energy
    (Thm 1 special case); results clamp to [0, total]."""
    R = rng(15)
    A = R.standard_normal((10, 2)) * 5; B = R.standard_normal((10, 3))
    sp, res = eval_pair([A, B], 5)
    EA, EB = np.sum(A * A), np.sum(B * B)
    assert abs(res.err2[0, 0] - min(EA, EB)) < 1e-11 * (EA + EB)
    assert np.all(res.err2[0] >= 0) and np.all(res.err2[0] <= res.total[0])


@pytest.mark.parametrize("r", [1, 9, 18, 21])
def test_zero_and_low_rank_blocks_vs_brute_force(r):
    """Rank-deficient concatenations (a zero block, a rank-2 block) converge
    and agree with LAPACK brute force on the plain definitions."""
    R = rng(1000)
    m, n = 34, 18
    Z = np.zeros((m, n)); A = R.standard_normal((m, n)); L2 = R.standard_normal((m, 2)) @ R.standard_normal((2, n))
    for X, Y in [(A, Z), (Z, A), (A, L2), (L2, A), (Z, Z)]:
        sp, res = eval_pair([X, Y], r)
        assert res.err2[0, 2] >= exact([X, Y], r) - 1e-10 * max(res.total[0], 1)
        UA, sA, _ = np.linalg.svd(X, full_matrices=False)
        rr = min(r, int(np.sum(sA > oracle.TAU * sA[0]))) if sA[0] > 0 else 0
        st = np.linalg.svd(np.concatenate([UA[:, :rr] * sA[:rr], Y], 1), compute_uv=False)[:r]
        st = np.pad(st, (0, r - st.size))
        assert np.allclose(res.sigma_tilde[0], st, atol=1e-12 * max(1, st[0]))


# ---------------------------------------------------------------------------
# N3 (beyond the paper): residual bound with the tracked basis U_r (A4) and the
# per-index Weyl bound (A8), oracle.pair_errors_tight
# ---------------------------------------------------------------------------
@pytest.mark.parametrize("seed", range(20))
def test_tight_variants_chain_and_definitions(seed):
    """Chain exact <= inc <= residual(U_r) <= residual(full) <= Weyl and
    exact <= per-index Weyl <= Weyl (Eq. 5); both variants against direct numpy
    evaluations of their definitions (LAPACK SVDs, independent of oracle.c)."""
    R = rng(700 + seed)
    m = int(R.integers(6, 20))
    n1, n2 = int(R.integers(1, 7)), int(R.integers(1, 7))
    if seed % 2:
        U = np.linalg.qr(R.standard_normal((m, 3)))[0]
        A = U @ R.standard_normal((3, n1)) + 0.05 * R.standard_normal((m, n1))
        B = U @ R.standard_normal((3, n2)) + 0.05 * R.standard_normal((m, n2))
    else:
        A = R.standard_normal((m, n1)); B = R.standard_normal((m, n2))
    r = int(R.integers(1, min(m, n1 + n2) + 1))
    sA = np.linalg.svd(A, compute_uv=False); sB = np.linalg.svd(B, compute_uv=False)
    if np.sum(sB[:r] ** 2) > np.sum(sA[:r] ** 2):
        A, B = B, A
        sA, sB = sB, sA
    sp = oracle.block_spectra([A, B])
    std = oracle.pair_errors(sp, [[0, 1]], r, 7)
    x, tot = oracle.pair_errors_tight(sp, [[0, 1]], r)
    res_ur, w_idx = x[0]
    w, res, inc = std.err2[0]
    ex = exact([A, B], r)
    tol = 1e-10 * tot[0]
    assert ex <= inc + tol and inc <= res_ur + tol and res_ur <= res + tol and res <= w + tol
    assert ex <= w_idx + tol and w_idx <= w + tol
    E = np.sum(A * A) + np.sum(B * B)
    # per-index Weyl by definition
    k = r
    sa = np.pad(sA, (0, max(0, k - sA.size)))[:k]; sb = np.pad(sB, (0, max(0, k - sB.size)))[:k]
    assert abs(w_idx - max(0.0, E - np.sum(np.maximum(sa, sb) ** 2))) < 1e-10 * E
    # residual with U_r by definition: Q = first min(r, rank) left singular vectors of A
    Ua, sa_full, _ = np.linalg.svd(A, full_matrices=False)
    rank = int(np.sum(sa_full > 1e-5 * sa_full[0]))
    Q = Ua[:, :min(r, rank)]
    Rr = B - Q @ (Q.T @ B)
    mu = np.sort(np.concatenate([sa_full, np.linalg.svd(Rr, compute_uv=False)]))[::-1][:r]
    assert abs(res_ur - max(0.0, E - np.sum(mu ** 2))) < 1e-9 * E


def test_tight_variants_closed_form_AA():
    """[A, A]: residual(U_r) = per-index Weyl = E_A + tail_r(A) (R = (I - U_r U_r^T)A
    has sigma_{>r}(A), so the top-r of mu are sigma_{<=r}(A))."""
    R = rng(41)
    A = R.standard_normal((18, 7)) @ np.diag([5, 4, 3, 2, 1, 0.5, 0.2])
    s = np.linalg.svd(A, compute_uv=False)
    EA = np.sum(A * A)
    for r in (1, 3, 6):
        sp = oracle.block_spectra([A])
        x, tot = oracle.pair_errors_tight(sp, [[0, 0]], r)
        t = np.sum(s[r:] ** 2)
        assert abs(x[0, 0] - (EA + t)) < 1e-10 * EA
        assert abs(x[0, 1] - (EA + t)) < 1e-10 * EA
