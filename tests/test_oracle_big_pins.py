"""Pins of the oracle parts added for blocks wider than 512 columns (reading
A15 / A22: own Householder tridiagonalisation + bisection + inverse iteration
on the m x m Gram), of the TRUNC operand (A6) with n > r, and of the
brute-force group errors (or_exact_groups).  CPU only (-m "not gpu").

Each test compares against something other than the oracle itself: a closed
form (the 1-D Laplacian's spectrum, a block built from a known SVD, a
hand-computed merge), an invariant (the energy split P1), or LAPACK (numpy).
"""
import numpy as np
import pytest

import oracle


def haar(R, m, k):
    q, rr = np.linalg.qr(R.standard_normal((m, k)))
    return q * np.sign(np.diag(rr))


# ------------------------------------------------------ symmetric eigensolver --
@pytest.mark.parametrize("n", [2, 3, 17, 60])
def test_sym_eig_laplacian_closed_form(n):
    """T = tridiag(-1, 2, -1) has lambda_k = 2 - 2 cos(k pi / (n + 1)) with eigenvectors
    sin(i k pi / (n + 1)); a Haar similarity Q T Q^T exercises the Householder reduction."""
    R = np.random.default_rng(n)
    T = 2 * np.eye(n) - np.eye(n, k=1) - np.eye(n, k=-1)
    Q = haar(R, n, n)
    G = Q @ T @ Q.T
    k = min(n, 5)
    lam, V = oracle.sym_eig_topk(G, k)
    kk = np.arange(n, 0, -1)                                   # non-increasing order
    lam_ref = 2 - 2 * np.cos(kk * np.pi / (n + 1))
    assert np.allclose(lam, lam_ref, rtol=0, atol=1e-13 * 4)
    for l in range(k):
        y = np.sin(np.arange(1, n + 1) * kk[l] * np.pi / (n + 1))
        u = Q @ (y / np.linalg.norm(y))
        assert abs(abs(u @ V[:, l]) - 1) < 1e-10, l
    assert np.abs(V.T @ V - np.eye(k)).max() < 1e-12


def test_sym_eig_repeated_eigenvalues():
    """A triple and a double eigenvalue: the top-5 vectors are orthonormal and span the
    constructed invariant subspaces (inverse iteration with re-orthogonalisation)."""
    R = np.random.default_rng(3)
    n = 40
    Q = haar(R, n, n)
    d = np.concatenate([[7.0, 7.0, 7.0, 3.0, 3.0], np.linspace(1.0, 0.1, n - 5)])
    G = (Q * d) @ Q.T
    lam, V = oracle.sym_eig_topk(G, 5)
    assert np.allclose(lam, np.sort(d)[::-1], atol=1e-13 * 7)
    assert np.abs(V.T @ V - np.eye(5)).max() < 1e-12
    P3 = Q[:, :3] @ Q[:, :3].T
    P2 = Q[:, 3:5] @ Q[:, 3:5].T
    assert np.linalg.norm(P3 @ V[:, :3] - V[:, :3]) < 1e-10
    assert np.linalg.norm(P2 @ V[:, 3:5] - V[:, 3:5]) < 1e-10


def test_sym_eig_diagonal_and_zero():
    lam, V = oracle.sym_eig_topk(np.diag([1.0, 4.0, 2.0]), 3)
    assert np.allclose(lam, [4, 2, 1], atol=1e-15)
    assert np.allclose(np.abs(V), np.eye(3)[:, [1, 2, 0]], atol=1e-14)
    lam, V = oracle.sym_eig_topk(np.zeros((4, 4)), 2)
    assert np.all(lam == 0)


# ----------------------------------------------------------- A22 block spectra --
def square_block(R, m, s):
    """A = U diag(s) V^T with Haar U, V (float32-representable after rounding: the pins
    compare against the SVD of the rounded matrix where the rounding matters)."""
    U = haar(R, m, m)
    V = haar(R, m, m)
    return (U * s) @ V.T, U


def test_big_block_known_sigma():
    """A 520 x 520 block (wider than BIG_N: the A22 route) built from a known SVD with
    sigma_l = l^-0.7 (config 3's decay): the oracle returns sigma (to the fp32 rounding of
    the block) and U_r = +-U[:, :r]; energy split sum sigma^2 = ||A||_F^2 (P1)."""
    R = np.random.default_rng(5)
    m = 520
    s = np.arange(1, m + 1, dtype=np.float64) ** -0.7
    A, U = square_block(R, m, s)
    A32 = A.astype(np.float32)
    r = 24
    sp = oracle.block_spectra([A32.astype(np.float64)], nvec=r)
    assert sp.rank[0] == m                                           # A22: range = R^m
    dA = np.linalg.norm(A32.astype(np.float64) - A, 2)               # fp32 rounding of the block
    assert np.all(np.abs(sp.sig[0] - s) <= dA + 1e-12)               # Weyl: |sigma(A32) - s| <= ||dA||
    assert np.all(np.abs(sp.sig[0][:r] - s[:r]) <= 1e-6 * s[:r])
    E = float(np.sum(A32.astype(np.float64) ** 2))
    assert abs(np.sum(sp.sig[0] ** 2) - E) <= 1e-12 * E             # P1 (trace of the Gram)
    # top-r vectors: the gaps of l^-0.7 at l <= 24 are >= 3% of sigma_l, far above the rounding
    c = np.abs(np.sum(sp.U[0] * U[:, :r], axis=0))
    assert np.all(c > 1 - 1e-6), c.min()


def test_big_block_vs_lapack():
    """Random 600 x 640 block: all sigma against LAPACK's SVD, U_r against the LAPACK vectors."""
    R = np.random.default_rng(6)
    A = R.standard_normal((600, 640)).astype(np.float32).astype(np.float64)
    sp = oracle.block_spectra([A], nvec=10)
    U, s, _ = np.linalg.svd(A)
    assert np.allclose(sp.sig[0], s, rtol=0, atol=1e-12 * s[0])
    assert np.all(np.abs(np.sum(sp.U[0] * U[:, :10], axis=0)) > 1 - 1e-9)


def test_big_pair_closed_forms():
    """A22 pair estimators on 530 x 530 blocks: residual = E_i + E_j - sum_{l<=r} sigma_l^2(A_i)
    (R = 0 on a full-range base), Weyl = Eq. 5, incremental = LAPACK SVD of [U_r S_r, F_j] with
    F_j = U_{j,r} S_{j,r} (TRUNC) built from the LAPACK factors."""
    R = np.random.default_rng(8)
    m, r = 530, 12
    A = (R.standard_normal((m, m)) @ np.diag(np.arange(1, m + 1) ** -0.5)).astype(np.float32).astype(np.float64)
    B = (R.standard_normal((m, m)) @ np.diag(np.arange(1, m + 1) ** -0.6)).astype(np.float32).astype(np.float64)
    sp = oracle.block_spectra([A, B], nvec=r)
    res = oracle.pair_errors(sp, [[0, 1]], r, 7, oracle.TRUNC)
    Ua, sa, _ = np.linalg.svd(A)
    Ub, sb, _ = np.linalg.svd(B)
    EA, EB = np.sum(A * A), np.sum(B * B)
    tot = EA + EB
    assert abs(res.err2[0, 0] - (tot - max(np.sum(sa[:r] ** 2), np.sum(sb[:r] ** 2)))) < 1e-10 * tot
    assert abs(res.err2[0, 1] - (tot - np.sum(sa[:r] ** 2))) < 1e-10 * tot
    X = np.concatenate([Ua[:, :r] * sa[:r], Ub[:, :r] * sb[:r]], axis=1)
    st = np.linalg.svd(X, compute_uv=False)[:r]
    assert np.allclose(res.sigma_tilde[0], st, rtol=1e-10)
    assert abs(res.err2[0, 2] - (tot - np.sum(st ** 2))) < 1e-10 * tot
    assert np.allclose(res.mu[0], sa[:r], rtol=1e-10)


# ------------------------------------------------------- TRUNC operand, n > r --
def test_trunc_operand_closed_form():
    """TRUNC keeps the TOP-r singular directions of the appended block (A6): with
    A = [10 e1, 9 e2, 0, ...] (rank 2) and B = U_B diag(4, 3, 1, 0.5) V_B^T where
    U_B = [e1, e3, e4, e5], r = 2, the operand is F = [4 e1, 3 e3] and by hand
      sigma~ = top-2 sigma([10 e1, 9 e2, 4 e1, 3 e3]) = (sqrt(116), 9)  -> inc = E - 197,
      mu = top-2 of {10, 9} u sigma((I - QQ^T) F) = {3}   = (10, 9)     -> res = E - 181,
      Weyl = E - max(181, 25) = E - 181.
    Truncating to the wrong directions (e.g. the tail [e4, e5]) would give sigma~ = (10, 9)."""
    m, n = 12, 6
    e = np.eye(m)
    A = np.zeros((m, n)); A[:, 0] = 10 * e[0]; A[:, 1] = 9 * e[1]
    R = np.random.default_rng(9)
    VB = haar(R, n, 4)
    UB = np.stack([e[0], e[2], e[3], e[4]], axis=1)
    B = (UB * np.array([4.0, 3.0, 1.0, 0.5])) @ VB.T
    sp = oracle.block_spectra([A, B])
    res = oracle.pair_errors(sp, [[0, 1]], 2, 7, oracle.TRUNC)
    E = 181.0 + 16 + 9 + 1 + 0.25
    assert abs(res.total[0] - E) < 1e-12 * E
    assert np.allclose(res.sigma_tilde[0], [np.sqrt(116.0), 9.0], rtol=1e-13)
    assert abs(res.err2[0, 2] - (E - 197.0)) < 1e-11 * E
    assert np.allclose(res.mu[0], [10.0, 9.0], rtol=1e-13)
    assert abs(res.err2[0, 1] - (E - 181.0)) < 1e-11 * E
    assert abs(res.err2[0, 0] - (E - 181.0)) < 1e-11 * E
    # RAW keeps the tail: sigma~ = top-2 sigma([10 e1, 9 e2, B]) = hand value via e1 and e2 blocks
    raw = oracle.pair_errors(sp, [[0, 1]], 2, 7, oracle.RAW)
    assert np.allclose(raw.sigma_tilde[0], [np.sqrt(116.0), 9.0], rtol=1e-13)
    assert abs(raw.err2[0, 2] - (E - 197.0)) < 1e-11 * E


# ---------------------------------------------------------------- exact groups --
def test_exact_groups_vs_lapack_and_union():
    """or_exact_groups: E_r^2 of the explicit concatenation of each group (Thm EYM) against
    LAPACK on random groups, and the union-spectrum closed form for blocks with mutually
    orthogonal column spaces (A2: sigma(M) = union of sigma(A_i))."""
    R = np.random.default_rng(10)
    m = 30
    blocks = [R.standard_normal((m, int(R.integers(1, 6)))) for _ in range(7)]
    sp = oracle.block_spectra(blocks)
    groups = [[0], [1, 2], [3, 0, 5], [6, 5, 4, 3, 2, 1, 0]]
    for r in (1, 3, 8):
        got = oracle.exact_groups(sp, groups, r)
        for g, v in zip(groups, got):
            s = np.linalg.svd(np.concatenate([blocks[i] for i in g], axis=1), compute_uv=False)
            assert abs(v - np.sum(s[r:] ** 2)) <= 1e-11 * np.sum(s ** 2)
    Q = haar(R, m, 9)
    sa, sb = np.array([5.0, 2.0, 0.5]), np.array([4.0, 3.0, 1.0, 0.2])
    A = (Q[:, :3] * sa) @ haar(R, 3, 3).T
    B = (Q[:, 3:7] * sb) @ haar(R, 4, 4).T
    sp = oracle.block_spectra([A, B])
    union = np.sort(np.concatenate([sa, sb]))[::-1]
    for r in range(0, 8):
        assert abs(oracle.exact_groups(sp, [[0, 1]], r)[0] - np.sum(union[r:] ** 2)) < 1e-12 * 60


def test_exact_groups_wide_gram_route():
    """Concatenations wider than 512 (both Gram orientations) take the Gram + own tridiagonal route:
    against LAPACK's SVD of the explicit concatenation."""
    R = np.random.default_rng(12)
    for m, widths in [(560, [300, 300]), (700, [200, 350, 100])]:
        blocks = [(R.standard_normal((m, w)) * np.linspace(2, 0.1, w)).astype(np.float32).astype(np.float64)
                  for w in widths]
        sp = oracle.block_spectra(blocks)
        M = np.concatenate(blocks, axis=1)
        s = np.linalg.svd(M, compute_uv=False)
        for r in (1, 40, 300):
            got = oracle.exact_groups(sp, [list(range(len(blocks)))], r)[0]
            assert abs(got - np.sum(s[r:] ** 2)) <= 1e-10 * np.sum(s ** 2), (m, r)
