"""A greedy run traced by hand (pins Algs 2-3 of Appendix E, with the
readings listed in oracle/cluster.py's header).

Five blocks whose columns are scaled coordinate axes of R^6, all rotated by one fixed orthogonal
matrix (every quantity of the method is invariant under it, and no SVD in the run is trivial):

    B0 = [10 e0, 5 e1]   E = 125      B1 = [3 e0]          E = 9      B2 = [1 e2]   E = 1
    B3 = [2 e1, 2 e3]    E = 8        B4 = [6 e4, 6 e5]    E = 72

With r = 2 every Gram matrix of a concatenation is diagonal in the axis frame, so sigma^2 of a
concatenation is the per-axis sum of the squared scales, and every estimate is integer arithmetic:

* Alg. 3 (Lemma 1 + Cor. 3): tentative err^2 = E_total - (two largest per-axis sums of
  [U_2 diag(sigma_2), F]); the state keeps those two axes after a commit.
* Alg. 2 (Thm 2): tentative err^2 = E_total - (two largest of mu(state) U sigma^2 of the residual
  of F outside the range basis Q); energy of F inside range(Q) is lost to the bound.

RUNS lists (algorithm, sort, eps, knn) -> the clusters in append order, their certificate err^2 and
energy, and every tentative evaluation (cluster, candidate, err^2, E_total, accepted) in the order
the algorithm makes them.  Example, Alg. 3 / Frobenius order / eps = 0.1 (eps^2 = 0.01): anchor B0;
candidates by ascending energy B2, B3, B1, B4; B2: axes (100, 25, 1) -> err^2 = 1 of 126 (0.0079,
accepted); B3: axes (100, 25 + 4, 4) -> err^2 = 134 - 129 = 5 (0.037, rejected: the cluster closes
at [0, 2] with err^2 = 126 - 125); anchor B4: B3 loses all of its 8 of 80; anchor B1 (E = 9 > 8):
B3: axes (9, 4, 4) -> 4 of 17; B3 stays alone.  The other runs are traced the same way; the
smallest margin of a decision from eps^2 is 20 %.
"""
import numpy as np

MAX_NORM, RESIDUAL_ALG, APPROX = 0, 1, 2
FROB, RESID = 0, 1
R = 2
M = 6

_COLS = [
    [(0, 10.0), (1, 5.0)],
    [(0, 3.0)],
    [(2, 1.0)],
    [(1, 2.0), (3, 2.0)],
    [(4, 6.0), (5, 6.0)],
]


def blocks(dtype=np.float64):
    """The five blocks (m x n_j, column-major like every collection of synth/), rotated."""
    rot = np.linalg.qr(np.random.default_rng(11626).standard_normal((M, M)))[0]
    out = []
    for cols in _COLS:
        a = np.zeros((M, len(cols)))
        for c, (axis, scale) in enumerate(cols):
            a[axis, c] = scale
        out.append(np.asfortranarray(rot @ a, dtype=dtype))
    return out


# (algorithm, sort, eps, knn): (clusters, err2, total, [(cluster, candidate, err2, total, accepted), ...])
RUNS = {
    (APPROX, FROB, 0.1, 1): (
        [[0, 2], [4], [1], [3]], [1, 0, 0, 0], [126, 72, 9, 8],
        [(0, 2, 1, 126, True), (0, 3, 5, 134, False), (1, 3, 8, 80, False), (2, 3, 4, 17, False)]),
    # residual order: B1 lies in range(B0) (key 0) and costs nothing; then B2 (key 1), B3 (key 4)
    (APPROX, RESID, 0.1, 1): (
        [[0, 1, 2], [4], [3]], [1, 0, 0], [135, 72, 8],
        [(0, 1, 0, 134, True), (0, 2, 1, 135, True), (0, 3, 5, 143, False), (1, 3, 8, 80, False)]),
    # window of 2: after B2 the window (B3, B1) rejects B3 and takes B1; (B3, B4) has no passing block
    (APPROX, FROB, 0.1, 2): (
        [[0, 2, 1], [4], [3]], [1, 0, 0], [135, 72, 8],
        [(0, 2, 1, 126, True), (0, 3, 5, 134, False), (0, 1, 1, 135, True), (0, 3, 5, 143, False),
         (0, 4, 62, 207, False), (1, 3, 8, 80, False)]),
    # eps^2 = 0.0484 lies between Alg. 3's 5 / 134 and Alg. 2's 9 / 134 for B3: the two algorithms part
    (APPROX, FROB, 0.22, 1): (
        [[0, 2, 3, 1], [4]], [5, 0], [143, 72],
        [(0, 2, 1, 126, True), (0, 3, 5, 134, True), (0, 1, 5, 143, True), (0, 4, 70, 215, False)]),
    (RESIDUAL_ALG, FROB, 0.22, 1): (
        [[0, 2], [4], [1], [3]], [1, 0, 0, 0], [126, 72, 9, 8],
        [(0, 2, 1, 126, True), (0, 3, 9, 134, False), (1, 3, 8, 80, False), (2, 3, 4, 17, False)]),
    # Alg. 2 loses the whole energy of the in-range B1 (9 of 134) and closes B0 at once; under anchor B1
    # the range basis is e0 only: B2 (key 1) is exact (mu = (3, 1)), B3 costs 18 - 13
    (RESIDUAL_ALG, RESID, 0.1, 1): (
        [[0], [4], [1, 2], [3]], [0, 0, 0, 0], [125, 72, 10, 8],
        [(0, 1, 9, 134, False), (1, 2, 1, 73, False), (2, 2, 0, 10, True), (2, 3, 5, 18, False)]),
}
