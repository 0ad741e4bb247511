"""Greedy certificate-driven clustering drivers (oracle side).

TEST INFRASTRUCTURE ONLY (see oracle/__init__.py).  Plain float64 host loops
over the oracle's own SVD; the order of operations follows Appendix E,
Algorithms 1-3 with SPEC.md's readings of the vague
steps and SURVEY.md A10/A11:

* anchor = largest remaining ||A||_F, ties -> smaller block id;
* ``frobenius`` mode: candidates in ascending ||A||_F (ties -> smaller id);
  ``residual`` mode: ascending ||(I - Q Q^T) A_j||_F against the *current*
  state (Q = Alg. 2 range basis, U = Alg. 3 tracked basis), re-ranked after
  every accept;
* a candidate is evaluated on a tentative append and accepted iff
  err^2 <= eps^2 * E_total (inclusive, A9); with ``knn = k`` the first k
  candidates in order form the window and the first passing one is
  accepted; a window with no passing candidate closes the cluster
  (``knn = 1`` is the paper's stop-on-first-rejection);
* zero-energy blocks are merged unconditionally.
"""
from __future__ import annotations

from dataclasses import dataclass, field

import numpy as np

from . import Spectra, TAU, svd, RAW, TRUNC

MAX_NORM, RESIDUAL_ALG, APPROX = 0, 1, 2
SORT_FROBENIUS, SORT_RESIDUAL = 0, 1


@dataclass
class ClusterResult:
    assign: np.ndarray                 # cluster id per block (creation order)
    order: np.ndarray                  # position of the block in its cluster's append order
    clusters: list = field(default_factory=list)   # member ids in append order
    err2: list = field(default_factory=list)       # certificate err^2 at close
    total: list = field(default_factory=list)      # cluster energy
    n_evals: int = 0                   # tentative merge evaluations performed
    decisions: list = field(default_factory=list)  # (cluster, candidate, key, err2, total, accepted)


def _desc_order(E: np.ndarray) -> list:
    return sorted(range(len(E)), key=lambda i: (-E[i], i))


def _operand(spec: Spectra, j: int, r: int, operand: int) -> np.ndarray:
    if operand == RAW:
        return spec.A[j]
    rr = min(r, int(spec.rank[j]))
    return spec.U[j][:, :rr] * spec.sig[j][:rr]


def _finish(res: ClusterResult, members: list, e2: float, tot: float):
    cid = len(res.clusters)
    for pos, b in enumerate(members):
        res.assign[b] = cid
        res.order[b] = pos
    res.clusters.append(list(members))
    res.err2.append(max(0.0, min(e2, tot)))
    res.total.append(tot)


def cluster_max_norm(spec: Spectra, r: int, eps: float) -> ClusterResult:
    """Algorithm 1, Weyl-based max-norm clustering.
    Head = anchor plus the next-largest blocks while total width <= r; if the
    anchor alone is wider than r the head is the anchor with head energy
    sum_{l<=r} sigma_l^2(anchor) (A11, Eq. 5 form).  Tail = smallest-norm
    remaining blocks added while (E_C - E_head)/E_C <= eps^2."""
    N = len(spec.A)
    E = spec.E
    res = ClusterResult(np.full(N, -1, np.int32), np.full(N, -1, np.int32))
    remaining = _desc_order(E)
    while remaining:
        anchor = remaining.pop(0)
        head = [anchor]
        width = int(spec.n[anchor])
        if width > r:
            e_head = float(np.sum(spec.sig[anchor][:r] ** 2))
        else:
            while remaining and width + int(spec.n[remaining[0]]) <= r:
                b = remaining.pop(0)
                head.append(b)
                width += int(spec.n[b])
            e_head = float(sum(E[b] for b in head))
        members = list(head)
        tot = float(sum(E[b] for b in head))
        while remaining:
            b = remaining[-1]                       # smallest norm remaining
            t2 = tot + E[b]
            e2 = t2 - e_head
            ok = (E[b] == 0.0) or (e2 <= eps * eps * t2)
            res.n_evals += 1
            res.decisions.append((len(res.clusters), b, E[b], e2, t2, ok))
            if not ok:
                break
            remaining.pop()
            members.append(b)
            tot = t2
        _finish(res, members, tot - e_head, tot)
    return res


class _ResidualState:
    """Alg. 2 state: range basis Q of the cluster (grows, <= m columns), the
    running top-r of the pooled residual spectrum mu (top_r(X u Y) =
    top_r(top_r(X) u Y), proof Step 5 PAPER.md:1694-1706), and energy E."""

    def __init__(self, spec: Spectra, anchor: int, r: int):
        q = int(spec.rank[anchor])
        self.Q = np.array(spec.U[anchor][:, :q])
        self.mu = np.array(spec.sig[anchor][:r])
        self.E = float(spec.E[anchor])
        self.r = r

    def residual(self, F):
        R = F - self.Q @ (self.Q.T @ F)
        R = R - self.Q @ (self.Q.T @ R)          # one re-orthogonalisation pass
        return R

    def key(self, F) -> float:
        R = self.residual(F)
        return float(np.sum(R * R))

    def tentative(self, F, Ej):
        R = self.residual(F)
        s, Ur = svd(R, want_u=True)
        mu = np.sort(np.concatenate([self.mu, s]))[::-1][: self.r]
        tot = self.E + Ej
        e2 = tot - float(np.sum(mu ** 2))
        return e2, tot, (R, s, Ur, mu)

    def commit(self, Ej, data):
        R, s, Ur, mu = data
        if s.size and s[0] > 0:
            keep = s > TAU * s[0]
            # the range basis grows to at most m columns ("Q grows to <= m
            # columns"): once Q spans R^m the residual is rounding noise and adds no direction
            room = self.Q.shape[0] - self.Q.shape[1]
            idx = np.flatnonzero(keep)[:max(room, 0)]
            self.Q = np.concatenate([self.Q, Ur[:, idx]], axis=1)
        self.mu = mu
        self.E += Ej

    def err2(self):
        return self.E - float(np.sum(self.mu ** 2))


class _IncrementalState:
    """Alg. 3 state: truncated incremental SVD (Lemma 1 + Cor. 3,
    PAPER.md:1297-1436) kept as U (m x r'), sigma (r'), E; appending F gives
    sigma~ = top-r sigma([U diag(sigma), F]) and U <- top-r left singular
    vectors (truncate after every append)."""

    def __init__(self, spec: Spectra, anchor: int, r: int):
        rr = min(r, int(spec.rank[anchor]))
        self.U = np.array(spec.U[anchor][:, :rr])
        self.s = np.array(spec.sig[anchor][:rr])
        self.E = float(spec.E[anchor])
        self.r = r

    def key(self, F) -> float:
        R = F - self.U @ (self.U.T @ F)
        return float(np.sum(R * R))

    def tentative(self, F, Ej):
        X = np.concatenate([self.U * self.s, F], axis=1)
        s, U = svd(X, want_u=True)
        st = s[: self.r]
        tot = self.E + Ej
        e2 = tot - float(np.sum(st ** 2))
        return e2, tot, (s, U)

    def commit(self, Ej, data):
        s, U = data
        k = min(self.r, s.size)
        keep = [l for l in range(k) if s[0] > 0 and s[l] > TAU * s[0]]
        self.U = U[:, keep]
        self.s = s[keep]
        self.E += Ej

    def err2(self):
        return self.E - float(np.sum(self.s ** 2))


def cluster_tracked(spec: Spectra, algorithm: int, r: int, eps: float, sort: int = SORT_FROBENIUS,
                    knn: int = 1, operand: int = RAW) -> ClusterResult:
    """Algorithms 2 (residual) and 3 (approximate)."""
    N = len(spec.A)
    E = spec.E
    res = ClusterResult(np.full(N, -1, np.int32), np.full(N, -1, np.int32))
    remaining = _desc_order(E)
    State = _ResidualState if algorithm == RESIDUAL_ALG else _IncrementalState
    while remaining:
        anchor = remaining.pop(0)
        st = State(spec, anchor, r)
        members = [anchor]
        while remaining:
            if sort == SORT_FROBENIUS:
                cand = sorted(remaining, key=lambda b: (E[b], b))
                keys = [E[b] for b in cand]
            else:
                kk = {b: st.key(_operand(spec, b, r, operand)) for b in remaining}
                cand = sorted(remaining, key=lambda b: (kk[b], b))
                keys = [kk[b] for b in cand]
            accepted = None
            for b, key in list(zip(cand, keys))[:knn]:
                F = _operand(spec, b, r, operand)
                e2, tot, data = st.tentative(F, E[b])
                ok = (E[b] == 0.0) or (e2 <= eps * eps * tot)
                res.n_evals += 1
                res.decisions.append((len(res.clusters), b, key, e2, tot, ok))
                if ok:
                    accepted = (b, data)
                    break
            if accepted is None:
                break
            b, data = accepted
            st.commit(E[b], data)
            remaining.remove(b)
            members.append(b)
        _finish(res, members, st.err2(), st.E)
    return res


def cluster(spec: Spectra, algorithm: int, r: int, eps: float, sort: int = SORT_FROBENIUS,
            knn: int = 1, operand: int = RAW) -> ClusterResult:
    if not (0.0 < eps < 1.0) or r < 1:
        raise ValueError("need 0 < eps < 1 and r >= 1")
    if algorithm == MAX_NORM:
        return cluster_max_norm(spec, r, eps)
    return cluster_tracked(spec, algorithm, r, eps, sort, knn, operand)


def compression(m: int, ncols, clusters, r: int):
    """Compression accounting of a partition (PAPER.md:158-162 mem_c = r_c (m + N_c);
    PAPER.md:590-597 ratio = parameters before / after).  Reading A23: a
    cluster is stored raw when that is smaller, mem_c = min(m N_c, r_c (m + N_c)) with
    r_c = min(r, m, N_c) -- consistent with Table 2's 1.000* for failed (all-singleton)
    clusterings.  Returns (mem per cluster, ratio)."""
    ncols = np.asarray(ncols, dtype=np.int64)
    mem = []
    for members in clusters:
        Nc = int(np.sum(ncols[list(members)]))
        rc = min(r, m, Nc)
        mem.append(min(m * Nc, rc * (m + Nc)))
    mem = np.array(mem, dtype=np.int64)
    return mem, float(m * np.sum(ncols)) / float(np.sum(mem))


def sequence_errors(spec: Spectra, seqs, r: int, kinds: int = 7, operand: int = RAW):
    """Predicted rank-r errors of given block sequences (clusters in append order) --
    the slack diagnostic's estimates: for each sequence
    (A_1, ..., A_K): Weyl = Eq. 5 over the K blocks; residual =
    Alg. 2's state after appending A_2..A_K to A_1 (Thm 2 / Cor 1); incremental =
    Alg. 3's state after the same appends (Lemma 1 + Cor 3 + Cor 2).  A single block
    gives its own truncation error for every kind.  Returns (err2 (S, 3), total (S,))."""
    S = len(seqs)
    err2 = np.full((S, 3), np.nan)
    total = np.zeros(S)
    for s, seq in enumerate(seqs):
        seq = [int(b) for b in seq]
        tot = float(sum(spec.E[b] for b in seq))
        total[s] = tot
        if kinds & 1:
            top = max(float(np.sum(spec.sig[b][:r] ** 2)) for b in seq)
            err2[s, 0] = min(max(tot - top, 0.0), tot)
        for bit, col, State in ((2, 1, _ResidualState), (4, 2, _IncrementalState)):
            if not kinds & bit:
                continue
            st = State(spec, seq[0], r)
            e2 = st.err2()
            for b in seq[1:]:
                e2, _, data = st.tentative(_operand(spec, b, r, operand), float(spec.E[b]))
                st.commit(float(spec.E[b]), data)
            err2[s, col] = min(max(e2, 0.0), tot)
    return err2, total
