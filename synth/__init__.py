"""Seeded synthetic collections shaped like the paper's workloads.

This module is shared by the oracle tests, the GPU parity tests and bench.py.
It holds NO arithmetic of the method (no energies, spectra, bounds or
estimators): it only draws matrices.  Recipes follow SURVEY.md §8(d) and are
restated in DESIGN.md ("Input recipe"); the paper's datasets (PAPER.md:550-575,
Table 1) are absent, these collections stand in for them.

Layout: every generator returns ``blocks``, a float32 array of shape
(N, n, m), C-contiguous, i.e. block ``i`` is the column-major m×n matrix
``blocks[i].T`` (column c of block i is ``blocks[i, c, :]``).  Column-major is
the layout the C ABI consumes (include/cmsvd.h) and makes horizontal
concatenation a contiguous append.
"""
from __future__ import annotations

import dataclasses
import numpy as np

__all__ = ["Collection", "haar", "config1", "config2", "config3", "config4",
           "config5", "make_config", "all_pairs_by_norm_order", "knn_pairs",
           "CONFIGS"]


@dataclasses.dataclass
class Collection:
    name: str
    blocks: np.ndarray          # (N, n, m) float32, block i column-major
    r: int                      # target rank
    eps: tuple                  # thresholds the config is quoted with
    operand: int                # 0 = RAW appended block, 1 = TRUNC (rank-r factor)
    groups: np.ndarray          # hidden group id per block (for reporting only)
    seed: int

    @property
    def N(self) -> int:
        return self.blocks.shape[0]

    @property
    def m(self) -> int:
        return self.blocks.shape[2]

    @property
    def n(self) -> int:
        return self.blocks.shape[1]

    def block(self, i: int) -> np.ndarray:
        """Block i as an m×n float32 array (a transposed view)."""
        return self.blocks[i].T


def haar(rng: np.random.Generator, m: int, k: int) -> np.ndarray:
    """m×k matrix with Haar-distributed orthonormal columns: QR of a Gaussian
    with column signs fixed by sign(diag R) (SURVEY.md §8(d) common rules)."""
    g = rng.standard_normal((m, k))
    q, rr = np.linalg.qr(g)
    s = np.sign(np.diag(rr))
    s[s == 0] = 1.0
    return q * s


def _unit_rms(signal_t: np.ndarray) -> np.ndarray:
    """Scale a (n, m) signal so that ||S||_F^2 = m*n ("unit-RMS signal")."""
    return signal_t * np.sqrt(signal_t.size / np.sum(signal_t * signal_t))


def config1(seed: int = 0) -> Collection:
    """BASELINE.json configs[0]: N=16, 64x32, 4 hidden groups, block =
    U_g(64x6 orthonormal) @ Gaussian(6x32) + 0.01*N(0,1); r=8, eps=0.05."""
    rng = np.random.default_rng(seed)
    N, m, n, G, k = 16, 64, 32, 4, 6
    U = [haar(rng, m, k) for _ in range(G)]
    out = np.empty((N, n, m), np.float32)
    for i in range(N):
        g = i % G
        c = rng.standard_normal((k, n))
        a = U[g] @ c + 0.01 * rng.standard_normal((m, n))
        out[i] = a.T
    return Collection("config1", out, 8, (0.05,), 0, np.arange(N) % G, seed)


def config2(seed: int = 1) -> Collection:
    """configs[1]: N=128, 512x128, 8 groups sharing rank-24 orthonormal bases,
    sigma_k ~ 1/k, unit-RMS signal, 0.02 Gaussian noise; r=32."""
    rng = np.random.default_rng(seed)
    N, m, n, G, k = 128, 512, 128, 8, 24
    U = [haar(rng, m, k) for _ in range(G)]
    sig = 1.0 / np.arange(1, k + 1)
    out = np.empty((N, n, m), np.float32)
    for i in range(N):
        g = i % G
        W = haar(rng, n, k)
        st = (W * sig) @ U[g].T                      # (n, m) = (U diag(sig) W^T)^T
        st = _unit_rms(st)
        out[i] = st + 0.02 * rng.standard_normal((n, m))
    return Collection("config2", out, 32, (0.02, 0.05, 0.1), 0, np.arange(N) % G, seed)


def config3(seed: int = 2, N: int = 256, m: int = 1024, shared: int = 128) -> Collection:
    """configs[2]: N=256 square 1024x1024, sigma_l ~ l^-0.7, unit-RMS; even
    blocks share a rank-128 column subspace (first 128 left singular vectors =
    U_s, rest Haar in U_s^perp); r=128, TRUNC operand (A6)."""
    rng = np.random.default_rng(seed)
    n = m
    Us = haar(rng, m, shared)
    sig = np.arange(1, n + 1, dtype=np.float64) ** -0.7
    out = np.empty((N, n, m), np.float32)
    for i in range(N):
        if i % 2 == 0:
            comp = haar(rng, m, m - shared)
            comp -= Us @ (Us.T @ comp)               # project to U_s^perp ...
            comp = np.linalg.qr(comp)[0]             # ... and re-orthonormalise
            Ui = np.concatenate([Us, comp], axis=1)
        else:
            Ui = haar(rng, m, m)
        Vi = haar(rng, n, n)
        st = (Vi * sig) @ Ui.T
        out[i] = _unit_rms(st)
    return Collection("config3", out, 128, (0.1, 0.3), 1, (np.arange(N) % 2 == 0).astype(int), seed)


def config4(seed: int = 3, N: int = 64, m: int = 4096, rank: int = 256, nu: float = 0.1) -> Collection:
    """configs[3]: 64 = 16 layers x {Q,K,V,O}, 4096x4096; 4 layer groups of 4
    consecutive layers share U_g (m x 256); W = U_g C_i (unit-RMS) + nu N(0,1),
    nu = 0.1 (proposed reading); r=256, TRUNC operand."""
    rng = np.random.default_rng(seed)
    n = m
    G = 4
    U = [haar(rng, m, rank) for _ in range(G)]
    out = np.empty((N, n, m), np.float32)
    for i in range(N):
        g = (i // 4) // 4
        c = rng.standard_normal((rank, n)).astype(np.float32)
        st = (c.T @ U[g].T.astype(np.float32))
        st *= np.float32(np.sqrt(st.size / np.sum(st.astype(np.float64) ** 2)))
        st += np.float32(nu) * rng.standard_normal((n, m), dtype=np.float32)
        out[i] = st
    return Collection("config4", out, 256, (0.15,), 1, (np.arange(N) // 16), seed)


def config5(seed: int = 4, N: int = 512, r: int = 16, m: int = 2048, n: int = 64) -> Collection:
    """configs[4]: N in {512, 2048} tall-thin 2048x64; 32 groups of rank 16:
    U_g (2048x16 Haar) @ Gaussian(16x64) * sqrt(m/16) (unit RMS) + 0.05 N(0,1);
    r in {16, 64}; eps = 0.1 (proposed)."""
    rng = np.random.default_rng(seed)
    G, k = 32, 16
    U = [haar(rng, m, k) for _ in range(G)]
    out = np.empty((N, n, m), np.float32)
    for i in range(N):
        g = i % G
        c = rng.standard_normal((k, n)) * np.sqrt(m / k)
        a = U[g] @ c + 0.05 * rng.standard_normal((m, n))
        out[i] = a.T
    return Collection(f"config5_N{N}_r{r}", out, r, (0.1,), 0, np.arange(N) % G, seed)


CONFIGS = {
    "config1": config1,
    "config2": config2,
    "config3": config3,
    "config4": config4,
    "config5": config5,
}


def make_config(name: str, **kw) -> Collection:
    return CONFIGS[name](**kw)


def all_pairs_by_norm_order(order: np.ndarray) -> np.ndarray:
    """All unordered pairs as (base, appended) with base = the earlier block in
    ``order`` (a permutation, normally blocks sorted by descending norm; A7).
    Returns int32 (P, 2)."""
    order = np.asarray(order, dtype=np.int64)
    N = order.size
    ii, jj = np.triu_indices(N, k=1)
    return np.stack([order[ii], order[jj]], axis=1).astype(np.int32)


def knn_pairs(neighbours: np.ndarray) -> np.ndarray:
    """(i, nbr) candidate pairs from an (N, k) neighbour table."""
    N, k = neighbours.shape
    base = np.repeat(np.arange(N, dtype=np.int32), k)
    return np.stack([base, neighbours.reshape(-1).astype(np.int32)], axis=1)
