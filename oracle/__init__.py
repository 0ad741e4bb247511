"""float64 CPU oracle for the merge-error evaluation path of arXiv 2601.11626.

TEST INFRASTRUCTURE ONLY.  Only ``tests/``, ``__graft_entry__.smoke()`` and
``bench.py``'s ``cpu_baseline`` / ``--impl reference`` legs may import this
package.  The product path (``paper_2601_11626_b200``) never imports it and
fails loudly when its CUDA library is missing.

The heavy numerics live in ``oracle.c`` (own Householder QR + one-sided
Jacobi SVD, float64, OpenMP over independent evaluations); this module only
marshals numpy arrays and holds the host-side greedy drivers
(``oracle.cluster``).  It shares no code with the CUDA path.

Every function cites the PAPER.md passage it follows; ambiguous passages use
the SURVEY.md §8(c) readings (A1..A21) and DESIGN.md's A22, restated in DESIGN.md.

Pins: tests/test_oracle_pins.py, tests/test_oracle_big_pins.py and
tests/test_oracle_cluster.py (closed forms, LAPACK cross-checks, brute force,
invariants, and a greedy run traced by hand: tests/axis_example.py fixes the
exact compositions, append orders and every tentative evaluation of Algs 2-3).
No function here is left without a pin.
"""
from __future__ import annotations

import ctypes
import os
import subprocess
from dataclasses import dataclass

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
_LIB_PATH = os.path.join(_HERE, "liboracle.so")
_lib = None

TAU = 1e-5          # numerical-rank rule (A5): keep sigma_l > TAU * sigma_1
BIG_N = 512         # blocks with more columns take reading A22 (range = R^m, spectra from the m x m Gram)
WEYL, RESIDUAL, INCREMENTAL = 1, 2, 4
RAW, TRUNC = 0, 1


def build(force: bool = False) -> str:
    """Compile oracle.c with gcc (plain C, -O2, OpenMP)."""
    src = os.path.join(_HERE, "oracle.c")
    if force or not os.path.exists(_LIB_PATH) or os.path.getmtime(_LIB_PATH) < os.path.getmtime(src):
        subprocess.check_call(["gcc", "-O2", "-fopenmp", "-fPIC", "-shared", "-o", _LIB_PATH, src, "-lm"])
    return _LIB_PATH


def lib():
    global _lib
    if _lib is None:
        build()
        L = ctypes.CDLL(_LIB_PATH)
        dp = ctypes.POINTER(ctypes.c_double)
        ip = ctypes.POINTER(ctypes.c_int32)
        pp = ctypes.POINTER(ctypes.c_void_p)
        i64 = ctypes.c_int64
        L.or_energy_f32.restype = ctypes.c_double
        L.or_energy_f32.argtypes = [ctypes.c_void_p, i64]
        L.or_svd.restype = ctypes.c_int
        L.or_svd.argtypes = [i64, i64, dp, i64, dp, dp, i64, dp, i64]
        L.or_exact_err2.restype = ctypes.c_int
        L.or_exact_err2.argtypes = [i64, i64, dp, i64, ctypes.c_int32, dp]
        L.or_pair_errors.restype = ctypes.c_int
        L.or_pair_errors.argtypes = [i64, ctypes.c_int32, ip, pp, dp, pp, pp, ip, ip, i64,
                                     ctypes.c_int32, ctypes.c_uint32, ctypes.c_int, dp, dp, dp, dp]
        L.or_pair_errors_tight.restype = ctypes.c_int
        L.or_pair_errors_tight.argtypes = [i64, ctypes.c_int32, ip, pp, dp, pp, pp, ip, ip, i64,
                                           ctypes.c_int32, ctypes.c_int, dp, dp]
        L.or_block_svds.restype = ctypes.c_int
        L.or_block_svds.argtypes = [i64, ctypes.c_int32, ip, pp, pp, pp]
        L.or_exact_groups.restype = ctypes.c_int
        L.or_exact_groups.argtypes = [i64, ip, pp, ip, ip, ctypes.c_int32, ctypes.c_int32, dp]
        L.or_num_threads.restype = ctypes.c_int
        L.or_sym_eig_topk.restype = ctypes.c_int
        L.or_sym_eig_topk.argtypes = [i64, dp, i64, i64, dp, dp, i64]
        L.or_block_spectra_big.restype = ctypes.c_int
        L.or_block_spectra_big.argtypes = [i64, i64, ctypes.c_void_p, i64, dp, dp]
        _lib = L
    return _lib


def _dp(a):
    return a.ctypes.data_as(ctypes.POINTER(ctypes.c_double)) if a is not None else None


def _ip(a):
    return a.ctypes.data_as(ctypes.POINTER(ctypes.c_int32))


def _ptrs(arrs):
    return (ctypes.c_void_p * len(arrs))(*[a.ctypes.data for a in arrs])


def num_threads() -> int:
    return lib().or_num_threads()


# --------------------------------------------------------------------------
# Primitives
# --------------------------------------------------------------------------
def energy(a) -> float:
    """||A||_F^2 in float64 (split PAPER.md:1484-1488)."""
    a32 = np.ascontiguousarray(a, dtype=np.float32)
    return lib().or_energy_f32(a32.ctypes.data, a32.size)


def svd(a: np.ndarray, want_u: bool = False, want_v: bool = False):
    """Thin SVD (own Householder QR + one-sided Jacobi, float64).
    Returns s (non-increasing) and optionally U (m×k), V (n×k)."""
    a = np.asfortranarray(a, dtype=np.float64)
    m, n = a.shape
    k = min(m, n)
    s = np.zeros(k)
    U = np.zeros((m, k), order="F") if want_u else None
    V = np.zeros((n, k), order="F") if want_v else None
    st = lib().or_svd(m, n, _dp(a), m, _dp(s), _dp(U), m, _dp(V), n)
    if st:
        raise RuntimeError(f"oracle SVD did not converge (status {st}) for {m}x{n}")
    out = [s]
    if want_u:
        out.append(U)
    if want_v:
        out.append(V)
    return out[0] if len(out) == 1 else tuple(out)


def exact_err2(M: np.ndarray, r: int) -> float:
    """E_r^2(M) = sum_{j>r} sigma_j^2(M) by SVD of the explicit matrix
    (Thm EYM)."""
    s = svd(M)
    return float(np.sum(s[r:] ** 2))


# --------------------------------------------------------------------------
# Block spectra (S2): sigma(A_i), U_r, full-range basis (A5)
# --------------------------------------------------------------------------
@dataclass
class Spectra:
    m: int
    n: np.ndarray        # int32 columns per block
    A: list              # float64 Fortran blocks (m × n_i)
    E: np.ndarray        # float64 energies
    sig: list            # per block: all min(m, n_i) singular values
    U: list              # per block: m × min(m, n_i) left singular vectors
    rank: np.ndarray     # int32 numerical rank (sigma_l > TAU sigma_1)


def sym_eig_topk(G: np.ndarray, k: int):
    """All eigenvalues (non-increasing) and the top-k eigenvectors of a
    symmetric matrix: textbook Householder tridiagonalisation, bisection on
    Sturm counts, inverse iteration + back-transformation (oracle.c,
    or_sym_eig_topk; reading A15)."""
    G = np.array(G, dtype=np.float64, order="F", copy=True)
    m = G.shape[0]
    lam = np.zeros(m)
    V = np.zeros((m, max(k, 1)), order="F")
    st = lib().or_sym_eig_topk(m, _dp(G), m, int(k), _dp(lam), _dp(V), m)
    if st:
        raise RuntimeError(f"oracle symmetric eigensolver failed (status {st})")
    return lam, V[:, :k]


def block_spectra(blocks, tau: float = TAU, nvec: int | None = None) -> Spectra:
    """Per-block thin SVD in float64 (the Weyl bound needs the blocks' leading
    singular values; the residual bound the range basis,
    PAPER.md:362-363; Alg. 3 starts from the anchor's top-r SVD,
    PAPER.md:1999).  ``blocks`` is the (N, n, m) float32 array of synth or a
    list of m×n_i arrays.  ``nvec``: left singular vectors kept per block
    wider than BIG_N (A22; default min(m, 256)); narrower blocks keep all."""
    if isinstance(blocks, np.ndarray) and blocks.ndim == 3:
        A = [np.asfortranarray(blocks[i].T, dtype=np.float64) for i in range(blocks.shape[0])]
    else:
        A = [np.asfortranarray(b, dtype=np.float64) for b in blocks]
    m = A[0].shape[0]
    n = np.array([a.shape[1] for a in A], dtype=np.int32)
    N = len(A)
    E = np.array([float(np.sum(a * a)) for a in A])   # fp64 sum of squares (exact products)
    big = [int(k) > BIG_N for k in n]
    if any(big) and not all(big):
        raise ValueError("collections mixing blocks wider than BIG_N columns with narrower ones (A22)")
    if all(big):
        return _block_spectra_big(blocks, A, m, n, E, min(m, 256) if nvec is None else int(nvec))
    sig = [np.zeros(min(m, int(k))) for k in n]
    U = [np.zeros((m, min(m, int(k))), order="F") for k in n]
    st = lib().or_block_svds(m, N, _ip(n), _ptrs(A), _ptrs(sig), _ptrs(U))
    if st:
        raise RuntimeError(f"oracle block SVD failed (status {st})")
    rank = np.array([int(np.sum(s > tau * s[0])) if s[0] > 0 else 0 for s in sig], dtype=np.int32)
    return Spectra(m, n, A, E, sig, U, rank)


def _block_spectra_big(blocks, A, m, n, E, nvec) -> Spectra:
    """Reading A22 for blocks wider than BIG_N columns (configs 3
    and 4, square weight-like blocks; n_i >= m required): the spectra follow
    A15's exact route in oracle.c (or_block_spectra_big): the m x m fp64 Gram
    A A^T, own Householder tridiagonalisation, bisection for every eigenvalue,
    inverse iteration for the top ``nvec`` eigenvectors (squaring costs
    relative accuracy (sigma_1/sigma_l)^2 * 1e-16 only).  The block's range is
    taken as all of R^m: rank_i = min(m, n_i) and the paper-literal residual
    R = (I - Q Q^T) F is identically 0 (oracle.c, pair_residual).  U keeps
    the top ``nvec`` left singular vectors (pair evaluations need r <= nvec)."""
    sig, U = [], []
    for i, a in enumerate(A):
        if a.shape[1] < m:
            raise ValueError("A22 blocks must have n_i >= m")
        a32 = np.asfortranarray(blocks[i].T if isinstance(blocks, np.ndarray) and blocks.ndim == 3 else a,
                                dtype=np.float32)
        s = np.zeros(m)
        u = np.zeros((m, max(nvec, 1)), order="F")
        st = lib().or_block_spectra_big(m, a32.shape[1], a32.ctypes.data, nvec, _dp(s), _dp(u))
        if st:
            raise RuntimeError(f"oracle big-block spectra failed (status {st})")
        sig.append(s)
        U.append(u[:, :nvec])
    rank = np.array([min(m, int(k)) for k in n], dtype=np.int32)
    return Spectra(m, n, A, E, sig, U, rank)


# --------------------------------------------------------------------------
# Pair evaluation (S3..S9)
# --------------------------------------------------------------------------
@dataclass
class PairResult:
    err2: np.ndarray          # (P, 3) weyl, residual, incremental (NaN if not requested)
    total: np.ndarray         # (P,)
    sigma_tilde: np.ndarray   # (P, r)
    mu: np.ndarray            # (P, r)


def _check_vectors(spec: Spectra, r: int):
    """The pair estimators read U_{i, 1..min(r, rank_i)}: blocks wider than BIG_N keep only nvec vectors."""
    for u, rk in zip(spec.U, spec.rank):
        if min(r, int(rk)) > u.shape[1]:
            raise ValueError(f"r = {r} needs more left singular vectors than block_spectra(nvec={u.shape[1]}) kept")


def pair_errors(spec: Spectra, pairs, r: int, kinds: int = 7, operand: int = RAW) -> PairResult:
    """Weyl (Eq. 5), residual (Eq. 6) and incremental (Cor. 2) estimates of
    E_r^2([A_i, F_j]) for ordered pairs (base i, appended j).  See oracle.c
    for the per-estimator definitions and citations."""
    pairs = np.ascontiguousarray(pairs, dtype=np.int32).reshape(-1, 2)
    _check_vectors(spec, r)
    P = pairs.shape[0]
    err2 = np.zeros((P, 3))
    total = np.zeros(P)
    st_ = np.zeros((P, r))
    mu = np.zeros((P, r))
    status = lib().or_pair_errors(spec.m, len(spec.A), _ip(spec.n), _ptrs(spec.A), _dp(spec.E),
                                  _ptrs(spec.sig), _ptrs(spec.U), _ip(spec.rank), _ip(pairs), P, r,
                                  kinds, operand, _dp(err2), _dp(total), _dp(st_), _dp(mu))
    if status:
        raise RuntimeError(f"oracle pair evaluation failed (status {status})")
    return PairResult(err2, total, st_, mu)


def pair_errors_tight(spec: Spectra, pairs, r: int, operand: int = RAW):
    """Beyond the paper: (P, 2) [residual bound with the tracked
    basis U_r (A4), per-index Weyl bound (A8)] and the totals.  See oracle.c
    or_pair_errors_tight."""
    pairs = np.ascontiguousarray(pairs, dtype=np.int32).reshape(-1, 2)
    _check_vectors(spec, r)
    P = pairs.shape[0]
    err2x = np.zeros((P, 2))
    total = np.zeros(P)
    st = lib().or_pair_errors_tight(spec.m, len(spec.A), _ip(spec.n), _ptrs(spec.A), _dp(spec.E),
                                    _ptrs(spec.sig), _ptrs(spec.U), _ip(spec.rank), _ip(pairs), P, r,
                                    operand, _dp(err2x), _dp(total))
    if st:
        raise RuntimeError(f"oracle tight pair evaluation failed (status {st})")
    return err2x, total


def exact_groups(spec: Spectra, groups, r: int) -> np.ndarray:
    """Exact E_r^2 of the explicit concatenation of each group of block ids
    (brute force, tiny inputs)."""
    offs = np.zeros(len(groups) + 1, dtype=np.int32)
    ids = np.concatenate([np.asarray(g, dtype=np.int32) for g in groups]) if groups else np.zeros(0, np.int32)
    offs[1:] = np.cumsum([len(g) for g in groups])
    out = np.zeros(len(groups))
    st = lib().or_exact_groups(spec.m, _ip(spec.n), _ptrs(spec.A), _ip(offs), _ip(ids), len(groups), r, _dp(out))
    if st:
        raise RuntimeError("oracle exact SVD failed")
    return out
