"""Thin ctypes binding of libcmsvd (include/cmsvd.h): argument marshalling
only -- every step of the path runs in the library's CUDA kernels.  There is
no CPU fallback: if the shared library or a CUDA device is missing, the calls
raise.

Torch is used only as plumbing: device tensors may be passed (their
``data_ptr()`` goes to the C ABI with ``where=DEVICE``) and the context can
borrow torch's current CUDA stream.
"""
from __future__ import annotations

import ctypes
import os

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(_HERE, "libcmsvd.so")

OK, E_ARG, E_SHAPE, E_NONFINITE, E_STATE, E_NOCONV, E_CUDA, E_NOMEM = range(8)
HOST, DEVICE = 0, 1
WEYL, RESIDUAL, INCREMENTAL, ALL = 1, 2, 4, 7
RAW, TRUNC = 0, 1
ALG_MAX_NORM, ALG_RESIDUAL, ALG_APPROX = 0, 1, 2
SORT_FROBENIUS, SORT_RESIDUAL = 0, 1

EXPORTS = ["cmsvd_status_string", "cmsvd_last_error", "cmsvd_version", "cmsvd_create", "cmsvd_destroy",
           "cmsvd_register", "cmsvd_block_spectra", "cmsvd_pair_errors", "cmsvd_pair_errors_tight",
           "cmsvd_cluster", "cmsvd_cluster_verify", "cmsvd_cluster_verify_ex", "cmsvd_cluster_factors", "cmsvd_sequence_errors",
           "cmsvd_launch_count", "cmsvd_sym_eigvals", "cmsvd_spectra_diagnostics",
           "cmsvd_profile_enable",
           "cmsvd_profile_read"]


class CmsvdError(RuntimeError):
    def __init__(self, status: int, msg: str):
        super().__init__(f"{_status_name(status)}: {msg}")
        self.status = status


class ClusterOpts(ctypes.Structure):
    _fields_ = [("algorithm", ctypes.c_int32), ("sort", ctypes.c_int32), ("knn", ctypes.c_int32),
                ("operand", ctypes.c_int32), ("r", ctypes.c_int32), ("eps", ctypes.c_double)]


_lib = None


def load(path: str = LIB_PATH):
    """Load libcmsvd.so (raises if it is missing -- no fallback)."""
    global _lib
    if _lib is not None:
        return _lib
    if not os.path.exists(path):
        raise ImportError(f"libcmsvd.so not built at {path}; run __graft_entry__.build()")
    L = ctypes.CDLL(path)
    vp, i64, i32, u32 = ctypes.c_void_p, ctypes.c_int64, ctypes.c_int32, ctypes.c_uint32
    L.cmsvd_status_string.restype = ctypes.c_char_p
    L.cmsvd_status_string.argtypes = [ctypes.c_int]
    L.cmsvd_last_error.restype = ctypes.c_char_p
    L.cmsvd_last_error.argtypes = [vp]
    L.cmsvd_version.restype = ctypes.c_char_p
    L.cmsvd_version.argtypes = []
    L.cmsvd_create.restype = ctypes.c_int
    L.cmsvd_create.argtypes = [ctypes.c_int, vp, ctypes.POINTER(vp)]
    L.cmsvd_destroy.restype = ctypes.c_int
    L.cmsvd_destroy.argtypes = [vp]
    L.cmsvd_register.restype = ctypes.c_int
    L.cmsvd_register.argtypes = [vp, i64, i32, vp, vp, vp, ctypes.c_int]
    L.cmsvd_block_spectra.restype = ctypes.c_int
    L.cmsvd_block_spectra.argtypes = [vp, i32, vp, vp, vp]
    L.cmsvd_pair_errors.restype = ctypes.c_int
    L.cmsvd_pair_errors.argtypes = [vp, vp, i64, i32, u32, ctypes.c_int, ctypes.c_int, vp, vp, vp, vp]
    L.cmsvd_cluster.restype = ctypes.c_int
    L.cmsvd_pair_errors_tight.argtypes = [vp, vp, i64, i32, ctypes.c_int, ctypes.c_int, vp, vp]
    L.cmsvd_pair_errors_tight.restype = ctypes.c_int
    L.cmsvd_cluster.argtypes = [vp, ctypes.POINTER(ClusterOpts), vp, vp, vp, vp, vp, vp]
    L.cmsvd_sequence_errors.restype = ctypes.c_int
    L.cmsvd_sequence_errors.argtypes = [vp, vp, vp, i32, i32, u32, ctypes.c_int, vp, vp]
    L.cmsvd_cluster_factors.restype = ctypes.c_int
    L.cmsvd_cluster_factors.argtypes = [vp, i32, vp, i32, vp, vp, vp]
    L.cmsvd_cluster_verify.restype = ctypes.c_int
    L.cmsvd_cluster_verify.argtypes = [vp, i32, vp, i32, vp, vp, vp]
    L.cmsvd_cluster_verify_ex.restype = ctypes.c_int
    L.cmsvd_cluster_verify_ex.argtypes = [vp, i32, vp, i32, vp, vp, vp, vp, vp]
    L.cmsvd_sym_eigvals.restype = ctypes.c_int
    L.cmsvd_sym_eigvals.argtypes = [vp, i32, i32, vp, vp, i32, vp, vp]
    L.cmsvd_spectra_diagnostics.restype = ctypes.c_int
    L.cmsvd_spectra_diagnostics.argtypes = [vp, vp, vp]
    L.cmsvd_launch_count.restype = i64
    L.cmsvd_launch_count.argtypes = [vp]
    L.cmsvd_profile_enable.restype = ctypes.c_int
    L.cmsvd_profile_enable.argtypes = [vp, ctypes.c_int]
    L.cmsvd_profile_read.restype = i32
    L.cmsvd_profile_read.argtypes = [vp, i32, ctypes.POINTER(ctypes.c_char_p), vp, vp]
    _lib = L
    return L


def _status_name(s: int) -> str:
    try:
        return load().cmsvd_status_string(s).decode()
    except Exception:
        return f"status {s}"


def _check_tensor(t, name, dtype, shape, device=None):
    """Device-path argument check (a torch tensor's raw pointer goes to the C ABI): dtype, contiguity,
    exact shape and device, so that a mismatched tensor raises instead of being misread or overrun."""
    if t is None:
        raise CmsvdError(E_ARG, f"{name} is required")
    if not hasattr(t, "data_ptr"):
        raise CmsvdError(E_ARG, f"{name}: expected a torch tensor")
    if str(t.dtype) != dtype:
        raise CmsvdError(E_ARG, f"{name}: dtype {t.dtype}, expected {dtype}")
    if tuple(t.shape) != tuple(shape):
        raise CmsvdError(E_SHAPE, f"{name}: shape {tuple(t.shape)}, expected {tuple(shape)}")
    if not t.is_contiguous():
        raise CmsvdError(E_ARG, f"{name}: not contiguous")
    if device is not None and (not t.is_cuda or t.device.index != device):
        raise CmsvdError(E_ARG, f"{name}: on {t.device}, expected cuda:{device}")


def _ptr(a):
    if a is None:
        return None
    if hasattr(a, "data_ptr"):
        return ctypes.c_void_p(a.data_ptr())
    return a.ctypes.data_as(ctypes.c_void_p)


class Context:
    """One cmsvd context = one registered collection on one device/stream."""

    def __init__(self, device: int = 0, stream=None):
        L = load()
        h = ctypes.c_void_p()
        s = L.cmsvd_create(device, ctypes.c_void_p(stream) if stream else None, ctypes.byref(h))
        if s != OK:
            raise CmsvdError(s, "cmsvd_create failed (is a CUDA device visible?)")
        self._h = h
        self._L = L
        self.device = device
        self.count = 0
        self.r = 0

    def _check(self, s):
        if s != OK:
            raise CmsvdError(s, self._L.cmsvd_last_error(self._h).decode())

    def close(self):
        if getattr(self, "_h", None):
            self._L.cmsvd_destroy(self._h)
            self._h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    def __enter__(self):
        return self

    def __exit__(self, *a):
        self.close()

    @property
    def launches(self) -> int:
        return int(self._L.cmsvd_launch_count(self._h))

    def profile(self, enable: bool = True):
        """Reset and enable/disable per-kernel-category CUDA-event timing."""
        self._check(self._L.cmsvd_profile_enable(self._h, 1 if enable else 0))

    def profile_read(self) -> dict:
        """{category: (ms, launch_groups)} accumulated since profile(True)."""
        mx = 64
        names = (ctypes.c_char_p * mx)()
        ms = np.zeros(mx)
        cnt = np.zeros(mx, np.int64)
        k = self._L.cmsvd_profile_read(self._h, mx, names, _ptr(ms), _ptr(cnt))
        return {names[i].decode(): (float(ms[i]), int(cnt[i])) for i in range(k)}

    def spectra_diagnostics(self):
        """(largest Ritz residual, power iterations) of the last big-block (A22) block_spectra."""
        res = ctypes.c_double()
        it = ctypes.c_int32()
        self._check(self._L.cmsvd_spectra_diagnostics(self._h, ctypes.byref(res), ctypes.byref(it)))
        return res.value, it.value

    # -- cmsvd_sym_eigvals (diagnostic) ------------------------------------
    def sym_eigvals(self, mats, kw: int):
        """Top-kw eigenvalues of symmetric matrices (list of n_p x n_p float64 arrays, n_p <= 512) through
        the pair path's batched eigensolver: returns (ev (count, kw) non-increasing, trace (count,))."""
        ns = np.array([m.shape[0] for m in mats], np.int32)
        nmax = int(max(1, ns.max()))
        G = np.zeros((len(mats), nmax, nmax))
        for p, m in enumerate(mats):
            G[p, :m.shape[0], :m.shape[0]] = np.asarray(m, np.float64).T    # column-major
        ev = np.zeros((len(mats), kw))
        tr = np.zeros(len(mats))
        self._check(self._L.cmsvd_sym_eigvals(self._h, len(mats), nmax, _ptr(ns), _ptr(G), int(kw), _ptr(ev),
                                              _ptr(tr)))
        return ev, tr

    # -- cmsvd_register --------------------------------------------------
    def register(self, blocks, where: int | None = None):
        """blocks: (N, n, m) float32 array/tensor (block i column-major), or a
        list of column-major m x n_i arrays (Fortran-ordered numpy or tensors
        holding the transposed (n_i, m) layout)."""
        if hasattr(blocks, "dim") and blocks.dim() == 3:          # torch tensor (N, n, m)
            N, n, m = blocks.shape
            _check_tensor(blocks, "blocks", "torch.float32", (N, n, m), self.device if blocks.is_cuda else None)
            dev = blocks.is_cuda
            base = blocks.data_ptr()
            stride = n * m * 4
            ptrs = [base + i * stride for i in range(N)]
            ns = np.full(N, n, np.int32)
            keep = blocks
        elif isinstance(blocks, np.ndarray) and blocks.ndim == 3:
            blocks = np.ascontiguousarray(blocks, dtype=np.float32)
            N, n, m = blocks.shape
            dev = False
            ptrs = [blocks.ctypes.data + i * n * m * 4 for i in range(N)]
            ns = np.full(N, n, np.int32)
            keep = blocks
        else:
            keep, ptrs, nl = [], [], []
            dev = False
            m = None
            for b in blocks:
                if hasattr(b, "data_ptr"):
                    dev = b.is_cuda
                    nn, mm = b.shape
                    _check_tensor(b, "blocks[i]", "torch.float32", (nn, mm), self.device if dev else None)
                    ptrs.append(b.data_ptr())
                else:
                    f = np.asfortranarray(b, dtype=np.float32)
                    mm, nn = f.shape
                    ptrs.append(f.ctypes.data)
                    b = f
                keep.append(b)
                nl.append(nn)
                m = mm
            N = len(ptrs)
            ns = np.array(nl, np.int32)
        w = (DEVICE if dev else HOST) if where is None else where
        arr = (ctypes.c_void_p * N)(*ptrs)
        self._check(self._L.cmsvd_register(self._h, int(m), int(N), _ptr(ns), arr, None, w))
        del keep
        self.count = N
        self.m = int(m)
        self._ncols = np.asarray(ns, np.int64)
        return self

    # -- cmsvd_block_spectra ---------------------------------------------
    def block_spectra(self, r: int):
        N = self.count
        E = np.zeros(N)
        sig = np.zeros((N, r), np.float32)
        rank = np.zeros(N, np.int32)
        self._check(self._L.cmsvd_block_spectra(self._h, int(r), _ptr(E), _ptr(sig), _ptr(rank)))
        self.r = r
        return E, sig, rank

    # -- cmsvd_pair_errors -----------------------------------------------
    def pair_errors(self, pairs, r: int | None = None, kinds: int = ALL, operand: int = RAW,
                    want_sigma: bool = True, want_mu: bool = True, out=None):
        """Host path: pairs (P,2) int32 numpy -> dict of numpy outputs.
        Device path: pairs as an int32 CUDA tensor and ``out`` a dict of CUDA
        tensors (err2 (P,3) f64, total (P,) f64, sigma_tilde/mu (P,r) f32)."""
        r = self.r if r is None else r
        if hasattr(pairs, "data_ptr") and pairs.is_cuda:
            P = pairs.shape[0]
            _check_tensor(pairs, "pairs", "torch.int32", (P, 2), self.device)
            _check_tensor(out.get("err2"), "out['err2']", "torch.float64", (P, 3), self.device)
            _check_tensor(out.get("total"), "out['total']", "torch.float64", (P,), self.device)
            for k in ("sigma_tilde", "mu"):
                if out.get(k) is not None:
                    _check_tensor(out[k], f"out['{k}']", "torch.float32", (P, r), self.device)
            self._check(self._L.cmsvd_pair_errors(self._h, _ptr(pairs), P, r, kinds, operand, DEVICE,
                                                  _ptr(out["err2"]), _ptr(out["total"]),
                                                  _ptr(out.get("sigma_tilde")), _ptr(out.get("mu"))))
            return out
        pairs = np.ascontiguousarray(pairs, dtype=np.int32).reshape(-1, 2)
        P = pairs.shape[0]
        err2 = np.zeros((P, 3))
        total = np.zeros(P)
        st = np.zeros((P, r), np.float32) if want_sigma else None
        mu = np.zeros((P, r), np.float32) if want_mu else None
        self._check(self._L.cmsvd_pair_errors(self._h, _ptr(pairs), P, r, kinds, operand, HOST, _ptr(err2),
                                              _ptr(total), _ptr(st), _ptr(mu)))
        return {"err2": err2, "total": total, "sigma_tilde": st, "mu": mu}

    # -- cmsvd_pair_errors_tight (N3, beyond the paper) -------------------
    def pair_errors_tight(self, pairs, r: int | None = None, operand: int = RAW):
        """Residual bound with the U_r basis and per-index Weyl bound (host path):
        returns {"err2x": (P, 2) f64 [residual_Ur, weyl_index], "total": (P,) f64}."""
        r = self.r if r is None else r
        pairs = np.ascontiguousarray(pairs, dtype=np.int32).reshape(-1, 2)
        P = pairs.shape[0]
        err2x = np.zeros((P, 2))
        total = np.zeros(P)
        self._check(self._L.cmsvd_pair_errors_tight(self._h, _ptr(pairs), P, r, operand, HOST, _ptr(err2x),
                                                    _ptr(total)))
        return {"err2x": err2x, "total": total}

    # -- cmsvd_sequence_errors (N2) ----------------------------------------
    def sequence_errors(self, seqs, r: int | None = None, kinds: int = ALL, operand: int = RAW):
        """Predicted errors of block sequences (lists of block ids in append order):
        {"err2": (S, 3) [weyl, residual, incremental], "total": (S,)}."""
        r = self.r if r is None else r
        offs = np.zeros(len(seqs) + 1, np.int32)
        offs[1:] = np.cumsum([len(q) for q in seqs])
        ids = np.ascontiguousarray(np.concatenate([np.asarray(q, np.int32) for q in seqs]) if seqs else
                                   np.zeros(0, np.int32), dtype=np.int32)
        e2 = np.zeros((len(seqs), 3))
        tot = np.zeros(len(seqs))
        self._check(self._L.cmsvd_sequence_errors(self._h, _ptr(offs), _ptr(ids), len(seqs), int(r), kinds, operand,
                                                  _ptr(e2), _ptr(tot)))
        return {"err2": e2, "total": tot}

    # -- cmsvd_cluster_factors (N1 codec) ----------------------------------
    def cluster_factors(self, assign, r: int | None = None):
        """Per-cluster factors of the rank-r truncated SVD of each concatenation: a list of
        (members, Ut (m x r_c), V (N_c x r_c)); block i is reconstructed as Ut @ V_i.T."""
        r = self.r if r is None else r
        assign = np.ascontiguousarray(assign, dtype=np.int32)
        nc = int(assign.max()) + 1 if assign.size else 0
        members = [np.flatnonzero(assign == c) for c in range(nc)]
        ncols = [int(np.sum(self._ncols[mb])) for mb in members]
        rcs = [min(r, self.m, n) for n in ncols]
        Ut = np.zeros(sum(self.m * k for k in rcs), np.float32)
        V = np.zeros(sum(n * k for n, k in zip(ncols, rcs)), np.float32)
        rc = np.zeros(nc, np.int32)
        self._check(self._L.cmsvd_cluster_factors(self._h, int(r), _ptr(assign), nc, _ptr(Ut), _ptr(V), _ptr(rc)))
        out, uo, vo = [], 0, 0
        for c in range(nc):
            k = int(rc[c])
            out.append((members[c], Ut[uo:uo + self.m * k].reshape(k, self.m).T,
                        V[vo:vo + ncols[c] * k].reshape(k, ncols[c]).T))
            uo += self.m * k
            vo += ncols[c] * k
        return out

    # -- cmsvd_cluster_verify (N1) -----------------------------------------
    def cluster_verify(self, assign, r: int | None = None):
        """Exact per-cluster rank-r errors of the explicit concatenations and the
        compression accounting: {"exact_err2", "total", "rel", "mem", "ratio"}."""
        r = self.r if r is None else r
        assign = np.ascontiguousarray(assign, dtype=np.int32)
        nc = int(assign.max()) + 1 if assign.size else 0
        e2 = np.zeros(nc)
        tot = np.zeros(nc)
        mem = np.zeros(nc, np.int64)
        rel = np.zeros(nc)
        ratio = ctypes.c_double(float("nan"))
        self._check(self._L.cmsvd_cluster_verify_ex(self._h, int(r), _ptr(assign), nc, _ptr(e2), _ptr(tot),
                                                    _ptr(mem), _ptr(rel), ctypes.byref(ratio)))
        return {"exact_err2": e2, "total": tot, "rel": rel, "mem": mem, "ratio": ratio.value}

    # -- cmsvd_cluster ---------------------------------------------------
    def cluster(self, algorithm: int, eps: float, r: int | None = None, sort: int = SORT_FROBENIUS,
                knn: int = 1, operand: int = RAW):
        r = self.r if r is None else r
        N = self.count
        o = ClusterOpts(algorithm, sort, knn, operand, r, eps)
        assign = np.zeros(N, np.int32)
        order = np.zeros(N, np.int32)
        K = ctypes.c_int32()
        ce = np.zeros(N)
        ct = np.zeros(N)
        ne = ctypes.c_int64()
        self._check(self._L.cmsvd_cluster(self._h, ctypes.byref(o), _ptr(assign), _ptr(order), ctypes.byref(K),
                                          _ptr(ce), _ptr(ct), ctypes.byref(ne)))
        k = K.value
        clusters = [[] for _ in range(k)]
        for b in np.argsort(order, kind="stable"):
            clusters[assign[b]].append(int(b))
        for c in clusters:
            c.sort(key=lambda b: order[b])
        return {"assign": assign, "order": order, "clusters": clusters, "err2": ce[:k], "total": ct[:k],
                "n_evals": ne.value}
