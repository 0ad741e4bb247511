"""The batched fp64 symmetric eigensolver of the core Grams (Lemma 1 / Cor. 3, PAPER.md:1325-1338,
1399-1436) through the diagnostic C-ABI entry cmsvd_sym_eigvals, against LAPACK (numpy eigvalsh) on
random Gram matrices: every size class of the dispatch (n <= 160 register / shared-memory kernels,
160 < n <= 512 the two-stage band reduction, and the one-stage in-place kernel behind CMSVD_EIG_SBR=0),
ragged batches and degenerate sizes.  Householder reduction + bisection are backward stable: the bar
is the bisection's stopping rule (1e-11 relative) plus 1e-12 of the largest eigenvalue."""
import numpy as np
import pytest

pytestmark = pytest.mark.gpu
torch = pytest.importorskip("torch")


@pytest.fixture(scope="module")
def cm():
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    import paper_2601_11626_b200 as cm
    cm.load()
    return cm


def gram(R, n, decay=0.0):
    X = R.standard_normal((n, n + 3)) * (np.arange(1, n + 4) ** -decay)
    return X @ X.T


def check(ev, mats, kw):
    for p, G in enumerate(mats):
        n = G.shape[0]
        if n == 0:
            continue
        ref = np.linalg.eigvalsh(G)[::-1][:kw]
        k = min(kw, n)
        err = np.abs(ev[p, :k] - ref[:k]).max()
        tol = 2e-11 * np.abs(ref[:k]) + 1e-12 * max(abs(ref[0]), 1e-300) * max(1.0, n / 64)
        assert np.all(np.abs(ev[p, :k] - ref[:k]) <= tol), (p, n, err, ref[0])
        assert np.all(np.diff(ev[p, :k]) <= 1e-12 * abs(ref[0]))


@pytest.mark.parametrize("n", [2, 3, 31, 64, 96, 128, 150, 160, 161, 176, 200, 255, 256, 300, 384, 500, 511, 512, 513, 700, 1024])
def test_eigvals_vs_lapack(cm, n):
    R = np.random.default_rng(n)
    mats = [gram(R, n), gram(R, n, decay=1.0)]
    kw = min(n, 128)
    with cm.Context(0) as ctx:
        ev, tr = ctx.sym_eigvals(mats, kw)
    check(ev, mats, kw)
    assert np.allclose(tr, [np.trace(G) for G in mats], rtol=1e-12)


@pytest.mark.parametrize("sbr", ["1", "0"])
def test_ragged_large_batch(cm, sbr, monkeypatch):
    """Ragged sizes in one launch (the pair path's nG = r'_i + w_j varies per pair), both large-n kernels."""
    monkeypatch.setenv("CMSVD_EIG_SBR", sbr)
    R = np.random.default_rng(7)
    sizes = [512, 300, 161, 17, 0, 450, 256, 512, 333, 1]
    mats = [gram(R, n, decay=0.5) if n else np.zeros((0, 0)) for n in sizes]
    with cm.Context(0) as ctx:
        ev, _ = ctx.sym_eigvals(mats, 256)
    check(ev, mats, 256)


def test_structured_spectra(cm):
    """Repeated and zero eigenvalues (rank-deficient Grams), a diagonal matrix (already tridiagonal) and a
    matrix that is already banded: the reduction must leave their eigenvalues exact to rounding."""
    R = np.random.default_rng(11)
    n = 400
    Q = np.linalg.qr(R.standard_normal((n, n)))[0]
    d = np.concatenate([np.full(50, 9.0), np.full(50, 4.0), np.linspace(3, 1, 200), np.zeros(100)])
    A = (Q * d) @ Q.T
    A = 0.5 * (A + A.T)
    D = np.diag(np.linspace(5, 1, 300))
    Bnd = np.triu(np.tril(gram(R, 260), 16), -16)
    with cm.Context(0) as ctx:
        ev, _ = ctx.sym_eigvals([A, D, Bnd], 200)
    check(ev, [A, D, Bnd], 200)
    assert np.allclose(ev[0, :50], 9.0, atol=1e-12 * 9) and np.allclose(ev[0, 50:100], 4.0, atol=1e-12 * 9)


@pytest.mark.parametrize("knob", ["", "CMSVD_SBR_FUSED=1", "CMSVD_SYMM_DMMA=0", "CMSVD_SYR2K_DMMA=0", "CMSVD_SYR2K_ROW=0",
                                  "CMSVD_SYMM_DMMA=0,CMSVD_SYR2K_DMMA=0,CMSVD_SYR2K_ROW=1", "CMSVD_CHASE2=1",
                                  "CMSVD_CHASE_FLAGS=1", "CMSVD_SBR_TMA=0", "CMSVD_SBR_PANEL_RR=0", "CMSVD_BISECT_P=0"])
def test_band_reduction_variants(cm, knob, monkeypatch):
    """Every selectable path of the two-stage reduction agrees with LAPACK on ragged sizes (including the
    global-memory panel / band above 512): the default (stage 1 on the fp64 tensor cores: DMMA product and
    row-persistent DMMA update), the scalar product / update kernels, the one-tile-per-CTA and row-persistent
    scalar updates, the look-ahead fused pass, the chase with per-sweep flags or with two problems in flight
    per CTA over the circular band buffer, the non-TMA staging, and the shared-memory panel QR (the default
    panel kernel keeps the panel in registers), and the pivot-form bisection with its fp32 coarse phase (the
    default is the division-free polynomial recurrence)."""
    for kv in filter(None, knob.split(",")):
        k, v = kv.split("=")
        monkeypatch.setenv(k, v)
    R = np.random.default_rng(31)
    sizes = [512, 400, 161, 257, 640]
    mats = [gram(R, n, decay=0.4) for n in sizes]
    with cm.Context(0) as ctx:
        ev, _ = ctx.sym_eigvals(mats, 160)
    check(ev, mats, 160)


@pytest.mark.parametrize("split", ["1", "0"])
def test_chase_split_boundaries(cm, split, monkeypatch):
    """256 < nmax <= 512: the chase runs sweeps 0 .. nmax - 257 on the full band and hands the trailing band
    matrix (written back into the lower storage) to the half-band kernel.  Sizes around the hand-over: problems
    that phase A finishes alone (n - 2 <= J), a trailing matrix of 3 rows (one sweep), one window step more,
    and the full size; nmax = 500 moves J off a multiple of the band width."""
    monkeypatch.setenv("CMSVD_CHASE_SPLIT", split)
    R = np.random.default_rng(47)
    for sizes in ([512, 259, 258, 257, 260, 273, 274, 290, 511, 3, 2, 0], [500, 245, 246, 247, 248, 263, 499, 300]):
        mats = [gram(R, n, decay=0.4) if n else np.zeros((0, 0)) for n in sizes]
        with cm.Context(0) as ctx:
            ev, tr = ctx.sym_eigvals(mats, 200)
        check(ev, mats, 200)


@pytest.mark.parametrize("groups", ["1", "3"])
def test_pipelined_groups_bitwise(cm, groups, monkeypatch):
    """CMSVD_SBR_GROUPS: the batch cut into groups whose chase + bisection run on a second stream under the
    next group's stage 1.  Same kernels per problem: the eigenvalues are bitwise those of the one-stream path
    (and within the LAPACK bar), on a ragged batch large enough for three groups (>= 2 x SM count each)."""
    R = np.random.default_rng(43)
    base = [300, 161, 256, 0, 200, 257, 170, 3]
    nsm = torch.cuda.get_device_properties(0).multi_processor_count
    sizes = (base * ((6 * nsm + 40) // len(base) + 1))[:6 * nsm + 37]
    protos = {n: (gram(R, n, decay=0.3) if n else np.zeros((0, 0))) for n in set(sizes)}
    mats = [protos[n] for n in sizes]
    monkeypatch.setenv("CMSVD_SBR_GROUPS", "1")
    with cm.Context(0) as ctx:
        ev1, tr1 = ctx.sym_eigvals(mats, 64)
    monkeypatch.setenv("CMSVD_SBR_GROUPS", groups)
    with cm.Context(0) as ctx:
        ev, tr = ctx.sym_eigvals(mats, 64)
        ev_b, _ = ctx.sym_eigvals(mats, 64)   # second call on the same context: streams and events reused
    assert np.array_equal(ev, ev1) and np.array_equal(tr, tr1) and np.array_equal(ev_b, ev1)
    check(ev[:len(base)], mats[:len(base)], 64)


def test_chase_two_in_flight_queue(cm, monkeypatch):
    """CMSVD_CHASE2=1 with more problems than SMs: every persistent CTA walks a queue of ragged problems
    through the circular band buffer (offsets 0, n_A, n_A + n_B mod 768, ...: column wrap inside a problem,
    early write-out of the finished columns before they are overwritten, empty and tiny problems in the
    queue).  Same bar as the default path."""
    monkeypatch.setenv("CMSVD_CHASE2", "1")
    R = np.random.default_rng(41)
    base = [512, 161, 400, 0, 512, 257, 200, 3, 333, 512, 170, 2, 480, 1]
    sizes = (base * 32)[:420]
    protos = {n: (gram(R, n, decay=0.3) if n else np.zeros((0, 0))) for n in set(sizes)}
    # distinct matrices per problem (scaled copies keep the LAPACK reference cheap)
    scale = 1.0 + 0.01 * np.arange(len(sizes))
    mats = [protos[n] * scale[i] for i, n in enumerate(sizes)]
    with cm.Context(0) as ctx:
        ev, _ = ctx.sym_eigvals(mats, 64)
    refs = {n: (np.linalg.eigvalsh(protos[n])[::-1][:64] if n else np.zeros(0)) for n in protos}
    for i, n in enumerate(sizes):
        k = min(64, n)
        if k == 0:
            continue
        ref = refs[n][:k] * scale[i]
        tol = 2e-11 * np.abs(ref) + 1e-12 * abs(ref[0]) * max(1.0, n / 64)
        assert np.all(np.abs(ev[i, :k] - ref) <= tol), (i, n, np.abs(ev[i, :k] - ref).max())


@pytest.mark.parametrize("colbt,qlf", [("1", "1"), ("0", "1"), ("1", "0"), ("0", "0")])
def test_syev_inplace_variants(cm, colbt, qlf, monkeypatch):
    """k_syev_ql<true> (160 < n <= 512, Z in place in global memory): the column-resident back-transformation
    and the fused four-sweep QL pass, and their one-at-a-time forms (CMSVD_SYEV_COLBT=0, CMSVD_SYEV_QLF=0),
    through the N1 codec (cmsvd_cluster_factors on a 300-column cluster, Thm EYM): the
    reconstruction from the returned factors has exactly the rank-r tail energy that LAPACK's singular
    values of the explicit concatenation give, and V has orthonormal columns."""
    monkeypatch.setenv("CMSVD_SYEV_COLBT", colbt)
    monkeypatch.setenv("CMSVD_SYEV_QLF", qlf)
    R = np.random.default_rng(300)
    m, n, r = 600, 150, 40
    dec = np.exp(-0.03 * np.arange(2 * n))
    X = (np.linalg.qr(R.standard_normal((m, 2 * n)))[0] * dec) @ np.linalg.qr(R.standard_normal((2 * n, 2 * n)))[0]
    blocks = np.ascontiguousarray(np.stack([X[:, :n].T, X[:, n:].T, R.standard_normal((n, m))]), dtype=np.float32)
    with cm.Context(0) as ctx:
        ctx.register(blocks)
        ctx.block_spectra(r)
        fac = ctx.cluster_factors(np.array([0, 0, 1], np.int32))
    members, Ut, V = fac[0]
    assert list(members) == [0, 1]
    X32 = np.concatenate([blocks[0].T, blocks[1].T], axis=1).astype(np.float64)
    s = np.linalg.svd(X32, compute_uv=False)
    tail = float(np.sum(s[r:] ** 2))
    Xh = Ut.astype(np.float64) @ V.astype(np.float64).T
    err2 = float(np.sum((X32 - Xh) ** 2))
    assert abs(err2 - tail) <= 1e-4 * tail + 1e-9 * float(np.sum(s ** 2)), (err2, tail)
    G = V.astype(np.float64).T @ V.astype(np.float64)
    assert np.allclose(G, np.eye(G.shape[0]), atol=1e-5)
