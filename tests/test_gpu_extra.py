"""GPU parity for SURVEY §8f: the reference's diagnostics on the device (row f1), solve_sqrt +
hpd_sqrt (row f2) and the pencil oracle solve_reference (row f3), each against the CPU oracle
(oracle/, the LAPACK restatement pinned to the reference's KATs) and numpy on the same inputs.

Tolerances: eigenvalues relative 1e-10 vs the oracle's same method (the squared SQRT method on
well-conditioned config-2 inputs; the direct pencil everywhere); residuals <= 100 n eps;
diagnostics to 1e-12 relative of numpy's value on the same arrays.
"""
import numpy as np
import pytest

import oracle
import paper_2008_08825_b200 as bse
from paper_2008_08825_b200 import configs
from tests.helpers import EPS, norm_h, residual, sigma_orthogonality_error, vector_phase_errors

pytestmark = pytest.mark.gpu
RNG = np.random.default_rng(2008)


def crand(*shape):
    return RNG.standard_normal(shape) + 1j * RNG.standard_normal(shape)


def assert_solution(a, b, r, ref_lam, lam_tol=1e-10):
    n = a.shape[0]
    assert r.lambda_.shape == (n,) and r.v.shape == (2 * n, n)
    assert np.all(np.isfinite(r.lambda_)) and np.all(np.isfinite(r.v))
    assert np.all(np.diff(r.lambda_) >= 0) and r.lambda_[0] > 0
    keep = np.setdiff1d(np.arange(n), r.near_singular)
    res = residual(a, b, r.lambda_[keep], r.v[:, keep])
    assert res.max() <= 100 * n * EPS, res.max()
    err = np.max(np.abs(r.lambda_ - ref_lam) / np.abs(ref_lam))
    assert err <= lam_tol, err


# ------------------------------------------------------------------ row f2: SQRT + hpd_sqrt
@pytest.mark.parametrize("n", [1, 2, 7, 33, 64, 65, 100, 129, 200])
def test_solve_sqrt_parity(n):
    a, b = configs.config2(3, n=n)
    r = bse.solve_sqrt(bse.from_blocks(a, b))
    lo, vo, nso = oracle.solve("sqrt", a, b)
    assert r.method == bse.Method.Sqrt
    assert_solution(a, b, r, lo)
    assert r.near_singular == list(nso)
    errs, bounds, sep = vector_phase_errors(r.v, vo, r.lambda_, norm_h(a, b))
    assert np.all(errs[sep] <= np.maximum(bounds[sep], 1e-10))
    assert sigma_orthogonality_error(r.v) <= 1e-9


def test_solve_sqrt_config1_real():
    a, b = configs.config1(0)
    r = bse.solve(bse.Method.Sqrt, bse.from_blocks(a, b))
    lo, _, _ = oracle.solve("sqrt", a, b)
    assert_solution(a, b, r, lo)


@pytest.mark.parametrize("n", [1, 3, 64, 65, 150])
def test_hpd_sqrt(n):
    x = crand(n, n)
    m = x @ x.conj().T + n * np.eye(n)
    s = bse.hpd_sqrt(m)
    assert np.array_equal(s, s.conj().T)  # hermitized exactly (backend.cpp:104-105)
    assert np.linalg.norm(s @ s - m) <= 100 * n * EPS * np.linalg.norm(m)
    w = np.linalg.eigvalsh(s)
    assert w.min() > 0
    w_ref, q = np.linalg.eigh(m)
    s_ref = (q * np.sqrt(w_ref)) @ q.conj().T
    assert np.linalg.norm(s - s_ref) <= 1e3 * n * EPS * np.linalg.norm(s_ref)


def test_hpd_sqrt_not_positive_definite():
    """backend.cpp:93-101: first eigenvalue at or below eps * lambda_max, with its index."""
    m = np.diag([1.0, 1e-20, 2.0, -1.0]).astype(complex)
    with pytest.raises(bse.NotPositiveDefinite) as e:
        bse.hpd_sqrt(m)
    assert e.value.pivot_index == 0  # ascending eigenvalues: -1 comes first
    with pytest.raises(bse.NotPositiveDefinite) as e:
        bse.hpd_sqrt(np.diag([1.0, 1e-20, 2.0]).astype(complex))
    assert e.value.pivot_index == 0


def test_solve_sqrt_error_payloads():
    # A-B passes the Cholesky certificate but its square root fails (solvers.cpp:96-101)
    a = np.diag([3.0, 2e-20]).astype(complex)  # A+B = diag(5, 3e-20), A-B = diag(1, 1e-20)
    b = np.diag([2.0, 1e-20]).astype(complex)
    with pytest.raises(bse.NotDefinite) as e:
        bse.solve_sqrt(bse.from_blocks(a, b))
    assert e.value.which == bse.Block.M2
    assert str(e.value).startswith("square root of A-B failed")
    # certificate order: A+B first (core.cpp:89-99)
    with pytest.raises(bse.NotDefinite) as e:
        bse.solve_sqrt(bse.from_blocks(np.eye(2), 2 * np.eye(2)))
    assert e.value.which == bse.Block.M2
    with pytest.raises(bse.NotDefinite) as e:
        bse.solve_sqrt(bse.from_blocks(-np.eye(2), 0.5 * np.eye(2)))
    assert e.value.which == bse.Block.M1


# ------------------------------------------------------------------ row f3: pencil oracle
@pytest.mark.parametrize("n", [1, 2, 7, 33, 64, 65, 100, 129])
def test_solve_reference_parity(n):
    a, b = configs.config2(5, n=n)
    r = bse.solve_reference(bse.from_blocks(a, b))
    lo, vo, _ = oracle.solve("reference", a, b)
    assert r.method == bse.Method.Reference and r.near_singular == []
    assert_solution(a, b, r, lo)
    errs, bounds, sep = vector_phase_errors(r.v, vo, r.lambda_, norm_h(a, b))
    assert np.all(errs[sep] <= np.maximum(bounds[sep], 1e-10))
    # the pencil normalisation: v^H Sigma v = +1 (solvers.cpp:203-208)
    assert sigma_orthogonality_error(r.v) <= 1e-9


def test_reference_agrees_with_chol_and_svd():
    a, b = configs.config2(11, n=96)
    h = bse.from_blocks(a, b)
    lr = bse.solve_reference(h).lambda_
    for m in (bse.Method.Chol, bse.Method.CholSvd, bse.Method.Sqrt):
        assert np.max(np.abs(bse.solve(m, h).lambda_ - lr) / lr) <= 1e-10


def test_reference_certificates():
    with pytest.raises(bse.NotDefinite) as e:
        bse.solve_reference(bse.from_blocks(np.eye(3), 2 * np.eye(3)))
    assert e.value.which == bse.Block.M2


# ------------------------------------------------------------------ row f1: diagnostics
@pytest.mark.parametrize("n,k", [(1, 1), (5, 3), (64, 64), (65, 40), (130, 130)])
def test_residual_matches_numpy(n, k):
    a, b = configs.config2(7, n=n)
    h = bse.from_blocks(a, b)
    v = crand(2 * n, k)
    lam = np.sort(RNG.uniform(0.5, 3.0, k))
    got = bse.residual(h, bse.SpectralResult(lam, v, bse.Method.Chol, []))
    hv_top = a @ v[:n] + b @ v[n:]
    hv_bot = -(b @ v[:n]) - a @ v[n:]
    want = np.sqrt(np.sum(np.abs(hv_top - lam * v[:n]) ** 2, axis=0) +
                   np.sum(np.abs(hv_bot - lam * v[n:]) ** 2, axis=0)) / norm_h(a, b)
    assert np.allclose(got, want, rtol=1e-12, atol=0)


def test_residual_of_a_solution():
    a, b = configs.config2(1, n=120)
    h = bse.from_blocks(a, b)
    r = bse.solve_chol(h)
    res = bse.residual(h, r)
    assert res.shape == (120,) and res.max() <= 100 * 120 * EPS
    with pytest.raises(bse.DimensionMismatch):
        bse.residual(h, bse.SpectralResult(r.lambda_[:3], r.v, r.method, []))


@pytest.mark.parametrize("rows,k", [(2, 1), (10, 4), (128, 64), (130, 130)])
def test_sigma_orthogonality_matches_numpy(rows, k):
    v = crand(rows, k)
    h = rows // 2
    g = v.conj().T @ np.concatenate([v[:h], -v[h:]])
    want = np.linalg.norm(g - np.eye(k))
    assert abs(bse.sigma_orthogonality_error(v) - want) <= 1e-12 * want


def test_sigma_orthogonality_of_a_solution_and_errors():
    a, b = configs.config2(2, n=100)
    r = bse.solve_chol_svd(bse.from_blocks(a, b))
    assert bse.sigma_orthogonality_error(r.v) <= 1e-10
    with pytest.raises(bse.OddDimension):
        bse.sigma_orthogonality_error(crand(5, 2))


def test_check_forms():
    a, b = configs.config2(4, n=40)
    hm = np.block([[a, b], [-b, -a]])  # H of the residual (verify.cpp:84-86), A, B Hermitian
    assert bse.check_form1(hm, 1e-12)
    pert = hm.copy()
    pert[0, 1] += 1e-3
    assert not bse.check_form1(pert, 1e-12)
    # form II uses the transpose in the J condition: a real BSE matrix satisfies both
    ar, br = configs.config1(0)
    hr = np.block([[ar, br], [-br, -ar]]).astype(complex)
    assert bse.check_form1(hr, 1e-12) and bse.check_form2(hr, 1e-12)
    with pytest.raises(bse.OddDimension):
        bse.check_form1(crand(3, 3), 1e-12)
    with pytest.raises(bse.DimensionMismatch):
        bse.check_form2(crand(4, 2), 1e-12)


def test_check_form_matches_reference_formula():
    """verify.cpp:46-68 restated with numpy on random (non-BSE) matrices near the threshold."""
    n = 6
    for trial in range(6):
        m = crand(2 * n, 2 * n)
        J = np.block([[np.zeros((n, n)), np.eye(n)], [-np.eye(n), np.zeros((n, n))]])
        S = np.diag(np.r_[np.ones(n), -np.ones(n)])
        norm = np.linalg.norm(m)
        for form, x in ((1, m.conj().T), (2, m.T)):
            dj = np.linalg.norm(J @ x @ J - m)
            ds = np.linalg.norm(S @ m.conj().T @ S - m)
            tol = max(dj, ds) / norm * (1.0 + 1e-9)  # just accepts
            assert bse._check_form(form, m, tol, None)
            assert not bse._check_form(form, m, 0.999 * max(dj, ds) / norm, None)


def test_negative_spectrum_device():
    lam = np.array([1.0, 2.0])
    v = np.arange(8, dtype=complex).reshape(4, 2) * (1 + 0.5j)
    h = bse.BseMatrixI(np.eye(2, dtype=complex), np.zeros((2, 2), complex))
    neg = bse.negative_spectrum(h, bse.SpectralResult(lam, v, bse.Method.Chol, [1]))
    assert np.array_equal(neg.lambda_, -lam)
    assert np.array_equal(neg.v[:2], v[2:]) and np.array_equal(neg.v[2:], v[:2])
    assert neg.near_singular == [1] and neg.method == bse.Method.Chol


def test_negative_spectrum_of_a_solution_pairs():
    a, b = configs.config2(9, n=80)
    h = bse.from_blocks(a, b)
    r = bse.solve_chol(h)
    neg = bse.negative_spectrum(h, r)
    res = bse.residual(h, neg)
    assert res.max() <= 100 * 80 * EPS
    assert bse.check_pairing(r.lambda_, neg.lambda_, 1e-14)
    with pytest.raises(bse.LengthMismatch):
        bse.check_pairing(r.lambda_, neg.lambda_[:3], 1e-14)


def test_predicted_error_formula():
    """verify.cpp:108-114."""
    e = bse.machine_eps()
    assert bse.predicted_error(10.0, 0.5, 0.5) == e * 10.0 / 0.5
    assert bse.predicted_error(10.0, 0.5, 0.5, squared_method=True) == e * 20.0 * min(20.0, 1 / np.sqrt(e))


def test_device_diagnostics_through_torch_buffers():
    """bse_residual_device / bse_sigma_orthogonality_error_device on device-resident data
    (the at-scale validation path of tools/big_check.py), against the host-pointer versions."""
    torch = pytest.importorskip("torch")
    a, b = configs.config2(13, n=300)
    h = bse.from_blocks(a, b)
    r = bse.solve_chol(h)
    dev = torch.device("cuda", 0)
    da = torch.from_numpy(np.ascontiguousarray(h.a.T)).to(dev)
    db = torch.from_numpy(np.ascontiguousarray(h.b.T)).to(dev)
    dv = torch.from_numpy(np.ascontiguousarray(r.v.T)).to(dev)
    dl = torch.from_numpy(r.lambda_.copy()).to(dev)
    out = torch.empty(300, dtype=torch.float64, device=dev)
    bse.residual_device(300, da.data_ptr(), db.data_ptr(), 300, dl.data_ptr(), dv.data_ptr(),
                        out.data_ptr())
    assert np.array_equal(out.cpu().numpy(), bse.residual(h, r))  # deterministic, same kernels
    s = bse.sigma_orthogonality_error_device(600, 300, dv.data_ptr())
    assert s == bse.sigma_orthogonality_error(r.v)


# ------------------------------------------------- streamed output into page-locked host memory
@pytest.mark.parametrize("method", [bse.Method.Chol, bse.Method.CholSvd])
@pytest.mark.parametrize("n", [700, 1500])
def test_pinned_output_streams_same_solution(method, n):
    """bse_solve into page-locked buffers copies V in column chunks while the recovery stage
    is still running (solvers.cu sink_columns); the result must match the pageable path."""
    import ctypes

    import torch

    a, b = configs.config2(5, n=n)
    ref = bse.solve(method, bse.from_blocks(a, b))  # numpy (pageable) output path
    ha = torch.from_numpy(np.asfortranarray(a).T.copy()).pin_memory()
    hb = torch.from_numpy(np.asfortranarray(b).T.copy()).pin_memory()
    hv = torch.full((n, 2 * n), complex("nan"), dtype=torch.complex128).pin_memory()
    hl = torch.empty(n, dtype=torch.float64).pin_memory()
    ctx = bse.default_context()
    lib = bse._lib.lib()
    st = bse.Status()
    ns = np.zeros(n, dtype=np.int64)
    nn = ctypes.c_int64(0)
    rc = lib.bse_solve(ctx.handle, int(method), n, ctypes.c_void_p(ha.data_ptr()), n,
                       ctypes.c_void_p(hb.data_ptr()), n, ctypes.c_void_p(hl.data_ptr()),
                       ctypes.c_void_p(hv.data_ptr()), 2 * n, ns.ctypes.data_as(ctypes.c_void_p),
                       ctypes.byref(nn), ctypes.byref(st))
    assert rc == 0, st.message
    lam = hl.numpy()
    v = hv.numpy().T  # (2n, n) column-major view
    assert np.array_equal(lam, ref.lambda_)
    assert np.all(np.isfinite(v))
    scale = np.abs(ref.v).max()
    assert np.abs(v - ref.v).max() <= 1e-9 * scale
    res = residual(a, b, lam, v)
    assert res.max() <= 100 * n * EPS


# ------------------------------------------------------------- batch driver
@pytest.mark.parametrize("lanes", [1, 2, 4])
@pytest.mark.parametrize("method", [bse.Method.Chol, bse.Method.CholSvd])
def test_solve_batched_matches_single_solves(method, lanes):
    """One lane runs the single-solve kernels: bit-identical. With L lanes the cooperative
    panel kernels run on 1/L of the SMs, which changes the partial-sum order of the
    reductions: equal to rounding, and every item still meets the residual bound."""
    ctx = bse.Context(0)
    ctx.set_batch_lanes(lanes)
    sizes = ((0, 150), (1, 150), (2, 150), (3, 150), (4, 150))
    hs = [bse.from_blocks(*configs.config2(s, n=n)) for s, n in sizes]
    out = bse.solve_batched(method, hs, ctx=ctx)
    assert len(out) == len(hs)
    for h, r in zip(hs, out):
        one = bse.solve(method, h)
        if lanes == 1:
            assert np.array_equal(r.lambda_, one.lambda_)
            assert np.array_equal(r.v, one.v)
        else:
            assert np.max(np.abs(r.lambda_ - one.lambda_) / one.lambda_) <= 1e-13
            assert np.abs(r.v - one.v).max() <= 1e-10 * np.abs(one.v).max()
        assert residual(h.a, h.b, r.lambda_, r.v).max() <= 100 * h.n * EPS
        assert r.near_singular == one.near_singular and r.method == method
    ctx.close()


def test_solve_batched_device_lanes():
    """bse_solve_batched_device on HBM-resident items equals bse_solve_device per item (one
    lane: bit-identical; two lanes: to rounding, residual-checked)."""
    import torch

    n, k = 300, 4
    dev = torch.device("cuda", 0)
    mats = [configs.config2(20 + s, n=n) for s in range(k)]
    da = [torch.from_numpy(a.T.copy()).to(dev) for a, _ in mats]
    db = [torch.from_numpy(b.T.copy()).to(dev) for _, b in mats]
    ref = []
    for i in range(k):
        lam = torch.empty(n, dtype=torch.float64, device=dev)
        v = torch.empty((n, 2 * n), dtype=torch.complex128, device=dev)
        bse.solve_device(bse.Method.Chol, n, da[i].data_ptr(), db[i].data_ptr(), lam.data_ptr(),
                         v.data_ptr())
        ref.append((lam.cpu().numpy(), v.cpu().numpy().T))
    for lanes in (1, 2):
        ctx = bse.Context(0)
        ctx.set_batch_lanes(lanes)
        lams = [torch.empty(n, dtype=torch.float64, device=dev) for _ in range(k)]
        vs = [torch.empty((n, 2 * n), dtype=torch.complex128, device=dev) for _ in range(k)]
        flags = bse.solve_batched_device(bse.Method.Chol, n, [x.data_ptr() for x in da],
                                         [x.data_ptr() for x in db], [x.data_ptr() for x in lams],
                                         [x.data_ptr() for x in vs], ctx=ctx)
        assert flags == [[]] * k
        for i in range(k):
            lam, v = lams[i].cpu().numpy(), vs[i].cpu().numpy().T
            if lanes == 1:
                assert np.array_equal(lam, ref[i][0]) and np.array_equal(v, ref[i][1])
            else:
                assert np.max(np.abs(lam - ref[i][0]) / ref[i][0]) <= 1e-13
                assert residual(mats[i][0], mats[i][1], lam, v).max() <= 100 * n * EPS
        ctx.close()
    for bad in (0, 9):
        with pytest.raises(bse.InvalidSpec):
            bse.default_context().set_batch_lanes(bad)


def test_solve_batched_reports_failing_item():
    n = 40
    good = bse.from_blocks(*configs.config2(4, n=n))
    a = np.eye(n, dtype=complex)
    bad = bse.from_blocks(a, 2 * a)  # A - B = -I: M2 not definite
    with pytest.raises(bse.BatchError) as ei:
        bse.solve_batched(bse.Method.Chol, [good, bad, good])
    assert ei.value.index == 1
    assert isinstance(ei.value.error, bse.NotDefinite)
    assert ei.value.error.which == bse.Block.M2
    assert len(ei.value.results) == 1
    assert np.allclose(ei.value.results[0].lambda_, bse.solve_chol(good).lambda_, rtol=1e-13, atol=0)
    with pytest.raises(bse.DimensionMismatch):
        bse.solve_batched(bse.Method.Chol, [good, bse.from_blocks(*configs.config2(0, n=30))])
    assert bse.solve_batched(bse.Method.Chol, []) == []


def test_solve_batched_pinned_overlap():
    """Page-locked batch: uploads/downloads overlap the solves; results equal single solves."""
    import ctypes

    import torch

    n, k = 1100, 3
    hs = [bse.from_blocks(*configs.config2(10 + s, n=n)) for s in range(k)]
    mats = [(h.a, h.b) for h in hs]
    pin = lambda x: torch.from_numpy(np.asfortranarray(x).T.copy()).pin_memory()  # noqa: E731
    ha = [pin(a) for a, _ in mats]
    hb = [pin(b) for _, b in mats]
    hv = [torch.empty((n, 2 * n), dtype=torch.complex128).pin_memory() for _ in range(k)]
    hl = [torch.empty(n, dtype=torch.float64).pin_memory() for _ in range(k)]
    arr = lambda ts: (ctypes.c_void_p * k)(*[t.data_ptr() for t in ts])  # noqa: E731
    st = bse.Status()
    failed = ctypes.c_int64(0)
    ns = np.zeros((k, n), dtype=np.int64)
    nn = np.zeros(k, dtype=np.int64)
    rc = bse._lib.lib().bse_solve_batched(
        bse.default_context().handle, int(bse.Method.Chol), n, k, arr(ha), n, arr(hb), n, arr(hl),
        arr(hv), 2 * n, ns.ctypes.data_as(ctypes.c_void_p), nn.ctypes.data_as(ctypes.c_void_p),
        ctypes.byref(failed), ctypes.byref(st))
    assert rc == 0, st.message
    assert failed.value == -1
    for i, h in enumerate(hs):
        one = bse.solve_chol(h)  # default two lanes: equal to rounding (see above)
        assert np.max(np.abs(hl[i].numpy() - one.lambda_) / one.lambda_) <= 1e-13
        assert residual(h.a, h.b, hl[i].numpy(), hv[i].numpy().T).max() <= 100 * n * EPS


@pytest.mark.parametrize("method", [bse.Method.Chol, bse.Method.CholSvd])
def test_both_blocks_indefinite_reports_m1(method):
    """core.cpp:89-99 certifies M1 before M2; CHOL derives the M1 certificate from the
    spectrum of L^H M1 L but must still report M1 first when both fail."""
    n = 12
    a = -np.eye(n, dtype=complex)
    with pytest.raises(bse.NotDefinite) as e:
        bse.solve(method, bse.from_blocks(a, np.zeros((n, n))))
    assert e.value.which == bse.Block.M1
    assert "leading minor of order 1 " in str(e.value)


# ------------------------------------------------------ large solves through device diagnostics
@pytest.mark.parametrize("method", [bse.Method.Chol, bse.Method.CholSvd])
def test_large_solve_device_residual(method):
    """n = 3072 through bse_solve_device, checked with the device residual.
    Regression: CHOL+SVD factors A+B and A-B concurrently on two streams, so the CTAs of one
    Cholesky panel launch need not be co-resident; the panel kernel must not overwrite the
    diagonal block before its last CTA has read it (potrf.cu). Three repetitions because
    that race depended on scheduling."""
    import torch

    n = 3072
    a, b = configs.config2(0, n=n)
    dev = torch.device("cuda", 0)
    da = torch.from_numpy(a.T.copy()).to(dev)
    db = torch.from_numpy(b.T.copy()).to(dev)
    lam = torch.empty(n, dtype=torch.float64, device=dev)
    v = torch.empty((n, 2 * n), dtype=torch.complex128, device=dev)
    res = torch.empty(n, dtype=torch.float64, device=dev)
    ref = None
    for _ in range(3):
        flags = bse.solve_device(method, n, da.data_ptr(), db.data_ptr(), lam.data_ptr(),
                                 v.data_ptr())
        assert flags == []
        bse.residual_device(n, da.data_ptr(), db.data_ptr(), n, lam.data_ptr(), v.data_ptr(),
                            res.data_ptr())
        assert res.max().item() <= 100 * n * EPS
        got = lam.cpu().numpy()
        if ref is None:
            ref = got
        assert np.array_equal(got, ref)  # bit-deterministic run to run


def test_solve_batched_edge_cases():
    """Batch driver corner cases: one item on a multi-lane context, tiny sizes, several
    failing items in different lanes (the first one is reported), lanes > items."""
    ctx = bse.Context(0)
    ctx.set_batch_lanes(4)
    one = bse.from_blocks(np.array([[2.0]]), np.array([[1.0]]))
    r = bse.solve_batched(bse.Method.CholSvd, [one], ctx=ctx)
    assert len(r) == 1 and abs(r[0].lambda_[0] - np.sqrt(3.0)) < 1e-13
    hs = [bse.from_blocks(*configs.config2(s, n=65)) for s in range(6)]
    out = bse.solve_batched(bse.Method.Chol, hs, ctx=ctx)
    for h, x in zip(hs, out):
        assert residual(h.a, h.b, x.lambda_, x.v).max() <= 100 * 65 * EPS
    good = hs[0]
    bad = bse.from_blocks(np.eye(65, dtype=complex), 2 * np.eye(65, dtype=complex))
    with pytest.raises(bse.BatchError) as ei:
        bse.solve_batched(bse.Method.Chol, [good, good, bad, bad, good], ctx=ctx)
    assert ei.value.index == 2 and len(ei.value.results) == 2
    ctx.close()


@pytest.mark.parametrize("pad", [0, 3])
def test_solve_batched_pinned_outputs_stream_same_bits(pad):
    """bse_solve_batched into page-locked V buffers downloads each item with the L2-streaming
    copy kernel (zcopy2d_to_host_streaming) instead of the copy engine; pageable outputs take
    cudaMemcpy2DAsync. Same lanes, same solves: the outputs must be bit-identical, also with a
    padded leading dimension (ldv = 2n + pad)."""
    import ctypes

    import torch

    n, k = 300, 4
    ctx = bse.Context(0)
    ctx.set_batch_lanes(2)
    hs = [bse.from_blocks(*configs.config2(40 + s, n=n)) for s in range(k)]
    ref = bse.solve_batched(bse.Method.Chol, hs, ctx=ctx)
    ldv = 2 * n + pad
    hv = [torch.zeros((n, ldv), dtype=torch.complex128).pin_memory() for _ in range(k)]
    hl = [torch.zeros(n, dtype=torch.float64).pin_memory() for _ in range(k)]
    arr = lambda ptrs: (ctypes.c_void_p * k)(*ptrs)  # noqa: E731
    ns = np.zeros((k, n), dtype=np.int64)
    nn = np.zeros(k, dtype=np.int64)
    failed = ctypes.c_int64(-1)
    st = bse.Status()
    rc = bse._lib.lib().bse_solve_batched(
        ctx.handle, int(bse.Method.Chol), n, k, arr([h.a.ctypes.data for h in hs]), n,
        arr([h.b.ctypes.data for h in hs]), n, arr([t.data_ptr() for t in hl]),
        arr([t.data_ptr() for t in hv]), ldv, ns.ctypes.data_as(ctypes.c_void_p),
        nn.ctypes.data_as(ctypes.c_void_p), ctypes.byref(failed), ctypes.byref(st))
    assert rc == 0, st.message
    for i in range(k):
        v = hv[i].numpy()[:, : 2 * n].T  # column-major 2n x n with ld 2n + pad
        assert np.array_equal(hl[i].numpy(), ref[i].lambda_)
        assert np.array_equal(v, ref[i].v)
    ctx.close()


@pytest.mark.parametrize("method", [bse.Method.Chol, bse.Method.CholSvd])
@pytest.mark.parametrize("n", [96, 640])
def test_degenerate_bse_spectrum(method, n):
    """Physically degenerate excitations: A with eigenvalues of multiplicity n/4 and B = 0 (the
    reference's decoupled case, test_solvers.cpp) and B a small multiple of A (commuting, the
    multiplicities kept). lambda against the oracle's same method (1e-10), every eigenpair's
    residual <= 100 n eps and Sigma-orthogonality <= 100 n eps (vectors inside a degenerate
    eigenspace are not unique, so they are not compared)."""
    q, _ = np.linalg.qr(crand(n, n))
    ev = np.repeat([1.0, 2.0, 3.5, 7.0], n // 4)
    a = (q * ev) @ q.conj().T
    a = (a + a.conj().T) / 2
    for b in (np.zeros_like(a), 0.25 * a):
        r = bse.solve(method, bse.from_blocks(a, b))
        ref, _, _ = oracle.solve("chol" if method == bse.Method.Chol else "chol-svd", a, b)
        assert np.max(np.abs(r.lambda_ - ref) / ref) <= 1e-10
        assert residual(a, b, r.lambda_, r.v).max() <= 100 * n * EPS
        assert sigma_orthogonality_error(r.v) <= 100 * n * EPS


def test_solve_batched_pinned_outputs_misaligned():
    """A page-locked output that is only 8-byte aligned (a view one double into a pinned
    buffer) takes the copy-engine download instead of the 16-byte streaming kernel: same bits."""
    import ctypes

    import torch

    n, k = 200, 4  # two items per lane: the first goes through the streaming path's check
    ctx = bse.Context(0)
    ctx.set_batch_lanes(2)
    hs = [bse.from_blocks(*configs.config2(60 + s, n=n)) for s in range(k)]
    ref = bse.solve_batched(bse.Method.Chol, hs, ctx=ctx)
    raw = [torch.zeros(2 * n * 2 * n + 2, dtype=torch.float64).pin_memory() for _ in range(k)]
    hl = [torch.zeros(n, dtype=torch.float64).pin_memory() for _ in range(k)]
    arr = lambda ptrs: (ctypes.c_void_p * k)(*ptrs)  # noqa: E731
    vptr = [t.data_ptr() + 8 for t in raw]  # 8-byte aligned complex128 output
    failed = ctypes.c_int64(-1)
    st = bse.Status()
    rc = bse._lib.lib().bse_solve_batched(
        ctx.handle, int(bse.Method.Chol), n, k, arr([h.a.ctypes.data for h in hs]), n,
        arr([h.b.ctypes.data for h in hs]), n, arr([t.data_ptr() for t in hl]), arr(vptr), 2 * n,
        None, None, ctypes.byref(failed), ctypes.byref(st))
    assert rc == 0, st.message
    for i in range(k):
        v = raw[i].numpy()[1: 1 + 2 * n * 2 * n].view(np.complex128).reshape(n, 2 * n).T
        assert np.array_equal(v, ref[i].v)
    ctx.close()
