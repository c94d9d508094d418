"""The reference's API contract beyond single-call numerics:

* threading: "pure functions; safe for concurrent invocation; no global state"
   - bse_solve called from several host threads at
  once, on distinct contexts and on one shared context, returns bitwise what serial calls
  return (deterministic per input and lane count);
* CHOL's certificate of A+B: the strict mode (bse_ctx_set_strict_certificates) factors A+B on
  every solve exactly as product_pair does (core.cpp:87-100); results are bitwise those of the
  default spectral certificate, and an indefinite A+B reports NotDefinite{M1} with the
  oracle's message (block and pivot).
"""
import threading

import numpy as np
import pytest

import oracle
import paper_2008_08825_b200 as bse
from paper_2008_08825_b200 import configs

pytestmark = pytest.mark.gpu


def _inputs():
    return [bse.from_blocks(*configs.config2(s, n=n)) for s, n in
            ((1, 96), (2, 200), (3, 257), (4, 300))]


def _run_threads(fn, k):
    out, err = [None] * k, [None] * k

    def work(i):
        try:
            out[i] = fn(i)
        except Exception as e:  # surfaced below
            err[i] = e
    ts = [threading.Thread(target=work, args=(i,)) for i in range(k)]
    for t in ts:
        t.start()
    for t in ts:
        t.join(timeout=240)
        assert not t.is_alive(), "concurrent solve did not return"
    for e in err:
        if e is not None:
            raise e
    return out


@pytest.mark.timeout(600)
@pytest.mark.parametrize("method", [bse.Method.Chol, bse.Method.CholSvd])
def test_concurrent_solves_distinct_contexts(method):
    hs = _inputs()
    serial = [bse.solve(method, h) for h in hs]
    ctxs = [bse.Context(0) for _ in hs]
    try:
        for rep in range(2):
            got = _run_threads(lambda i: bse.solve(method, hs[i], ctx=ctxs[i]), len(hs))
            for r, s in zip(got, serial):
                assert np.array_equal(r.lambda_, s.lambda_)
                assert np.array_equal(r.v, s.v)
                assert r.near_singular == s.near_singular
    finally:
        for c in ctxs:
            c.close()


@pytest.mark.timeout(600)
def test_concurrent_solves_shared_context():
    hs = _inputs()
    ctx = bse.Context(0)
    try:
        serial = [bse.solve(bse.Method.Chol, h, ctx=ctx) for h in hs]
        got = _run_threads(lambda i: bse.solve(bse.Method.Chol, hs[i % len(hs)], ctx=ctx),
                           2 * len(hs))
        for i, r in enumerate(got):
            s = serial[i % len(hs)]
            assert np.array_equal(r.lambda_, s.lambda_) and np.array_equal(r.v, s.v)
    finally:
        ctx.close()


@pytest.mark.timeout(600)
def test_concurrent_batched_calls():
    """Two host threads each drive a 2-lane batch on their own context."""
    items = [configs.config2(s, n=160) for s in range(4)]
    serial = [bse.solve(bse.Method.Chol, bse.from_blocks(a, b)) for a, b in items]
    ctxs = [bse.Context(0), bse.Context(0)]
    try:
        for c in ctxs:
            c.set_batch_lanes(2)
        got = _run_threads(lambda i: bse.solve_batched(bse.Method.Chol,
                                                       [bse.from_blocks(a, b) for a, b in items],
                                                       ctx=ctxs[i]), 2)
        for res in got:
            for r, s in zip(res, serial):
                np.testing.assert_allclose(r.lambda_, s.lambda_, rtol=1e-12)
    finally:
        for c in ctxs:
            c.close()


def test_strict_certificates_same_result():
    h = bse.from_blocks(*configs.config2(7, n=320))
    ctx = bse.Context(0)
    try:
        r0 = bse.solve_chol(h, ctx=ctx)
        ctx.set_strict_certificates(True)
        r1 = bse.solve_chol(h, ctx=ctx)
        assert np.array_equal(r0.lambda_, r1.lambda_) and np.array_equal(r0.v, r1.v)
    finally:
        ctx.close()


@pytest.mark.parametrize("strict", [False, True])
def test_indefinite_m1_reported_like_the_reference(strict):
    """A+B indefinite by a clear margin (A-B definite): both certificates report
    NotDefinite{M1} with zpotrf's pivot, as the oracle's product_pair does."""
    n = 40
    rng = np.random.default_rng(5)
    q, _ = np.linalg.qr(rng.standard_normal((n, n)) + 1j * rng.standard_normal((n, n)))
    mu = np.linspace(1.0, 3.0, n)
    mu[n // 2] = -1e-3
    m1 = (q * mu) @ q.conj().T
    m1 = 0.5 * (m1 + m1.conj().T)
    m2 = np.diag(np.linspace(1.0, 2.0, n)).astype(complex)
    a, b = 0.5 * (m1 + m2), 0.5 * (m1 - m2)
    with pytest.raises(oracle.OracleError) as eo:
        oracle.solve("chol", a, b)
    ctx = bse.Context(0)
    try:
        ctx.set_strict_certificates(strict)
        with pytest.raises(bse.NotDefinite) as eg:
            bse.solve_chol(bse.from_blocks(a, b), ctx=ctx)
    finally:
        ctx.close()
    assert eg.value.which == bse.Block.M1 and eo.value.block == 0
    assert str(eg.value) == str(eo.value)


def test_device_pointers_must_be_16_byte_aligned():
    """bse_solve_device / bse_solve_batched_device read and write complex128 as 16-byte
    vectors: an 8-byte-aligned device operand is rejected with InvalidSpec (no launch)."""
    import torch

    n = 64
    a, b = configs.config2(5, n=n)
    dev = torch.device("cuda", 0)
    buf = torch.zeros(2 * n * n + 2, dtype=torch.float64, device=dev)
    da = torch.from_numpy(a.T.copy()).to(dev)
    lam = torch.empty(n, dtype=torch.float64, device=dev)
    v = torch.empty((n, 2 * n), dtype=torch.complex128, device=dev)
    with pytest.raises(bse.InvalidSpec):
        bse.solve_device(bse.Method.Chol, n, da.data_ptr(), buf.data_ptr() + 8, lam.data_ptr(),
                         v.data_ptr())
    with pytest.raises(bse.InvalidSpec):
        bse.solve_batched_device(bse.Method.Chol, n, [da.data_ptr()], [buf.data_ptr() + 8],
                                 [lam.data_ptr()], [v.data_ptr()])
