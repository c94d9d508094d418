"""Seeded synthetic inputs: BASELINE.json configs 1-5 and the reference's test families.

Input synthesis only (host numpy + the counter-based generator in ``libbse_gen.so``, a
host-only library built from csrc/gen.cpp without any CUDA code, so loading the inputs never
maps the GPU library ``libbse_b200.so``); not part of the timed hot path. The reference's public benchmark has no dataset: these generators stand in
for it with its stated shapes, sizes and value distributions (BASELINE.json "configs").
"""
from __future__ import annotations

import ctypes
import os
import threading

import numpy as np

_GEN_PATH = os.path.join(os.path.dirname(os.path.abspath(__file__)), "libbse_gen.so")
_gen = None
_gen_lock = threading.Lock()


def gen_lib():
    """The host generator library (same bse_gen_* entry points as include/bse_gpu.h)."""
    global _gen
    with _gen_lock:
        if _gen is None:
            if not os.path.exists(_GEN_PATH):
                raise RuntimeError(f"{_GEN_PATH} is missing: build it with `make -C "
                                   f"{os.path.dirname(_GEN_PATH)}`")
            L = ctypes.CDLL(_GEN_PATH)
            c_u64, c_i64, c_dp, c_d = ctypes.c_uint64, ctypes.c_int64, ctypes.c_void_p, ctypes.c_double
            L.bse_gen_dominant.argtypes = [c_i64, c_u64, ctypes.c_int, c_d, c_d, c_d, c_dp, c_dp]
            for name in ("bse_gen_gaussian_stream", "bse_gen_normal", "bse_gen_uniform"):
                getattr(L, name).argtypes = [c_u64, c_u64, c_i64, c_dp]
            for name in ("bse_gen_dominant", "bse_gen_gaussian_stream", "bse_gen_normal",
                         "bse_gen_uniform"):
                getattr(L, name).restype = ctypes.c_int
            _gen = L
    return _gen


def _gen_dominant(n: int, seed: int, is_complex: bool, scale: float, dlo: float, dhi: float):
    a = np.zeros((n, n), dtype=np.complex128, order="F")
    b = np.zeros((n, n), dtype=np.complex128, order="F")
    rc = gen_lib().bse_gen_dominant(n, seed, 1 if is_complex else 0, scale, dlo, dhi,
                                     a.ctypes.data_as(ctypes.c_void_p),
                                     b.ctypes.data_as(ctypes.c_void_p))
    if rc != 0:
        raise ValueError("bse_gen_dominant failed")
    return a, b


def normal(seed: int, stream: int, count: int) -> np.ndarray:
    out = np.zeros(count)
    gen_lib().bse_gen_normal(seed, stream, count, out.ctypes.data_as(ctypes.c_void_p))
    return out


def uniform(seed: int, stream: int, count: int) -> np.ndarray:
    out = np.zeros(count)
    gen_lib().bse_gen_uniform(seed, stream, count, out.ctypes.data_as(ctypes.c_void_p))
    return out


def config1(seed: int = 0, n: int = 512):
    """Real fp64 n=512: A = diag(d) + 0.05 (X+X^T)/2, X ~ N(0,1)/sqrt(n), d ~ U[1,10];
    B = 0.05 (X'+X'^T)/2 (independent stream). Returned as complex with zero imag."""
    return _gen_dominant(n, seed, False, 0.05, 1.0, 10.0)


def config2(seed: int = 0, n: int = 2048, dhi: float = 20.0):
    """Complex n=2048: A = diag(d) + 0.1 (Z+Z^H)/2, Re/Im Z ~ N(0,1)/sqrt(2n), d ~ U[1,20];
    B = 0.1 (W+W^H)/2."""
    return _gen_dominant(n, seed, True, 0.1, 1.0, dhi)


def config4(seed: int = 0, n: int = 16384):
    """Config-2 generator at n=16384 with d ~ U[1,50]."""
    return _gen_dominant(n, seed, True, 0.1, 1.0, 50.0)


def config5(seed: int, n: int = 4096):
    """Batch member `seed` (0..63) of config 5: the config-2 generator at n=4096."""
    return _gen_dominant(n, seed, True, 0.1, 1.0, 20.0)


def haar_unitary(n: int, seed: int, stream: int = 3) -> np.ndarray:
    """Haar unitary: complex Gaussian fill, QR, columns phased by diag(R)/|diag(R)|
    (the recipe of proj/src/gen.cpp:40-58)."""
    z = (normal(seed, stream, n * n) + 1j * normal(seed, stream + 1, n * n)) * np.sqrt(0.5)
    z = z.reshape((n, n), order="F")
    q, r = np.linalg.qr(z)
    d = np.diag(r)
    ph = np.where(np.abs(d) > 0, d / np.maximum(np.abs(d), 1e-300), 1.0)
    return np.asfortranarray(q * ph[None, :])


def config3(seed: int = 0, n: int = 4096):
    """Ill-conditioned complex n=4096: A-B = Q diag(logspace(-6,1,n)) Q^H (Q Haar),
    A+B = (A-B) + diag(U[0.5,2]); smallest eigenvalues of H ~ 1e-3."""
    q = haar_unitary(n, seed)
    s = np.logspace(-6, 1, n)
    m2 = (q * s[None, :]) @ q.conj().T
    m2 = 0.5 * (m2 + m2.conj().T)
    m1 = m2 + np.diag(0.5 + 1.5 * uniform(seed, 2, n))
    a = np.asfortranarray(0.5 * (m1 + m2))
    b = np.asfortranarray(0.5 * (m1 - m2))
    return a, b


# ---------------------------------------------------------------- reference test families
def gaussian_stream(seed: int, stream: int, count: int) -> np.ndarray:
    """proj/src/gen.cpp:19-38 GaussianStream::next_complex() x count (bit-exact port)."""
    out = np.zeros(2 * count)
    gen_lib().bse_gen_gaussian_stream(seed, stream, count, out.ctypes.data_as(ctypes.c_void_p))
    return out[0::2] + 1j * out[1::2]


def random_hermitian(n: int, seed: int) -> np.ndarray:
    """proj/tests/test_backend.cpp:16-22."""
    m = gaussian_stream(seed, 0, n * n).reshape((n, n), order="F")
    return np.asfortranarray(0.5 * (m + m.conj().T))


def generate_random_definite(n: int, seed: int, shift_margin: float = 1.0):
    """proj/src/gen.cpp:74-96."""
    a = gaussian_stream(seed, 0, n * n).reshape((n, n), order="F")
    b = gaussian_stream(seed, 1, n * n).reshape((n, n), order="F")
    a = 0.5 * (a + a.conj().T)
    b = 0.5 * (b + b.conj().T)
    rho = np.abs(a).sum(axis=0).max() + np.abs(b).sum(axis=0).max()
    a = a + (rho + shift_margin) * np.eye(n)
    return np.asfortranarray(a), np.asfortranarray(b)


def random_unitary(n: int, seed: int) -> np.ndarray:
    """proj/src/gen.cpp:40-58 (Householder QR via numpy/LAPACK instead of Eigen)."""
    z = gaussian_stream(seed, 0, n * n).reshape((n, n), order="F")
    q, r = np.linalg.qr(z)
    d = np.diag(r)
    ph = np.where(np.abs(d) > 0, d / np.maximum(np.abs(d), 1e-300), 1.0)
    return np.asfortranarray(q * ph[None, :])


def generate_conditioned(n: int, kappa: float, seed: int):
    """proj/src/gen.cpp:60-72: A = Q^H D Q, B = A/2, spectrum (sqrt(3)/2) linspace(1,kappa/3,n)."""
    d = np.linspace(1.0, kappa / 3.0, n)
    q = random_unitary(n, seed)
    a = (q.conj().T * d[None, :]) @ q
    a = 0.5 * (a + a.conj().T)
    return np.asfortranarray(a), np.asfortranarray(0.5 * a)
