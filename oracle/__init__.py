"""CPU oracle for Lloyd's K-means (arXiv 2405.12052) -- TEST INFRASTRUCTURE ONLY.

Only ``tests/``, ``__graft_entry__.smoke()`` and ``bench.py``'s cpu_baseline /
``--impl reference`` leg may import this package.  The product package
``paper_2405_12052_b200`` never imports it, and the two share no code.

This module is a thin ctypes marshalling layer over ``lloyd_oracle.c`` (plain
single-threaded C, fp32 form-D distances, fp64 sums; see the header comment of
that file and DESIGN.md "Readings").  Arrays are numpy; points are N x d
row-major float32.
"""
from __future__ import annotations

import ctypes
import os
import subprocess

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
_SRC = os.path.join(_HERE, "lloyd_oracle.c")
_LIB = os.path.join(_HERE, "liblloyd_oracle.so")

ORACLE_CFLAGS = ["-std=c11", "-O2", "-ffp-contract=off", "-fno-fast-math",
                 "-fPIC", "-shared"]


class OracleError(RuntimeError):
    pass


def build(force: bool = False) -> str:
    """Compile the oracle with gcc (no contraction, no fast-math)."""
    if force or not os.path.exists(_LIB) or os.path.getmtime(_LIB) < os.path.getmtime(_SRC):
        tmp = _LIB + f".tmp{os.getpid()}"
        subprocess.check_call(["gcc", *ORACLE_CFLAGS, "-o", tmp, _SRC, "-lm"])
        os.replace(tmp, _LIB)
    return _LIB


_lib = None


def _load():
    global _lib
    if _lib is None:
        build()
        lib = ctypes.CDLL(_LIB)
        P = ctypes.c_void_p
        i64 = ctypes.c_int64
        ci = ctypes.c_int
        lib.oracle_dist.restype = ctypes.c_float
        lib.oracle_dist.argtypes = [P, P, ci]
        lib.oracle_shift_error.restype = ctypes.c_double
        lib.oracle_shift_error.argtypes = [P, P, ci, ci]
        lib.oracle_partials.restype = ci
        lib.oracle_partials.argtypes = [P, i64, ci, ci, P, P, P, P, P, P]
        lib.oracle_update.restype = ci
        lib.oracle_update.argtypes = [P, P, P, ci, ci, P, P]
        lib.oracle_step.restype = ci
        lib.oracle_step.argtypes = [P, i64, ci, ci, P, P, P, P, P, P, P, P]
        lib.oracle_fit.restype = ci
        lib.oracle_fit.argtypes = [P, i64, ci, ci, P, ctypes.c_double, ci,
                                   P, P, P, P, P, P]
        _lib = lib
    return _lib


def _ptr(a):
    return ctypes.c_void_p(a.ctypes.data) if a is not None else None


def _points(X):
    X = np.ascontiguousarray(X, dtype=np.float32)
    if X.ndim == 1:
        X = X.reshape(-1, 1)
    return X


def _check(rc, what):
    if rc != 0:
        raise OracleError(f"{what} returned {rc} "
                          f"({'invalid argument' if rc == -1 else 'non-finite input'})")


def dist(x, c) -> np.float32:
    """Form-D squared distance between one fp32 point and one fp32 centroid."""
    x = np.ascontiguousarray(x, dtype=np.float32).ravel()
    c = np.ascontiguousarray(c, dtype=np.float32).ravel()
    assert x.shape == c.shape
    return np.float32(_load().oracle_dist(_ptr(x), _ptr(c), x.size))


def shift_error(mu_prev, mu_next) -> float:
    a = np.ascontiguousarray(mu_prev, dtype=np.float64)
    b = np.ascontiguousarray(mu_next, dtype=np.float64)
    assert a.shape == b.shape and a.ndim == 2
    return _load().oracle_shift_error(_ptr(a), _ptr(b), a.shape[0], a.shape[1])


def partials(X, mu):
    """Per-slice sums/counts/J at centroids mu (K x d fp64).

    Returns dict(labels, dmin, sums, counts, J)."""
    X = _points(X)
    mu = np.ascontiguousarray(mu, dtype=np.float64)
    n, d = X.shape
    K = mu.shape[0]
    labels = np.empty(n, np.int32)
    dmin = np.empty(n, np.float32)
    sums = np.empty((K, d), np.float64)
    counts = np.empty(K, np.int64)
    J = np.zeros(1, np.float64)
    rc = _load().oracle_partials(_ptr(X), n, d, K, _ptr(mu), _ptr(labels), _ptr(dmin),
                                 _ptr(sums), _ptr(counts), _ptr(J))
    _check(rc, "oracle_partials")
    return dict(labels=labels, dmin=dmin, sums=sums, counts=counts, J=float(J[0]))


def update(sums, counts, mu_prev):
    sums = np.ascontiguousarray(sums, dtype=np.float64)
    counts = np.ascontiguousarray(counts, dtype=np.int64)
    mu_prev = np.ascontiguousarray(mu_prev, dtype=np.float64)
    K, d = mu_prev.shape
    mu_next = np.empty_like(mu_prev)
    E = np.zeros(1, np.float64)
    rc = _load().oracle_update(_ptr(sums), _ptr(counts), _ptr(mu_prev), K, d,
                               _ptr(mu_next), _ptr(E))
    _check(rc, "oracle_update")
    return mu_next, float(E[0])


def step(X, mu):
    """One Lloyd iteration at mu^t.  Returns dict(labels, dmin, sums, counts, J,
    mu_next, E)."""
    X = _points(X)
    mu = np.ascontiguousarray(mu, dtype=np.float64)
    N, d = X.shape
    K = mu.shape[0]
    labels = np.empty(N, np.int32)
    dmin = np.empty(N, np.float32)
    sums = np.empty((K, d), np.float64)
    counts = np.empty(K, np.int64)
    J = np.zeros(1, np.float64)
    mu_next = np.empty_like(mu)
    E = np.zeros(1, np.float64)
    rc = _load().oracle_step(_ptr(X), N, d, K, _ptr(mu), _ptr(labels), _ptr(dmin),
                             _ptr(sums), _ptr(counts), _ptr(J), _ptr(mu_next), _ptr(E))
    _check(rc, "oracle_step")
    return dict(labels=labels, dmin=dmin, sums=sums, counts=counts, J=float(J[0]),
                mu_next=mu_next, E=float(E[0]))


def fit(X, K, init_idx, tol, max_iter):
    """The serial Lloyd loop.  Returns dict(labels, centroids,
    iters, inertia, E_trace, J_trace)."""
    X = _points(X)
    N, d = X.shape
    init_idx = np.ascontiguousarray(init_idx, dtype=np.int64)
    assert init_idx.shape == (K,)
    labels = np.empty(N, np.int32)
    cent = np.empty((K, d), np.float64)
    iters = ctypes.c_int(0)
    inertia = ctypes.c_double(0.0)
    Et = np.zeros(max_iter, np.float64)
    Jt = np.zeros(max_iter, np.float64)
    rc = _load().oracle_fit(_ptr(X), N, d, K, _ptr(init_idx), float(tol), int(max_iter),
                            _ptr(labels), _ptr(cent), ctypes.byref(iters),
                            ctypes.byref(inertia), _ptr(Et), _ptr(Jt))
    _check(rc, "oracle_fit")
    T = iters.value
    return dict(labels=labels, centroids=cent, iters=T, inertia=inertia.value,
                E_trace=Et[:T].copy(), J_trace=Jt[:T].copy())
