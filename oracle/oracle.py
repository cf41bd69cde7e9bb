"""ctypes wrapper around the fp64 CPU oracle (oracle/blr_oracle.c).

TEST INFRASTRUCTURE ONLY.  Only tests/, ``__graft_entry__.smoke()`` and bench.py's
``cpu_baseline`` / ``--impl reference`` legs may import this module.  Nothing here is shared
with the CUDA path (paper_2512_20861_b200/csrc); the product path never imports it.

All functions take numpy arrays (any float dtype; widened to float64 exactly) in the paper's
storage layouts and return float64 numpy arrays.
"""
from __future__ import annotations

import ctypes
import os
import subprocess

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
_SRC = os.path.join(_HERE, "blr_oracle.c")
_LIB = os.path.join(_HERE, "liboracle.so")
_lib = None

# Monarch V composite-index layouts (reading R2).
B2_FASTEST = 0
RPRIME_FASTEST = 1


def build(force: bool = False) -> str:
    """Compile blr_oracle.c -> liboracle.so with gcc (fp64, OpenMP over token rows)."""
    if force or not os.path.exists(_LIB) or os.path.getmtime(_LIB) < os.path.getmtime(_SRC):
        cmd = ["gcc", "-O2", "-fopenmp", "-fPIC", "-shared", "-std=c11", "-o", _LIB, _SRC]
        subprocess.check_call(cmd)
    return _LIB


def _load():
    global _lib
    if _lib is None:
        build()
        lib = ctypes.CDLL(_LIB)
        i64, dp = ctypes.c_int64, ctypes.POINTER(ctypes.c_double)
        lib.orc_dense_forward.argtypes = [i64, i64, i64, dp, dp, dp]
        lib.orc_lowrank_weight.argtypes = [i64, i64, i64, dp, dp, dp]
        lib.orc_lowrank_forward.argtypes = [i64, i64, i64, i64, dp, dp, dp, dp, dp]
        lib.orc_monarch_weight.argtypes = [i64, i64, i64, i64, i64, dp, dp, ctypes.c_int, dp]
        lib.orc_monarch_forward.argtypes = [i64, i64, i64, i64, i64, i64, dp, dp, dp, ctypes.c_int, dp]
        lib.orc_blast_weight.argtypes = [i64, i64, i64, i64, i64, dp, dp, dp, dp]
        lib.orc_blast_forward.argtypes = [i64, i64, i64, i64, i64, i64, dp, dp, dp, dp, dp, dp]
        lib.orc_num_threads.restype = ctypes.c_int
        lib.orc_set_num_threads.argtypes = [ctypes.c_int]
        _lib = lib
    return _lib


def _f64(a) -> np.ndarray:
    a = np.ascontiguousarray(np.asarray(a, dtype=np.float64))
    return a


def _p(a: np.ndarray):
    return a.ctypes.data_as(ctypes.POINTER(ctypes.c_double))


def num_threads() -> int:
    return int(_load().orc_num_threads())


def set_num_threads(n: int) -> None:
    """Thread count of later calls (timing only; results do not depend on it). n <= 0: default."""
    _load().orc_set_num_threads(int(n))


# ---------------------------------------------------------------- dense ------------------------
def dense_forward(X, W) -> np.ndarray:
    """Y = X W."""
    X, W = _f64(X), _f64(W)
    n, i = X.shape
    i2, o = W.shape
    assert i == i2
    Y = np.empty((n, o), np.float64)
    _load().orc_dense_forward(n, i, o, _p(X), _p(W), _p(Y))
    return Y


# ---------------------------------------------------------------- low rank ---------------------
def lowrank_weight(V, U) -> np.ndarray:
    """W = V U, V [i, r], U [r, o]."""
    V, U = _f64(V), _f64(U)
    i, r = V.shape
    r2, o = U.shape
    assert r == r2
    W = np.empty((i, o), np.float64)
    _load().orc_lowrank_weight(i, o, r, _p(V), _p(U), _p(W))
    return W


def lowrank_forward(X, V, U) -> np.ndarray:
    """Y = (X V) U, structured."""
    X, V, U = _f64(X), _f64(V), _f64(U)
    n, i = X.shape
    i2, r = V.shape
    r2, o = U.shape
    assert i == i2 and r == r2
    Y = np.empty((n, o), np.float64)
    scratch = np.empty((max(n, 1), r), np.float64)
    _load().orc_lowrank_forward(n, i, o, r, _p(X), _p(V), _p(U), _p(Y), _p(scratch))
    return Y


# ---------------------------------------------------------------- Monarch ----------------------
def _monarch_dims(V, U, b1, b2):
    V, U = _f64(V), _f64(U)
    assert V.ndim == 3 and U.ndim == 3 and V.shape[0] == b1 and U.shape[0] == b2
    R, p = V.shape[1], V.shape[2]
    q, K2 = U.shape[1], U.shape[2]
    assert R % b2 == 0 and K2 % b1 == 0
    rp = R // b2
    assert K2 // b1 == rp, "U inner dim must be b1*r'"
    return V, U, rp, p, q


def monarch_weight(V, U, b1: int, b2: int, layout: int = B2_FASTEST) -> np.ndarray:
    """Dense W (i x o) of a Monarch layer; V [b1, r'b2, p], U [b2, q, b1 r']."""
    V, U, rp, p, q = _monarch_dims(V, U, b1, b2)
    W = np.empty((b1 * p, b2 * q), np.float64)
    _load().orc_monarch_weight(b1, b2, rp, p, q, _p(V), _p(U), int(layout), _p(W))
    return W


def monarch_forward(X, V, U, b1: int, b2: int, layout: int = B2_FASTEST) -> np.ndarray:
    """Y_k = sum_l X_l V_{l,k} U_{l,k}, canonical output order Y[t, k*q + c]."""
    V, U, rp, p, q = _monarch_dims(V, U, b1, b2)
    X = _f64(X)
    n = X.shape[0]
    assert X.shape[1] == b1 * p
    Y = np.empty((n, b2 * q), np.float64)
    _load().orc_monarch_forward(n, b1, b2, rp, p, q, _p(X), _p(V), _p(U), int(layout), _p(Y))
    return Y


def monarch_forward_transposed(X, V, U, b1: int, b2: int, layout: int = B2_FASTEST) -> np.ndarray:
    """The same product in the "transposed" output order the paper's optimization (3) leaves in
    place (PAPER.md L45 footnote, L219-220): output block k, column c lands at Y[t, c*b2 + k]
    instead of Y[t, k*q + c], i.e. the (b2, q) column grid of the canonical output read
    column-major.  Written out element by element from that definition."""
    Yc = monarch_forward(X, V, U, b1, b2, layout)
    n, o = Yc.shape
    q = o // b2
    Yt = np.empty_like(Yc)
    for k in range(b2):
        for c in range(q):
            Yt[:, c * b2 + k] = Yc[:, k * q + c]
    return Yt


# ---------------------------------------------------------------- BLAST ------------------------
def _blast_dims(V, S, U):
    V, S, U = _f64(V), _f64(S), _f64(U)
    b1, p, r = V.shape
    b1s, b2, rs = S.shape
    b2u, ru, q = U.shape
    assert b1 == b1s and r == rs and b2 == b2u and r == ru
    return V, S, U, b1, b2, r, p, q


def blast_weight(V, S, U) -> np.ndarray:
    """Dense W of a BLAST layer; V [b1,p,r], S [b1,b2,r], U [b2,r,q]."""
    V, S, U, b1, b2, r, p, q = _blast_dims(V, S, U)
    W = np.empty((b1 * p, b2 * q), np.float64)
    _load().orc_blast_weight(b1, b2, r, p, q, _p(V), _p(S), _p(U), _p(W))
    return W


def blast_forward(X, V, S, U) -> np.ndarray:
    """Y_k = (sum_l (X_l V_l) S_{l,k}) U_k."""
    V, S, U, b1, b2, r, p, q = _blast_dims(V, S, U)
    X = _f64(X)
    n = X.shape[0]
    assert X.shape[1] == b1 * p
    Y = np.empty((n, b2 * q), np.float64)
    scratch = np.empty((max(n, 1), b1 * r + r), np.float64)
    _load().orc_blast_forward(n, b1, b2, r, p, q, _p(X), _p(V), _p(S), _p(U), _p(Y), _p(scratch))
    return Y
