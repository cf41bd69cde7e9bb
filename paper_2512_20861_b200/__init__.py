"""B200-native block-low-rank (BLR) prefill forward (arXiv 2512.20861).

Thin Python binding over the C ABI of ``libblr.so`` (include/blr.h).  It only marshals
arguments: every step of the path runs in the library's sm_100a kernels.  torch is used for
device memory (output and workspace allocation through the caching allocator) and streams.
There is no CPU fallback: a missing or unloadable library raises.

    Y = lowrank_matmul(X, V, U)
    Y = monarch_matmul(X, V, U, b1, b2, v_layout=0)
    Y = blast_matmul(X, V, S, U)
"""
from __future__ import annotations

import ctypes
import os

import torch

from .build import LIB_PATH, build  # noqa: F401

__all__ = ["load", "lowrank_matmul", "monarch_matmul", "blast_matmul", "blast_kmajor_factors", "BLRError",
           "B2_FASTEST", "RPRIME_FASTEST", "OUT_CANONICAL", "OUT_TRANSPOSED", "last_launch_count",
           "lib_path", "transposed_row_perm", "permute_rows_for_transposed_input"]

B2_FASTEST = 0       # BLR_MON_V_B2_FASTEST   (original layout)
RPRIME_FASTEST = 1   # BLR_MON_V_RPRIME_FASTEST (after re-layout (1))
OUT_CANONICAL = 0    # BLR_OUT_CANONICAL   Y[t, k q + c]
OUT_TRANSPOSED = 1   # BLR_OUT_TRANSPOSED  Y[t, c b2 + k]

_lib = None


class BLRError(RuntimeError):
    def __init__(self, fn: str, code: int, msg: str):
        super().__init__(f"{fn} failed: {msg} ({code})")
        self.code = code


def lib_path() -> str:
    return LIB_PATH


def load():
    """Load libblr.so (raises if it is missing; never falls back).  BLR_LIB=<path> loads another
    build of the same library instead (A/B timing of two builds only)."""
    global _lib
    if _lib is not None:
        return _lib
    path = os.environ.get("BLR_LIB", LIB_PATH)
    if not os.path.exists(path):
        raise RuntimeError(f"libblr.so not found at {path}; run __graft_entry__.build()")
    lib = ctypes.CDLL(path)
    i64, vp, sz = ctypes.c_int64, ctypes.c_void_p, ctypes.c_size_t
    lib.blr_lowrank_matmul.argtypes = [vp, i64, i64, i64, i64, vp, vp, vp, vp, sz, vp]
    lib.blr_monarch_matmul.argtypes = [vp, i64, i64, i64, i64, i64, i64, vp, vp, ctypes.c_int,
                                       ctypes.c_int, vp, vp, sz, vp]
    lib.blr_blast_matmul.argtypes = [vp, i64, i64, i64, i64, i64, i64, vp, vp, vp, vp, vp, sz, vp]
    lib.blr_blast_matmul_fp8z.argtypes = lib.blr_blast_matmul.argtypes
    fns = ["blr_lowrank_matmul", "blr_monarch_matmul", "blr_blast_matmul", "blr_blast_matmul_fp8z"]
    # (an older build loaded through BLR_LIB for an A/B may predate the K-major entry point)
    if path == LIB_PATH or hasattr(lib, "blr_blast_matmul_kmajor"):
        lib.blr_blast_matmul_kmajor.argtypes = lib.blr_blast_matmul.argtypes
        fns.append("blr_blast_matmul_kmajor")
    for fn in fns:
        getattr(lib, fn).restype = ctypes.c_int
    lib.blr_lowrank_workspace_size.argtypes = [i64, i64, i64, i64]
    lib.blr_monarch_workspace_size.argtypes = [i64, i64, i64, i64, i64, i64]
    lib.blr_blast_workspace_size.argtypes = [i64, i64, i64, i64, i64, i64]
    for fn in ("blr_lowrank_workspace_size", "blr_monarch_workspace_size", "blr_blast_workspace_size"):
        getattr(lib, fn).restype = sz
    lib.blr_status_string.argtypes = [ctypes.c_int]
    lib.blr_status_string.restype = ctypes.c_char_p
    lib.blr_version.restype = ctypes.c_char_p
    lib.blr_last_launch_count.restype = ctypes.c_int
    lib.blr_profile_begin.argtypes = [ctypes.c_void_p, ctypes.c_int]
    lib.blr_profile_begin.restype = None
    lib.blr_profile_end.restype = ctypes.c_int
    lib.blr_transposed_row_perm.argtypes = [i64, i64, ctypes.POINTER(ctypes.c_int64)]
    lib.blr_transposed_row_perm.restype = ctypes.c_int
    _lib = lib
    return lib


def last_launch_count() -> int:
    return int(load().blr_last_launch_count())


def _check(fn: str, code: int):
    if code != 0:
        raise BLRError(fn, code, load().blr_status_string(code).decode())


def _dev_bf16(name: str, t: torch.Tensor) -> int:
    if not isinstance(t, torch.Tensor) or t.dtype != torch.bfloat16 or not t.is_cuda:
        raise TypeError(f"{name} must be a CUDA bf16 tensor")
    if not t.is_contiguous():
        raise ValueError(f"{name} must be contiguous")
    return t.data_ptr()


def _stream_ptr(device) -> int:
    return torch.cuda.current_stream(device).cuda_stream


def _out(X, n, o, out):
    if out is None:
        return torch.empty((n, o), dtype=torch.bfloat16, device=X.device)
    if tuple(out.shape) != (n, o):
        raise ValueError(f"out must have shape {(n, o)}")
    return out


def _ws(X, nbytes, workspace):
    if workspace is not None:
        return workspace
    return torch.empty(max(int(nbytes), 16), dtype=torch.uint8, device=X.device)


def lowrank_matmul(X: torch.Tensor, V: torch.Tensor, U: torch.Tensor, out=None, workspace=None):
    """Y = (X V) U with X [n, i], V [i, r], U [r, o]."""
    lib = load()
    n, i = X.shape
    i2, r = V.shape
    r2, o = U.shape
    if i2 != i or r2 != r:
        raise ValueError("shape mismatch")
    Y = _out(X, n, o, out)
    ws = _ws(X, lib.blr_lowrank_workspace_size(n, i, o, r), workspace)
    with torch.cuda.device(X.device):
        code = lib.blr_lowrank_matmul(_dev_bf16("X", X), n, i, o, r, _dev_bf16("V", V), _dev_bf16("U", U),
                                      _dev_bf16("out", Y), ws.data_ptr(), ws.numel() * ws.element_size(),
                                      _stream_ptr(X.device))
    _check("blr_lowrank_matmul", code)
    return Y


def transposed_row_perm(b2: int, q: int) -> torch.Tensor:
    """perm[c*b2 + k] = k*q + c (blr_transposed_row_perm): the canonical input column of each
    position of a BLR_OUT_TRANSPOSED Monarch output."""
    perm = torch.empty(b2 * q, dtype=torch.int64)
    _check("blr_transposed_row_perm",
           load().blr_transposed_row_perm(b2, q, ctypes.cast(perm.data_ptr(), ctypes.POINTER(ctypes.c_int64))))
    return perm


def permute_rows_for_transposed_input(W: torch.Tensor, b2: int, q: int) -> torch.Tensor:
    """The next layer's static weight (rows = input features) re-laid out once, offline, so it
    consumes a BLR_OUT_TRANSPOSED Monarch output directly (optimization (3)):
    W'[j] = W[perm[j]]."""
    perm = transposed_row_perm(b2, q).to(W.device)
    return W.index_select(0, perm).contiguous()


def monarch_matmul(X: torch.Tensor, V: torch.Tensor, U: torch.Tensor, b1: int, b2: int,
                   v_layout: int = B2_FASTEST, out=None, workspace=None, out_order: int = OUT_CANONICAL):
    """Monarch Y_k = sum_l X_l V_{l,k} U_{l,k}; V [b1, r'b2, p], U [b2, q, b1 r'].
    out_order OUT_TRANSPOSED writes Y[t, c*b2 + k] instead of Y[t, k*q + c]."""
    lib = load()
    n, i = X.shape
    if V.dim() != 3 or U.dim() != 3 or V.shape[0] != b1 or U.shape[0] != b2:
        raise ValueError("factor shapes must be V [b1, r'*b2, p], U [b2, q, b1*r']")
    rp = V.shape[1] // b2
    p, q = V.shape[2], U.shape[1]
    if V.shape[1] != rp * b2 or U.shape[2] != b1 * rp or p * b1 != i:
        raise ValueError("inconsistent Monarch factor shapes")
    o = q * b2
    Y = _out(X, n, o, out)
    ws = _ws(X, lib.blr_monarch_workspace_size(n, i, o, b1, b2, rp), workspace)
    with torch.cuda.device(X.device):
        code = lib.blr_monarch_matmul(_dev_bf16("X", X), n, i, o, b1, b2, rp, _dev_bf16("V", V),
                                      _dev_bf16("U", U), int(v_layout), int(out_order), _dev_bf16("out", Y),
                                      ws.data_ptr(), ws.numel() * ws.element_size(), _stream_ptr(X.device))
    _check("blr_monarch_matmul", code)
    return Y


def blast_kmajor_factors(V: torch.Tensor, U: torch.Tensor):
    """The one-time static re-layout of blr_blast_matmul_kmajor (paper's optimization (1) applied to
    BLAST): Vt [b1, r, p] = V^T per block, Ut [b2, q, r] = U^T per block."""
    return V.transpose(1, 2).contiguous(), U.transpose(1, 2).contiguous()


def blast_matmul(X: torch.Tensor, V: torch.Tensor, S: torch.Tensor, U: torch.Tensor, out=None,
                 workspace=None, fp8_intermediate: bool = False, kmajor: bool = False):
    """BLAST Y_k = (sum_l (X_l V_l) S_{l,k}) U_k; V [b1,p,r], S [b1,b2,r], U [b2,r,q].
    fp8_intermediate=True calls blr_blast_matmul_fp8z (e4m3 Z; its own accuracy contract, blr.h).
    kmajor=True: V, U are blast_kmajor_factors(V, U) (Vt [b1,r,p], Ut [b2,q,r]) and the call goes to
    blr_blast_matmul_kmajor (split tensor-core path only; same result)."""
    lib = load()
    n, i = X.shape
    if kmajor:
        if fp8_intermediate:
            raise ValueError("kmajor and fp8_intermediate are separate entry points")
        b1, r, p = V.shape
        b2u, q, ru = U.shape
    else:
        b1, p, r = V.shape
        b2u, ru, q = U.shape
    b1s, b2, rs = S.shape
    if b1s != b1 or rs != r or b2u != b2 or ru != r or b1 * p != i:
        raise ValueError("inconsistent BLAST factor shapes")
    o = b2 * q
    Y = _out(X, n, o, out)
    ws = _ws(X, lib.blr_blast_workspace_size(n, i, o, b1, b2, r), workspace)
    with torch.cuda.device(X.device):
        fn = (lib.blr_blast_matmul_kmajor if kmajor else
              lib.blr_blast_matmul_fp8z if fp8_intermediate else lib.blr_blast_matmul)
        code = fn(_dev_bf16("X", X), n, i, o, b1, b2, r, _dev_bf16("V", V),
                  _dev_bf16("S", S), _dev_bf16("U", U), _dev_bf16("out", Y),
                  ws.data_ptr(), ws.numel() * ws.element_size(), _stream_ptr(X.device))
    _check("blr_blast_matmul_kmajor" if kmajor else
           "blr_blast_matmul_fp8z" if fp8_intermediate else "blr_blast_matmul", code)
    return Y
