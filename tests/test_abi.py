"""C-ABI checks that need no GPU: the library loads, exports every symbol include/blr.h declares,
and host-side validation returns the documented status codes before touching CUDA."""
import ctypes
import os
import re

import pytest

import paper_2512_20861_b200 as blr

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
HDR = os.path.join(ROOT, "include", "blr.h")


def declared_symbols():
    src = open(HDR).read()
    src = re.sub(r"/\*.*?\*/", "", src, flags=re.S)
    return sorted(set(re.findall(r"\b(blr_[a-z_]+)\s*\(", src)))


def test_header_declares_entry_points():
    syms = declared_symbols()
    for s in ("blr_lowrank_matmul", "blr_monarch_matmul", "blr_blast_matmul", "blr_status_string",
              "blr_lowrank_workspace_size", "blr_monarch_workspace_size", "blr_blast_workspace_size"):
        assert s in syms


def test_library_exports_every_declared_symbol():
    blr.build()
    lib = ctypes.CDLL(blr.lib_path())
    for s in declared_symbols():
        assert hasattr(lib, s), s


def test_status_strings_and_version():
    lib = blr.load()
    names = [lib.blr_status_string(c).decode() for c in range(8)]
    assert names == ["BLR_OK", "BLR_ERR_NULL", "BLR_ERR_SHAPE", "BLR_ERR_ALIGN", "BLR_ERR_UNSUPPORTED",
                     "BLR_ERR_WORKSPACE", "BLR_ERR_ARCH", "BLR_ERR_CUDA"]
    assert re.match(r"\d+\.\d+\.\d+", lib.blr_version().decode())


def test_workspace_sizes():
    lib = blr.load()
    # n above the weight-streaming path's range (DTC_MAX_N = 4096): only the tcgen05 path's intermediate
    n = 5000
    # S3 contraction >= 128: one bf16 intermediate
    assert lib.blr_lowrank_workspace_size(n, 64, 64, 128) == n * 128 * 2
    assert lib.blr_monarch_workspace_size(n, 64, 64, 4, 2, 32) == 2 * n * 4 * 32 * 2
    # BLAST with b1*r <= 512 fuses S1+S2 (only Z''); larger b1*r also keeps the S1 output Z_l
    assert lib.blr_blast_workspace_size(n, 64, 64, 2, 2, 192) == 2 * n * 192 * 2
    # split path: Z'' and fp16 Z (R13), token rows padded to whole 128-row tiles (tile-blocked, §5.4),
    # then the pipelined layer's counters (ticket + 2 x 40 token tiles of 4 B, rounded up to 256 B)
    assert lib.blr_blast_workspace_size(n, 64, 64, 4, 2, 192) == 2 * 5120 * 192 * 2 + 4 * 5120 * 192 * 2 + 512
    # shorter contractions keep a compensated hi|lo pair: twice the bytes
    assert lib.blr_lowrank_workspace_size(n, 64, 64, 16) == 2 * n * 16 * 2
    assert lib.blr_monarch_workspace_size(n, 64, 64, 4, 2, 8) == 2 * 2 * n * 4 * 8 * 2
    assert lib.blr_blast_workspace_size(n, 64, 64, 4, 2, 16) == 2 * 2 * n * 16 * 2  # fused (b1 r <= 512)
    assert lib.blr_blast_workspace_size(0, 64, 64, 4, 2, 16) == 0
    # n <= DTC_MAX_N: the larger of the tcgen05 intermediate and the fp32 weight-streaming one
    assert lib.blr_lowrank_workspace_size(100, 64, 64, 128) == max(100 * 128 * 2, 100 * 128 * 4)


def test_workspace_sizes_cover_the_decode_path():
    """n <= 16 (decode path): fp32 intermediates (+ split-K partials) must fit too."""
    lib = blr.load()
    n, i, o, r = 8, 4096, 11008, 1488
    assert lib.blr_lowrank_workspace_size(n, i, o, r) >= n * r * 4          # fp32 Z
    assert lib.blr_blast_workspace_size(n, i, o, 16, 16, r) >= (16 + 16) * n * r * 4  # fp32 Z, Z''
    assert lib.blr_monarch_workspace_size(n, i, o, 16, 16, 96) >= 16 * n * 16 * 96 * 4  # fp32 Z'
    # above the weight-streaming range only the tcgen05 path's bf16 intermediate is needed
    assert lib.blr_lowrank_workspace_size(4097, i, o, r) == 4097 * r * 2


FAKE = 0x10000  # 16-B aligned, never dereferenced: validation fails before any CUDA call


@pytest.mark.parametrize("args,code", [
    # (n, i, o, b1, b2, r) -> expected status
    ((-1, 64, 64, 2, 2, 16), 2),   # n < 0
    ((8, 64, 64, 3, 2, 16), 2),    # b1 does not divide d_in
    ((8, 64, 64, 2, 3, 16), 2),    # b2 does not divide d_out
    ((8, 64, 64, 2, 2, 12), 3),    # r not a multiple of 8
    ((8, 48, 64, 4, 2, 16), 3),    # p = 12 not a multiple of 8
    ((8, 544, 64, 17, 2, 16), 4),  # b1 > 16 unsupported
])
def test_blast_validation(args, code):
    lib = blr.load()
    n, i, o, b1, b2, r = args
    st = lib.blr_blast_matmul(FAKE, n, i, o, b1, b2, r, FAKE, FAKE, FAKE, FAKE, FAKE, 1 << 40, None)
    assert st == code, (args, lib.blr_status_string(st))


def test_null_and_workspace_errors():
    lib = blr.load()
    assert lib.blr_blast_matmul(None, 8, 64, 64, 2, 2, 16, FAKE, FAKE, FAKE, FAKE, FAKE, 1 << 40, None) == 1
    assert lib.blr_blast_matmul(FAKE, 8, 64, 64, 2, 2, 16, FAKE, FAKE, FAKE, FAKE, FAKE, 10, None) == 5
    assert lib.blr_lowrank_matmul(FAKE, 8, 64, 64, 16, FAKE, FAKE, FAKE, FAKE, 10, None) == 5
    assert lib.blr_lowrank_matmul(FAKE + 8, 8, 64, 64, 16, FAKE, FAKE, FAKE, FAKE, 1 << 40, None) == 3
    # n_tok == 0 is a successful no-op even with NULL pointers
    assert lib.blr_lowrank_matmul(None, 0, 64, 64, 16, None, None, None, None, 0, None) == 0


def test_monarch_validation():
    lib = blr.load()
    # an out_order outside {CANONICAL, TRANSPOSED} is rejected before any device access
    assert lib.blr_monarch_matmul(FAKE, 8, 64, 64, 2, 2, 8, FAKE, FAKE, 0, 5, FAKE, FAKE, 1 << 40, None) == 2
    # invalid V layout flag
    assert lib.blr_monarch_matmul(FAKE, 8, 64, 64, 2, 2, 8, FAKE, FAKE, 7, 0, FAKE, FAKE, 1 << 40, None) == 2
    # r' not a multiple of 8
    assert lib.blr_monarch_matmul(FAKE, 8, 64, 64, 2, 2, 4, FAKE, FAKE, 0, 0, FAKE, FAKE, 1 << 40, None) == 3


@pytest.mark.skipif(__import__("torch").cuda.is_available(), reason="CPU-only check")
def test_no_gpu_fails_loudly():
    """Without a device the valid call returns an error code (no silent CPU fallback)."""
    lib = blr.load()
    st = lib.blr_lowrank_matmul(FAKE, 8, 64, 64, 16, FAKE, FAKE, FAKE, FAKE, 1 << 40, None)
    assert st in (6, 7)


def test_transposed_row_perm_closed_form_and_errors():
    """blr_transposed_row_perm: perm[c*b2 + k] = k*q + c, a bijection."""
    import ctypes
    lib = blr.load()
    perm = blr.transposed_row_perm(3, 5)
    assert perm.tolist() == [k * 5 + c for c in range(5) for k in range(3)]
    assert sorted(perm.tolist()) == list(range(15))
    buf = (ctypes.c_int64 * 4)()
    assert lib.blr_transposed_row_perm(0, 4, buf) == 2
    assert lib.blr_transposed_row_perm(2, 2, None) == 1
