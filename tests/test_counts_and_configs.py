"""Host-logic pins: closed-form counts (§2, Table 2) and the Table 3 shapes."""
import json
import os

import pytest

from paper_2512_20861_b200 import configs, roofline

GOLD = os.path.join(os.path.dirname(__file__), "golden")


def test_p10_table2_llama7b_qkvo():
    g = json.load(open(os.path.join(GOLD, "table2_llama7b_qkvo.json")))
    s = g["shape"]
    n, i, o, r, b = s["n"], s["i"], s["o"], s["r"], s["b"]
    for m in ("dense", "lowrank", "monarch", "blast"):
        fl = roofline.flops(m, n, i, o, r, b, b)
        by = roofline.table2_bytes(m, n, i, o, r, b)
        assert fl == g["flops"][m], m
        assert by == g["bytes"][m], m
        assert abs(roofline.intensity(fl, by) - g["alpha"][m]) <= 0.05 + 1e-9, m
    assert roofline.params("lowrank", 4096, 4096, 1024) == g["params"]["lowrank_4096_4096_r1024"]
    assert roofline.params("blast", 4096, 4096, 1024, 16, 16) == g["params"]["blast_4096_4096_r1024_b16"]


def test_p10_param_identities():
    # Monarch with b1 = b2 = b, r = r' b recovers the low-rank complexity r(i+o)
    for (i, o, r, b) in [(4096, 11008, 1536, 16), (768, 3072, 192, 4), (2048, 2048, 256, 16)]:
        assert roofline.params("monarch", i, o, r, b, b) == roofline.params("lowrank", i, o, r)
    # BLAST = LR + r b1 b2 diagonal entries (reading R1)
    assert roofline.params("blast", 4096, 11008, 1488, 16, 16) - roofline.params("lowrank", 4096, 11008, 1488) == 1488 * 256
    # fused bytes = Table 2 minus the underlined intermediate terms
    n, i, o, r, b = 1024, 4096, 4096, 1024, 16
    assert roofline.table2_bytes("lowrank", n, i, o, r) - roofline.fused_bytes("lowrank", n, i, o, r) == 2 * 2 * n * r
    assert roofline.table2_bytes("monarch", n, i, o, r, b) - roofline.fused_bytes("monarch", n, i, o, r, b, b) == 2 * 4 * b * n * r
    assert roofline.table2_bytes("blast", n, i, o, r, b) - roofline.fused_bytes("blast", n, i, o, r, b, b) == 2 * 8 * b * n * r


def test_table3_matches_paper_rows():
    rows = []
    for line in open(os.path.join(GOLD, "table3.txt")):
        line = line.split("#")[0].strip()
        if not line:
            continue
        m, nm, i, o, meth, r, b = [f.strip() for f in line.split("|")]
        rows.append((m, nm, int(i), int(o), meth, int(r), int(b)))
    got = [(L.model, L.name, L.i, L.o, L.method, L.r, L.b) for L in configs.TABLE3]
    assert got == rows


def test_derived_block_sizes():
    L = configs.table3("Llama-7B", "gate_up_proj", "blast")
    assert (L.p, L.q) == (256, 688)
    M = configs.table3("Llama-7B", "down_proj", "monarch")
    assert (M.p, M.q, M.r_blk) == (688, 256, 96)
    G = configs.table3("GPT2-S", "c_fc", "monarch")
    assert (G.p, G.q, G.r_blk) == (192, 768, 48)
    assert configs.C2.n == 8192 and configs.C4.n == 65536


def test_roofline_time():
    peaks = {"hbm_gbs": 8000.0, "bf16_tflops": 2250.0}
    assert roofline.roofline_time_s(2250e12, 1, peaks) == pytest.approx(1.0)
    assert roofline.roofline_time_s(1, 8e12, peaks) == pytest.approx(1.0)
