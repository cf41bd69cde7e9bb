"""Workload shapes: PAPER.md Table 3 (L316-413) and BASELINE.json ``configs`` C1..C5.

Host-side data only (no method arithmetic).  Derived block sizes follow PAPER.md L48:
p = i/b1, q = o/b2; Monarch per-block rank r' = r/b (L59, symmetric b1 = b2 = b).
"""
from __future__ import annotations

from dataclasses import dataclass


@dataclass(frozen=True)
class Layer:
    model: str
    name: str
    i: int          # input features
    o: int          # output features
    method: str     # "lowrank" | "monarch" | "blast"
    r: int          # rank (Monarch: total rank r = r' b)
    b: int = 1      # blocks, b1 = b2 = b (Table 3 "(r, b)")

    @property
    def b1(self) -> int:
        return self.b if self.method != "lowrank" else 1

    @property
    def b2(self) -> int:
        return self.b if self.method != "lowrank" else 1

    @property
    def p(self) -> int:
        return self.i // self.b1

    @property
    def q(self) -> int:
        return self.o // self.b2

    @property
    def r_blk(self) -> int:
        """Monarch per-block rank r' = r / b."""
        assert self.method == "monarch"
        return self.r // self.b


def _rows(model, name, i, o, lr, mon, bl):
    out = []
    if lr is not None:
        out.append(Layer(model, name, i, o, "lowrank", lr, 1))
    if mon is not None:
        out.append(Layer(model, name, i, o, "monarch", mon[0], mon[1]))
    if bl is not None:
        out.append(Layer(model, name, i, o, "blast", bl[0], bl[1]))
    return out


# PAPER.md Table 3 (L330-407), one entry per (model, layer, method).
TABLE3 = (
    _rows("Llama-7B", "qkvo_proj", 4096, 4096, 1024, (1024, 16), (1024, 16))
    + _rows("Llama-7B", "gate_up_proj", 4096, 11008, 1488, (1536, 16), (1488, 16))
    + _rows("Llama-7B", "down_proj", 11008, 4096, 1488, (1536, 16), (1488, 16))
    + _rows("Llama-3.2-1B", "q_o_proj", 2048, 2048, 256, (256, 16), (256, 16))
    + _rows("Llama-3.2-1B", "gate_proj", 2048, 8192, 512, (512, 16), (512, 16))
    + _rows("Llama-3.2-1B", "up_proj", 2048, 8192, 768, (768, 16), (768, 16))
    + _rows("Llama-3.2-1B", "down_proj", 8192, 2048, 768, (768, 16), (768, 16))
    + _rows("GPT2-S", "c_attn", 768, 2304, 192, (192, 4), (192, 6))
    + _rows("GPT2-S", "c_fc", 768, 3072, 192, (192, 4), (192, 6))
    + _rows("GPT2-S", "c_proj", 3072, 768, 192, (192, 4), (192, 6))
    + _rows("ViT-B", "attn_qkv", 768, 2304, 128, (128, 4), (128, 3))
    + _rows("ViT-B", "fc1", 768, 3072, 128, (128, 4), (128, 3))
    + _rows("ViT-B", "fc2", 3072, 768, 128, (128, 4), (128, 3))
    + _rows("DiT-XL/2", "qkv_proj", 1152, 3456, 384, None, (384, 9))
    + _rows("DiT-XL/2", "fc1", 1152, 4608, 256, None, (256, 9))
    + _rows("DiT-XL/2", "adaLN_proj", 1152, 6912, 256, None, (256, 9))
)


def table3(model: str, name: str, method: str) -> Layer:
    for L in TABLE3:
        if L.model == model and L.name == name and L.method == method:
            return L
    raise KeyError((model, name, method))


@dataclass(frozen=True)
class Workload:
    key: str
    desc: str
    n: int                      # tokens in one step (batch x seq)
    layers: tuple               # Layer objects run back to back in one step
    fp8z: bool = False          # BLAST layers through blr_blast_matmul_fp8z (e4m3 Z)
    kmajor: bool = False        # BLAST layers through blr_blast_matmul_kmajor (statically re-laid-out V, U)


# BASELINE.json configs (SURVEY.md §8 labels C1..C5).
C1 = Workload("C1", "single BLAST linear 768x768, b=4, r=16, 128 tokens", 128,
              (Layer("synthetic", "blast768", 768, 768, "blast", 16, 4),))

# configs[1]: GPT2-S MLP c_fc (768->3072) then c_proj (3072->768), batch 8 x seq 1024.
C2 = Workload("C2", "GPT2-S MLP (768->3072->768) Monarch and BLAST (+LR), batch 8 x seq 1024",
              8 * 1024,
              tuple(table3("GPT2-S", nm, m) for m in ("lowrank", "monarch", "blast")
                    for nm in ("c_fc", "c_proj")))

C3 = Workload("C3", "Llama-3.2-1B q/o, gate, up, down projections, prefill seq 4096", 4096,
              tuple(table3("Llama-3.2-1B", nm, m) for m in ("lowrank", "monarch", "blast")
                    for nm in ("q_o_proj", "gate_proj", "up_proj", "down_proj")))

C4 = Workload("C4", "Llama-7B MLP (4096<->11008) BLAST prefill seq 8192 x batch 8", 8 * 8192,
              (table3("Llama-7B", "gate_up_proj", "blast"), table3("Llama-7B", "down_proj", "blast")))

C4_MONARCH = Workload("C4M", "Llama-7B MLP (4096<->11008) Monarch prefill seq 8192 x batch 8",
                      8 * 8192,
                      (table3("Llama-7B", "gate_up_proj", "monarch"),
                       table3("Llama-7B", "down_proj", "monarch")))


# >= 2x parameter compression at the Llama-7B MLP (north_star target; SURVEY §8(d) compression
# note): BLAST r = 1456 (CF 2.016) and Monarch r' = 88 (r = 1408, CF 2.12).  Table 3's own ranks
# (C4 / C4M) give CF 1.97 / 1.94.
C4_2X = Workload("C4X", "Llama-7B MLP (4096<->11008) at >=2x compression: BLAST r=1456, Monarch r'=88, seq 8192 x batch 8",
                 8 * 8192,
                 (Layer("Llama-7B", "gate_up_proj", 4096, 11008, "blast", 1456, 16),
                  Layer("Llama-7B", "down_proj", 11008, 4096, "blast", 1456, 16),
                  Layer("Llama-7B", "gate_up_proj", 4096, 11008, "monarch", 1408, 16),
                  Layer("Llama-7B", "down_proj", 11008, 4096, "monarch", 1408, 16)))


# C4 through the FP8-intermediate entry point (its own accuracy contract, include/blr.h)
C4_FP8 = Workload("C4F8", "Llama-7B MLP (4096<->11008) BLAST prefill seq 8192 x batch 8, e4m3 first-stage intermediate",
                  8 * 8192, C4.layers, fp8z=True)


# C4 with the BLAST factors statically re-laid-out K-major once (blr_blast_matmul_kmajor, the
# paper's optimization (1) applied to BLAST)
C4_KMAJOR = Workload("C4K", "Llama-7B MLP (4096<->11008) BLAST prefill seq 8192 x batch 8, K-major factor storage",
                     8 * 8192, C4.layers, kmajor=True)


def c5(images: int) -> Workload:
    """ViT-B layers (197 tokens per image, Table 3): qkv, fc1, fc2 in Monarch
    (r = 128, b = 4) and BLAST (r = 128, b = 3)."""
    vit = tuple(table3("ViT-B", nm, m) for m in ("monarch", "blast") for nm in ("attn_qkv", "fc1", "fc2"))
    return Workload(f"C5V-{images}", f"ViT-B layers, {images} images x 197 tokens", 197 * images, vit)


def c5_dit(images: int) -> Workload:
    """DiT-XL/2 layers (256 tokens per image at 256x256 / patch 2, reading
    R15): QKV (r = 384, b = 9) and fc1 (r = 256, b = 9), BLAST (the paper has no DiT Monarch)."""
    dit = (table3("DiT-XL/2", "qkv_proj", "blast"), table3("DiT-XL/2", "fc1", "blast"))
    return Workload(f"C5D-{images}", f"DiT-XL/2 layers, {images} images x 256 tokens", 256 * images, dit)


C5_IMAGES = (1, 8, 64, 256)   # BASELINE.json configs[4]: batch sweep 1-256 images

WORKLOADS = {w.key: w for w in (C1, C2, C3, C4, C4_MONARCH, C4_2X, C4_FP8, C4_KMAJOR)}
for _im in C5_IMAGES:
    WORKLOADS[f"C5V-{_im}"] = c5(_im)
    WORKLOADS[f"C5D-{_im}"] = c5_dit(_im)
