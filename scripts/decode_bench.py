"""Small-token (decode) path measurement: per-layer time at n_tok in {1, 8, 16}
(graph replay, L2 flushed between calls), the factor bytes it must stream, and the fraction of
the measured HBM peak that achieves (the path's roofline: params bytes / HBM bandwidth).  The
prefill (tcgen05) path is timed on the same calls for comparison (BLR_DECODE=0 in a subprocess).

    python scripts/decode_bench.py [--child]     (writes a table to stdout)
"""
import json
import os
import subprocess
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import paper_2512_20861_b200 as blr  # noqa: E402
from paper_2512_20861_b200 import configs, roofline, synth  # noqa: E402

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
LAYERS = [("lowrank", "Llama-7B", "gate_up_proj"), ("monarch", "Llama-7B", "gate_up_proj"),
          ("blast", "Llama-7B", "gate_up_proj"), ("blast", "Llama-7B", "down_proj"),
          ("lowrank", "GPT2-S", "c_fc"), ("blast", "GPT2-S", "c_fc")]
NS = [int(x) for x in os.environ.get("DECODE_NS", "1,8,16").split(",")]


def measure():
    dev = torch.device("cuda")
    blr.load()
    flush = torch.empty(256 << 20, dtype=torch.uint8, device=dev)
    R = 20
    out = {}

    def gtime(fn):
        fn()
        torch.cuda.synchronize()
        g = torch.cuda.CUDAGraph()
        with torch.cuda.graph(g):
            fn()
        best = 1e9
        for _ in range(5):
            a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            a.record()
            g.replay()
            b.record()
            torch.cuda.synchronize()
            best = min(best, a.elapsed_time(b))
        return best * 1e3

    def fl():
        for _ in range(R):
            flush.zero_()

    t_fl = gtime(fl)
    for method, model, layer in LAYERS:
        L = configs.table3(model, layer, method)
        if L.method == "lowrank":
            fac = [t.to(dev) for t in synth.lowrank_factors(L.i, L.o, L.r)]
        elif L.method == "monarch":
            fac = [t.to(dev) for t in synth.monarch_factors(L.i, L.o, L.b1, L.b2, L.r_blk)]
        else:
            fac = [t.to(dev) for t in synth.blast_factors(L.i, L.o, L.b1, L.b2, L.r)]
        for n in NS:
            X = synth.make_x(n, L.i, device=dev)
            Y = torch.empty(n, L.o, dtype=torch.bfloat16, device=dev)
            if L.method == "lowrank":
                call = lambda: blr.lowrank_matmul(X, *fac, out=Y)
            elif L.method == "monarch":
                call = lambda: blr.monarch_matmul(X, *fac, L.b1, L.b2, out=Y)
            else:
                call = lambda: blr.blast_matmul(X, *fac, out=Y)

            def body():
                for _ in range(R):
                    flush.zero_()
                    call()

            out[f"{model}.{layer}.{method}.{n}"] = (gtime(body) - t_fl) / R
    return out


def main():
    if "--child" in sys.argv:
        print(json.dumps(measure()))
        return
    res = {}
    for mode in ("decode", "tcgen05"):
        env = dict(os.environ, BLR_DECODE="1" if mode == "decode" else "0")  # force each path
        p = subprocess.run([sys.executable, __file__, "--child"], env=env, capture_output=True, text=True)
        if p.returncode:
            print(p.stderr[-2000:])
            sys.exit(1)
        res[mode] = json.loads(p.stdout.strip().splitlines()[-1])
    peaks = roofline.load_peaks(ROOT)
    bw = peaks["hbm_gbs"]
    print(f"# decode path (SURVEY §8 f2): graph replay, L2 flushed; roofline = factor bytes / {bw:.0f} GB/s "
          f"({peaks.get('source', 'measured')})")
    print("# layer                              n   decode_us  tcgen05_us  factor_MB  roof_us  frac(decode)")
    for method, model, layer in LAYERS:
        L = configs.table3(model, layer, method)
        pbytes = roofline.BF16 * roofline.params(L.method, L.i, L.o, L.r, L.b1, L.b2)
        for n in NS:
            k = f"{model}.{layer}.{method}.{n}"
            td, tt = res["decode"][k], res["tcgen05"][k]
            troof = (pbytes + roofline.BF16 * n * (L.i + L.o)) / (bw * 1e3)  # us
            print(f"{model + '.' + layer + '.' + method:36s} {n:3d} {td:10.1f} {tt:11.1f} {pbytes / 1e6:10.1f} "
                  f"{troof:8.1f} {troof / td:12.2f}")


if __name__ == "__main__":
    main()
