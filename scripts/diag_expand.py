"""Time one LR layer's launches under debug variants (env set per subprocess) + pure write bandwidth."""
import os, subprocess, sys, json
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
variants = [("base", {}), ("nostore", {"BLR_DBG": "1"}), ("nostage", {"BLR_DBG": "2"}), ("neither", {"BLR_DBG": "3"}),
            ("noresident", {"BLR_NO_RESIDENT": "1"}), ("pair2", {"BLR_PAIR": "2"}), ("nopdl", {"BLR_NO_PDL": "1"})]
layer = sys.argv[1] if len(sys.argv) > 1 else "c_fc"
method = sys.argv[2] if len(sys.argv) > 2 else "lowrank"
for name, env in variants:
    e = dict(os.environ, SCAN_N="8192,32768", **env)
    out = subprocess.run([sys.executable, "scripts/scan.py", method, "GPT2-S", layer], env=e, capture_output=True, text=True)
    print(f"--- {name} {env}\n" + out.stdout.strip() + ("\n" + out.stderr[-500:] if out.returncode else ""), flush=True)
import torch
for mb in (50, 200):
    b = torch.empty(mb << 20, dtype=torch.uint8, device="cuda"); src = torch.empty_like(b)
    fl = torch.empty(512 << 20, dtype=torch.uint8, device="cuda")
    for what in ("fill", "copy"):
        ts = []
        for _ in range(10):
            fl.zero_(); s = torch.cuda.Event(enable_timing=True); t = torch.cuda.Event(enable_timing=True)
            s.record(); (b.fill_(1) if what == "fill" else b.copy_(src)); t.record(); torch.cuda.synchronize()
            ts.append(s.elapsed_time(t))
        ts.sort(); ms = ts[len(ts) // 2]
        gb = (mb << 20) * (1 if what == "fill" else 2) / ms / 1e6
        print(f"{what} {mb} MiB after dirty flush: {ms*1e3:.1f} us  {gb:.0f} GB/s")
