"""Top CUDA source lines by warp-stall samples from an `ncu --page source --csv --print-source cuda,sass` export.
usage: python scripts/ncu_stalls.py export.csv [top]"""
import csv
import sys
from collections import defaultdict

rows = list(csv.reader(open(sys.argv[1])))
top = int(sys.argv[2]) if len(sys.argv) > 2 else 25
tot = defaultdict(int)
src = {}
fname = "?"
col = 4
for r in rows:
    if not r:
        continue
    if r[0] in ("File Path", "File Name"):
        fname = r[1].split("/")[-1]
        continue
    if r[0] == "Line No":
        col = r.index("Warp Stall Sampling (All Samples)")
        continue
    if r[0] in ("Function Name", "Kernel Name") or not r[0].isdigit():
        continue
    try:
        v = int(r[col])
    except (ValueError, IndexError):
        v = 0
    key = (fname, int(r[0]))
    tot[key] += v
    src[key] = r[1][:100]
s = sum(tot.values())
print(f"total samples {s}")
for k, v in sorted(tot.items(), key=lambda kv: -kv[1])[:top]:
    print(f"  {v:8d} {100.0 * v / max(s, 1):5.1f}%  {k[0]}:{k[1]:<5} {src[k]}")
