"""Warp-stall samples per kernel source line with inlined helpers charged to their call site.

From an `ncu --page source --csv --print-source cuda,sass` export (one kernel): every SASS
instruction is mapped to its source line; instructions of inlined helpers (another file) are
charged to the kernel-file line that precedes them in address order, and out-of-line spin loops
(after the function's last EXIT) to the line of the address they branch back to.
usage: python scripts/ncu_lines.py export.csv kernel_file.cuh [ranges...]
  a range is name=lo-hi over kernel-file lines; stall totals and reasons are printed per range."""
import csv
import re
import sys
from collections import Counter, defaultdict

rows = list(csv.reader(open(sys.argv[1])))
kfile = sys.argv[2]
ranges = []
for a in sys.argv[3:]:
    n, lh = a.split("=")
    lo, hi = lh.split("-")
    ranges.append((n, int(lo), int(hi)))
fname = "?"
line = None
hdr = None
ins = {}
for r in rows:
    if not r:
        continue
    if r[0] in ("File Path", "File Name"):
        fname = r[1].split("/")[-1]
        continue
    if r[0] == "Line No":
        hdr = r
        continue
    if r[0].isdigit():
        line = (fname, int(r[0]))
        continue
    if r[0] == "" and len(r) > 3 and r[2].startswith("0x"):
        st = {}
        for i, h in enumerate(hdr):
            if i > 3 and h.startswith("stall_") and "Not Issued" not in h:
                st[h] = int(r[i] or 0)
        v = int(r[4] or 0)
        ins[int(r[2], 16)] = (line, r[3].strip(), v, st)
addrs = sorted(ins)
exit_at = max([a for a in addrs if "EXIT" in ins[a][1]] or [addrs[-1]])
charge = {}
last_k = None
for a in addrs:
    ln = ins[a][0]
    if ln and ln[0] == kfile:
        last_k = ln[1]
    charge[a] = last_k
block = []
for a in addrs:
    if a <= exit_at:
        continue
    block.append(a)
    m = re.match(r"(?:@!?U?P\d+\s+)?BRA (0x[0-9a-f]+)", ins[a][1])
    if m and not ins[a][1].startswith("@"):
        tgt = int(m.group(1), 16)
        for b in block:
            charge[b] = charge.get(tgt)
        block = []
per = defaultdict(int)
reasons = defaultdict(Counter)
for a in addrs:
    per[charge[a]] += ins[a][2]
    for h, x in ins[a][3].items():
        reasons[charge[a]][h] += x
tot = sum(per.values())
print("total samples", tot)
for n, lo, hi in ranges:
    v = sum(c for l, c in per.items() if l is not None and lo <= l <= hi)
    rc = Counter()
    for l, c in reasons.items():
        if l is not None and lo <= l <= hi:
            rc.update(c)
    print(f"  {n:10s} {v:8d} {100.0 * v / max(tot, 1):5.1f}%  {rc.most_common(4)}")
print("top lines:")
for l, c in sorted(per.items(), key=lambda kv: -kv[1])[:25]:
    print(f"  {c:8d} {100.0 * c / max(tot, 1):5.1f}%  L{l}  {reasons[l].most_common(2)}")
