"""Warp-stall samples of a warp-specialised kernel split by role, from an
`ncu --page source --csv --print-source sass` export (first kernel in the file).
Roles are assigned by landmark instructions in address order (UTMALDG -> producer,
UTCHMMA/UTCBAR -> mma, LDTM/UTMASTG -> epilogue); out-of-line spin loops inherit the role of
the code they branch back to.
usage: python scripts/ncu_roles.py export.csv [kernel_index]"""
import csv
import re
import sys
from collections import Counter, defaultdict

rows = list(csv.reader(open(sys.argv[1])))
kidx = int(sys.argv[2]) if len(sys.argv) > 2 else 0
kernels = []
cur = None
for r in rows:
    if r and r[0] == "Kernel Name":
        cur = {"name": r[1], "rows": []}
        kernels.append(cur)
    elif r and r[0] == "Address":
        cur["hdr"] = r
    elif r and r[0].startswith("0x") and cur is not None:
        cur["rows"].append(r)
k = kernels[kidx]
hdr = k["hdr"]
ci = hdr.index("Warp Stall Sampling (All Samples)")
ie = hdr.index("Instructions Executed")
st = [h for h in hdr if h.startswith("stall_") and "Not Issued" not in h]
sidx = [hdr.index(h) for h in st]
ins = [(int(r[0], 16), r[1].strip(), int(r[ci] or 0), int(r[ie] or 0), [int(r[i] or 0) for i in sidx]) for r in k["rows"]]
addr_role = {}
role = "prologue"
for a, s, *_ in ins:
    if "UTMALDG" in s:
        role = "producer"
    elif "UTCHMMA" in s or "UTCBAR" in s:
        role = "mma"
    elif "LDTM" in s or "UTMASTG" in s or "UBLKCP" in s:
        role = "epilogue"
    addr_role[a] = role
# out-of-line blocks: an unconditional BRA back into the body gives the block its role
last_body = max(a for a, s, *_ in ins if "EXIT" in s) if any("EXIT" in s for _, s, *_ in ins) else ins[-1][0]
block = []
for a, s, *_ in ins:
    if a <= last_body:
        continue
    block.append(a)
    m = re.match(r"BRA (0x[0-9a-f]+)", s)
    if m:
        tgt = int(m.group(1), 16)
        r = addr_role.get(tgt, "?")
        for b in block:
            addr_role[b] = r + "(wait)"
        block = []
tot = defaultdict(int)
stalls = defaultdict(Counter)
for a, s, v, e, sv in ins:
    r = addr_role.get(a, "?")
    tot[r] += v
    for h, x in zip(st, sv):
        stalls[r][h] += x
print(k["name"][:100])
S = sum(tot.values())
for r, v in sorted(tot.items(), key=lambda kv: -kv[1]):
    print(f"  {r:18s} {v:8d} {100.0 * v / S:5.1f}%  {stalls[r].most_common(4)}")
