"""Aggregate an ncu `--page source --csv --print-source sass` dump by opcode:
instructions executed and stall samples per opcode, for the first kernel
in the file (or the one whose name contains argv[2])."""
import csv
import sys
from collections import defaultdict

path = sys.argv[1]
want = sys.argv[2] if len(sys.argv) > 2 else None
rows = list(csv.reader(open(path)))
cnt, smp = defaultdict(int), defaultdict(int)
active, hdr, total = None, None, 0
for r in rows:
    if r and r[0] == "Kernel Name":
        active = (want is None and active is None) or (want is not None and want in r[1])
        hdr = None
        continue
    if r and r[0] == "Address":
        hdr = {h: i for i, h in enumerate(r)}
        continue
    if not active or hdr is None or len(r) < 5:
        continue
    op = r[hdr["Source"]].strip().split()
    if not op:
        continue
    o = op[0]
    if o.startswith("@"):
        o = op[1] if len(op) > 1 else o
    o = o.split(".")[0]
    n = int(r[hdr["Instructions Executed"]] or 0)
    s = int(r[hdr["Warp Stall Sampling (All Samples)"]] or 0)
    cnt[o] += n
    smp[o] += s
    total += n
print(f"total warp instructions {total}")
for o in sorted(cnt, key=lambda k: -cnt[k])[:40]:
    print(f"{o:12s} {cnt[o]:12d} {100.0 * cnt[o] / max(total, 1):6.2f}%  stall samples {smp[o]}")
