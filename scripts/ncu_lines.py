"""Per-CUDA-source-line totals from `ncu -i X --page source --csv
--print-source sass,cuda` (first function in the dump, or the one whose name
contains argv[2]): instructions executed and stall samples per line."""
import csv
import sys
from collections import defaultdict

rows = list(csv.reader(open(sys.argv[1])))
want = sys.argv[2] if len(sys.argv) > 2 else None
cnt, smp, text = defaultdict(int), defaultdict(int), {}
active, hdr, seen, cur = False, None, 0, '?'
for r in rows:
    if not r:
        continue
    if r[0] == "Function Name":
        seen += 1
        active = (want in r[1]) if want else (seen == 1)
        continue
    if r[0] == "Line No":
        hdr = r
        continue
    if not active or hdr is None or len(r) < 8:
        continue
    # rows: line no, cuda source, address, sass, samples..., inst executed
    if r[0]:
        cur = r[0]
        if r[1]:
            text[cur] = r[1]
        if not r[2]:        # a CUDA line row without its own SASS
            continue
    line = cur
    try:
        cnt[line] += int(r[7] or 0)
        smp[line] += int(r[4] or 0)
    except ValueError:
        pass
tot = sum(cnt.values())
print("total", tot)
for l in sorted(cnt, key=lambda k: -cnt[k])[:int(sys.argv[3]) if len(sys.argv) > 3 else 50]:
    print(f"{l:>5} {cnt[l]:10d} {100.0 * cnt[l] / tot:5.1f}% samp {smp[l]:5d}  {text.get(l, '')[:90].strip()}")
