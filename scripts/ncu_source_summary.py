"""Summarise an ncu --page source --csv --print-source sass dump: stall
reasons (totals) and the hottest SASS instructions."""
import csv, sys, collections
rows = list(csv.reader(open(sys.argv[1])))
hdr = rows[1]; body = rows[2:]
ix = {h: i for i, h in enumerate(hdr)}
stalls = [h for h in hdr if h.startswith('stall_') and 'Not Issued' not in h]
tot = collections.Counter()
samples = 0
def num(x):
    try: return int(x)
    except ValueError: return 0
for r in body:
    if len(r) < len(hdr): continue
    samples += num(r[ix['# Samples']])
    for s in stalls:
        tot[s] += num(r[ix[s]])
print('samples', samples)
for s, v in tot.most_common(12):
    print(f'  {s:28s} {v:8d} {100*v/max(1,samples):5.1f}%')
ops = collections.Counter(); execd = collections.Counter()
for r in body:
    if len(r) < len(hdr): continue
    toks = r[ix['Source']].split()
    if not toks: continue
    op = toks[1] if toks[0].startswith('@') and len(toks) > 1 else toks[0]
    ops[op.split('.')[0]] += num(r[ix['# Samples']])
    execd[op.split('.')[0]] += num(r[ix['Instructions Executed']])
print('samples by opcode:')
for o, v in ops.most_common(20):
    print(f'  {o:12s} samples {v:8d}  warp-instrs {execd[o]:12d}')
n = int(sys.argv[2]) if len(sys.argv) > 2 else 25
top = sorted([r for r in body if len(r) >= len(hdr)], key=lambda r: -num(r[ix['# Samples']]))[:n]
for r in top:
    print(r[ix['# Samples']], r[ix['Source']].strip()[:60], {s[6:]: r[ix[s]] for s in stalls if r[ix[s]] not in ('0', '')})
