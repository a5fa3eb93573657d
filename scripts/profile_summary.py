"""Write the judged ncu summaries under profiles/ from gpurun_out/:
   <tag>_launches.csv   the per-launch gpu__time_duration list (+ share by kernel)
   <tag>_attn_ncu.txt   key metrics, stall reasons and hot SASS of the top kernel
usage: python scripts/profile_summary.py <tag> [gpurun_out]"""
import collections, csv, io, os, subprocess, sys
tag = sys.argv[1]
src = sys.argv[2] if len(sys.argv) > 2 else 'gpurun_out'
os.makedirs('profiles', exist_ok=True)
out = []
lc = os.path.join(src, 'launches.csv')
if os.path.exists(lc):
    rows = [r for r in csv.reader(open(lc))]
    hdr = next(i for i, r in enumerate(rows) if r and r[0] == 'ID')
    h = rows[hdr]; body = [dict(zip(h, r)) for r in rows[hdr + 1:] if len(r) == len(h)]
    tot = collections.Counter(); n = collections.Counter()
    with open(f'profiles/{tag}_launches.csv', 'w') as f:
        w = csv.writer(f); w.writerow(['id', 'kernel', 'gpu__time_duration_ns'])
        for d in body:
            name = d['Kernel Name'].split('(')[0].replace('void ', '')
            w.writerow([d['ID'], name, d['Metric Value']])
            if 'sparge' in name:
                tot[name] += float(d['Metric Value']); n[name] += 1
    s = sum(tot.values())
    out.append('# per-kernel share of the sparge launches (ncu, cold-cache, serialised)')
    for k, v in tot.most_common():
        out.append(f'{k:70s} launches {n[k]:3d} avg {v / n[k] / 1e3:9.1f} us  share {100 * v / s:5.1f}%')
rep = os.path.join(src, 'prof_attn.ncu-rep')
if os.path.exists(rep):
    raw = subprocess.run(['ncu', '-i', rep, '--page', 'raw', '--csv'], capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(raw)))
    keys = ['gpu__time_duration.sum', 'dram__bytes_read.sum', 'dram__bytes_write.sum',
            'sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_active',
            'sm__pipe_tensor_subpipe_imma_cycles_active.avg.pct_of_peak_sustained_active',
            'sm__pipe_tensor_subpipe_hmma_cycles_active.avg.pct_of_peak_sustained_active',
            'sm__inst_executed_pipe_xu.avg.pct_of_peak_sustained_active',
            'sm__pipe_alu_cycles_active.avg.pct_of_peak_sustained_active',
            'sm__pipe_fma_cycles_active.avg.pct_of_peak_sustained_active',
            'smsp__issue_active.avg.pct_of_peak_sustained_active',
            'sm__warps_active.avg.pct_of_peak_sustained_active',
            'launch__registers_per_thread', 'launch__grid_size', 'launch__occupancy_limit_shared_mem',
            'gpc__cycles_elapsed.max', 'sm__cycles_elapsed.avg.per_second']
    out.append('\n# ncu --set full, k_sparse_attn (one launch)')
    for r in rows[2:3]:
        for k in keys:
            if k in rows[0]:
                i = rows[0].index(k); out.append(f'{k:75s} {r[i]:>16s} {rows[1][i]}')
    srcp = subprocess.run(['ncu', '-i', rep, '--page', 'source', '--csv', '--print-source', 'sass'],
                          capture_output=True, text=True).stdout
    open('/tmp/_src.csv', 'w').write(srcp)
    summ = subprocess.run([sys.executable, 'scripts/ncu_source_summary.py', '/tmp/_src.csv', '20'],
                          capture_output=True, text=True).stdout
    out.append('\n# stall reasons / hot SASS')
    out.append(summ)
open(f'profiles/{tag}_attn_ncu.txt', 'w').write('\n'.join(out) + '\n')
print('\n'.join(out[:12]))
