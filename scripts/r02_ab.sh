#!/bin/bash
# A/B helper: GPU suite (optional -k filter in $K), stage times per workload for
# each library in $LIBS (default libsparge.so), optional ncu launch list ($LL=workload)
O=gpurun_out
LIBS=${LIBS:-libsparge.so}
WL=${WL:-"llama31_8b_32k cogvideox_2b mochi sweep_128k"}
if [ -n "$K" ]; then python -m pytest tests -m gpu -q -x --timeout 1500 -k "$K" > $O/ab_pytest.log 2>&1;
else python -m pytest tests -m gpu -q -x --timeout 1500 > $O/ab_pytest.log 2>&1; fi
tail -3 $O/ab_pytest.log
rm -f $O/ab.txt
for lib in $LIBS; do for w in $WL; do
  SPARGE_LIB=$lib python bench.py --workload $w --profile --steps 10 --warmup 3 --no-sweep --no-cpu-baseline --no-f1 --no-e2e --no-dense \
    --out $O/ab_$w.json > /dev/null 2>&1
  python -c "import json; r=json.load(open('$O/ab_$w.json')); print('$lib $w', round(r['value'],1), {k: round(v,4) for k,v in r['stages_ms'].items()})" >> $O/ab.txt 2>&1
done; done
cat $O/ab.txt
if [ -n "$LL" ]; then
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $O/ab_launch.csv \
  python bench.py --workload $LL --profile --steps 1 --warmup 0 --no-sweep --no-cpu-baseline --no-f1 --no-e2e --no-dense > /dev/null 2>&1
python - <<'PY'
import csv
rows=list(csv.reader(open('gpurun_out/ab_launch.csv'))); hdr=None
for r in rows:
    if 'Kernel Name' in r: hdr={h:i for i,h in enumerate(r)}; continue
    if hdr and len(r)>5 and r[hdr['Metric Name']]=='gpu__time_duration.sum':
        print(f"{r[hdr['Kernel Name']][:50]:50s} {r[hdr['Metric Value']]:>12s}")
PY
fi
