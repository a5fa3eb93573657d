#!/bin/bash
# attention kernel capped at 128 registers (libsparge_r128.so: any 2-CTA warp placement fits)
# vs the 170-register launch bound (libsparge.so, 154 used)
O=gpurun_out/s21
mkdir -p $O
SPARGE_LIB=libsparge_r128.so timeout 900 python -m pytest tests -m gpu -q -x --timeout 600 -k "parity or edge or mpv or pdl or f1 or f4" > $O/pytest_r128.log 2>&1; tail -2 $O/pytest_r128.log
rm -f $O/ab.txt
for w in ${WL:-mochi_22k cogvideox_2b llama31_8b_32k flux mochi sweep_8k}; do
for lib in libsparge.so libsparge_r128.so; do
  SPARGE_LIB=$lib timeout 300 python bench.py --workload $w --profile --steps 20 --warmup 3 --no-sweep --no-cpu-baseline --no-f1 --no-e2e --no-dense \
    --out $O/ab_$w.json > /dev/null 2>&1
  python -c "import json; r=json.load(open('$O/ab_$w.json')); print('$lib $w', round(r['value'],1), round(r['ms_per_step'],4), {k: round(v,4) for k,v in r['stages_ms'].items()}, 'frac', round(r['roofline']['frac'],3), r['clocks'].get('sm_mhz'))" >> $O/ab.txt 2>&1
done; done
cat $O/ab.txt
