#!/bin/bash
# launch order: remaining items per L2 group longest first (default) vs shortest first (SPARGE_ORDER_ASC=1)
O=gpurun_out/s22
mkdir -p $O
rm -f $O/ab.txt
for w in ${WL:-mochi_22k cogvideox_2b mochi llama31_8b_32k flux sweep_8k sweep_32k}; do
for a in 0 1; do
  SPARGE_ORDER_ASC=$a timeout 300 python bench.py --workload $w --profile --steps 20 --warmup 3 --no-sweep --no-cpu-baseline --no-f1 --no-e2e --no-dense \
    --out $O/ab_$w.json > /dev/null 2>&1
  python -c "import json; r=json.load(open('$O/ab_$w.json')); print('asc=$a $w', round(r['value'],1), round(r['ms_per_step'],4), {k: round(v,4) for k,v in r['stages_ms'].items()}, r['clocks'].get('sm_mhz'))" >> $O/ab.txt 2>&1
done; done
cat $O/ab.txt
