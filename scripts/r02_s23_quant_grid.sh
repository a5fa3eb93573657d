#!/bin/bash
# quantiser grid: min(jobs, 4 x SMs) (default) vs the same job count per CTA (SPARGE_QUANT_BALANCED=1)
O=gpurun_out/s23
mkdir -p $O
rm -f $O/ab.txt
for w in ${WL:-flux sweep_8k cogvideox_2b mochi_22k llama31_8b_32k mochi}; do
for b in 0 1 0 1; do
  SPARGE_QUANT_BALANCED=$b timeout 300 python bench.py --workload $w --profile --steps 20 --warmup 3 --no-sweep --no-cpu-baseline --no-f1 --no-e2e --no-dense \
    --out $O/ab_$w.json > /dev/null 2>&1
  python -c "import json; r=json.load(open('$O/ab_$w.json')); print('bal=$b $w', round(r['value'],1), round(r['ms_per_step'],4), {k: round(v,4) for k,v in r['stages_ms'].items()})" >> $O/ab.txt 2>&1
done; done
cat $O/ab.txt
