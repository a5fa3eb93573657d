#!/bin/bash
# PDL per-site A/B (SPARGE_PDL bit mask: 1 quant Q, 2 quant K, 4 predict, 8 V stage, 16 order, 32 attention)
O=gpurun_out/s11
mkdir -p $O
python -m pytest tests -m gpu -q -x --timeout 1500 > $O/pytest.log 2>&1; tail -3 $O/pytest.log
rm -f $O/ab.txt
for w in ${WL:-flux sweep_8k cogvideox_2b mochi_22k llama31_8b_32k}; do
for m in ${MASKS:-0 0x3f 0x3e 0x3c 0x38}; do
  SPARGE_PDL=$m python bench.py --workload $w --profile --steps 30 --warmup 3 --no-sweep --no-cpu-baseline --no-f1 --no-e2e --no-dense \
    --out $O/ab_$w.json > /dev/null 2>&1
  python -c "import json; r=json.load(open('$O/ab_$w.json')); print('pdl=$m $w', round(r['value'],1), round(r['ms_per_step'],4), {k: round(v,4) for k,v in r['stages_ms'].items()})" >> $O/ab.txt 2>&1
done; done
cat $O/ab.txt
