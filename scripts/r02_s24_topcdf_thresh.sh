#!/bin/bash
# TopCdf kernel choice after the bulk row copy: warp-per-row below T_n=1024 (default) vs CTA-per-row from T_n > 256
O=gpurun_out/s24
mkdir -p $O
rm -f $O/ab.txt
for w in ${WL:-llama31_8b_32k mochi cogvideox_2b sweep_64k mochi_22k}; do
for t in 1024 256 1024 256; do
  SPARGE_TOPCDF_CTA_MIN_TN=$t timeout 300 python bench.py --workload $w --profile --steps 20 --warmup 3 --no-sweep --no-cpu-baseline --no-f1 --no-e2e --no-dense \
    --out $O/ab_$w.json > /dev/null 2>&1
  python -c "import json; r=json.load(open('$O/ab_$w.json')); print('ctamin=$t $w', round(r['value'],1), round(r['ms_per_step'],4), {k: round(v,4) for k,v in r['stages_ms'].items()})" >> $O/ab.txt 2>&1
done; done
cat $O/ab.txt
