#!/bin/bash
# 8-warp attention CTA: setmaxnreg split softmax/other 160/96, 168/88 (libsparge.so), 176/80 vs 6 warps
O=gpurun_out/s18
mkdir -p $O
rm -f $O/ab.txt
for w in ${WL:-mochi_22k cogvideox_2b llama31_8b_32k flux}; do
for lib in libsparge_6w.so libsparge_r160.so libsparge.so libsparge_r176.so; do
  SPARGE_LIB=$lib python bench.py --workload $w --profile --steps 20 --warmup 3 --no-sweep --no-cpu-baseline --no-f1 --no-e2e --no-dense \
    --out $O/ab_$w.json > /dev/null 2>&1
  python -c "import json; r=json.load(open('$O/ab_$w.json')); print('$lib $w', round(r['value'],1), round(r['ms_per_step'],4), {k: round(v,4) for k,v in r['stages_ms'].items()}, r['clocks'].get('sm_mhz'))" >> $O/ab.txt 2>&1
done; done
cat $O/ab.txt
