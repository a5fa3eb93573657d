#!/bin/bash
# attention CTA padded to 8 warps with setmaxnreg (libsparge.so) vs 6 warps (libsparge_6w.so)
O=gpurun_out/s19
mkdir -p $O
python -m pytest tests -m gpu -q -x --timeout 1500 > $O/pytest.log 2>&1; tail -3 $O/pytest.log
for w in mochi_22k cogvideox_2b llama31_8b_32k; do python scripts/cta_timeline.py $w; done > $O/cta.txt 2>&1; cat $O/cta.txt
rm -f $O/ab.txt
for w in ${WL:-mochi_22k cogvideox_2b mochi flux llama31_8b_32k sweep_8k sweep_128k}; do
for lib in libsparge_6w.so libsparge.so; do
  SPARGE_LIB=$lib python bench.py --workload $w --profile --steps 20 --warmup 3 --no-sweep --no-cpu-baseline --no-f1 --no-e2e --no-dense \
    --out $O/ab_$w.json > /dev/null 2>&1
  python -c "import json; r=json.load(open('$O/ab_$w.json')); print('$lib $w', round(r['value'],1), round(r['ms_per_step'],4), {k: round(v,4) for k,v in r['stages_ms'].items()}, 'frac', round(r['roofline']['frac'],3), r['clocks'].get('sm_mhz'))" >> $O/ab.txt 2>&1
done; done
cat $O/ab.txt
