#!/bin/bash
# quantiser: HEAD library (two launches) vs new kernel (runtime block size) two launches / joint launch
O=gpurun_out/s13
mkdir -p $O
python -m pytest tests -m gpu -q -x --timeout 1500 -k "quant or parity or smooth or f1 or edge" > $O/pytest.log 2>&1; tail -3 $O/pytest.log
rm -f $O/ab.txt
for w in ${WL:-flux sweep_8k cogvideox_2b mochi_22k llama31_8b_32k mochi}; do
for cfg in "libsparge_base.so 1" "libsparge.so 1" "libsparge.so 0"; do
  set -- $cfg
  SPARGE_LIB=$1 SPARGE_BENCH_SPLIT_QK=$2 python bench.py --workload $w --profile --steps 30 --warmup 3 --no-sweep --no-cpu-baseline --no-f1 --no-e2e --no-dense \
    --out $O/ab_$w.json > /dev/null 2>&1
  python -c "import json; r=json.load(open('$O/ab_$w.json')); print('$1 split=$2 $w', round(r['value'],1), round(r['ms_per_step'],4), {k: round(v,4) for k,v in r['stages_ms'].items()})" >> $O/ab.txt 2>&1
done; done
cat $O/ab.txt
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $O/launch_llama.csv \
  python bench.py --profile --steps 2 --warmup 1 --no-sweep --no-cpu-baseline --no-f1 --no-e2e --no-dense > /dev/null 2>&1
