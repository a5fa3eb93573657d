#!/bin/bash
# e2e (HostPipeline) with / without the tail split; GPU suite subset
O=gpurun_out/s14
mkdir -p $O
python -m pytest tests -m gpu -q -x --timeout 1500 -k "host_pipeline or parity" > $O/pytest.log 2>&1; tail -3 $O/pytest.log
rm -f $O/ab.txt
for w in llama31_8b_32k mochi cogvideox_2b flux; do
for ts in 0 1; do
  SPARGE_E2E_TAIL_SPLIT=$ts python bench.py --workload $w --steps 10 --warmup 3 --no-sweep --no-cpu-baseline --no-f1 --no-dense \
    --out $O/ab_$w.json > /dev/null 2>&1
  python -c "import json; r=json.load(open('$O/ab_$w.json')); print('tail_split=$ts $w', round(r['value'],1), 'e2e', round(r['e2e']['value'],1), round(r['e2e']['ms_per_step'],3))" >> $O/ab.txt 2>&1
done; done
cat $O/ab.txt
