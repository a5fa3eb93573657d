#!/bin/bash
# PDL A/B: GPU suite on the new library, then stage times per workload for
# base library / new library with SPARGE_PDL=0 / new library (PDL on)
O=gpurun_out/s10
mkdir -p $O
python -m pytest tests -m gpu -q -x --timeout 1500 > $O/pytest.log 2>&1; tail -3 $O/pytest.log
python -c "import __graft_entry__ as g; g.smoke()" 2>&1 | tail -1
rm -f $O/ab.txt
for w in ${WL:-flux cogvideox_2b mochi_22k llama31_8b_32k sweep_8k sweep_128k}; do
for cfg in "libsparge_base.so 1" "libsparge.so 0" "libsparge.so 1"; do
  set -- $cfg
  SPARGE_LIB=$1 SPARGE_PDL=$2 python bench.py --workload $w --profile --steps 20 --warmup 3 --no-sweep --no-cpu-baseline --no-f1 --no-e2e --no-dense \
    --out $O/ab_$w.json > /dev/null 2>&1
  python -c "import json; r=json.load(open('$O/ab_$w.json')); print('$1 pdl=$2 $w', round(r['value'],1), round(r['ms_per_step'],4), {k: round(v,4) for k,v in r['stages_ms'].items()})" >> $O/ab.txt 2>&1
done; done
cat $O/ab.txt
