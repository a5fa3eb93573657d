#!/bin/bash
# Round-2 checkpoint on the GPU box: GPU suite, default bench line, per-workload stage times.
O=gpurun_out
python -m pytest tests -m gpu -q -x --timeout 1500 > $O/ckpt_pytest.log 2>&1; tail -3 $O/ckpt_pytest.log
python -c "import __graft_entry__ as g; g.smoke()" > $O/ckpt_smoke.log 2>&1; tail -1 $O/ckpt_smoke.log
python bench.py --out $O/ckpt_bench.json > $O/ckpt_bench.log 2>&1; tail -c 600 $O/ckpt_bench.log
rm -f $O/ckpt_stages.txt
for w in llama31_8b_32k cogvideox_2b mochi flux sweep_8k sweep_32k sweep_128k; do
  python bench.py --workload $w --profile --steps 10 --warmup 3 --no-sweep --no-cpu-baseline --no-f1 --no-e2e \
    --out $O/ckpt_bench_$w.json > /dev/null 2>&1
  python -c "import json; r=json.load(open('$O/ckpt_bench_$w.json')); print('$w', round(r['value'],1), round(r['sparsity'],3), r['roofline']['frac'], {k: round(v,4) for k,v in r['stages_ms'].items()})" >> $O/ckpt_stages.txt 2>&1
done
cat $O/ckpt_stages.txt
