#!/bin/bash
# joint Q+K quantisation launch (sparge_quantize_qk) vs two launches: GPU suite, then step / stage times
O=gpurun_out/s12
mkdir -p $O
python -m pytest tests -m gpu -q -x --timeout 1500 > $O/pytest.log 2>&1; tail -3 $O/pytest.log
rm -f $O/ab.txt
for w in ${WL:-flux sweep_8k cogvideox_2b mochi_22k llama31_8b_32k mochi sweep_128k}; do
for split in 1 0; do
  SPARGE_BENCH_SPLIT_QK=$split python bench.py --workload $w --profile --steps 30 --warmup 3 --no-sweep --no-cpu-baseline --no-f1 --no-e2e --no-dense \
    --out $O/ab_$w.json > /dev/null 2>&1
  python -c "import json; r=json.load(open('$O/ab_$w.json')); print('split=$split $w', round(r['value'],1), round(r['ms_per_step'],4), {k: round(v,4) for k,v in r['stages_ms'].items()})" >> $O/ab.txt 2>&1
done; done
cat $O/ab.txt
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $O/launch_flux.csv \
  python bench.py --workload flux --profile --steps 2 --warmup 1 --no-sweep --no-cpu-baseline --no-f1 --no-e2e --no-dense > /dev/null 2>&1
ncu --set full --clock-control none --import-source on -k regex:k_quant_pool_sim -c 1 \
  -o $O/qk_llama -f python bench.py --profile --steps 1 --warmup 0 --no-sweep --no-cpu-baseline --no-f1 --no-e2e --no-dense > /dev/null 2>&1
ncu -i $O/qk_llama.ncu-rep --page details --csv > $O/qk_llama_details.csv 2>/dev/null
ncu -i $O/qk_llama.ncu-rep --page raw --csv > $O/qk_llama_raw.csv 2>/dev/null
ncu -i $O/qk_llama.ncu-rep --page source --csv --print-source sass > $O/qk_llama_sass.csv 2>/dev/null
rm -f $O/qk_llama.ncu-rep
