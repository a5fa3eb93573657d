#!/bin/bash
# predict-stage A/B: prediction parity tests, predict time and predict/attn over the workloads
O=gpurun_out
python -m pytest tests -m gpu -q -x --timeout 1500 -k "topcdf or fullsize or long or parity or edge" > $O/pa_pytest.log 2>&1; tail -1 $O/pa_pytest.log
rm -f $O/pa.txt
for ct in ${CTS:-1024}; do
for w in llama31_8b_32k cogvideox_2b mochi sweep_8k sweep_16k sweep_32k sweep_64k sweep_128k; do
  SPARGE_TOPCDF_CTA_MIN_TN=$ct python bench.py --workload $w --profile --steps 10 --warmup 3 --no-sweep --no-cpu-baseline --no-f1 --no-e2e --no-dense \
    --out $O/pa_$w.json > /dev/null 2>&1
  python -c "import json; r=json.load(open('$O/pa_$w.json')); st=r['stages_ms']; print('ctamin=$ct', '$w', round(st['predict_ms'],4), round(st['predict_ms']/st['attn_ms'],4))" >> $O/pa.txt 2>&1
done; done
cat $O/pa.txt
