#!/bin/bash
# Table 3 analogue: prediction time over full (dense) attention time, 8K..128K (+ TopCdf kernel threshold A/B)
O=gpurun_out
python -m pytest tests -m gpu -q -x --timeout 1500 -k "topcdf or fullsize or long or parity" 2>&1 | tail -1
rm -f $O/t3.txt
for ct in ${CTS:-1024}; do for w in sweep_8k sweep_16k sweep_32k sweep_64k sweep_128k; do
  SPARGE_TOPCDF_CTA_MIN_TN=$ct python bench.py --workload $w --steps 10 --warmup 3 --no-sweep --no-cpu-baseline --no-f1 --no-e2e --out $O/t3_$w.json > /dev/null 2>&1
  python -c "import json; r=json.load(open('$O/t3_$w.json')); st=r['stages_ms']; print('ctamin=$ct $w predict', round(st['predict_ms'],4), 'attn', round(st['attn_ms'],3), 'dense_attn', round(r['dense']['attn_ms'],3), 'pred/attn', round(r['predict_over_attn'],4), 'pred/dense_attn', round(r['predict_over_dense_attn'],5))" >> $O/t3.txt 2>&1
done; done
cat $O/t3.txt
