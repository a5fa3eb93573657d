#!/bin/bash
# Prediction kernels: GPU parity (default and CTA-forced TopCdf paths) + stage timing.
O=gpurun_out
python -m pytest tests -m gpu -q -x --timeout 1200 2>&1 | tail -3 > $O/r02_pred_ab_pytest.log
SPARGE_TOPCDF_CTA_MIN_TN=0 python -m pytest tests -m gpu -q -x --timeout 1200 -k "parity or edge or mpv or long or fullsize" 2>&1 | tail -3 > $O/r02_pred_ab_pytest_cta.log
rm -f $O/r02_pred_ab.txt
for w in llama31_8b_32k mochi cogvideox_2b sweep_8k sweep_32k sweep_64k sweep_128k; do
  for thr in 1024 100000; do
    SPARGE_TOPCDF_CTA_MIN_TN=$thr python bench.py --workload $w --profile --steps 10 --warmup 3 --no-sweep \
      | python -c "import json,sys; r=json.loads(sys.stdin.readlines()[-1]); print('$w thr=$thr', {k: round(v,4) for k,v in r['stages_ms'].items()})" >> $O/r02_pred_ab.txt 2>&1
  done
done
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $O/r02_launches_128k_v2.csv \
  python bench.py --workload sweep_128k --profile --steps 1 --warmup 1 --no-sweep > /dev/null 2>&1
