#!/bin/bash
O=gpurun_out
python -m pytest tests -m gpu -q -x --timeout 1200 2>&1 | tail -3 > $O/r02_pred_ab2_pytest.log
rm -f $O/r02_pred_ab2.txt
for w in llama31_8b_32k mochi sweep_64k sweep_128k; do
  python bench.py --workload $w --profile --steps 10 --warmup 3 --no-sweep \
    | python -c "import json,sys; r=json.loads(sys.stdin.readlines()[-1]); print('$w', {k: round(v,4) for k,v in r['stages_ms'].items()})" >> $O/r02_pred_ab2.txt 2>&1
done
ncu --set full --clock-control none --import-source on -k regex:"k_topcdf_cta|k_shat_dmma" -c 2 \
  -o $O/r02_pred128k_v2 -f python bench.py --workload sweep_128k --profile --steps 1 --warmup 0 --no-sweep > /dev/null 2>&1
