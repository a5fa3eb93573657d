#!/bin/bash
# quant v7 vs v6 (libsparge_qv6.so): GPU suite, per-workload stage times, ncu of the new kernel
O=gpurun_out
python -m pytest tests -m gpu -q -x --timeout 1500 -k "quant or parity or smooth or f1 or fullsize" > $O/qab_pytest.log 2>&1; tail -3 $O/qab_pytest.log
rm -f $O/qab.txt
for lib in libsparge.so libsparge_qv6.so; do
for w in llama31_8b_32k cogvideox_2b mochi sweep_128k; do
  SPARGE_LIB=$lib python bench.py --workload $w --profile --steps 10 --warmup 3 --no-sweep --no-cpu-baseline --no-f1 --no-e2e --no-dense \
    --out $O/qab_$w.json > /dev/null 2>&1
  python -c "import json; r=json.load(open('$O/qab_$w.json')); print('$lib $w', {k: round(v,4) for k,v in r['stages_ms'].items()})" >> $O/qab.txt 2>&1
done; done
cat $O/qab.txt
ncu --set full --clock-control none --import-source on -k regex:k_quant_pool_sim -c 2 \
  -o $O/qv14 -f python bench.py --profile --steps 1 --warmup 0 --no-sweep --no-cpu-baseline --no-f1 --no-e2e --no-dense > /dev/null 2>&1
ncu -i $O/qv14.ncu-rep --page details --csv > $O/qv14_details.csv; ncu -i $O/qv14.ncu-rep --page raw --csv > $O/qv14_raw.csv; ncu -i $O/qv14.ncu-rep --page source --csv --print-source sass > $O/qv14_sass.csv 2>&1; ls -la $O/qv14*
