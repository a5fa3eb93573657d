#!/bin/bash
# prediction-stage profile at 128K and 32K: launch lists + ncu --set full of the two kernels
O=gpurun_out
for w in sweep_128k sweep_32k llama31_8b_32k; do
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $O/pp_launch_$w.csv \
  python bench.py --workload $w --profile --steps 1 --warmup 0 --no-sweep --no-cpu-baseline --no-f1 --no-e2e --no-dense > /dev/null 2>&1
done
ncu --set full --clock-control none --import-source on -k regex:"k_shat_dmma|k_topcdf" -c 2 \
  -o $O/pp128k -f python bench.py --workload sweep_128k --profile --steps 1 --warmup 0 --no-sweep --no-cpu-baseline --no-f1 --no-e2e --no-dense > /dev/null 2>&1
ncu -i $O/pp128k.ncu-rep --page details --csv > $O/pp128k_details.csv
ncu -i $O/pp128k.ncu-rep --page raw --csv > $O/pp128k_raw.csv
ncu -i $O/pp128k.ncu-rep --page source --csv --print-source sass,cuda > $O/pp128k_mix.csv
ls -la $O/pp*
