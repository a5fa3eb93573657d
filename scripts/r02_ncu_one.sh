#!/bin/bash
# ncu --set full of kernels matching $KRE (count $KC) in one bench step of workload $WL -> gpurun_out/$TAG.*
O=gpurun_out
ncu --set full --clock-control none --import-source on -k regex:"$KRE" -c ${KC:-1} \
  -o $O/$TAG -f python bench.py --workload $WL --profile --steps 1 --warmup 0 --no-sweep --no-cpu-baseline --no-f1 --no-e2e --no-dense > /dev/null 2>&1
ncu -i $O/$TAG.ncu-rep --page details --csv > $O/${TAG}_details.csv
ncu -i $O/$TAG.ncu-rep --page raw --csv > $O/${TAG}_raw.csv
ncu -i $O/$TAG.ncu-rep --page source --csv --print-source sass,cuda > $O/${TAG}_mix.csv
ls -la $O/$TAG*
