#!/bin/bash
# prediction-stage profile at 128K: launch list + ncu --set full of k_topcdf_cta (current build)
O=gpurun_out
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $O/pq_launch_128k.csv \
  python bench.py --workload sweep_128k --profile --steps 1 --warmup 0 --no-sweep --no-cpu-baseline --no-f1 --no-e2e --no-dense > /dev/null 2>&1
ncu --set full --clock-control none --import-source on -k regex:"k_topcdf_cta|k_shat" -c 2 \
  -o $O/pq128k -f python bench.py --workload sweep_128k --profile --steps 1 --warmup 0 --no-sweep --no-cpu-baseline --no-f1 --no-e2e --no-dense > /dev/null 2>&1
ncu -i $O/pq128k.ncu-rep --page raw --csv > $O/pq128k_raw.csv
ncu -i $O/pq128k.ncu-rep --page source --csv --print-source sass > $O/pq128k_sass.csv
ls -la $O/pq*
