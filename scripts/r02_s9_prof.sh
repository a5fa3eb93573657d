#!/bin/bash
# launch lists of the small shapes (kernel time vs event-timed step) + source-level ncu of the TopCdf CTA kernel at 128K
O=gpurun_out/s9
mkdir -p $O
for w in flux cogvideox_2b llama31_8b_32k; do
  python bench.py --workload $w --profile --steps 20 --warmup 3 --no-sweep --no-cpu-baseline --no-f1 --no-e2e --no-dense --out $O/b_$w.json > /dev/null 2>&1
  ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $O/launch_$w.csv \
    python bench.py --workload $w --profile --steps 2 --warmup 1 --no-sweep --no-cpu-baseline --no-f1 --no-e2e --no-dense > /dev/null 2>&1
done
ncu --set full --clock-control none --import-source on -k regex:"k_topcdf_cta" -c 1 \
  -o $O/tc128k -f python bench.py --workload sweep_128k --profile --steps 1 --warmup 0 --no-sweep --no-cpu-baseline --no-f1 --no-e2e --no-dense > /dev/null 2>&1
ncu -i $O/tc128k.ncu-rep --page source --csv --print-source sass,cuda > $O/tc128k_src.csv 2>&1
ncu -i $O/tc128k.ncu-rep --page source --csv --print-source sass > $O/tc128k_sass.csv 2>&1
rm -f $O/tc128k.ncu-rep
ls -la $O
