#!/bin/bash
# Standard GPU measurement pass: default bench line, other workloads, ncu.
set -u
mkdir -p gpurun_out
timeout 900 python bench.py --steps 30 --warmup 5 --out gpurun_out/bench.json > gpurun_out/bench.log 2>&1; echo bench_rc=$?
for w in cogvideox_2b mochi sweep_8k sweep_32k; do
  timeout 600 python bench.py --workload $w --steps 10 --warmup 3 --no-e2e --no-cpu-baseline --out gpurun_out/bench_$w.json > gpurun_out/bench_$w.log 2>&1; echo ${w}_rc=$?
done
timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none -c 40 --csv --log-file gpurun_out/launches.csv python bench.py --profile --steps 2 --warmup 1 > /dev/null 2>&1; echo ncu1_rc=$?
timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_sparse_attn -s 1 -c 1 -o gpurun_out/prof_attn python bench.py --profile --steps 1 --warmup 1 > gpurun_out/ncu_full.log 2>&1; echo ncu2_rc=$?
