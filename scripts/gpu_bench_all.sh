#!/bin/bash
# Standard GPU measurement pass: GPU tests, default bench line, other
# workloads, the reference arm, ncu launch list and one --set full capture.
set -u
mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -q > gpurun_out/pytest_gpu.log 2>&1; echo pytest_rc=$?; tail -1 gpurun_out/pytest_gpu.log
timeout 900 python bench.py --steps 30 --warmup 5 --out gpurun_out/bench.json > gpurun_out/bench.log 2>&1; echo bench_rc=$?
for w in cogvideox_2b mochi mochi_22k sweep_8k sweep_16k sweep_32k sweep_64k sweep_128k; do
  timeout 900 python bench.py --workload $w --steps 10 --warmup 3 --no-e2e --no-cpu-baseline --out gpurun_out/bench_$w.json > gpurun_out/bench_$w.log 2>&1; echo ${w}_rc=$?
done
timeout 600 python bench.py --impl reference --steps 3 --warmup 1 > gpurun_out/bench_reference.log 2>&1; echo ref_rc=$?
timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none -c 40 --csv --log-file gpurun_out/launches.csv python bench.py --profile --steps 2 --warmup 1 > /dev/null 2>&1; echo ncu1_rc=$?
timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_sparse_attn -s 1 -c 1 -o gpurun_out/prof_attn python bench.py --profile --steps 1 --warmup 1 > gpurun_out/ncu_full.log 2>&1; echo ncu2_rc=$?
