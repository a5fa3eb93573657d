#!/bin/bash
# Round-2 profiling pass (run on the GPU box via gpurun from the repo root).
set -x
O=gpurun_out
NCU=ncu
# launch lists (per-launch device time, cold-cache serialised)
$NCU --metrics gpu__time_duration.sum --clock-control none --csv --log-file $O/r02_launches_llama.csv \
  python bench.py --profile --steps 3 --warmup 1 --no-sweep > $O/r02_prof_llama.log 2>&1
$NCU --metrics gpu__time_duration.sum --clock-control none --csv --log-file $O/r02_launches_128k.csv \
  python bench.py --workload sweep_128k --profile --steps 1 --warmup 1 --no-sweep > $O/r02_prof_128k.log 2>&1
# full sets of the prediction kernels at 128K
$NCU --set full --clock-control none --import-source on -k regex:"k_topcdf_rows|k_shat_dmma" -c 2 \
  -o $O/r02_pred128k -f python bench.py --workload sweep_128k --profile --steps 1 --warmup 0 --no-sweep > $O/r02_prof_pred.log 2>&1
# multi-rank plumbing on one GPU (gloo; timings meaningless): gathered O == single-GPU O
SPARGE_BENCH_ONE_GPU=1 timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 \
  --master-addr 127.0.0.1 --master-port 29517 bench.py --gpus 2 --steps 3 --warmup 3 --no-sweep \
  --no-f1 --no-e2e --no-dense --out $O/r02_2rank_onegpu.json > $O/r02_2rank.log 2>&1
