set -u
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_f1.py -x -q > gpurun_out/pytest_parity.log 2>&1; echo rc=$?; tail -2 gpurun_out/pytest_parity.log
for w in llama31_8b_32k mochi cogvideox_2b; do
timeout 300 python bench.py --workload $w --steps 20 --warmup 3 --no-e2e --no-cpu-baseline --no-dense --no-f1 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.readline()); print('$w', {k:round(v,3) for k,v in d['stages_ms'].items()})"
done
