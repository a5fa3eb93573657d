set -u
timeout 1200 python -m pytest tests/test_gpu_parity.py tests/test_gpu_fullsize.py tests/test_gpu_tuner.py -x -q > gpurun_out/pytest_pred.log 2>&1; echo rc=$?; tail -4 gpurun_out/pytest_pred.log
for lib in "libsparge_sparge_topcdf_binned=0.so" libsparge.so; do for w in llama31_8b_32k mochi cogvideox_2b sweep_128k; do
SPARGE_LIB=$lib timeout 300 python bench.py --workload $w --steps 10 --warmup 3 --no-e2e --no-cpu-baseline --no-dense --no-f1 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.readline()); print('$lib', '$w', {k:round(v,3) for k,v in d['stages_ms'].items()}, d['parity']['mask_mismatch'] if 'parity' in d else '')"
done; done
