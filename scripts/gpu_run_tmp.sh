set -u
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_f4.py tests/test_gpu_f1.py -x -q > gpurun_out/pytest_parity.log 2>&1; echo parity_rc=$?; tail -2 gpurun_out/pytest_parity.log
for w in llama31_8b_32k mochi cogvideox_2b sweep_8k; do
timeout 300 python scripts/variant_bench.py $w libsparge_lpt.so libsparge.so 2>&1 | grep attn
done
