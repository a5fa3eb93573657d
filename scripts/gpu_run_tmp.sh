set -u
timeout 900 python -m pytest tests/test_gpu_smooth.py -x -q > gpurun_out/pytest_smooth.log 2>&1; echo rc=$?; tail -25 gpurun_out/pytest_smooth.log
