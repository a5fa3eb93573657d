#!/bin/bash
# last check at the final commit: GPU suite, smoke, the driver's default bench line, the reference arm
O=gpurun_out/final4
mkdir -p $O
python -m pytest tests -m gpu -q --timeout 1500 > $O/pytest_gpu.log 2>&1; tail -2 $O/pytest_gpu.log
python -c "import __graft_entry__ as g; g.smoke()" > $O/smoke.log 2>&1; tail -1 $O/smoke.log
python bench.py > $O/bench.json 2> $O/bench.err; tail -c 300 $O/bench.json
python bench.py --impl reference --steps 2 --warmup 1 > $O/bench_reference.json 2>&1; tail -c 200 $O/bench_reference.json
