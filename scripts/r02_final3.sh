#!/bin/bash
# Round-2 measurement pass: GPU suite, smoke, the default bench line (+ sweep, e2e, host baseline),
# per-workload lines, the reference arm, an ncu launch list and full captures of the top kernels.
O=gpurun_out/final3
mkdir -p $O
python -m pytest tests -m gpu -q --timeout 1500 > $O/pytest_gpu.log 2>&1; tail -2 $O/pytest_gpu.log
python -c "import __graft_entry__ as g; g.smoke()" > $O/smoke.log 2>&1; tail -1 $O/smoke.log
python bench.py --out $O/bench.json > $O/bench.log 2>&1; tail -c 300 $O/bench.log
for w in cogvideox_2b mochi mochi_22k flux; do
  python bench.py --workload $w --no-sweep --out $O/bench_$w.json > $O/bench_$w.log 2>&1
done
python bench.py --impl reference --steps 2 --warmup 1 > $O/bench_reference.log 2>&1; tail -c 200 $O/bench_reference.log
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $O/launches.csv \
  python bench.py --steps 2 --warmup 1 --no-sweep --no-cpu-baseline --no-f1 --no-e2e --no-dense > /dev/null 2>&1
for spec in "k_sparse_attn llama31_8b_32k attn_llama" "k_sparse_attn cogvideox_2b attn_cogvideox" "k_quant_pool_sim llama31_8b_32k quant_llama" "k_shat_dmma|k_topcdf sweep_128k predict_128k"; do
  set -- $spec
  KC=1; [ "$3" = "quant_llama" ] && KC=2; [ "$3" = "predict_128k" ] && KC=2
  ncu --set full --clock-control none --import-source on -k regex:"$1" -c $KC -o $O/$3 -f \
    python bench.py --workload $2 --profile --steps 1 --warmup 0 --no-sweep --no-cpu-baseline --no-f1 --no-e2e --no-dense > /dev/null 2>&1
  ncu -i $O/$3.ncu-rep --page details --csv > $O/$3_details.csv 2>/dev/null
  ncu -i $O/$3.ncu-rep --page raw --csv > $O/$3_raw.csv 2>/dev/null
  rm -f $O/$3.ncu-rep
done
ls $O
