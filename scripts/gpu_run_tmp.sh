set -u
for w in llama31_8b_32k mochi cogvideox_2b sweep_8k sweep_32k sweep_128k; do
for cfg in "48 296" "1000000 0" "48 592"; do set -- $cfg
SPARGE_ORDER_BUDGET_MB=$1 SPARGE_ORDER_LONG=$2 timeout 300 python scripts/variant_bench.py $w libsparge.so 2>&1 | grep attn | sed "s/^/budget=$1 long=$2 /"
done; done
