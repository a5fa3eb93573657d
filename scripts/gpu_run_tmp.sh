set -u
for w in llama31_8b_32k mochi cogvideox_2b; do
timeout 400 python scripts/variant_bench.py $w libsparge.so "libsparge_sparge_bias_mma=0.so" "libsparge_sparge_poly_every=4.so" "libsparge_sparge_poly_every=0.so" "libsparge_sparge_rescale_thr=16.so" 2>&1 | grep attn
done
