for k in 0 2 0 2; do
 AUTOSAGE_DEV_LONG_FPL=$k python tools/c1_latency.py --reps 200 2>&1 | grep -E "spmm_fixed_cold|spmm_fixed_b2b|choices" | sed "s/^/fpl=$k /"
done
