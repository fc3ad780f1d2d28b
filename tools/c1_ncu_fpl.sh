cmd="python tools/profile_kernels.py --config c1 --spmm spmm:hubsplit:ft=64:rpc=1:vec=1:hubt=256 --reps 3"
for k in 0 2; do
AUTOSAGE_DEV_LONG_FPL=$k $cmd > gpurun_out/r02g_fpl${k}_plain.log 2>&1 && AUTOSAGE_DEV_LONG_FPL=$k ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/r02g_fpl${k}.csv $cmd > /dev/null 2>&1
echo fpl=$k rc=$?
done
