cmd="python tools/profile_kernels.py --config c1 --spmm spmm:hubsplit:ft=32:rpc=1:vec=1:hubt=256,spmm:rowparallel:ft=64:rpc=1:vec=1:hubt=256 --sddmm sddmm:rowparallel:ft=32:rpc=1:vec=0:hubt=256 --reps 3"
$cmd > gpurun_out/r02g_c1_plain.log 2>&1 && ncu --metrics gpu__time_duration.sum,sm__warps_active.avg.pct_of_peak_sustained_active --clock-control none --csv --log-file gpurun_out/r02g_c1_launches.csv $cmd > gpurun_out/r02g_c1_ncu.log 2>&1
echo rc=$?
