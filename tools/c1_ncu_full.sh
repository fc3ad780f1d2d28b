# ncu --set full of the c1 ring kernel (long rows) + group kernel, source lines summarised on the box
cmd="python tools/profile_kernels.py --config c1 --spmm spmm:rowparallel:ft=64:rpc=1:vec=1:hubt=256 --reps 3"
tag=${1:-r02g}
$cmd > gpurun_out/${tag}_c1full_plain.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:"spmm_longrow|spmm_seg" -s 2 -c 2 -f -o gpurun_out/${tag}_c1full $cmd > gpurun_out/${tag}_c1full_ncu.log 2>&1
echo ncu rc=$?
ncu -i gpurun_out/${tag}_c1full.ncu-rep --page raw --csv > gpurun_out/${tag}_c1full_raw.csv 2>/dev/null
python tools/ncu_lines.py gpurun_out/${tag}_c1full.ncu-rep 25 > gpurun_out/${tag}_c1full_lines.txt 2>&1
ncu -i gpurun_out/${tag}_c1full.ncu-rep --page details --csv > gpurun_out/${tag}_c1full_details.csv 2>/dev/null
rm -f gpurun_out/${tag}_c1full.ncu-rep
