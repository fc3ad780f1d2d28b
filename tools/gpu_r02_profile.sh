#!/bin/bash
# Round-2 profiling pass (no code change needed): the on-chip roofs
# (tools/gather_roofline), and ncu full captures of the kernels round 1 left
# unprofiled -- the Reddit SpMM pieces kernel, the Products F=100 SpMM (c3)
# and the fused-attention kernels (c5).  Every ncu command is preceded by the
# same command run plain (&&), as the profiling recipe requires.
#   gpurun --timeout 2400 -- 'bash tools/gpu_r02_profile.sh r02a'
tag=${1:-r02a}
out=gpurun_out
mkdir -p $out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,power.draw --format=csv > $out/nvsmi_$tag.txt 2>&1

timeout 300 ./tools/gather_roofline > $out/${tag}_gather_roofline.txt 2>&1
echo "gather_roofline rc=$?" | tee -a $out/status_$tag.txt

red_spmm="spmm:hubsplit:ft=64:rpc=1:vec=1:hubt=256"
prod_spmm="spmm:hubsplit:ft=128:rpc=1:vec=1:hubt=256"

# Reddit SpMM: both spmm_seg launches of the 3rd rep (light rows + pieces)
cmd="python tools/profile_kernels.py --config reddit --spmm $red_spmm --reps 3"
timeout 600 $cmd > $out/${tag}_plain_red.log 2>&1 &&
timeout 900 ncu --set full --clock-control none --import-source on -k regex:spmm_seg -s 4 -c 2 \
    -f -o $out/${tag}_spmm_red $cmd > $out/${tag}_ncu_red.log 2>&1
echo "ncu reddit spmm rc=$?" | tee -a $out/status_$tag.txt

# Products F=100 SpMM (c3, 1 GPU)
cmd="python tools/profile_kernels.py --config products --spmm $prod_spmm --reps 3"
timeout 600 $cmd > $out/${tag}_plain_prod.log 2>&1 &&
timeout 900 ncu --set full --clock-control none --import-source on -k regex:spmm_seg -s 4 -c 2 \
    -f -o $out/${tag}_spmm_prod $cmd > $out/${tag}_ncu_prod.log 2>&1
echo "ncu products spmm rc=$?" | tee -a $out/status_$tag.txt

# c5 fused attention: decide once (cache), then replay-only under ncu
rm -f $out/${tag}_att.cache
timeout 600 python tools/profile_attention.py --config reddit --fused 1 --reps 2 --cache $out/${tag}_att.cache \
    > $out/${tag}_plain_att0.log 2>&1
cmd="python tools/profile_attention.py --config reddit --fused 1 --reps 2 --cache $out/${tag}_att.cache --replay-only"
timeout 600 $cmd > $out/${tag}_plain_att.log 2>&1 &&
timeout 900 ncu --set full --clock-control none --import-source on -k regex:'spmm_seg|sddmm_pair|softmax' \
    -s 0 -c 6 -f -o $out/${tag}_att $cmd > $out/${tag}_ncu_att.log 2>&1
echo "ncu attention rc=$?" | tee -a $out/status_$tag.txt

# per-kernel DRAM traffic + duration of every launch of a replayed bench step
rm -f $out/${tag}_bench.cache
timeout 600 python bench.py --steps 3 --warmup 3 --no-e2e --no-cpu --cache $out/${tag}_bench.cache \
    > $out/${tag}_bench_plain0.json 2>&1
cmd="python bench.py --steps 3 --warmup 3 --no-e2e --no-cpu --cache $out/${tag}_bench.cache --replay-only"
timeout 600 $cmd > $out/${tag}_bench_plain.json 2>&1 &&
timeout 900 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum \
    --clock-control none --csv --log-file $out/${tag}_launches_traffic.csv $cmd > $out/${tag}_ncu_traffic.log 2>&1
echo "ncu traffic rc=$?" | tee -a $out/status_$tag.txt

# summaries on the box (raw pages), then drop the big reports if over budget
for r in spmm_red spmm_prod att; do
  if [ -f $out/${tag}_$r.ncu-rep ]; then
    ncu -i $out/${tag}_$r.ncu-rep --page raw --csv > $out/${tag}_${r}_raw.csv 2>/dev/null
    ncu -i $out/${tag}_$r.ncu-rep --page details --csv > $out/${tag}_${r}_details.csv 2>/dev/null
    ncu -i $out/${tag}_$r.ncu-rep --page source --csv > $out/${tag}_${r}_source.csv 2>/dev/null
    rm -f $out/${tag}_$r.ncu-rep   # gpurun merges back at most 64 MiB
  fi
done
du -sh $out
