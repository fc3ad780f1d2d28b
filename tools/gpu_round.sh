#!/bin/bash
# One GPU session: parity suite, bench (ours + reference arm), ncu launch
# list of the bench command, and one `ncu --set full` capture per dominant
# kernel.  Outputs land in gpurun_out/ (scratch); summaries are copied to
# profiles/ by tools/summarize_ncu.py.
#   gpurun --timeout 3000 -- 'bash tools/gpu_round.sh [config] [tag]'
cfg=${1:-reddit}
tag=${2:-r01}
out=gpurun_out
mkdir -p $out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,power.draw --format=csv > $out/nvsmi_$tag.txt 2>&1

timeout 900 python -m pytest tests -m gpu -q > $out/pytest_gpu_$tag.log 2>&1
echo "pytest rc=$?" | tee -a $out/status_$tag.txt
tail -3 $out/pytest_gpu_$tag.log

rm -f $out/sched_$tag.cache
timeout 900 python bench.py --config $cfg --cache $out/sched_$tag.cache > $out/bench_$tag.json 2> $out/bench_$tag.err
echo "bench rc=$?" | tee -a $out/status_$tag.txt
timeout 900 python bench.py --impl reference --config $cfg --steps 2 --warmup 3 > $out/bench_ref_$tag.json 2> $out/bench_ref_$tag.err
echo "bench_ref rc=$?" | tee -a $out/status_$tag.txt

# launch list of the same bench command (cold-cache, serialised per launch)
timeout 1200 ncu --metrics gpu__time_duration.sum --clock-control none --csv \
    --log-file $out/launches_$tag.csv python bench.py --config $cfg --steps 3 --warmup 3 \
    --no-e2e --no-cpu --cache $out/sched_$tag.cache --replay-only > $out/ncu_launch_$tag.log 2>&1
echo "ncu_launch rc=$?" | tee -a $out/status_$tag.txt

spmm=$(python -c "import json;print(json.load(open('$out/bench_$tag.json'))['config']['spmm_choice'])" 2>/dev/null)
sddmm=$(python -c "import json;print(json.load(open('$out/bench_$tag.json'))['config']['sddmm_choice'])" 2>/dev/null)
echo "choices spmm=$spmm sddmm=$sddmm" | tee -a $out/status_$tag.txt
timeout 900 ncu --set full --clock-control none --import-source on -k regex:sddmm -s 2 -c 1 \
    -f -o $out/sddmm_full_$tag python tools/profile_kernels.py --config $cfg --sddmm "$sddmm" --reps 3 \
    > $out/ncu_sddmm_$tag.log 2>&1
echo "ncu_sddmm rc=$?" | tee -a $out/status_$tag.txt
timeout 900 ncu --set full --clock-control none --import-source on -k regex:spmm_seg -s 2 -c 1 \
    -f -o $out/spmm_full_$tag python tools/profile_kernels.py --config $cfg --spmm "$spmm" --reps 3 \
    > $out/ncu_spmm_$tag.log 2>&1
echo "ncu_spmm rc=$?" | tee -a $out/status_$tag.txt
