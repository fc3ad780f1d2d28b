#!/bin/bash
# Round-2 final evidence pass (r02ac): both bench arms (default config), c1 / products lines,
# the ncu launch list with DRAM traffic of a replayed bench step, and one
# `ncu --set full` per dominant kernel (SDDMM pair kernel, SpMM pieces +
# light rows), summarised on the box (reports dropped: 64 MiB merge cap).
#   gpurun --timeout 3000 -- 'bash tools/gpu_r02_round.sh r02ac'
tag=${1:-r02ac}
out=gpurun_out
mkdir -p $out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,power.draw --format=csv > $out/${tag}_nvsmi.txt 2>&1
timeout 900 python bench.py --impl reference --steps 5 --warmup 3 > $out/${tag}_bench_ref.json 2> $out/${tag}_bench_ref.err
echo "bench_ref rc=$?"
rm -f $out/${tag}_bench.cache
timeout 900 python bench.py --steps 20 --warmup 5 --cache $out/${tag}_bench.cache > $out/${tag}_bench.json 2> $out/${tag}_bench.err
echo "bench rc=$?"
for cfg in c1 products; do
  timeout 900 python bench.py --config $cfg --steps 20 --warmup 5 --no-e2e > $out/${tag}_bench_$cfg.json 2> $out/${tag}_bench_$cfg.err
  echo "bench $cfg rc=$?"
done
for cfg in products c1; do
  rm -f $out/${tag}_$cfg.cache
  timeout 900 python bench.py --config $cfg --steps 3 --warmup 3 --no-e2e --no-cpu --cache $out/${tag}_$cfg.cache \
      > $out/${tag}_${cfg}_plain0.json 2>&1
  c2="python bench.py --config $cfg --steps 3 --warmup 3 --no-e2e --no-cpu --cache $out/${tag}_$cfg.cache --replay-only"
  timeout 600 $c2 > $out/${tag}_${cfg}_plain.json 2>&1 &&
  timeout 900 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum \
      --clock-control none --csv --log-file $out/${tag}_${cfg}_launches_traffic.csv $c2 > $out/${tag}_ncu_$cfg.log 2>&1
  echo "ncu $cfg rc=$?"
done
cmd="python bench.py --steps 3 --warmup 3 --no-e2e --no-cpu --cache $out/${tag}_bench.cache --replay-only"
timeout 600 $cmd > $out/${tag}_bench_plain.json 2>&1 &&
timeout 900 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum \
    --clock-control none --csv --log-file $out/${tag}_launches_traffic.csv $cmd > $out/${tag}_ncu_traffic.log 2>&1
echo "ncu traffic rc=$?"
sd=$(python -c "import json;print(json.loads(open('$out/${tag}_bench.json').read().strip().splitlines()[-1])['config']['sddmm_choice'])")
sp=$(python -c "import json;print(json.loads(open('$out/${tag}_bench.json').read().strip().splitlines()[-1])['config']['spmm_choice'])")
cmd="python tools/profile_kernels.py --config reddit --sddmm $sd --reps 3"
timeout 600 $cmd > $out/${tag}_plain_sd.log 2>&1 &&
timeout 900 ncu --set full --clock-control none --import-source on -k regex:sddmm_pair -s 2 -c 1 -f -o $out/${tag}_sddmm $cmd > $out/${tag}_ncu_sd.log 2>&1
echo "ncu sddmm rc=$?"
cmd="python tools/profile_kernels.py --config reddit --spmm $sp --reps 3"
timeout 600 $cmd > $out/${tag}_plain_sp.log 2>&1 &&
timeout 900 ncu --set full --clock-control none --import-source on -k regex:spmm_seg -s 2 -c 1 -f -o $out/${tag}_spmm $cmd > $out/${tag}_ncu_sp.log 2>&1
echo "ncu spmm rc=$?"
# pass-major SDDMM at F=256 (auto there): two passes (f0 = 0, then a carried one)
cmd="python tools/profile_kernels.py --config reddit --f 256 --sddmm sddmm:rowparallel:ft=32:rpc=1:vec=0:hubt=256 --reps 3"
timeout 600 $cmd > $out/${tag}_plain_pm.log 2>&1 &&
timeout 900 ncu --set full --clock-control none --import-source on -k regex:sddmm_pair1_pm -s 4 -c 2 -f -o $out/${tag}_pm $cmd > $out/${tag}_ncu_pm.log 2>&1
echo "ncu pm rc=$?"
timeout 300 python -c "import __graft_entry__ as g; g.smoke(); print('smoke ok')" > $out/${tag}_smoke.log 2>&1
echo "smoke rc=$?"
for r in sddmm spmm pm; do
  if [ -f $out/${tag}_$r.ncu-rep ]; then
    ncu -i $out/${tag}_$r.ncu-rep --page raw --csv > $out/${tag}_${r}_raw.csv 2>/dev/null
    python tools/ncu_lines.py $out/${tag}_$r.ncu-rep 20 > $out/${tag}_${r}_lines.txt 2>&1
    rm -f $out/${tag}_$r.ncu-rep
  fi
done
du -sh $out
