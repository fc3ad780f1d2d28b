#!/bin/bash
# ncu launch lists with DRAM bytes for the c1 and Products bench lines (roofline.traffic of those
# configs), each after the same command exited 0 without ncu
tag=${1:-r02t}
out=gpurun_out
mkdir -p $out
for cfg in products c1; do
  rm -f $out/${tag}_$cfg.cache
  timeout 900 python bench.py --config $cfg --steps 3 --warmup 3 --no-e2e --no-cpu --cache $out/${tag}_$cfg.cache \
      > $out/${tag}_${cfg}_plain0.json 2>&1
  cmd="python bench.py --config $cfg --steps 3 --warmup 3 --no-e2e --no-cpu --cache $out/${tag}_$cfg.cache --replay-only"
  timeout 600 $cmd > $out/${tag}_${cfg}_plain.json 2>&1 &&
  timeout 900 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum \
      --clock-control none --csv --log-file $out/${tag}_${cfg}_launches_traffic.csv $cmd > $out/${tag}_ncu_$cfg.log 2>&1
  echo "ncu $cfg rc=$?"
done
