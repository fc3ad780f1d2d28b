#!/bin/bash
# The N-GPU bench path (NCCL process group, sharded layout, rank-0 decisions
# broadcast, all-gather / blocked exchange, max-over-ranks timing) run at
# world size 1 on one B200 (AUTOSAGE_BENCH_DIST1=1), with the N=1 parity check.
tag=${1:-r02r}
out=gpurun_out
mkdir -p $out
for cfg in reddit products; do
  AUTOSAGE_BENCH_DIST1=1 timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node 1 \
      --master-addr 127.0.0.1 --master-port 29541 bench.py --gpus 1 --config $cfg --steps 5 --warmup 3 \
      > $out/${tag}_dist1_$cfg.json 2> $out/${tag}_dist1_$cfg.err
  echo "dist1 $cfg rc=$?"
  grep -c "NCCL INFO" $out/${tag}_dist1_$cfg.err
done
