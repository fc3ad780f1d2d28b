#!/bin/bash
# Parity suite + smoke + both bench arms on one GPU (no profiler).
#   gpurun --timeout 2400 -- 'bash tools/gpu_check.sh r02b'
tag=${1:-r02}
out=gpurun_out
mkdir -p $out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,power.draw --format=csv > $out/${tag}_nvsmi.txt 2>&1
timeout 1500 python -m pytest tests -m gpu -q -x ${PYTEST_ARGS:-} > $out/${tag}_pytest_gpu.log 2>&1
echo "pytest rc=$?" | tee -a $out/${tag}_status.txt
tail -5 $out/${tag}_pytest_gpu.log
timeout 300 python -c 'import __graft_entry__ as g; g.smoke()' > $out/${tag}_smoke.log 2>&1
echo "smoke rc=$?" | tee -a $out/${tag}_status.txt
timeout 900 python bench.py --impl reference --steps ${REF_STEPS:-5} --warmup 3 > $out/${tag}_bench_ref.json 2> $out/${tag}_bench_ref.err
echo "bench_ref rc=$?" | tee -a $out/${tag}_status.txt
timeout 900 python bench.py --steps 20 --warmup 5 > $out/${tag}_bench.json 2> $out/${tag}_bench.err
echo "bench rc=$?" | tee -a $out/${tag}_status.txt
tail -c 600 $out/${tag}_bench.err
