#!/bin/bash
# full GPU suite + c1 / reddit benches (no cpu leg) + c1 latency
tag=${1:-r02}
out=gpurun_out
timeout 1500 python -m pytest tests -m gpu -q > $out/${tag}_pytest_gpu.log 2>&1
echo "pytest rc=$?"; tail -2 $out/${tag}_pytest_gpu.log
for cfg in c1 reddit; do
timeout 600 python bench.py --config $cfg --steps 20 --warmup 5 --no-cpu --no-e2e > $out/${tag}_bench_$cfg.json 2> $out/${tag}_bench_$cfg.err
echo "bench $cfg rc=$?"; python -c "import json;d=json.loads(open('$out/${tag}_bench_$cfg.json').read().strip().splitlines()[-1]);print(d['ms_per_step'], d['ms_per_op'], d['config']['spmm_choice'], d['config']['sddmm_choice'])"
done
