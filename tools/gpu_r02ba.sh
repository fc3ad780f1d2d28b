#!/bin/bash
# Round-2 re-entry check on the restored tree: GPU suite, smoke, default bench (both arms).
tag=${1:-r02ba}
out=gpurun_out
mkdir -p $out
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > $out/${tag}_smoke.log 2>&1
echo "smoke rc=$?"
timeout 2400 python -m pytest tests -m gpu -q > $out/${tag}_pytest.log 2>&1
echo "pytest rc=$?"; tail -3 $out/${tag}_pytest.log
timeout 900 python bench.py > $out/${tag}_bench.json 2> $out/${tag}_bench.err
echo "bench rc=$?"
timeout 900 python bench.py --impl reference > $out/${tag}_bench_ref.json 2> $out/${tag}_bench_ref.err
echo "bench ref rc=$?"
timeout 900 python bench.py --config products --steps 20 --warmup 5 --no-e2e > $out/${tag}_bench_products.json 2> $out/${tag}_bench_products.err
echo "bench products rc=$?"
