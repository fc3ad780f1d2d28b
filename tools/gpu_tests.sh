#!/bin/bash
out=gpurun_out; tag=$1
timeout 1800 python -m pytest tests -m gpu -q > $out/${tag}_pytest_gpu.log 2>&1
echo "pytest rc=$?"
tail -15 $out/${tag}_pytest_gpu.log
