#!/bin/bash
# r02o: GPU suite with the F=100 pair kernel, its A/B, and the finite-scan cap A/B
mkdir -p gpurun_out
timeout 1500 python -m pytest tests -m gpu -x -q -p no:cacheprovider > gpurun_out/r02o_pytest.log 2>&1
echo "pytest rc=$?" >> gpurun_out/r02o_pytest.log
timeout 900 python tools/ab_sddmm_f100.py > gpurun_out/r02o_ab_f100.log 2>&1
echo "ab f100 rc=$?" >> gpurun_out/r02o_ab_f100.log
timeout 1200 python tools/ab_mix_scan.py > gpurun_out/r02o_ab_mix.log 2>&1
echo "ab mix rc=$?" >> gpurun_out/r02o_ab_mix.log
tail -3 gpurun_out/r02o_pytest.log; cat gpurun_out/r02o_ab_f100.log gpurun_out/r02o_ab_mix.log
