#!/bin/bash
# r02m: full GPU suite after tile-major SpMM + pass-major SDDMM, then the pass-major A/B
mkdir -p gpurun_out
timeout 1500 python -m pytest tests -m gpu -x -q -p no:cacheprovider > gpurun_out/r02m_pytest.log 2>&1
echo "pytest rc=$?" >> gpurun_out/r02m_pytest.log
timeout 900 python tools/ab_sddmm_pm.py > gpurun_out/r02m_ab_pm.log 2>&1
echo "ab rc=$?" >> gpurun_out/r02m_ab_pm.log
tail -3 gpurun_out/r02m_pytest.log; cat gpurun_out/r02m_ab_pm.log
