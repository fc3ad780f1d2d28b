#!/bin/bash
# gpu_round.sh, then the ncu summaries are written ON the box and the large
# .ncu-rep files dropped, so gpurun_out/ stays under gpurun's 64 MiB merge cap.
#   gpurun --timeout 3300 -- 'bash tools/gpu_round_small.sh reddit r01k'
cfg=${1:-reddit}
tag=${2:-r01}
bash tools/gpu_round.sh $cfg $tag
python tools/summarize_ncu.py --tag $tag > gpurun_out/summarize_$tag.log 2>&1
echo "summarize rc=$?" | tee -a gpurun_out/status_$tag.txt
mkdir -p gpurun_out/profiles_$tag
cp profiles/${tag}_* profiles/ncu_traffic.json gpurun_out/profiles_$tag/ 2>/dev/null
rm -f gpurun_out/*.ncu-rep
