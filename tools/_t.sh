for cfg in c1 reddit; do
timeout 200 python tools/profile_kernels.py --config $cfg --reps 4 --spmm spmm:hubsplit:ft=64:rpc=4:vec=1:hubt=256,spmm:rowparallel:ft=64:rpc=4:vec=1:hubt=256 2>&1 | awk -v c=$cfg '{print c, $0}'
AUTOSAGE_DEV_LONG_ROW=2048 timeout 200 python tools/profile_kernels.py --config $cfg --reps 3 --spmm spmm:rowparallel:ft=64:rpc=4:vec=1:hubt=256 2>&1 | awk -v c=$cfg '{print c, "LR2048", $0}'
done
