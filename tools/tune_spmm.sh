cfg=${1:-reddit}
for lr in 0 2048 4096; do
  AUTOSAGE_DEV_LONG_ROW=$lr timeout 120 python tools/profile_kernels.py --config $cfg --reps 3 --spmm spmm:rowparallel:ft=64:rpc=4:vec=1:hubt=256,spmm:hubsplit:ft=64:rpc=4:vec=1:hubt=256 2>&1 | awk -v c=$cfg -v lr=$lr '{print c, "lr="lr, "tune=", $0}'
done
for tma in 1 0; do
AUTOSAGE_DEV_SDDMM_TMA=$tma timeout 120 python tools/profile_kernels.py --config $cfg --reps 3 --sddmm sddmm:rowparallel:ft=64:rpc=4:vec=1:hubt=256,sddmm:rowparallel:ft=64:rpc=1:vec=1:hubt=256,sddmm:rowparallel:ft=64:rpc=16:vec=1:hubt=256,sddmm:rowparallel:ft=64:rpc=4:vec=0:hubt=256 2>&1 | awk -v c=$cfg -v t=$tma '{print c, "tma="t, "tune=", $0}'
done
