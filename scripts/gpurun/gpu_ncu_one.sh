# ncu --set full of one config's apply kernel: bash scripts/gpurun/gpu_ncu_one.sh <config> <kernel regex> <tag>
python scripts/profile_apply.py --config $1 --reps 2 > gpurun_out/plain_$3.log 2>&1 || exit 1
ncu --set full --clock-control none --import-source on -k regex:"$2" -s 1 -c 1 -o gpurun_out/ncu_$3 -f \
  python scripts/profile_apply.py --config $1 --reps 2 > gpurun_out/ncu_$3.log 2>&1
echo rc $?
