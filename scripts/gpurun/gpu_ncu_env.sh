# ncu --set full of one config's apply kernel with env settings: bash scripts/gpurun/gpu_ncu_env.sh <config> <kernel regex> <tag> [ENV=VAL ...]
c=$1; k=$2; tag=$3; shift 3
env "$@" python scripts/profile_apply.py --config $c --reps 2 > gpurun_out/plain_$tag.log 2>&1 || exit 1
env "$@" ncu --set full --clock-control none --import-source on -k regex:"$k" -s 1 -c 1 -o gpurun_out/ncu_$tag -f \
  python scripts/profile_apply.py --config $c --reps 2 > gpurun_out/ncu_$tag.log 2>&1
echo rc $?
