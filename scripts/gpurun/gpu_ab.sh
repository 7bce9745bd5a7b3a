# A/B timing of library variants: gpu_ab.sh "<pytest -k expr>" "<configs>" lib1.so lib2.so ...
# (libs prebuilt in-tree; the first one also runs the parity tests).  A lib argument "VAR=v,lib.so"
# runs that variant with the environment variable set (e.g. SKETCH_F4_DEBUG=2).
K="$1"; CFGS="$2"; shift 2
out=gpurun_out/ab.log; : > $out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv >> $out
if [ -n "$K" ]; then
  SKETCH_LIB="${1##*,}" timeout 600 python -m pytest tests/test_gpu_parity.py -x -q -k "$K" > gpurun_out/ab_tests.log 2>&1
  echo "tests rc $? ($1)" >> $out; tail -3 gpurun_out/ab_tests.log >> $out
fi
for rep in 1 2; do
  for lib in "$@"; do
    for c in $CFGS; do
      envs=""; l="$lib"; case "$lib" in *,*) envs="${lib%,*}"; l="${lib##*,}";; esac
      echo "$lib $c $(env $envs SKETCH_LIB=$l timeout 300 python scripts/profile_apply.py --config $c --reps 5 | grep ms)" >> $out
    done
  done
done
