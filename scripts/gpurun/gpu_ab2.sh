# A/B of library variants: gpu_ab2.sh "lib:config,config ..." ...  (each lib runs its configs, 3 rounds)
out=gpurun_out/ab2.log; : > $out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv >> $out
python -c "import __graft_entry__ as g; g.build()" > /dev/null 2>&1
for rep in 1 2 3; do
  for spec in "$@"; do
    lib="${spec%%:*}"; cfgs="${spec#*:}"
    for c in ${cfgs//,/ }; do
      echo "$lib $c $(SKETCH_LIB=$lib timeout 300 python scripts/profile_apply.py --config $c --reps 7 2>&1 | grep '^ms')" >> $out
    done
  done
done
cat $out
