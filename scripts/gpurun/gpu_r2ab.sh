mkdir -p gpurun_out/r2ab
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/r2ab/build.log 2>&1 || { echo build failed; exit 1; }
for pm in 0 1; do for args in "12 3000 2000" "30 1500 700" "7 200000 2000"; do
  echo "== bw4 persist=$pm $args $(SKETCH_LIB=variants_tmp/libsk_bw4.so SKETCH_F4_PERSIST=$pm SKETCH_F4_PGRID=4 timeout 120 python scripts/f4p_probe.py $args 2>&1 | grep -v Warning | tail -1)"
done; done
for rep in 1 2; do
  for lib in paper_2310_15419_b200/libsketch.so variants_tmp/libsk_bw4.so; do for pm in 0 1; do
    echo "$lib persist=$pm c5 $(SKETCH_LIB=$lib SKETCH_F4_PERSIST=$pm timeout 120 python scripts/profile_apply.py --config c5 --reps 7 2>&1 | grep '^ms')"
    echo "$lib persist=$pm c5/8 $(SKETCH_LIB=$lib SKETCH_F4_PERSIST=$pm timeout 120 python scripts/profile_apply.py --config c5 --rows 6250000 --reps 7 2>&1 | grep '^ms')"
  done; done
done
