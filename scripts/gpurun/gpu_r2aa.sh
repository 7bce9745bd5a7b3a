mkdir -p gpurun_out/r2aa
O=gpurun_out/r2aa
python -c "import __graft_entry__ as g; g.build()" > $O/build.log 2>&1 || { echo build failed; exit 1; }
for args in "12 3000 2000" "30 1500 700"; do
  echo "== $args"; SKETCH_F4_PERSIST=1 SKETCH_F4_PGRID=4 timeout 120 python scripts/f4p_probe.py $args 2>&1 | grep -v Warning | tail -1
done
for rep in 1 2; do
  for pm in 0 1; do
    echo "persist=$pm c5 $(SKETCH_F4_PERSIST=$pm timeout 120 python scripts/profile_apply.py --config c5 --reps 7 2>&1 | grep '^ms')"
    echo "persist=$pm c5/8 $(SKETCH_F4_PERSIST=$pm timeout 120 python scripts/profile_apply.py --config c5 --rows 6250000 --reps 7 2>&1 | grep '^ms')"
  done
done
