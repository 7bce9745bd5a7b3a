mkdir -p gpurun_out/r2af
O=gpurun_out/r2af
python -c "import __graft_entry__ as g; g.build()" > $O/build.log 2>&1 || { echo build failed; exit 1; }
for args in "12 3000 2000" "30 1500 700" "7 200000 2000"; do
  echo "== $args $(SKETCH_F4_PERSIST=1 SKETCH_F4_PGRID=4 timeout 120 python scripts/f4p_probe.py $args 2>&1 | grep -v Warning | tail -1)"
done
timeout 900 python -m pytest tests/test_gpu_parity.py -x -q -p no:faulthandler -k "f4 or rad_f64 or infinite or nan or config_c5" > $O/tests.log 2>&1; echo "tests rc $?"; tail -1 $O/tests.log
for rep in 1 2; do
  for rows in 50000000 25000000 6250000; do for pm in 0 1; do
    echo "rows=$rows persist=$pm $(SKETCH_F4_PERSIST=$pm timeout 120 python scripts/profile_apply.py --config c5 --rows $rows --reps 7 2>&1 | grep '^ms')"
  done; done
done
