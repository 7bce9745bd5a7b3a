# persistent kernel with 4 K-steps per stage (its own constants; the per-item kernel unchanged)
mkdir -p gpurun_out/r2as
O=gpurun_out/r2as
python -c "import __graft_entry__ as g; g.build()" > $O/build.log 2>&1 || { echo build failed; exit 1; }
for args in "12 3000 2000" "30 1500 700" "7 200000 2000" "200 1300 300"; do
  echo "== $args $(SKETCH_F4_PERSIST=1 SKETCH_F4_PGRID=4 timeout 120 python scripts/f4p_probe.py $args 2>&1 | grep -v Warning | tail -1)"
done
timeout 1500 python -m pytest tests -m gpu -q -p no:faulthandler > $O/tests.log 2>&1; echo "tests rc $?"; tail -1 $O/tests.log; grep -E "^FAILED" $O/tests.log | head
for rep in 1 2; do for rows in 50000000 25000000 6250000; do for pm in 0 1; do
  echo "rows=$rows persist=$pm $(SKETCH_F4_PERSIST=$pm timeout 120 python scripts/profile_apply.py --config c5 --rows $rows --reps 7 2>&1 | grep '^ms')"
done; done; done
