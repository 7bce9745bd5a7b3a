mkdir -p gpurun_out/r2u
O=gpurun_out/r2u
python -c "import __graft_entry__ as g; g.build()" > $O/build.log 2>&1 || { echo build failed; exit 1; }
for args in "4 3000 2000" "12 3000 2000" "40 3000 2000" "40 3000 1000"; do
  echo "== $args"; SKETCH_F4_PERSIST=1 SKETCH_F4_PGRID=4 timeout 120 python scripts/f4p_probe.py $args 2>&1 | tail -2
done
SKETCH_F4_PERSIST=1 SKETCH_F4_PGRID=4 timeout 300 compute-sanitizer --tool memcheck python scripts/f4p_probe.py 12 3000 2000 > $O/memcheck.log 2>&1; echo "memcheck rc $?"; grep -m5 -A12 "Invalid\|Error\|error" $O/memcheck.log | head -40
