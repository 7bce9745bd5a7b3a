# flakiness check: the GPU suite twice in a row, then the driver's round-end sequence
mkdir -p gpurun_out/r2bs
O=gpurun_out/r2bs
python -c "import __graft_entry__ as g; g.build()" > $O/build.log 2>&1 || { echo build failed; exit 1; }
for k in 1 2; do timeout 1500 python -m pytest tests -m gpu -q -p no:faulthandler > $O/tests$k.log 2>&1; echo "tests$k rc $?"; tail -1 $O/tests$k.log; done
python -c "import __graft_entry__ as g; g.smoke()" > $O/smoke.log 2>&1; echo "smoke rc $?"
timeout 900 python bench.py > $O/bench.json 2> $O/bench.err; echo "bench rc $?"; tail -c 300 $O/bench.json
