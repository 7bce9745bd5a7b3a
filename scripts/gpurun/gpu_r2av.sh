# thresholds 896 (persistent) / 1280 (per-item): full GPU suite + smoke + c5 bench
mkdir -p gpurun_out/r2av
O=gpurun_out/r2av
python -c "import __graft_entry__ as g; g.build()" > $O/build.log 2>&1 || { echo build failed; exit 1; }
timeout 1500 python -m pytest tests -m gpu -q -p no:faulthandler > $O/tests.log 2>&1; echo "tests rc $?"; tail -1 $O/tests.log; grep -E "^FAILED" $O/tests.log | head
python -c "import __graft_entry__ as g; g.smoke()" > $O/smoke.log 2>&1; echo "smoke rc $?"
SKETCH_F4_MIN_COL= timeout 600 python scripts/f4_threshold_sweep.py 2>&1 | grep "^L" | head -8
