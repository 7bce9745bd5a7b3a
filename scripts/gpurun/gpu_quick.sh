# quick GPU check: build, selected parity tests, per-config apply times (args: pytest -k expr, configs)
K="$1"; shift
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1 || { echo build failed; exit 1; }
timeout 600 python -m pytest tests/test_gpu_parity.py -x -q -k "$K" > gpurun_out/quick_tests.log 2>&1; echo "tests rc $?" > gpurun_out/quick.log
tail -3 gpurun_out/quick_tests.log >> gpurun_out/quick.log
for c in "$@"; do echo "$c $(timeout 300 python scripts/profile_apply.py --config $c --reps 5 | grep ms)" >> gpurun_out/quick.log; done
