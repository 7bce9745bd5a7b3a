python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1
timeout 900 python -m pytest tests/test_gpu_parity.py -x -q -k "jki" > gpurun_out/jki_tests.log 2>&1; echo "tests rc $?" > gpurun_out/jki.log
tail -3 gpurun_out/jki_tests.log >> gpurun_out/jki.log
for dist in uniform gaussian; do timeout 600 python scripts/abnormal_bench.py --dist $dist 2>&1 | grep pattern >> gpurun_out/jki.log; done
