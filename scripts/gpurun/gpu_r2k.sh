mkdir -p gpurun_out/r2k
O=gpurun_out/r2k
python -c "import __graft_entry__ as g; g.build()" > $O/build.log 2>&1 || { echo build failed; exit 1; }
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_multigpu.py -x -q -k "jki or multirank or backend" -p no:faulthandler > $O/tests.log 2>&1; echo "tests rc $?" > $O/summary.txt
tail -2 $O/tests.log >> $O/summary.txt; grep -E "^FAILED|^ERROR" $O/tests.log | head >> $O/summary.txt
for dist in uniform gaussian; do timeout 600 python scripts/abnormal_bench.py --dist $dist 2>&1 | grep pattern >> $O/summary.txt; done

timeout 900 python scripts/jki_configs.py c2 c3 >> $O/summary.txt 2>&1
cat $O/summary.txt
