mkdir -p gpurun_out/r2ad
O=gpurun_out/r2ad
python -c "import __graft_entry__ as g; g.build()" > $O/build.log 2>&1 || { echo build failed; exit 1; }
timeout 1500 python -m pytest tests -m gpu -q -p no:faulthandler > $O/tests.log 2>&1; echo "tests rc $?" > $O/summary.txt
tail -1 $O/tests.log >> $O/summary.txt; grep -E "^FAILED|^ERROR" $O/tests.log | head >> $O/summary.txt
python -c "import __graft_entry__ as g; g.smoke()" > $O/smoke.log 2>&1; echo "smoke rc $?" >> $O/summary.txt
timeout 900 python bench.py > $O/bench.json 2> $O/bench.err; echo "bench rc $?" >> $O/summary.txt
timeout 900 python bench.py --gpus 2 > $O/bench_g2.json 2> $O/bench_g2.err; echo "g2 rc $?" >> $O/summary.txt
cat $O/summary.txt
