mkdir -p gpurun_out/r2i
O=gpurun_out/r2i
python -c "import __graft_entry__ as g; g.build()" > $O/build.log 2>&1 || { echo build failed; exit 1; }
timeout 1500 python -m pytest tests -m gpu -q -p no:faulthandler > $O/gputests.log 2>&1; echo "tests rc $?" > $O/summary.txt
tail -2 $O/gputests.log >> $O/summary.txt; grep -E "^FAILED" $O/gputests.log | head >> $O/summary.txt
python -c "import __graft_entry__ as g; g.smoke()" > $O/smoke.log 2>&1; echo "smoke rc $?" >> $O/summary.txt
timeout 900 python bench.py > $O/bench_default.json 2> $O/bench_default.err; echo "bench rc $?" >> $O/summary.txt
timeout 900 python bench.py --impl reference > $O/bench_ref.json 2> $O/bench_ref.err; echo "ref rc $?" >> $O/summary.txt
cat $O/summary.txt; tail -c 600 $O/bench_default.json
