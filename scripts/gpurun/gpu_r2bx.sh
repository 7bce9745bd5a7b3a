# final-state validation: full GPU suite, smoke, default bench, a 200-step soak, N=2 (shared GPU), reference arm
mkdir -p gpurun_out/r2bx
O=gpurun_out/r2bx
python -c "import __graft_entry__ as g; g.build()" > $O/build.log 2>&1 || { echo build failed; exit 1; }
timeout 1500 python -m pytest tests -m gpu -q -p no:faulthandler > $O/gputests.log 2>&1; echo "tests rc $?" > $O/summary.txt
tail -1 $O/gputests.log >> $O/summary.txt; grep -E "^FAILED|^ERROR" $O/gputests.log | head >> $O/summary.txt
python -c "import __graft_entry__ as g; g.smoke()" > $O/smoke.log 2>&1; echo "smoke rc $?" >> $O/summary.txt
timeout 900 python bench.py > $O/bench1.json 2> $O/bench1.err; echo "bench1 rc $?" >> $O/summary.txt
timeout 900 python bench.py --steps 200 --warmup 5 --no-per-config > $O/soak.json 2> $O/soak.err; echo "soak rc $?" >> $O/summary.txt
timeout 900 python bench.py --gpus 2 > $O/bench2.json 2> $O/bench2.err; echo "bench2 rc $?" >> $O/summary.txt
timeout 900 python bench.py --impl reference > $O/ref.json 2> $O/ref.err; echo "ref rc $?" >> $O/summary.txt
cat $O/summary.txt
