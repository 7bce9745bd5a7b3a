# Algorithm 4: one record load per entry, S reused across a row: jki tests, Abnormal patterns, reuse sweep
mkdir -p gpurun_out/r2bg
O=gpurun_out/r2bg
python -c "import __graft_entry__ as g; g.build()" > $O/build.log 2>&1 || { echo build failed; exit 1; }
timeout 900 python -m pytest tests/test_gpu_parity.py -x -q -k "jki or cuda_graph or sap" -p no:faulthandler > $O/tests.log 2>&1; echo "tests rc $?"; tail -1 $O/tests.log; grep -E "^FAILED" $O/tests.log | head -3
for dist in uniform gaussian; do timeout 600 python scripts/abnormal_bench.py --dist $dist 2>&1 | grep pattern; done > $O/abnormal.jsonl
cat $O/abnormal.jsonl | cut -c1-250
cd scripts && timeout 1200 python jki_reuse_sweep.py > ../$O/sweep.jsonl 2>&1; cd ..
cat $O/sweep.jsonl | cut -c1-200
