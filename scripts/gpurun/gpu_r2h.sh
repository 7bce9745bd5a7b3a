# round 2, call H: tests, bench N=1 / N=2, calibration benches, oracle timings, ncu captures
mkdir -p gpurun_out/r2h
O=gpurun_out/r2h
python -c "import __graft_entry__ as g; g.build()" > $O/build.log 2>&1 || { echo build failed; exit 1; }
timeout 1500 python -m pytest tests -m gpu -q -p no:faulthandler > $O/gputests.log 2>&1; echo "tests rc $?" > $O/summary.txt
tail -2 $O/gputests.log >> $O/summary.txt; grep -E "^FAILED" $O/gputests.log | head >> $O/summary.txt
python -c "import __graft_entry__ as g; g.smoke()" > $O/smoke.log 2>&1; echo "smoke rc $?" >> $O/summary.txt
timeout 900 python bench.py --steps 20 --warmup 5 > $O/bench1.json 2> $O/bench1.err; echo "bench1 rc $?" >> $O/summary.txt
timeout 900 python bench.py --gpus 2 --steps 5 --warmup 3 > $O/bench2.json 2> $O/bench2.err; echo "bench2 rc $?" >> $O/summary.txt
timeout 600 python scripts/abnormal_bench.py --dist uniform > $O/abnormal_uniform.jsonl 2>&1; echo "abn u rc $?" >> $O/summary.txt
timeout 600 python scripts/abnormal_bench.py --dist gaussian > $O/abnormal_gaussian.jsonl 2>&1; echo "abn g rc $?" >> $O/summary.txt
for pp in kji jki; do SKETCH_PAIR_PATH=$pp timeout 300 python scripts/profile_apply.py --config c2 --dist gaussian --reps 5 | grep -E "^ms|kernel" > $O/c2_gauss_$pp.txt 2>&1; done
timeout 900 python scripts/oracle_times.py > $O/oracle_times.jsonl 2> $O/oracle_times.err; echo "oracle rc $?" >> $O/summary.txt
python bench.py --steps 2 --warmup 3 --no-cpu-baseline --no-e2e --no-per-config > $O/plain_bench.log 2>&1 && \
ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file $O/launches_bench.csv python bench.py --steps 2 --warmup 3 --no-cpu-baseline --no-e2e --no-per-config > $O/ncu_bench.log 2>&1
for c in c5 c3 c4 c2; do
  python scripts/profile_apply.py --config $c --reps 3 > $O/plain_$c.log 2>&1 && \
  ncu --set full --clock-control none --import-source on -k regex:"sk_rad_f4_kernel|sk_pair_kernel|sk_rad_kernel|sk_jki_kernel" -s 1 -c 1 -o $O/full_$c python scripts/profile_apply.py --config $c --reps 3 > $O/ncu_full_$c.log 2>&1
done
cat $O/summary.txt
