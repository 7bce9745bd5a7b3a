# round 2, call BZ: persistent tensor-core kernel as the c5 default -- tests, smoke, bench, launch list, ncu of c5
mkdir -p gpurun_out/r2bz
O=gpurun_out/r2bz
python -c "import __graft_entry__ as g; g.build()" > $O/build.log 2>&1 || { echo build failed; exit 1; }
timeout 1500 python -m pytest tests -m gpu -q -p no:faulthandler > $O/gputests.log 2>&1; echo "tests rc $?" > $O/summary.txt
tail -2 $O/gputests.log >> $O/summary.txt; grep -E "^FAILED" $O/gputests.log | head >> $O/summary.txt
python -c "import __graft_entry__ as g; g.smoke()" > $O/smoke.log 2>&1; echo "smoke rc $?" >> $O/summary.txt
timeout 900 python bench.py > $O/bench1.json 2> $O/bench1.err; echo "bench1 rc $?" >> $O/summary.txt
timeout 900 python bench.py --gpus 2 --steps 5 --warmup 3 > $O/bench2.json 2> $O/bench2.err; echo "bench2 rc $?" >> $O/summary.txt
python bench.py --steps 2 --warmup 3 --no-cpu-baseline --no-e2e --no-per-config > $O/plain_bench.log 2>&1 && \
ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file $O/launches_bench.csv python bench.py --steps 2 --warmup 3 --no-cpu-baseline --no-e2e --no-per-config > $O/ncu_bench.log 2>&1
python scripts/profile_apply.py --config c5 --reps 3 > $O/plain_c5.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:"sk_rad_f4p_kernel" -s 1 -c 1 -o $O/full_c5 python scripts/profile_apply.py --config c5 --reps 3 > $O/ncu_full_c5.log 2>&1
echo "ncu rc $?" >> $O/summary.txt
cat $O/summary.txt
timeout 900 python bench.py --steps 200 --warmup 5 --no-per-config > $O/soak.json 2> $O/soak.err; echo "soak rc $?" >> $O/summary.txt; timeout 900 python bench.py --impl reference > $O/ref.json 2> $O/ref.err; echo "ref rc $?" >> $O/summary.txt; cat $O/summary.txt
