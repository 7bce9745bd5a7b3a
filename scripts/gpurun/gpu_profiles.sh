# Round profile artifacts (each ncu step runs only after its command exited 0 without ncu):
#   bench line, per-config apply times, ncu launch list of the bench, ncu --set full of the headline kernel.
set -x
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1 || exit 1
python bench.py > gpurun_out/bench_c5.log 2>&1; tail -1 gpurun_out/bench_c5.log > gpurun_out/bench_c5.json
for c in c1 c2 c3 c4 c5; do echo "$c $(timeout 300 python scripts/profile_apply.py --config $c --reps 5 | grep ms)"; done > gpurun_out/apply_times.log 2>&1
python bench.py --steps 3 --warmup 3 > gpurun_out/bench_small.log 2>&1 && \
  ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_c5.csv \
    python bench.py --steps 3 --warmup 3 > gpurun_out/ncu_launch.log 2>&1
python scripts/profile_apply.py --config c5 --reps 2 > gpurun_out/plain_head.log 2>&1 && \
  ncu --set full --clock-control none --import-source on -k regex:"sk_rad_f4_kernel" -s 1 -c 1 -o gpurun_out/ncu_head -f \
    python scripts/profile_apply.py --config c5 --reps 2 > gpurun_out/ncu_head.log 2>&1
echo done
