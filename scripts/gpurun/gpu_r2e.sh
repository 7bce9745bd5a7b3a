mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1 || { echo build failed; exit 1; }
timeout 1500 python -m pytest tests -m gpu -q > gpurun_out/gputests_e.log 2>&1; echo "tests rc $?" > gpurun_out/summary_e.txt
tail -3 gpurun_out/gputests_e.log >> gpurun_out/summary_e.txt
grep -E "^FAILED|Error" gpurun_out/gputests_e.log | head -20 >> gpurun_out/summary_e.txt
bash scripts/gpurun/gpu_ab2.sh variants_tmp/lib_r1.so:c2,c5 variants_tmp/lib_cur4.so:c2,c5 > /dev/null 2>&1
python scripts/profile_apply.py --config c5 --reps 2 > gpurun_out/plain_c5.log 2>&1 && \
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_c5.csv python scripts/profile_apply.py --config c5 --reps 2 > gpurun_out/ncu_c5.log 2>&1
python scripts/profile_apply.py --config c2 --reps 2 > gpurun_out/plain_c2.log 2>&1 && \
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_c2.csv python scripts/profile_apply.py --config c2 --reps 2 > gpurun_out/ncu_c2.log 2>&1
cat gpurun_out/summary_e.txt gpurun_out/ab2.log
