mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1 || { echo build failed; exit 1; }
timeout 1200 python -m pytest tests/test_gpu_parity.py tests/test_multigpu.py -q -x -k "rad or inf or nan or f4 or extreme or repeated or config_c3 or config_c4 or config_c5 or gaussian or multirank or small" > gpurun_out/gputests_c.log 2>&1; echo "tests rc $?" > gpurun_out/summary_c.txt
tail -3 gpurun_out/gputests_c.log >> gpurun_out/summary_c.txt
bash scripts/gpurun/gpu_ab2.sh variants_tmp/lib_r1.so:c3,c4,c5 variants_tmp/lib_cur2.so:c3,c4,c5 > /dev/null 2>&1
cat gpurun_out/summary_c.txt gpurun_out/ab2.log
