mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1 || { echo build failed; exit 1; }
timeout 1500 python -m pytest tests -m gpu -q -x > gpurun_out/gputests_d.log 2>&1; echo "tests rc $?" > gpurun_out/summary_d.txt
tail -3 gpurun_out/gputests_d.log >> gpurun_out/summary_d.txt
grep -E "FAILED|Error|error" gpurun_out/gputests_d.log | head -20 >> gpurun_out/summary_d.txt
bash scripts/gpurun/gpu_ab2.sh variants_tmp/lib_r1.so:c2,c3,c4,c5 variants_tmp/lib_cur3.so:c2,c3,c4,c5 variants_tmp/lib_g_p0s8.so:c3 variants_tmp/lib_g_p1s0.so:c3 variants_tmp/lib_g_p0s0.so:c3 > /dev/null 2>&1
cat gpurun_out/summary_d.txt gpurun_out/ab2.log
