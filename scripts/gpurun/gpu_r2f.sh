mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1 || { echo build failed; exit 1; }
timeout 1500 python -m pytest tests -m gpu -q -p no:faulthandler > gpurun_out/gputests_f.log 2>&1; echo "tests rc $?" > gpurun_out/summary_f.txt
tail -3 gpurun_out/gputests_f.log >> gpurun_out/summary_f.txt
grep -E "^FAILED|Error" gpurun_out/gputests_f.log | head -20 >> gpurun_out/summary_f.txt
bash scripts/gpurun/gpu_ab2.sh variants_tmp/lib_r1.so:c2,c3,c5 variants_tmp/lib_cur5.so:c2,c5 variants_tmp/lib_g_l0s8.so:c3 variants_tmp/lib_g_l0s0.so:c3 variants_tmp/lib_g_l16s8.so:c3 variants_tmp/lib_g_l0s8p1.so:c3 > /dev/null 2>&1
cat gpurun_out/summary_f.txt gpurun_out/ab2.log
