mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1 || { echo build failed; exit 1; }
bash scripts/gpurun/gpu_ab2.sh variants_tmp/lib_r1.so:c2,c3,c4,c5 variants_tmp/lib_cur6.so:c2,c3,c4,c5 > /dev/null 2>&1
python scripts/profile_apply.py --config c2 --reps 1 > gpurun_out/plain_c2g.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:sk_jki_kernel -c 1 -o gpurun_out/jki_c2 python scripts/profile_apply.py --config c2 --reps 1 > gpurun_out/ncu_jki.log 2>&1
cat gpurun_out/ab2.log; tail -3 gpurun_out/ncu_jki.log
