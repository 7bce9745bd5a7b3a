python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1
for dbg in 0 2; do echo "dbg $dbg $(SKETCH_F4_DEBUG=$dbg timeout 60 python scripts/profile_apply.py --config c5 --reps 3 | grep ms)"; done > gpurun_out/f4n_small.log 2>&1
timeout 300 python -m pytest tests/test_gpu_parity.py -x -q -k "rad_f64_kernel_paths and fp4" >> gpurun_out/f4n_small.log 2>&1
