python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1
for lib in libsketch.so libsketch_t32.so libsketch_t16.so; do echo "$lib $(SKETCH_LIB=paper_2310_15419_b200/$lib SKETCH_RAD_F64_PATH=fp4t timeout 120 python scripts/profile_apply.py --config c5 --reps 3 | grep ms)"; done > gpurun_out/f4n_small.log 2>&1
