python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1
for lib in libsketch.so libsketch_g128.so; do for c in c3; do echo "$lib $(SKETCH_LIB=paper_2310_15419_b200/$lib timeout 60 python scripts/profile_apply.py --config $c --reps 3 | grep ms)"; done; done > gpurun_out/f4n_small.log 2>&1
