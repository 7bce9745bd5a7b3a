python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1
for i in 0 1 2 3 4; do timeout 60 python scripts/f4n_cases.py $i 2>&1 | grep -v Warning | grep -o 'max err.*\|illegal[a-z ]*' | head -1; done > gpurun_out/f4n_small.log 2>&1
for np in 8 16; do for dbg in 0 5; do echo "np $np dbg $dbg $(SKETCH_F4N_NP=$np SKETCH_F4N_DEBUG=$dbg timeout 120 python scripts/profile_apply.py --config c5 --reps 3 | grep ms)"; done; done >> gpurun_out/f4n_small.log 2>&1
