python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1
for args in "--dist uniform" "--dist uniform24" "--dist uniform --f32" "--dist uniform24 --f32" "--dist gaussian" "--dist gaussian --f32"; do echo "$args $(timeout 60 python scripts/profile_apply.py --config c2 --reps 3 $args | grep ms)"; done > gpurun_out/f4n_small.log 2>&1
