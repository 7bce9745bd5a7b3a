set -x
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv
python -c "import __graft_entry__ as g; g.build(); g.smoke()" > gpurun_out/smoke.log 2>&1; echo smoke $?
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/gputests.log 2>&1; echo tests $?
for c in c1 c2 c3 c4 c5; do timeout 300 python scripts/profile_apply.py --config $c --reps 5; done > gpurun_out/apply.log 2>&1
timeout 600 python bench.py > gpurun_out/bench.log 2>&1; echo bench $?
