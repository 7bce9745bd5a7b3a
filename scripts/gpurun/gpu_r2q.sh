mkdir -p gpurun_out/r2q
O=gpurun_out/r2q
python -c "import __graft_entry__ as g; g.build()" > $O/build.log 2>&1 || { echo build failed; exit 1; }
for k in 1 2; do
for pool in lib default; do
SKETCH_SCRATCH_POOL=$pool timeout 600 python bench.py --steps 10 --warmup 3 > $O/bench_$pool.json 2>/dev/null
python -c "
import json; d=json.loads(open('$O/bench_$pool.json').read().strip().splitlines()[-1]); print('$pool', d['ms_per_step'], d['e2e']['ms_per_step'])"
done; done
SKETCH_TIMING=1 timeout 600 python scripts/e2e_probe.py > $O/probe_lib.txt 2>&1
SKETCH_SCRATCH_POOL=default SKETCH_TIMING=1 timeout 600 python scripts/e2e_probe.py > $O/probe_default.txt 2>&1
tail -5 $O/probe_lib.txt $O/probe_default.txt
