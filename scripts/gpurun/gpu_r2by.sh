# bench variance: default bench 4x on one box
python -c "import __graft_entry__ as g; g.build()" > /dev/null 2>&1 || { echo build failed; exit 1; }
for k in 1 2 3 4; do
  timeout 600 python bench.py --no-per-config --no-cpu-baseline --no-e2e > /tmp/b$k.json 2>/dev/null
  python -c "
import json; d=json.loads(open('/tmp/b$k.json').read().strip().splitlines()[-1]); print($k, d['ms_per_step'], d['roofline']['frac'], d['clocks'])"
done
