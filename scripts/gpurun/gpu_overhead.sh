# c5 apply time vs column length (rows [0, R) of c5): separates per-item fixed cost from the
# per-nonzero cost of the default ±1 fp64 kernel
for r in 50000000 25000000 12500000 6250000; do
  echo "$r $(timeout 300 python scripts/profile_apply.py --config c5 --reps 5 --rows $r | grep '^ms')"
done > gpurun_out/overhead.log 2>&1
