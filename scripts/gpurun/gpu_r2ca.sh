# per-rank share of c5 under row sharding (N = 1, 2, 4, 8) with the final kernels
python -c "import __graft_entry__ as g; g.build()" > /dev/null 2>&1 || { echo build failed; exit 1; }
for rows in 50000000 25000000 12500000 6250000; do
  echo "rows=$rows $(timeout 120 python scripts/profile_apply.py --config c5 --rows $rows --reps 9 2>&1 | grep '^ms')"
done
