python -c "import __graft_entry__ as g; g.build()" > /dev/null 2>&1 || { echo build failed; exit 1; }
for rows in 50000000 25000000 12500000 6250000 3125000; do
  for pm in 0 1; do
    echo "rows=$rows persist=$pm $(SKETCH_F4_PERSIST=$pm timeout 120 python scripts/profile_apply.py --config c5 --rows $rows --reps 7 2>&1 | grep '^ms')"
  done
done
