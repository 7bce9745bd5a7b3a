# persistent kernel tail: K-split of the last wave on (default) vs off
python -c "import __graft_entry__ as g; g.build()" > /dev/null 2>&1 || { echo build failed; exit 1; }
for rep in 1 2; do for sp in 1 0; do for rows in 50000000 6250000; do
  if [ $sp = 0 ]; then export SKETCH_F4_SPLIT=0; else unset SKETCH_F4_SPLIT; fi
  echo "split=$sp rows=$rows $(timeout 120 python scripts/profile_apply.py --config c5 --rows $rows --reps 7 2>&1 | grep '^ms')"
done; done; done
