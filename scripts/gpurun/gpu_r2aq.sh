# tensor-core row tiling: (6, 6, 4) tiles per column of c5 (default) vs balanced (6, 5, 5)
python -c "import __graft_entry__ as g; g.build()" > /dev/null 2>&1 || { echo build failed; exit 1; }
echo "bal probe $(SKETCH_LIB=variants_tmp/libsk_bal.so timeout 120 python scripts/f4p_probe.py 12 3000 2000 2>&1 | tail -1)"
for rep in 1 2; do
  for lib in paper_2310_15419_b200/libsketch.so variants_tmp/libsk_bal.so; do for rows in 50000000 6250000; do
    echo "$lib rows=$rows $(SKETCH_LIB=$lib timeout 120 python scripts/profile_apply.py --config c5 --rows $rows --reps 7 2>&1 | grep '^ms')"
  done; done
done
