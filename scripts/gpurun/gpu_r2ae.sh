python -c "import __graft_entry__ as g; g.build()" > /dev/null 2>&1 || { echo build failed; exit 1; }
echo "blean probe $(SKETCH_LIB=variants_tmp/libsk_blean.so timeout 120 python scripts/f4p_probe.py 12 3000 2000 2>&1 | tail -1)"
echo "blean probe $(SKETCH_LIB=variants_tmp/libsk_blean.so SKETCH_F4_PERSIST=0 timeout 120 python scripts/f4p_probe.py 30 1500 700 2>&1 | tail -1)"
for rep in 1 2 3; do
  for lib in paper_2310_15419_b200/libsketch.so variants_tmp/libsk_blean.so; do
    echo "$lib c5 $(SKETCH_LIB=$lib timeout 120 python scripts/profile_apply.py --config c5 --reps 7 2>&1 | grep '^ms')"
  done
done
