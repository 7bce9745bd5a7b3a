# persistent kernel: 4 K-steps per stage with the digits split over 4 B warps (one per SM sub-partition)
python -c "import __graft_entry__ as g; g.build()" > /dev/null 2>&1 || { echo build failed; exit 1; }
for lib in variants_tmp/libsk_s4b4.so variants_tmp/libsk_s4.so; do
  echo "$lib probe $(SKETCH_LIB=$lib SKETCH_F4_PERSIST=1 SKETCH_F4_PGRID=4 timeout 120 python scripts/f4p_probe.py 12 3000 2000 2>&1 | tail -1)"
  echo "$lib probe $(SKETCH_LIB=$lib SKETCH_F4_PERSIST=1 SKETCH_F4_PGRID=4 timeout 120 python scripts/f4p_probe.py 30 1500 700 2>&1 | tail -1)"
done
for rep in 1 2; do
  for lib in paper_2310_15419_b200/libsketch.so variants_tmp/libsk_s4b4.so variants_tmp/libsk_s4.so; do for rows in 50000000 6250000; do
    echo "$lib rows=$rows $(SKETCH_LIB=$lib timeout 120 python scripts/profile_apply.py --config c5 --rows $rows --reps 7 2>&1 | grep '^ms')"
  done; done
done
