for lib in paper_2310_15419_b200/libsketch.so variants_tmp/libsk_idle.so; do
for args in "4 3000 2000" "12 3000 2000"; do
  echo "== $lib $args"; SKETCH_LIB=$lib SKETCH_F4_PERSIST=1 SKETCH_F4_PGRID=4 timeout 120 python scripts/f4p_probe.py $args 2>&1 | grep -v Warning | tail -2
done; done
