# persistent kernel: S transpose one stage short with paired 8-byte stores (SK_F4P_T4) vs full transpose
python -c "import __graft_entry__ as g; g.build()" > /dev/null 2>&1 || { echo build failed; exit 1; }
for args in "12 3000 2000" "30 1500 700" "7 200000 2000" "200 1300 300"; do
  echo "bt4 probe $args $(SKETCH_LIB=variants_tmp/libsk_bt4.so SKETCH_F4_PERSIST=1 SKETCH_F4_PGRID=4 timeout 120 python scripts/f4p_probe.py $args 2>&1 | tail -1)"
done
for rep in 1 2; do
  for lib in paper_2310_15419_b200/libsketch.so variants_tmp/libsk_bt4.so; do for rows in 50000000 6250000; do
    echo "$lib rows=$rows $(SKETCH_LIB=$lib timeout 120 python scripts/profile_apply.py --config c5 --rows $rows --reps 7 2>&1 | grep '^ms')"
  done; done
done
