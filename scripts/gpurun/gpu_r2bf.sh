# persistent kernel: nibble shifts as funnel rotates (SHF, SK_F4P_ROT=1) vs IMAD.SHL
python -c "import __graft_entry__ as g; g.build()" > /dev/null 2>&1 || { echo build failed; exit 1; }
echo "rot probe $(SKETCH_LIB=variants_tmp/libsk_rot.so SKETCH_F4_PERSIST=1 SKETCH_F4_PGRID=4 timeout 120 python scripts/f4p_probe.py 12 3000 2000 2>&1 | tail -1)"
for rep in 1 2; do
  for lib in paper_2310_15419_b200/libsketch.so variants_tmp/libsk_rot.so; do for rows in 50000000 6250000; do
    echo "$lib rows=$rows $(SKETCH_LIB=$lib timeout 120 python scripts/profile_apply.py --config c5 --rows $rows --reps 7 2>&1 | grep '^ms')"
  done; done
done
