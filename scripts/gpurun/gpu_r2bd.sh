# persistent kernel tail policy: current (split the last wave along K when N mod W < W/2) vs
# SK_F4P_TAIL=1 (always split the last W items along K) vs 2 (and the last W halves by row tiles)
python -c "import __graft_entry__ as g; g.build()" > /dev/null 2>&1 || { echo build failed; exit 1; }
for m in 1 2; do for args in "200 3000 2000" "400 1500 700" "160 2100 700"; do
  echo "tail$m probe $args $(SKETCH_LIB=variants_tmp/libsk_tail$m.so timeout 120 python scripts/f4p_probe.py $args 2>&1 | tail -1)"
done; done
for rep in 1 2; do
  for lib in paper_2310_15419_b200/libsketch.so variants_tmp/libsk_tail1.so variants_tmp/libsk_tail2.so; do for rows in 50000000 25000000 6250000; do
    echo "$lib rows=$rows $(SKETCH_LIB=$lib timeout 120 python scripts/profile_apply.py --config c5 --rows $rows --reps 7 2>&1 | grep '^ms')"
  done; done
done
