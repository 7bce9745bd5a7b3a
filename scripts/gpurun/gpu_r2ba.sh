# upper bound of what less digit work could give the persistent kernel (results invalid in the variants)
python -c "import __graft_entry__ as g; g.build()" > /dev/null 2>&1 || { echo build failed; exit 1; }
for rep in 1 2; do
  for lib in paper_2310_15419_b200/libsketch.so variants_tmp/libsk_nob1.so variants_tmp/libsk_nob2.so; do
    echo "$lib c5 $(SKETCH_LIB=$lib timeout 120 python scripts/profile_apply.py --config c5 --reps 7 2>&1 | grep '^ms')"
  done
done
