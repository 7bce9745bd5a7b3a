# SIMT kernels (sketch_kernels.cu) under other ptxas levels / a register cap: c2, c3, c4 apply times
python -c "import __graft_entry__ as g; g.build()" > /dev/null 2>&1 || { echo build failed; exit 1; }
for rep in 1 2; do
  for lib in paper_2310_15419_b200/libsketch.so variants_tmp/libsk_k_o2.so variants_tmp/libsk_k_o1.so variants_tmp/libsk_k_r96.so; do for c in c2 c3 c4; do
    echo "$lib $c $(SKETCH_LIB=$lib timeout 120 python scripts/profile_apply.py --config $c --reps 7 2>&1 | grep '^ms')"
  done; done
done
