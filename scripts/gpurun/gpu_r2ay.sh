# uniform53 from the Philox bits (no I2F.F64.U64) vs the conversion: c2 / c3 apply times, bit-exact check
python -c "import __graft_entry__ as g; g.build()" > /dev/null 2>&1 || { echo build failed; exit 1; }
SKETCH_LIB=variants_tmp/libsk_u53.so timeout 600 python -m pytest tests/test_gpu_parity.py -q -x -p no:faulthandler -k "fill_s or small or gaussian_entries or curand or config_c2 or config_c3 or jki_matches" 2>&1 | tail -1
for rep in 1 2; do
  for lib in paper_2310_15419_b200/libsketch.so variants_tmp/libsk_u53.so; do for c in c2 c3; do
    echo "$lib $c $(SKETCH_LIB=$lib timeout 120 python scripts/profile_apply.py --config $c --reps 7 2>&1 | grep '^ms')"
  done; done
done
