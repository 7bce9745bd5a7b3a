# persistent kernel: next-item scan started SK_F4P_SCANLEAD stages before the running item ends
mkdir -p gpurun_out/r2bj
O=gpurun_out/r2bj
python -c "import __graft_entry__ as g; g.build()" > /dev/null 2>&1 || { echo build failed; exit 1; }
for lib in variants_tmp/libsk_lead64.so variants_tmp/libsk_lead128.so; do
  echo "$lib probe $(SKETCH_LIB=$lib SKETCH_F4_PERSIST=1 SKETCH_F4_PGRID=4 timeout 120 python scripts/f4p_probe.py 12 3000 2000 2>&1 | tail -1)"
done
for rep in 1 2; do
  for lib in paper_2310_15419_b200/libsketch.so variants_tmp/libsk_lead64.so variants_tmp/libsk_lead128.so; do for rows in 50000000 6250000; do
    echo "$lib rows=$rows $(SKETCH_LIB=$lib timeout 120 python scripts/profile_apply.py --config c5 --rows $rows --reps 7 2>&1 | grep '^ms')"
  done; done
done
for lib in variants_tmp/libsk_lead64.so variants_tmp/libsk_lead128.so; do
  SKETCH_LIB=$lib timeout 300 ncu --metrics dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum --clock-control none -k regex:"sk_rad_f4p" -s 1 -c 1 python scripts/profile_apply.py --config c5 --reps 2 2>&1 | grep -E "dram__bytes|duration" | sed "s#^#$lib #"
done
