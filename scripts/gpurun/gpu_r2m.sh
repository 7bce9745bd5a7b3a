mkdir -p gpurun_out/r2m
O=gpurun_out/r2m
python -c "import __graft_entry__ as g; g.build()" > $O/build.log 2>&1 || { echo build failed; exit 1; }
python scripts/profile_apply.py --config c3 --dist uniform --jki --reps 3 > $O/plain.log 2>&1; echo "plain rc $?"; cat $O/plain.log | cut -c1-300
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $O/launches.csv python scripts/profile_apply.py --config c3 --dist uniform --jki --reps 2 > /dev/null 2>&1
grep -v "^==" $O/launches.csv | awk -F'","' '{print $5, $NF}' | cut -c1-120 | tail -12
ncu --set full --clock-control none --import-source on -k regex:"sk_jki_kernel" -s 1 -c 1 -o $O/ncu_jki_c3 -f \
  python scripts/profile_apply.py --config c3 --dist uniform --jki --reps 2 > $O/ncu.log 2>&1; echo "ncu rc $?"
