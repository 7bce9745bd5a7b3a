# ncu --set full of the default ±1 fp64 kernel on c5 (after a plain run of the same command)
python scripts/profile_apply.py --config c5 --reps 2 > gpurun_out/plain_c5.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:sk_rad_f4 -s 1 -c 1 \
  -o gpurun_out/f4_c5 -f python scripts/profile_apply.py --config c5 --reps 2 > gpurun_out/ncu_f4.log 2>&1
echo rc $?
