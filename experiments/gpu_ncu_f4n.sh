python scripts/profile_apply.py --config c5 --reps 2 > gpurun_out/plain_c5n.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:sk_rad_f4n -s 1 -c 1 \
  -o gpurun_out/f4n_c5 -f python scripts/profile_apply.py --config c5 --reps 2 > gpurun_out/ncu_f4n.log 2>&1
echo rc $?
