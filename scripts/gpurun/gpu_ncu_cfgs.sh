# ncu --set full of the apply kernel of c2, c3, c4 (after plain runs of the same commands)
for c in c2 c3 c4; do python scripts/profile_apply.py --config $c --reps 2 > gpurun_out/plain_$c.log 2>&1 || exit 1; done
for c in c2 c3 c4; do
  ncu --set full --clock-control none --import-source on -k regex:"sk_(pair|rad)_kernel" -s 1 -c 1 \
    -o gpurun_out/ncu_$c -f python scripts/profile_apply.py --config $c --reps 2 > gpurun_out/ncu_$c.log 2>&1
done
echo done
