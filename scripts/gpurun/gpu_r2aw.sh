# ncu --set full of the Algorithm 4 kernel on Abnormal_A (Gaussian and uniform), d = 2000
mkdir -p gpurun_out/r2aw
O=gpurun_out/r2aw
python -c "import __graft_entry__ as g; g.build()" > $O/build.log 2>&1 || { echo build failed; exit 1; }
for dist in gaussian uniform; do
  python scripts/jki_profile.py --dist $dist > $O/plain_$dist.log 2>&1 && cat $O/plain_$dist.log && \
  ncu --set full --clock-control none --import-source on -k regex:"sk_jki_kernel" -s 1 -c 1 -o $O/jki_$dist python scripts/jki_profile.py --dist $dist > $O/ncu_$dist.log 2>&1
  echo "ncu $dist rc $?"
done
