# ncu --set full of the persistent tensor-core kernel on the 8-way row shard of c5 (rows [0, 6.25e6))
mkdir -p gpurun_out/r2an
O=gpurun_out/r2an
python -c "import __graft_entry__ as g; g.build()" > $O/build.log 2>&1 || { echo build failed; exit 1; }
python scripts/profile_apply.py --config c5 --rows 6250000 --reps 3 > $O/plain.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:"sk_rad_f4" -s 1 -c 1 -o $O/full_c5s8 python scripts/profile_apply.py --config c5 --rows 6250000 --reps 3 > $O/ncu.log 2>&1
echo "ncu rc $?"; cat $O/plain.log | tail -1
SKETCH_F4_PERSIST=0 python scripts/profile_apply.py --config c5 --rows 6250000 --reps 3 > $O/plain0.log 2>&1 && \
SKETCH_F4_PERSIST=0 ncu --set full --clock-control none --import-source on -k regex:"sk_rad_f4" -s 1 -c 1 -o $O/full_c5s8_peritem python scripts/profile_apply.py --config c5 --rows 6250000 --reps 3 > $O/ncu0.log 2>&1
echo "ncu0 rc $?"
