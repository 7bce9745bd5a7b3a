mkdir -p gpurun_out/r2y
O=gpurun_out/r2y
python -c "import __graft_entry__ as g; g.build()" > $O/build.log 2>&1 || { echo build failed; exit 1; }
SKETCH_F4_PERSIST=1 timeout 600 ncu --set full --import-source on --clock-control none -k regex:"sk_rad_f4" -s 1 -c 1 -o $O/ncu_p1 -f python scripts/profile_apply.py --config c5 --reps 2 > $O/ncu_p1.log 2>&1; echo "ncu rc $?"
