mkdir -p gpurun_out/r2s
O=gpurun_out/r2s
python -c "import __graft_entry__ as g; g.build()" > $O/build.log 2>&1 || { echo build failed; exit 1; }
SKETCH_F4_PERSIST=1 timeout 900 python -m pytest tests/test_gpu_parity.py -x -q -p no:faulthandler -k "rad_f64 or nan or infinite or f4 or config or extreme_value or repeated or randomized or tiling or small or exact or shards or degenerate or index" > $O/tests.log 2>&1; echo "tests rc $?"; tail -2 $O/tests.log
for pm in 0 1; do
SKETCH_F4_PERSIST=$pm timeout 600 ncu --set full --clock-control none -k regex:"sk_rad_f4" -s 1 -c 1 -o $O/ncu_p$pm -f python scripts/profile_apply.py --config c5 --reps 2 > $O/ncu_p$pm.log 2>&1; echo "ncu $pm rc $?"
done
