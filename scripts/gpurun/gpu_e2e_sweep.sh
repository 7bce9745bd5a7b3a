# sketch_apply_host sweep on c5: column groups x size ratio (SKETCH_HOST_RATIO)
for r in 0.80 0.84 0.88; do echo "ratio $r"; SKETCH_HOST_RATIO=$r python scripts/e2e_probe.py 2>&1 | grep "groups=\(0\|8\|16\)"; done > gpurun_out/e2e_sweep.txt
