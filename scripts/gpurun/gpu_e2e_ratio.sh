# sketch_apply_host group-size ratio sweep on c5 (SKETCH_HOST_RATIO)
for r in 1.0 0.9 0.84 0.75; do echo "ratio $r"; SKETCH_HOST_RATIO=$r SKETCH_TIMING=1 python scripts/e2e_probe.py 2>&1 | grep "groups=\(0\|8\|16\)" ; done > gpurun_out/e2e_ratio.txt
