# round 2, GPU call A: build, full GPU tests, smoke, bench N=1 and N=2 (shared GPU), microbenchmarks
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1 || { echo build failed; tail gpurun_out/build.log; exit 1; }
nvidia-smi > gpurun_out/smi.txt 2>&1
(cd scripts && nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -o microbench_f32 microbench_f32.cu && timeout 120 ./microbench_f32) > gpurun_out/microbench_f32.txt 2>&1
timeout 1500 python -m pytest tests -m gpu -q -x > gpurun_out/gputests.log 2>&1; echo "tests rc $?" > gpurun_out/summary.txt
tail -15 gpurun_out/gputests.log >> gpurun_out/summary.txt
python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1; echo "smoke rc $?" >> gpurun_out/summary.txt
timeout 600 python bench.py --steps 20 --warmup 5 > gpurun_out/bench1.json 2> gpurun_out/bench1.err; echo "bench1 rc $?" >> gpurun_out/summary.txt
timeout 600 python bench.py --gpus 2 --steps 5 --warmup 3 --no-per-config > gpurun_out/bench2.json 2> gpurun_out/bench2.err; echo "bench2 rc $?" >> gpurun_out/summary.txt
SKETCH_F4_MIN_COL=1 timeout 600 python scripts/f4_threshold_sweep.py > gpurun_out/f4_sweep.txt 2>&1; echo "sweep rc $?" >> gpurun_out/summary.txt
cat gpurun_out/summary.txt
