python -c "import __graft_entry__ as g; g.build()" > /dev/null 2>&1 || { echo build failed; exit 1; }
timeout 600 python -m pytest tests/test_gpu_parity.py -x -q -p no:faulthandler -k "cuda_graph" 2>&1 | tail -30
