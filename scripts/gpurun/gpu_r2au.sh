# tensor-core vs SIMT per column length with the persistent tensor-core kernel (threshold re-measure)
python -c "import __graft_entry__ as g; g.build()" > /dev/null 2>&1 || { echo build failed; exit 1; }
SKETCH_F4_MIN_COL=1 timeout 1200 python scripts/f4_threshold_sweep.py 2>&1 | grep "^L"
