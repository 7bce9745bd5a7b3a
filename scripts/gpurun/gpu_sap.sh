python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1
timeout 600 python -m pytest tests/test_gpu_parity.py -x -q -k "sap" > gpurun_out/sap_tests.log 2>&1; echo "tests rc $?" > gpurun_out/sap.log
tail -3 gpurun_out/sap_tests.log >> gpurun_out/sap.log
for cfg in "--dist gaussian --method qr" "--dist rademacher --method qr" "--dist gaussian --method svd"; do timeout 600 python scripts/sap_demo.py $cfg 2>&1 | grep -v Warn | tail -1 >> gpurun_out/sap.log; done
