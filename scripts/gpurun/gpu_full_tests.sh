python -c "import __graft_entry__ as g; g.build(); g.smoke()" > gpurun_out/smoke.log 2>&1; echo "smoke $?" > gpurun_out/full_tests.log
timeout 1500 python -m pytest tests -m gpu -q > gpurun_out/gputests.log 2>&1; echo "tests $?" >> gpurun_out/full_tests.log
tail -5 gpurun_out/gputests.log >> gpurun_out/full_tests.log
