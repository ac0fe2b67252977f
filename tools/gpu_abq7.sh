cp abtest/B.so paper_2412_07894_b200/libhyd.so
timeout 900 python -m pytest tests/test_parity_gpu.py tests/test_ragged_gpu.py tests/test_digests_gpu.py -k "not digests or cfg2 or cfg3" -q -x --timeout 800 > gpurun_out/pytest_abq7.log 2>&1; echo "pytest rc=$?"; tail -3 gpurun_out/pytest_abq7.log
CFG=4 bash tools/ab.sh
