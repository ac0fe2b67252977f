cp abtest/B.so paper_2412_07894_b200/libhyd.so
timeout 900 python -m pytest tests/test_small_gpu.py tests/test_parity_gpu.py tests/test_digests_gpu.py -k "not digests or cfg2 or cfg6 or cfg1" -q -x --timeout 800 > gpurun_out/pytest_abq8.log 2>&1; echo "pytest rc=$?"; tail -3 gpurun_out/pytest_abq8.log
CFG=2 bash tools/ab.sh
CFG=6 bash tools/ab.sh
