cp abtest/B.so paper_2412_07894_b200/libhyd.so
timeout 900 python -m pytest tests/test_parity_gpu.py tests/test_digests_gpu.py tests/test_pipe_index_gpu.py tests/test_race_gpu.py -k "not digests or cfg5 or cfg3 or cfg4" -q -x --timeout 800 > gpurun_out/pytest_abq5.log 2>&1; echo "pytest rc=$?"; tail -3 gpurun_out/pytest_abq5.log

CFG=4 EXTRA="--candidates 512" bash tools/ab.sh
CFG=5 bash tools/ab.sh
