for v in A B; do cp abtest/$v.so paper_2412_07894_b200/libhyd.so
timeout 900 python -m pytest tests/test_small_gpu.py tests/test_ragged_gpu.py tests/test_digests_gpu.py -k "not digests or cfg1 or cfg6" -q -x --timeout 800 > gpurun_out/pytest_s4$v.log 2>&1; echo "pytest $v rc=$?"; tail -2 gpurun_out/pytest_s4$v.log; done
CFG=6 bash tools/abc.sh
CFG=1 bash tools/abc.sh
