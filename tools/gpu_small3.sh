timeout 900 python -m pytest tests/test_small_gpu.py tests/test_ragged_gpu.py tests/test_digests_gpu.py -k "not digests or cfg1 or cfg6" -q -x --timeout 800 > gpurun_out/pytest_small3.log 2>&1; echo "pytest rc=$?"
tail -15 gpurun_out/pytest_small3.log
CFG=6 bash tools/ab.sh
