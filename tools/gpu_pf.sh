# unstaged-lanes prefetch: config-5 parity (full digests, prefix parity), then A/B on config 5
timeout 1200 python -m pytest tests/test_digests_gpu.py tests/test_parity_gpu.py -q -x -m gpu --timeout 1100 -k "5 or cfg5 or prefix or big" > gpurun_out/pytest_pf.log 2>&1; echo "pytest rc=$?"; tail -3 gpurun_out/pytest_pf.log
VARIANTS="A B" CFG=5 bash tools/abc.sh
