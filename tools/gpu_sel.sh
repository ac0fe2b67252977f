# select change: parity (keys in every digest, edge cases, multi-rank offsets), then A/B
timeout 1200 python -m pytest tests/test_parity_gpu.py tests/test_digests_gpu.py tests/test_race_gpu.py -q -x -m gpu --timeout 1100 > gpurun_out/pytest_sel.log 2>&1; echo "pytest rc=$?"; tail -3 gpurun_out/pytest_sel.log
for c in 5 4 6; do VARIANTS="A B" CFG=$c bash tools/abc.sh; done
