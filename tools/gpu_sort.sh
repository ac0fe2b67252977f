# sort change: parity (every config's digests incl. sorted_len / perm / cost, edge cases), then A/B
timeout 1200 python -m pytest tests/test_parity_gpu.py tests/test_digests_gpu.py tests/test_small_gpu.py tests/test_ragged_gpu.py -q -x -m gpu --timeout 1100 > gpurun_out/pytest_sort.log 2>&1; echo "pytest rc=$?"; tail -3 gpurun_out/pytest_sort.log
for c in 2 6 3 4; do VARIANTS="A B" CFG=$c bash tools/abc.sh; done
