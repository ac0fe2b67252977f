# small flagged sets to the warp queue: parity (digests of every config, reduced / edge cases), then A/B
timeout 1500 python -m pytest tests/test_digests_gpu.py tests/test_parity_gpu.py tests/test_pipe_index_gpu.py tests/test_ragged_gpu.py tests/test_bb_gpu.py -q -x -m gpu --timeout 1400 > gpurun_out/pytest_fq.log 2>&1; echo "pytest rc=$?"; tail -3 gpurun_out/pytest_fq.log
for c in 2 3 4; do VARIANTS="A B" CFG=$c bash tools/abc.sh; done
