# dispatch change: parity on the general (MODE 1/2, windowed) paths, then A/B timing
timeout 1200 python -m pytest tests/test_parity_gpu.py tests/test_digests_gpu.py tests/test_pipe_index_gpu.py tests/test_ragged_gpu.py -q -x -m gpu --timeout 1100 > gpurun_out/pytest_disp.log 2>&1; echo "pytest rc=$?"; tail -3 gpurun_out/pytest_disp.log
for c in 5 3 2 4; do VARIANTS="A B" CFG=$c bash tools/abc.sh; done
