set -x
timeout 900 python -m pytest tests/test_small_gpu.py tests/test_ragged_gpu.py tests/test_parity_gpu.py tests/test_bb_gpu.py tests/test_pipe_index_gpu.py tests/test_digests_gpu.py -k "not digests or cfg1 or cfg2 or cfg6" -q -x --timeout 800 > gpurun_out/pytest_small.log 2>&1; echo "pytest rc=$?"
tail -30 gpurun_out/pytest_small.log
for c in 6 1; do timeout 600 python bench.py --config $c --steps 10 --warmup 3 --no-cpu > gpurun_out/bench_small_cfg$c.json 2> gpurun_out/bench_small_cfg$c.err; echo "bench cfg$c rc=$?"; tail -c 2500 gpurun_out/bench_small_cfg$c.json; done
