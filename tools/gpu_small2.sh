timeout 900 python -m pytest tests/test_small_gpu.py tests/test_ragged_gpu.py tests/test_digests_gpu.py -k "not digests or cfg1 or cfg6" -q -x --timeout 800 > gpurun_out/pytest_small2.log 2>&1; echo "pytest rc=$?"
tail -15 gpurun_out/pytest_small2.log
for c in 6 1; do timeout 600 python bench.py --config $c --steps 10 --warmup 3 --no-cpu > gpurun_out/bench_small2_cfg$c.json 2> gpurun_out/bench_small2_cfg$c.err; echo "bench cfg$c rc=$?"; python -c "
import json; d=json.load(open('gpurun_out/bench_small2_cfg$c.json')); print(d['value']/1e6, d['kernel_ms'], d['roofline']['frac'], d['e2e']['value']/1e6)"; done
