timeout 900 python -m pytest tests/test_parity_gpu.py tests/test_digests_gpu.py tests/test_pipe_index_gpu.py -k "not digests or cfg2 or cfg3" -q -x --timeout 800 > gpurun_out/pytest_c5.log 2>&1; echo "pytest rc=$?"
tail -5 gpurun_out/pytest_c5.log
CFG=4 bash tools/ab.sh
for v in A B; do cp abtest/$v.so paper_2412_07894_b200/libhyd.so; timeout 600 python bench.py --config 5 --steps 4 --warmup 2 --no-cpu --no-e2e > gpurun_out/bench_c5_$v.json 2>&1; python -c "
import json; d=json.loads(open('gpurun_out/bench_c5_$v.json').read().strip().splitlines()[-1]); print('$v', d['value']/1e6, {k: round(x,2) for k,x in d['kernel_ms'].items()}, d['roofline']['handoff'])"; done
