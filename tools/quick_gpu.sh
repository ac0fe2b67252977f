#!/bin/bash
# quick GPU check: parity tests + cfg4 bench kernel times
timeout 400 python -m pytest tests -m gpu -q -x --timeout 300 2>&1 | tail -1 | sed "s/^/TESTS: /"
for c in ${CFGS:-4}; do
timeout 240 python bench.py --config $c --steps 3 --warmup 3 --no-cpu --no-e2e 2>&1 | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(d['config']['workload'], round(d['value']/1e6,2), {k:round(v,3) for k,v in d['kernel_ms'].items()})"
done
