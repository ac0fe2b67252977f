#!/bin/bash
# A/B/C timing of three builds of libhyd.so on one box (abtest/{A,B,C}.so), alternating
for r in 1 2; do
for v in ${VARIANTS:-A B C}; do
cp abtest/$v.so paper_2412_07894_b200/libhyd.so
timeout 240 python bench.py --config ${CFG:-4} --steps 10 --warmup 3 --no-cpu --no-e2e ${EXTRA:-} 2>&1 | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('$v', round(d['value']/1e6,2), {k:round(v,3) for k,v in d['kernel_ms'].items()})"
done
done
