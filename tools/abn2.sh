#!/bin/bash
# A/B of library builds (abtest/{A,B}.so) at N GPUs (torchrun), alternating
N=${N:-2}
for r in 1 2; do
for v in ${VARIANTS:-A B}; do
cp abtest/$v.so paper_2412_07894_b200/libhyd.so
timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node $N --master-addr 127.0.0.1 --master-port 29517 bench.py --gpus $N --config ${CFG:-5} --steps 6 --warmup 3 --no-cpu --no-e2e 2>/dev/null | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('$v', round(d['value']/1e6,3), {k:round(v,2) for k,v in d['kernel_ms'].items()})"
done
done
