for n in 512 1024; do
timeout 300 python bench.py --config 4 --candidates $n --steps 5 --warmup 2 --no-cpu --no-e2e > gpurun_out/sh$n.json 2>&1
python -c "
import json; d=json.loads(open('gpurun_out/sh$n.json').read().strip().splitlines()[-1]); print($n, round(d['value']/1e6,2), round(d['ms_per_step'],3), {k: round(x,3) for k,x in d['kernel_ms'].items()})"
CFG=4 EXTRA="--candidates $n" bash tools/launches.sh | head -12
done
