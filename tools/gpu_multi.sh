# usage: bash tools/gpu_multi.sh N "configs"
N=${1:-2}; CFGS=${2:-4}
HYD_TEST_GPUS=$N timeout 900 python -m pytest tests/test_multigpu_gpu.py -q --timeout 800 > gpurun_out/pytest_mgpu$N.log 2>&1; echo "mgpu pytest rc=$?"; tail -5 gpurun_out/pytest_mgpu$N.log
for c in $CFGS; do
timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node $N --master-addr 127.0.0.1 --master-port 29511 bench.py --gpus $N --config $c --steps 10 --warmup 3 > gpurun_out/bench_cfg${c}_n$N.json 2> gpurun_out/bench_cfg${c}_n$N.err; echo "bench cfg$c N=$N rc=$?"
python -c "
import json; d=json.loads(open('gpurun_out/bench_cfg${c}_n$N.json').read().strip().splitlines()[-1]); print(d['value']/1e6, d['ms_per_step'], d['rank_ms'], d.get('a6_check'), d['e2e']['value']/1e6 if d.get('e2e') else None)"
tail -3 gpurun_out/bench_cfg${c}_n$N.err
done
