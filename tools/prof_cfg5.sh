timeout 600 python bench.py --config 5 --steps 5 --warmup 2 --no-cpu > gpurun_out/bench_cfg5_n1.json 2> gpurun_out/bench_cfg5.err; echo "bench rc=$?"
python -c "
import json; d=json.load(open('gpurun_out/bench_cfg5_n1.json')); print(d['value']/1e6, d['kernel_ms']); print(d['roofline']['handoff'], d['roofline']['frac'], d['roofline']['executed_evals_per_ci'])"
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_cfg5_r02.csv python bench.py --config 5 --profile --steps 1 --warmup 1 > gpurun_out/ncu5l.log 2>&1; echo "launch rc=$?"
python tools/ncu_summary.py --launches gpurun_out/launches_cfg5_r02.csv -o gpurun_out/launches_cfg5_summary.json > /dev/null; cat gpurun_out/launches_cfg5_summary.json | head -60
