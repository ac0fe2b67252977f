timeout 300 python bench.py --config 4 --candidates 1024 --profile --steps 1 --warmup 1 > gpurun_out/plain_sh.log 2>&1 && \
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_shard.csv python bench.py --config 4 --candidates 1024 --profile --steps 1 --warmup 1 > gpurun_out/ncu_sh.log 2>&1; echo "launch rc=$?"
python tools/ncu_summary.py --launches gpurun_out/launches_shard.csv -o gpurun_out/launches_shard_summary.json > /dev/null; python -c "
import json; d=json.load(open('gpurun_out/launches_shard_summary.json'))['launch_list']
for k,v in d.items(): print(k[:40], round(v['mean_ms'],3), v['launches'])"
