timeout 300 python bench.py --config 5 --profile --steps 1 --warmup 1 > gpurun_out/plain5.log 2>&1 && \
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_cfg5_r02b.csv python bench.py --config 5 --profile --steps 1 --warmup 1 > gpurun_out/ncu5l.log 2>&1; echo "launch rc=$?"
python tools/ncu_summary.py --launches gpurun_out/launches_cfg5_r02b.csv -o gpurun_out/launches_cfg5b_summary.json > /dev/null; python -c "
import json; d=json.load(open('gpurun_out/launches_cfg5b_summary.json'))['launch_list']
for k,v in d.items(): print(k[:40], round(v['mean_ms'],2))"
timeout 1200 ncu --set full --import-source on --clock-control none -k regex:"k_pack_big|k_dispatch" -c 2 -o gpurun_out/full_cfg5_big -f python bench.py --config 5 --profile --steps 1 --warmup 0 > gpurun_out/ncu5f.log 2>&1; echo "full rc=$?"
