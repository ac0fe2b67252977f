#!/bin/bash
# Round measurement: default bench line (N=1, cfg4), ncu launch list, one `ncu --set full` step,
# summary JSON.  Outputs under gpurun_out/prof/ (copy what is judged into profiles/rNN/).
set -e
CFG=${CFG:-4}
O=gpurun_out/prof
mkdir -p $O
timeout 600 python bench.py --config $CFG > $O/bench_cfg${CFG}_n1.json 2> $O/bench_cfg${CFG}.err
tail -1 $O/bench_cfg${CFG}_n1.json | cut -c1-300
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $O/launches_cfg${CFG}.csv \
  python bench.py --config $CFG --profile --steps 2 --warmup 1 > $O/ncu_launch.log 2>&1
timeout 1200 ncu --set full --import-source on --clock-control none -k regex:"k_(pack|dispatch|sort|select)" -c 8 \
  -o $O/full_cfg${CFG} -f python bench.py --config $CFG --profile --steps 1 --warmup 0 > $O/ncu_full.log 2>&1
python tools/ncu_summary.py --launches $O/launches_cfg${CFG}.csv --rep $O/full_cfg${CFG}.ncu-rep \
  -o $O/ncu_cfg${CFG}_summary.json --note "cfg${CFG} N=1: launch list = ncu --metrics gpu__time_duration.sum --clock-control none (cold-cache, serialised), bench.py --profile --steps 2 --warmup 1; full_capture = ncu --set full --clock-control none, one step (bench.py --profile --steps 1 --warmup 0), kernels k_(pack|dispatch|sort|select)" > /dev/null
echo done
