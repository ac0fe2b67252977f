# final round-2 measurement: N=1 bench lines, cfg4 launch list + ncu --set full, summaries
set -x
mkdir -p gpurun_out/final2
timeout 900 python bench.py > gpurun_out/final2/bench_cfg4_n1.json 2> gpurun_out/final2/bench_cfg4.err; echo "cfg4 rc=$?"
for c in 1 2 3 5 6; do timeout 900 python bench.py --config $c > gpurun_out/final2/bench_cfg${c}_n1.json 2> gpurun_out/final2/bench_cfg$c.err; echo "cfg$c rc=$?"; done
timeout 900 python bench.py --impl reference --steps 20 --warmup 5 > gpurun_out/final2/bench_reference.json 2> gpurun_out/final2/bench_ref.err; echo "ref rc=$?"
timeout 600 python bench.py --config 4 --profile --steps 2 --warmup 1 > gpurun_out/final2/plain4.log 2>&1 && \
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/final2/launches_cfg4.csv python bench.py --config 4 --profile --steps 2 --warmup 1 > gpurun_out/final2/ncu_launch.log 2>&1; echo "launch rc=$?"
timeout 1500 ncu --set full --import-source on --clock-control none -k regex:"k_(pack|dispatch|sort|select|flag)" -c 10 -o gpurun_out/final2/full_cfg4 -f python bench.py --config 4 --profile --steps 1 --warmup 0 > gpurun_out/final2/ncu_full.log 2>&1; echo "full rc=$?"
python tools/ncu_summary.py --launches gpurun_out/final2/launches_cfg4.csv --rep gpurun_out/final2/full_cfg4.ncu-rep -o gpurun_out/final2/ncu_cfg4_summary.json --note "cfg4 N=1 (round 2 final build): launch list = ncu --metrics gpu__time_duration.sum --clock-control none (cold-cache, serialised), bench.py --profile --steps 2 --warmup 1; full_capture = ncu --set full --clock-control none, one step (bench.py --profile --steps 1 --warmup 0), kernels k_(pack|dispatch|sort|select|flag)" > /dev/null; echo "summary rc=$?"
