# final: cfg4/cfg5/cfg6 N=1 lines with the final build + cfg6 fused-kernel ncu capture
mkdir -p gpurun_out/final3
for c in 4 5 6 1 2 3; do timeout 900 python bench.py --config $c > gpurun_out/final3/bench_cfg${c}_n1.json 2> gpurun_out/final3/bench_cfg$c.err; echo "cfg$c rc=$?"; done
timeout 300 python bench.py --config 6 --profile --steps 1 --warmup 1 > gpurun_out/final3/plain6.log 2>&1 && \
timeout 900 ncu --set full --import-source on --clock-control none -k regex:"k_assign_small|k_sort|k_select" -c 3 -o gpurun_out/final3/full_cfg6 -f python bench.py --config 6 --profile --steps 1 --warmup 0 > gpurun_out/final3/ncu6.log 2>&1; echo "ncu6 rc=$?"
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/final3/launches_cfg6.csv python bench.py --config 6 --profile --steps 1 --warmup 1 > gpurun_out/final3/ncu6l.log 2>&1; echo "launch6 rc=$?"
python tools/ncu_summary.py --launches gpurun_out/final3/launches_cfg6.csv --rep gpurun_out/final3/full_cfg6.ncu-rep -o gpurun_out/final3/ncu_cfg6_summary.json --note "cfg6 N=1 (round 2 final build): launch list = ncu --metrics gpu__time_duration.sum --clock-control none; full_capture = ncu --set full --clock-control none, one step, kernels k_assign_small / k_sort / k_select" > /dev/null; echo "sum rc=$?"
