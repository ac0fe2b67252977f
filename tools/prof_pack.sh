timeout 300 python bench.py --config 4 --profile --steps 1 --warmup 1 > gpurun_out/plain4.log 2>&1 && \
timeout 1200 ncu --set full --import-source on --clock-control none -k regex:"k_pack_lanes|k_dispatch|k_pack_big" -c 4 -o gpurun_out/full_cfg4_r02 -f python bench.py --config 4 --profile --steps 1 --warmup 0 > gpurun_out/ncu4.log 2>&1
echo "rc=$?"; tail -3 gpurun_out/ncu4.log
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_cfg4_r02.csv python bench.py --config 4 --profile --steps 2 --warmup 1 > gpurun_out/ncu4l.log 2>&1; echo "launch rc=$?"
