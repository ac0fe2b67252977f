# launch list (ncu gpu__time_duration, cold-cache, serialised) of the default bench config
mkdir -p gpurun_out/final4
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/final4/launches_cfg${CFG:-4}.csv \
  python bench.py --config ${CFG:-4} --profile --steps 2 --warmup 1 > gpurun_out/final4/ncu_launch_cfg${CFG:-4}.log 2>&1; echo "ncu rc=$?"
