# one ncu --set full capture of one config-4 step (pack / dispatch / sort / select kernels)
mkdir -p gpurun_out/final4
timeout 1800 ncu --set full --import-source on --clock-control none -k regex:"k_(pack|dispatch|sort|select|flag)" -c 12 \
  -o gpurun_out/final4/full_cfg${CFG:-4} -f python bench.py --config ${CFG:-4} --profile --steps 1 --warmup 0 --no-e2e --no-cpu \
  > gpurun_out/final4/ncu_full_cfg${CFG:-4}.log 2>&1; echo "ncu rc=$?"
