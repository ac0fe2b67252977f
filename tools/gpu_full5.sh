# one ncu --set full capture of one config-5 step (lanes, warp-queue and dispatch kernels)
mkdir -p gpurun_out/final4
timeout 2400 ncu --set full --import-source on --clock-control none -k regex:"k_(pack|dispatch)" -c 10 \
  -o gpurun_out/final4/full_cfg5 -f python bench.py --config 5 --profile --steps 1 --warmup 0 --no-e2e --no-cpu \
  > gpurun_out/final4/ncu_full_cfg5.log 2>&1; echo "ncu rc=$?"
