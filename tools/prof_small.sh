set -x
timeout 300 python bench.py --config 6 --profile --steps 1 --warmup 1 > gpurun_out/plain6.log 2>&1 && \
timeout 900 ncu --set full --import-source on --clock-control none -k regex:"k_assign_small" -c 1 -o gpurun_out/full_cfg6_small -f python bench.py --config 6 --profile --steps 1 --warmup 0 > gpurun_out/ncu6.log 2>&1
echo "rc=$?"; tail -5 gpurun_out/ncu6.log
