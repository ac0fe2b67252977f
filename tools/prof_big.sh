timeout 300 python bench.py --config 5 --profile --steps 1 --warmup 1 > gpurun_out/plain5b.log 2>&1 && \
timeout 1500 ncu --set full --import-source on --clock-control none -k regex:"k_pack_big" -c 1 -o gpurun_out/full_cfg5_pbig -f python bench.py --config 5 --profile --steps 1 --warmup 0 > gpurun_out/ncu5pb.log 2>&1; echo "full rc=$?"; tail -2 gpurun_out/ncu5pb.log
