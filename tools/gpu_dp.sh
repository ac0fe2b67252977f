# DP pruning: bit-exact DP parity (incl. the paper's grid), then A/B of bench.py --dp
timeout 1200 python -m pytest tests/test_dp_gpu.py -q -x -m gpu --timeout 1100 > gpurun_out/pytest_dp.log 2>&1; echo "pytest rc=$?"; tail -2 gpurun_out/pytest_dp.log
for r in 1 2; do for v in A B; do cp abtest/$v.so paper_2412_07894_b200/libhyd.so; timeout 600 python bench.py --dp --steps 10 --warmup 3 2>/dev/null | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('$v', d.get('ms_per_step'), d.get('value'))"; done; done
cp abtest/B.so paper_2412_07894_b200/libhyd.so
