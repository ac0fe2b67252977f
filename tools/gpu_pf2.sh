# warp-queue member prefetch: config-5 parity on each variant, then A/B/C timing on config 5
for v in B C; do cp abtest/$v.so paper_2412_07894_b200/libhyd.so; timeout 900 python -m pytest tests/test_digests_gpu.py -q -x -m gpu -k "5" > gpurun_out/pytest_pf2_$v.log 2>&1; echo "$v pytest rc=$?"; tail -1 gpurun_out/pytest_pf2_$v.log; done
CFG=5 bash tools/abc.sh
