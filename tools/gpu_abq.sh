# quick A/B (abtest/A.so vs B.so) on CFG with a parity gate on B
cp abtest/B.so paper_2412_07894_b200/libhyd.so
timeout 900 python -m pytest tests/test_parity_gpu.py tests/test_small_gpu.py tests/test_digests_gpu.py -k "not digests or cfg2 or cfg3 or cfg6" -q -x --timeout 800 > gpurun_out/pytest_abq.log 2>&1; echo "pytest rc=$?"
tail -3 gpurun_out/pytest_abq.log
for c in ${CFGS:-4}; do CFG=$c bash tools/ab.sh; done
