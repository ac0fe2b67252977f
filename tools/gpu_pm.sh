# pipeline-major member rows for big batches: full GPU suite, then A/B on config 5 (N=1 and a 2-GPU shard)
timeout 1500 python -m pytest tests -m gpu -q -x --timeout 1400 > gpurun_out/pytest_pm.log 2>&1; echo "pytest rc=$?"; tail -3 gpurun_out/pytest_pm.log
VARIANTS="A B" CFG=5 bash tools/abc.sh
VARIANTS="A B" CFG=5 EXTRA="--candidates 8192" bash tools/abc.sh
