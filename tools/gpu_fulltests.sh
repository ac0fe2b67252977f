# the whole GPU suite (as the driver runs it) + smoke
timeout 2400 python -m pytest tests -m gpu -q --timeout 1200 > gpurun_out/pytest_gpu_full.log 2>&1; echo "pytest rc=$?"; tail -15 gpurun_out/pytest_gpu_full.log
timeout 600 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke_full.log 2>&1; echo "smoke rc=$?"; tail -3 gpurun_out/smoke_full.log
