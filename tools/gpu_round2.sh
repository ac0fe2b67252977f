set -x
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv
timeout 900 python -m pytest tests -m gpu -q -k "not digests or cfg1 or cfg2" --timeout 800 > gpurun_out/pytest1.log 2>&1; echo "pytest rc=$?"
tail -30 gpurun_out/pytest1.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke1.log 2>&1; echo "smoke rc=$?"; tail -5 gpurun_out/smoke1.log
timeout 300 python tools/int_peak.py --out gpurun_out/int_peak.json > gpurun_out/int_peak.log 2>&1; echo "intpeak rc=$?"; tail -c 1500 gpurun_out/int_peak.log
timeout 600 python bench.py --steps 10 --warmup 3 > gpurun_out/bench1.json 2> gpurun_out/bench1.err; echo "bench rc=$?"; tail -c 3000 gpurun_out/bench1.json
