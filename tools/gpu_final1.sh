# round-2 measurement batch: bench lines per config, gap study, DP line, debug-checked build cases
mkdir -p gpurun_out/final
timeout 300 python -m pytest tests/test_race_gpu.py -q -x --timeout 280 > gpurun_out/final/pytest_race.log 2>&1; echo "race rc=$?"; tail -2 gpurun_out/final/pytest_race.log
HYD_LIB=paper_2412_07894_b200/libhyd_debug.so timeout 900 python tools/sanitize_cases.py > gpurun_out/final/sanitize_debug_build.log 2>&1; echo "debug-build cases rc=$?"; tail -3 gpurun_out/final/sanitize_debug_build.log
timeout 900 python bench.py > gpurun_out/final/bench_cfg4_n1.json 2> gpurun_out/final/bench_cfg4.err; echo "cfg4 rc=$?"
for c in 1 2 3 6 5; do timeout 900 python bench.py --config $c > gpurun_out/final/bench_cfg${c}_n1.json 2> gpurun_out/final/bench_cfg$c.err; echo "cfg$c rc=$?"; done
timeout 600 python bench.py --dp --steps 10 --warmup 3 > gpurun_out/final/bench_dp.json 2> gpurun_out/final/bench_dp.err; echo "dp rc=$?"
timeout 1200 python bench.py --gap --gap-batch 32 --gap-cands 1024 --gap-iters 64 --gap-no-eq1 > gpurun_out/final/bench_gap_b32.json 2> gpurun_out/final/bench_gap_b32.err; echo "gap32 rc=$?"
timeout 1200 python bench.py --gap --gap-batch 48 --gap-cands 256 --gap-iters 16 --gap-no-eq1 > gpurun_out/final/bench_gap_b48.json 2> gpurun_out/final/bench_gap_b48.err; echo "gap48 rc=$?"
for f in gpurun_out/final/bench_*.json; do echo "== $f"; tail -c 600 $f; echo; done
