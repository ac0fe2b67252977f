# round-2 final build: N=1 bench lines of every config (with the oracle's cpu_baseline)
mkdir -p gpurun_out/final4
for c in 4 5 6 1 2 3; do timeout 900 python bench.py --config $c > gpurun_out/final4/bench_cfg${c}_n1.json 2> gpurun_out/final4/bench_cfg$c.err; echo "cfg$c rc=$?"; done
