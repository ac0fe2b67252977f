#!/bin/bash
# ncu A/B of the VMAX-16 lane pass: abtest/A.so vs abtest/B.so, one launch each at 512 candidates
# (diagnostic; key metrics printed one line per build)
mkdir -p gpurun_out/ab
for v in ${VARS:-A B}; do
cp abtest/$v.so paper_2412_07894_b200/libhyd.so
timeout 600 ncu --set full --import-source on --clock-control none -k regex:k_pack_lanes -c 1 \
  -o gpurun_out/ab/$v -f python bench.py --config ${CFG:-4} --candidates ${NC:-512} --profile --steps 1 --warmup 0 \
  > gpurun_out/ab/$v.log 2>&1
ncu -i gpurun_out/ab/$v.ncu-rep --page raw --csv --metrics gpu__time_duration.sum,smsp__inst_executed.sum,smsp__issue_active.avg.pct_of_peak_sustained_active,sm__warps_active.avg.pct_of_peak_sustained_active,smsp__thread_inst_executed_per_inst_executed.ratio,launch__registers_per_thread 2>/dev/null | tail -1 | cut -d, -f12- | sed "s/^/$v /"
done
