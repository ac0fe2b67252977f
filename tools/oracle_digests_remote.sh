#!/bin/bash
# Oracle digests of config 5 iteration ranges on the box's host cores (CPU only; the GPU is idle).
# usage: bash tools/oracle_digests_remote.sh "8 10" "10 12" ...
mkdir -p gpurun_out/dig5
nproc
for r in "$@"; do
  timeout 3000 python tools/make_golden_digests.py --configs 5 --iter-range $r --chunk 1 --out gpurun_out/dig5 \
    >> gpurun_out/dig5/log.txt 2>&1
  echo "range $r rc=$?"
done
tail -20 gpurun_out/dig5/log.txt
