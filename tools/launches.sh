#!/bin/bash
# per-kernel launch times (ncu, cold-cache, serialised) of one short bench run: diagnostic
mkdir -p gpurun_out/ll
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/ll/l.csv \
  python bench.py --config ${CFG:-4} ${EXTRA:-} --profile --steps 1 --warmup 0 > gpurun_out/ll/l.log 2>&1
python - <<'PY'
import csv, collections
rows = [r for r in csv.reader(open("gpurun_out/ll/l.csv")) if len(r) > 10]
h = rows[0]; ki = h.index("Kernel Name"); vi = h.index("Metric Value")
agg = collections.defaultdict(list)
for r in rows[1:]:
    try: agg[r[ki][:60]].append(float(r[vi].replace(",", "")))
    except ValueError: pass
for k, v in sorted(agg.items(), key=lambda kv: -sum(kv[1])):
    print(f"{sum(v)/1e6:9.3f} ms  x{len(v)}  {k}")
PY
