#!/bin/bash
# tools/launches.sh TAG [bench args] -- on the GPU box: ncu kernel-duration
# list of a short fma bench, summarised (the top kernels by total time).
v=$1; shift
for _ in 1; do
  timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none ${NCU_EXTRA} --csv \
    --log-file gpurun_out/launch_$v.csv python bench.py --steps 1 --warmup 1 --iters 20 \
    --no-cpu-baseline --no-e2e --no-bitexact "$@" > /dev/null 2>&1
  python - "$v" <<'PY'
import csv, sys, collections
v = sys.argv[1]
rows = [r for r in csv.reader(open(f"gpurun_out/launch_{v}.csv")) if len(r) > 10]
h = rows[0]; ki = h.index("Kernel Name"); mi = h.index("Metric Value")
t = collections.defaultdict(list)
for r in rows[1:]:
    t[r[ki].split("(")[0][:60]].append(float(r[mi].replace(",", "")))
for k, x in sorted(t.items(), key=lambda kv: -sum(kv[1]))[:6]:
    x = sorted(x); print(f"{v:8s} {k:60s} n={len(x):4d} median={x[len(x)//2]/1e3:8.1f} us")
PY
done
