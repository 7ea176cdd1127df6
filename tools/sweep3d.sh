#!/bin/bash
# tools/sweep3d.sh -- on the GPU box: 3D BP3 / BP5 throughput at ~10M DOFs
# (GDOF/s, operator and CG roofline fractions, operator us).
run() {
  timeout 600 python bench.py --no-cpu-baseline --no-e2e --no-bitexact --no-extra --steps 3 --iters 100 "$@" 2>/dev/null \
    | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('$*', round(d['value'],2), 'op', round(d['roofline']['frac'],3), 'cg', round(d['cg_roofline']['frac'],3), 'op_us', round(d['roofline']['ms_per_launch']*1e3,1))" \
    || echo "$* FAILED"
}
# tools/sweep3d.sh [P...] -- only the listed BP3 orders
if [ $# -gt 0 ]; then
  for p in "$@"; do run --dim 3 --order $p; done
  exit 0
fi
for p in 2 3 4 5 6 7 8; do run --dim 3 --order $p; done
for p in 2 4 5 6 7 8; do run --dim 3 --order $p --bp 5; done
