#!/bin/bash
# tools/run1.sh [bench args] -- one short bench line (GDOF/s, operator and
# CG roofline fractions, operator us) for A/B runs on the GPU box.
timeout 600 python bench.py --no-cpu-baseline --no-e2e --no-bitexact --no-extra --steps 3 --iters 100 "$@" 2>/dev/null \
  | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('$*', round(d['value'],2), 'op', round(d['roofline']['frac'],3), 'cg', round(d['cg_roofline']['frac'],3), 'op_us', round(d['roofline']['ms_per_launch']*1e3,1))" \
  || echo "$* FAILED"
