#!/bin/bash
# tools/sweep50.sh -- on the GPU box: BASELINE config C3 (order sweep at ~50M
# DOFs; 2D n = round(7071/p), 3D n = round(368/p)), 50 iterations, FMA.
run() {
  timeout 600 python bench.py --no-cpu-baseline --no-e2e --no-bitexact --no-extra --steps 2 --iters 50 "$@" 2>/dev/null \
    | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('$*', d['config']['dofs_per_rank'], round(d['value'],2), 'op', round(d['roofline']['frac'],3), 'cg', round(d['cg_roofline']['frac'],3), 'fp64', round(d['roofline']['fp64']['frac'],3))" \
    || echo "$* FAILED"
}
for p in 1 2 3 4 5 6 7 8; do run --dim 2 --order $p --cells $(( (7071 + p / 2) / p )); done
for p in 1 2 3 4 5 6 7 8; do run --dim 3 --order $p --cells $(( (368 + p / 2) / p )); done
