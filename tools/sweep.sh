#!/bin/bash
# tools/sweep.sh -- on the GPU box: the DESIGN.md §5 order sweep (GDOF/s and CG
# roofline fraction per configuration), FMA numerics, ~10M DOFs.
run() {
  timeout 300 python bench.py --no-cpu-baseline --no-e2e --no-bitexact --no-extra --steps 3 --iters 100 "$@" 2>/dev/null \
    | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('$*', round(d['value'],2), 'op', round(d['roofline']['frac'],3), 'cg', round(d['cg_roofline']['frac'],3), 'fp64', round(d['roofline']['fp64']['achieved'],2), round(d['roofline']['fp64']['frac'],3))" \
    || echo "$* FAILED"
}
for p in 1 2 3 4 6 8; do run --dim 2 --order $p; done
for p in 1 2 3 4 6 8; do run --dim 3 --order $p; done
run --dim 2 --order 3 --bp 5; run --dim 2 --order 4 --bp 5
run --dim 3 --order 2 --bp 5; run --dim 3 --order 4 --bp 5
run --dim 3 --order 2 --bp 1 --iters 50
run --dim 2 --order 3 --cells 3334
