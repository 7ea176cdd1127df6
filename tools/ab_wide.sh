#!/bin/bash
# tools/ab_wide.sh -- A/B of the 2D p>=4 warp cap (main vs build/w11 = -DTFEM_HI_WIDE=11), ~10M DOFs
run() {
  timeout 300 python bench.py --no-cpu-baseline --no-e2e --no-bitexact --steps 3 --iters 100 "$@" 2>/dev/null \
    | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('$V $*', round(d['value'],2), round(d['cg_roofline']['frac'],3))" \
    || echo "$V $* FAILED"
}
for V in main w11 main; do
  if [ $V = main ]; then unset TFEM_LIB; else export TFEM_LIB=build/w11/libtfem_cuda.so; fi
  run --dim 2 --order 5; run --dim 2 --order 7; run --dim 2 --order 8 --bp 5
done
