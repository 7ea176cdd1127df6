#!/bin/bash
# tools/ab_w15p4.sh -- A/B of 15 computing warps at 2D p=4 BP5 (q=5), ~10M DOFs
run() {
  timeout 300 python bench.py --no-cpu-baseline --no-e2e --no-bitexact --steps 3 --iters 100 "$@" 2>/dev/null \
    | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('$V $*', round(d['value'],2), round(d['cg_roofline']['frac'],3))" \
    || echo "$V $* FAILED"
}
for V in main w15p4 main w15p4; do
  if [ $V = main ]; then unset TFEM_LIB; else export TFEM_LIB=build/$V/libtfem_cuda.so; fi
  run --dim 2 --order 4 --bp 5
done
