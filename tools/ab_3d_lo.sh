#!/bin/bash
# tools/ab_3d_lo.sh VARIANT... -- A/B of low-order 3D kernel variants
# (TFEM_LIB builds from tools/variants.sh), ~10M DOFs
run() {
  timeout 300 python bench.py --no-cpu-baseline --no-e2e --no-bitexact --steps 3 --iters 100 "$@" 2>/dev/null \
    | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('$V $*', round(d['value'],2), round(d['cg_roofline']['frac'],3), 'fp64', round(d['roofline']['fp64']['frac'],3))" \
    || echo "$V $* FAILED"
}
for V in main "$@"; do
  if [ $V = main ]; then unset TFEM_LIB; else export TFEM_LIB=build/$V/libtfem_cuda.so; fi
  for p in 1 2 3; do run --dim 3 --order $p; done
  run --dim 3 --order 2 --bp 5
done
