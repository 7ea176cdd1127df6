#!/bin/bash
# tools/ab.sh ROUNDS VARIANT... -- on the GPU box: fma bench (operator ms and
# GDOF/s) for the in-tree build ("main") and each build/VARIANT, interleaved.
R=$1; shift
for r in $(seq $R); do
  for v in main "$@"; do
    if [ "$v" = main ]; then L=""; else L="build/$v/libtfem_cuda.so"; fi
    TFEM_LIB=$L timeout 120 python bench.py --no-cpu-baseline --no-e2e --no-bitexact --steps 5 ${BENCH_ARGS} \
      | python -c "import json,sys; d=json.loads(sys.stdin.readlines()[-1]); print('$v', d['config']['numerics'], round(d['value'],3), round(d['ms_per_step'],2), 'op', round(d['roofline']['ms_per_launch'],4))"
  done
done
