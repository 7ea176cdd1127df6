#!/bin/bash
# tools/abenv.sh ROUNDS 'ENV=..' ... -- on the GPU box: fma bench per env setting
R=$1; shift
for r in $(seq $R); do
  for e in "$@"; do
    env $e timeout 120 python bench.py --no-cpu-baseline --no-e2e --no-bitexact --steps 5 ${BENCH_ARGS} \
      | python -c "import json,sys; d=json.loads(sys.stdin.readlines()[-1]); print('$e', d['config']['numerics'], round(d['value'],3), round(d['ms_per_step'],2), 'op', round(d['roofline']['ms_per_launch'],4))"
  done
done
