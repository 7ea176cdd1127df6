#!/bin/bash
# tools/ncu_one.sh NAME KERNEL_REGEX [bench args] -- on the GPU box: one
# `ncu --set full` capture of KERNEL_REGEX in a short bench run (after the
# same command exits 0 without ncu), exported as raw csv into gpurun_out/.
name=$1 kern=$2; shift 2
O=gpurun_out
B="python bench.py --steps 1 --warmup 1 --iters 20 --no-e2e --no-cpu-baseline --no-bitexact --no-extra"
$B "$@" > $O/${name}_cmd.json 2>&1 || { echo "$name: command failed"; exit 1; }
timeout 900 ncu --set full --clock-control none --import-source on -k regex:$kern -s 40 -c 1 \
   -o /tmp/${name} -f $B "$@" > $O/${name}_ncu.log 2>&1 || echo "$name: ncu failed"
ncu -i /tmp/${name}.ncu-rep --page raw --csv > $O/${name}_raw.csv 2>/dev/null
ncu -i /tmp/${name}.ncu-rep --page source --csv > $O/${name}_source.csv 2>/dev/null
