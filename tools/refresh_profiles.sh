#!/bin/bash
# tools/refresh_profiles.sh -- on the GPU box: the default bench line, then the
# ncu launch list and full captures behind profiles/ (each ncu command only
# after the same command exited 0 without ncu).
set -e
O=gpurun_out
python bench.py > $O/bench_default.json 2> $O/bench_default.err
CMD="python bench.py --steps 1 --warmup 1 --iters 20 --no-e2e --no-cpu-baseline"
$CMD > $O/cmd.json 2> $O/cmd.err
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $O/launches.csv $CMD > /dev/null 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:apply2d_tma -s 40 -c 1 -o $O/elem_full -f $CMD > /dev/null 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:scatter_kernel -s 40 -c 1 -o $O/scatter_full -f $CMD > /dev/null 2>&1
CMD3="python bench.py --dim 3 --steps 1 --warmup 1 --iters 20 --no-e2e --no-cpu-baseline --no-bitexact"
$CMD3 > $O/cmd3.json 2> $O/cmd3.err
timeout 600 ncu --set full --clock-control none --import-source on -k regex:apply3d_tma -s 40 -c 1 -o $O/elem3d_full -f $CMD3 > /dev/null 2>&1
echo refreshed
