#!/bin/bash
# tools/refresh_profiles.sh TAG -- on the GPU box: the default bench line,
# the ncu launch list of the headline config, and one `ncu --set full`
# capture per dominant kernel of the headline and the north-star configs
# (each ncu command only after the same command exited 0 without ncu).
T=${1:-r02}
O=gpurun_out
python bench.py > $O/${T}_bench_default.json 2> $O/${T}_bench_default.err
B="python bench.py --steps 1 --warmup 1 --iters 20 --no-e2e --no-cpu-baseline --no-bitexact --no-extra"
full() { # name, kernel regex, bench args
  local name=$1 kern=$2; shift 2
  $B "$@" > $O/${T}_${name}_cmd.json 2>&1 || { echo "$name: command failed"; return; }
  # the reports stay on the box (gpurun copies back <= 64 MiB): raw csv here
  timeout 900 ncu --set full --clock-control none --import-source on -k regex:$kern -s 40 -c 1 \
     -o /tmp/${T}_${name} -f $B "$@" > $O/${T}_${name}_ncu.log 2>&1 || echo "$name: ncu failed"
  ncu -i /tmp/${T}_${name}.ncu-rep --page raw --csv > $O/${T}_${name}_raw.csv 2>/dev/null
}
$B > /dev/null 2>&1 && timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv \
   --log-file $O/${T}_launches.csv $B > /dev/null 2>&1
full elem2d_p3 apply2d_tma
full scatter2d_p3 scatter_kernel
full elem3d_p3 apply3d_tma --dim 3 --order 3
full elem3d_p5 apply3d_tma --dim 3 --order 5
full elem3d_p6_qg apply3d_tma --dim 3 --order 6
full elem3d_p7_qg apply3d_tma --dim 3 --order 7
full elem3d_p8_qg apply3d_tma --dim 3 --order 8
full elem2d_bp5_p4 apply2d_hi --dim 2 --order 4 --bp 5
full elem3d_bp5_p4 apply3d_tma --dim 3 --order 4 --bp 5
du -sh $O; ls -la $O/${T}_*
