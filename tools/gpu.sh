#!/bin/bash
# tools/gpu.sh LOG TIMEOUT 'command'  -- rebuild, then run on the GPU box from the repo root
cd /root/repo || exit 1
make -s -j8 -C paper_1911_09220_b200/csrc 2>&1 | grep -E "error" && exit 1
mkdir -p gpurun_out
timeout $(( $2 + 900 )) /usr/local/graft/bin/gpurun --timeout "$2" -- "$3" > "gpurun_out/$1" 2>&1
tail -n 12 "gpurun_out/$1"
