#!/bin/bash
out=gpurun_out/ncuc2
mkdir -p $out
B="python bench.py --steps 1 --warmup 1 --no-cpu-baseline --no-secondary --no-big --no-oneshot --arith exact --config 2"
$B > $out/pre.log 2>&1 && \
ncu --section WarpStateStats --section SourceCounters --warp-sampling-interval 0 --clock-control none --import-source on \
    -k regex:"chain_kernel" -s 10 -c 2 -o $out/chain -f $B > $out/ncu.log 2>&1
echo done > $out/status.txt
