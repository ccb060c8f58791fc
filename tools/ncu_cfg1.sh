#!/bin/bash
# ncu full captures of the cfg 1 (n = 4096) A.D kernels, exact and fast.
out=gpurun_out/ncu1
mkdir -p $out
B="python bench.py --config 1 --steps 1 --warmup 1 --no-cpu-baseline --no-secondary --no-big --no-oneshot"
export COOPCG_LIB_PATH=${COOPCG_LIB_PATH:-}
$B --arith exact > $out/pre_exact.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:"ad_exact_pipe|chain_kernel" -s 40 -c 4 \
    -o $out/exact_cfg1 -f $B --arith exact > $out/ncu_exact.log 2>&1
$B --arith fast > $out/pre_fast.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:"ad_fast|fast_iter" -s 40 -c 2 \
    -o $out/fast_cfg1 -f $B --arith fast > $out/ncu_fast.log 2>&1
echo done > $out/status.txt
