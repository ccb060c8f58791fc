#!/bin/bash
# ncu of the exact chain kernels at cfg 2 (and cfg 1) for a library variant.
out=gpurun_out/ncuc
mkdir -p $out
B="python bench.py --steps 1 --warmup 1 --no-cpu-baseline --no-secondary --no-big --no-oneshot --arith exact"
for c in 2 1; do
  $B --config $c > $out/pre_cfg$c.log 2>&1 && \
  ncu --set full --clock-control none --import-source on -k regex:"chain_kernel" -s 10 -c 2 \
      -o $out/chain_cfg$c -f $B --config $c > $out/ncu_cfg$c.log 2>&1
done
ncu --metrics gpu__time_duration.sum --clock-control none -s 200 -c 60 --csv \
    --log-file $out/launches_exact_cfg2.csv $B --config 2 > /dev/null 2>&1
echo done > $out/status.txt
