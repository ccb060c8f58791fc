#!/bin/bash
# Round refresh on the GPU box: every config's bench line (exact headline +
# fast secondary), the reference arm (cfg 2), launch lists for cfg 1 / 2
# (exact and fast) and full ncu captures of the top kernels at cfg 2.
# Runs ON the box: gpurun -- bash tools/gpu_round.sh
mkdir -p gpurun_out/round
rm -f gpurun_out/sweep_status.log
bash tools/sweep_configs.sh
timeout 600 python bench.py --impl reference --steps 3 --warmup 1 > gpurun_out/round/reference_cfg2.log 2>&1
B="python bench.py --steps 1 --warmup 1 --no-cpu-baseline --no-secondary"
for c in 1 2; do for a in exact fast; do
  timeout 600 $B --config $c --arith $a > gpurun_out/round/pre_ncu_${a}_cfg$c.log 2>&1 && \
  ncu --metrics gpu__time_duration.sum --clock-control none -s 300 -c 80 --csv \
      --log-file gpurun_out/round/launches_${a}_cfg$c.csv $B --config $c --arith $a > /dev/null 2>&1
done; done
ncu --set full --clock-control none --import-source on -k regex:"ad_exact_pipe|chain_kernel" -s 6 -c 3 \
    -o gpurun_out/round/exact_cfg2 -f $B > gpurun_out/round/ncu_full_exact.log 2>&1
ncu --set full --clock-control none --import-source on -k regex:ad_fast -s 3 -c 1 \
    -o gpurun_out/round/fast_cfg2 -f $B --arith fast > gpurun_out/round/ncu_full_fast.log 2>&1
echo done
