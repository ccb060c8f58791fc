#!/bin/bash
# Round refresh on the GPU box: every config's bench line, the reference arm
# (cfg 2), launch lists for cfg 0 / 1 / 2 (exact) and one full ncu capture of
# the exact A.D kernel at cfg 2.  Runs ON the box (gpurun -- bash tools/gpu_round.sh).
mkdir -p gpurun_out/round
bash tools/sweep_configs.sh
timeout 600 python bench.py --impl reference --steps 3 --warmup 1 > gpurun_out/round/reference_cfg2.log 2>&1
for c in 0 1 2; do
  timeout 600 python bench.py --config $c --steps 1 --warmup 1 --no-cpu-baseline --no-secondary > gpurun_out/round/pre_ncu_cfg$c.log 2>&1 && \
  ncu --metrics gpu__time_duration.sum --clock-control none -s 300 -c 80 --csv --log-file gpurun_out/round/launches_cfg$c.csv \
      python bench.py --config $c --steps 1 --warmup 1 --no-cpu-baseline --no-secondary > gpurun_out/round/ncu_cfg$c.log 2>&1
done
ncu --set full --clock-control none --import-source on -k regex:ad_exact_pipe -s 3 -c 1 -o gpurun_out/round/ad_pipe_cfg2 -f \
    python bench.py --steps 1 --warmup 1 --no-cpu-baseline --no-secondary > gpurun_out/round/ncu_full.log 2>&1
echo done
