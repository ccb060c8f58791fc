#!/bin/bash
# Bench every BASELINE config (exact headline + fast secondary).  Runs on the GPU box.
for c in 0 1 2 3 4; do
  extra=""
  if [ $c -ge 3 ]; then extra="--no-cpu-baseline"; fi
  timeout 900 python bench.py --config $c --steps 3 --warmup 2 $extra > gpurun_out/sweep_cfg$c.log 2>&1
  echo "cfg$c rc=$?" >> gpurun_out/sweep_status.log
done
