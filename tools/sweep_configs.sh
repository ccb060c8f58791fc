#!/bin/bash
# Bench every BASELINE config (exact headline + fast secondary), one line each,
# plus the reference arm at cfg 0-2.  Runs on the GPU box:
#   gpurun -- bash tools/sweep_configs.sh [tag]
tag=${1:-sweep}
out=gpurun_out/$tag
mkdir -p $out
for c in 0 1 2 3 4; do
  extra="--no-big"
  if [ $c -ge 3 ]; then extra="$extra --no-cpu-baseline --no-oneshot"; fi
  timeout 900 python bench.py --config $c --steps 3 --warmup 3 $extra > $out/cfg$c.json 2> $out/cfg$c.err
  echo "cfg$c rc=$?" >> $out/status.log
done
for c in 0 1 2; do
  timeout 900 python bench.py --impl reference --config $c --steps 5 --warmup 3 > $out/reference_cfg$c.json 2>&1
done
