#!/bin/bash
# Launch list of whole cfg 0 solves (n = 1000, p = 3, 8 iterations): where a short solve's time goes.
out=gpurun_out/cfg0
mkdir -p $out
for a in exact fast; do
  B="python bench.py --config 0 --arith $a --steps 2 --warmup 1 --no-cpu-baseline --no-secondary --no-big --no-oneshot"
  ncu --metrics gpu__time_duration.sum --clock-control none -s 150 -c 150 --csv \
      --log-file $out/launches_$a.csv $B > /dev/null 2>&1
  python tools/launches.py $out/launches_$a.csv > $out/launches_$a.txt 2>&1
done
