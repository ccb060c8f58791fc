#!/bin/bash
# Launch lists of the fast and exact iterations at cfg 3 / cfg 4 (per-kernel
# times; the A.D dominates, the list shows what the rest costs).
out=gpurun_out/lbig
mkdir -p $out
for c in ${CFGS:-4 3}; do for a in ${ARITHS:-fast}; do
  B="python bench.py --config $c --arith $a --steps 1 --warmup 1 --no-cpu-baseline --no-secondary --no-big --no-oneshot"
  ncu --metrics gpu__time_duration.sum --clock-control none -s ${SKIP:-60} -c ${COUNT:-40} --csv \
      --log-file $out/launches_${a}_cfg$c.csv $B > /dev/null 2>&1
  python tools/launches.py $out/launches_${a}_cfg$c.csv > $out/launches_${a}_cfg$c.txt 2>&1
done; done
