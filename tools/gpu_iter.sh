#!/bin/bash
# One build -> measure cycle on the GPU box (runs ON the box:
#   gpurun -- bash tools/gpu_iter.sh [tag] [pytest selection...]).
# Tests first; then the cfg 2 bench line (both modes, no cfg4 object) and
# ncu launch lists (per-kernel durations) of one solve in each mode.
tag=${1:-iter}; shift
sel=${@:-tests -m gpu}
out=gpurun_out/$tag
mkdir -p $out
python -m pytest $sel -q -x -p no:cacheprovider > $out/tests.log 2>&1; echo "rc=$?" >> $out/tests.log
B="python bench.py --steps 3 --warmup 3 --no-cpu-baseline --no-big --no-oneshot"
timeout 600 $B > $out/bench_cfg2.json 2> $out/bench_cfg2.err
for a in exact fast; do
  ncu --metrics gpu__time_duration.sum --clock-control none -s 400 -c 120 --csv \
      --log-file $out/launches_${a}_cfg2.csv $B --no-secondary --arith $a > /dev/null 2>&1
  python tools/launches.py $out/launches_${a}_cfg2.csv > $out/launches_${a}_cfg2.txt 2>&1
done
echo done
