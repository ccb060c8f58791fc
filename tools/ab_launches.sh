#!/bin/bash
# Per-kernel launch times (ncu launch list) for library variants: cfg 1 / 2.
out=gpurun_out/abl
mkdir -p $out
for v in ${VARIANTS:-old}; do
  export COOPCG_LIB_PATH=$PWD/paper_1204_0069_b200/_lib/variants/$v/libcoopcg_gpu.so
  for c in ${CFGS:-1 2}; do for a in ${ARITH:-exact}; do
    B="python bench.py --config $c --arith $a --steps 1 --warmup 1 --no-cpu-baseline --no-secondary --no-big --no-oneshot"
    ncu --metrics gpu__time_duration.sum --clock-control none -s 300 -c 60 --csv \
        --log-file $out/${v}_cfg${c}_$a.csv $B > /dev/null 2>&1
    python tools/launches.py $out/${v}_cfg${c}_$a.csv > $out/${v}_cfg${c}_$a.txt 2>&1
  done; done
done
