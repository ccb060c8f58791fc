#!/bin/bash
# fast_iter phase times (COOPCG_PHASE_TIMES build) against the L2-resident share of A, cfg 1.
out=gpurun_out/phase_res
mkdir -p $out
export COOPCG_LIB_PATH=$PWD/paper_1204_0069_b200/_lib/variants/phase/libcoopcg_gpu.so
for mb in 0 48 63 80; do
  export COOPCG_L2_RES_MB=$mb
  echo "== resident $mb MB" >> $out/summary.txt
  timeout 300 python bench.py --config 1 --arith fast --steps 3 --warmup 3 --no-big --no-oneshot \
      --no-cpu-baseline --no-secondary > $out/res_$mb.json 2> $out/res_$mb.err
  grep -h "fast_iter phases\|C-solve:" $out/res_$mb.err | tail -2 >> $out/summary.txt
  python -c "
import json,sys
d=json.loads(open('$out/res_$mb.json').read().strip().splitlines()[-1]); print(round(d['value'],1),'it/s  A.D', round(d['roofline']['ad_ms_per_launch']*1e3,2),'us')" >> $out/summary.txt
done
