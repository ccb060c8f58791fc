#!/bin/bash
# fast-mode tail tuning sweep (k-split cap, row-pass grid) at cfg 2 and cfg 1
mkdir -p gpurun_out/fsweep
B="python bench.py --steps 3 --warmup 3 --no-cpu-baseline --no-big --no-oneshot --no-secondary --arith fast"
for c in 2 1; do
for kmax in 16 8 4 2 1; do for rg in 0 256; do
  COOPCG_FAST_KMAX=$kmax COOPCG_FAST_RG=$rg timeout 300 $B --config $c > gpurun_out/fsweep/c${c}_k${kmax}_rg${rg}.json 2>&1
  python -c "import json;d=json.loads(open('gpurun_out/fsweep/c${c}_k${kmax}_rg${rg}.json').read().strip().splitlines()[-1]);print('cfg$c kmax=$kmax rg=$rg', round(d['value'],1), 'ad_ms', round(d['roofline']['ad_ms_per_launch'],4))" >> gpurun_out/fsweep/summary.txt 2>&1
done; done; done
