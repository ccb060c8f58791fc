#!/bin/bash
# Fast-mode A-in-L2 residency A/B with the per-unit resident range (round 2,
# session 4): cfg 1 fast at several evict-last budgets.  Runs ON the GPU box.
out=gpurun_out/l2res_fast
mkdir -p $out
for c in ${CFGS:-1}; do for mb in ${MBS:-0 32 64 80 96 112}; do
  COOPCG_L2_RES_MB=$mb timeout 300 python bench.py --config $c --arith fast --steps ${STEPS:-3} --warmup 3 --no-big --no-oneshot \
      --no-cpu-baseline --no-secondary > $out/cfg${c}_${mb}.json 2> $out/cfg${c}_${mb}.err
  python - $out/cfg${c}_${mb}.json $c $mb >> $out/summary.txt <<'PY'
import json, sys
try:
    d = json.loads(open(sys.argv[1]).read().strip().splitlines()[-1])
    r = d["roofline"]
    print(f"cfg{sys.argv[2]} fast res {sys.argv[3]:>4s} MB: {d['value']:9.1f} it/s  A.D {r['ad_ms_per_launch']*1e3:8.2f} us  frac {r['frac']:.3f}")
except Exception as e:
    print(f"cfg{sys.argv[2]} {sys.argv[3]}: failed {e}")
PY
done; done
