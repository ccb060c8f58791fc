#!/bin/bash
# L2 residency A/B (round 2): the streaming probe, then cfg 1 / 2 in both modes
# at several evict-last budgets (COOPCG_L2_RES_MB).  Runs ON the GPU box.
out=gpurun_out/l2res
mkdir -p $out
(cd tools/probe && timeout 300 ./l2res_probe) > $out/probe.txt 2>&1
for c in 1 2; do for a in exact fast; do for mb in ${MBS:-0 48 80 96}; do
  COOPCG_L2_RES_MB=$mb timeout 300 python bench.py --config $c --arith $a --steps ${STEPS:-3} --warmup 3 --no-big --no-oneshot \
      --no-cpu-baseline --no-secondary > $out/cfg${c}_${a}_${mb}.json 2> $out/cfg${c}_${a}_${mb}.err
  python - $out/cfg${c}_${a}_${mb}.json $c $a $mb >> $out/summary.txt <<'PY'
import json, sys
try:
    d = json.loads(open(sys.argv[1]).read().strip().splitlines()[-1])
    r = d["roofline"]
    print(f"cfg{sys.argv[2]} {sys.argv[3]:5s} res {sys.argv[4]:>4s} MB: {d['value']:9.1f} it/s  A.D {r['ad_ms_per_launch']*1e3:8.2f} us  frac {r['frac']:.3f}  clocks {d.get('clocks')}")
except Exception as e:
    print(f"cfg{sys.argv[2]} {sys.argv[3]} {sys.argv[4]}: failed {e}")
PY
done; done; done
