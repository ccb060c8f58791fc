#!/bin/bash
# Alternating A/B of the fast-mode L2-resident share of A at cfg 1 (run-to-run noise check).
out=gpurun_out/l2res_ab2
mkdir -p $out
for rep in 1 2 3 4; do for mb in 0 default 48; do
  if [ $mb = default ]; then unset COOPCG_L2_RES_MB; else export COOPCG_L2_RES_MB=$mb; fi
  timeout 300 python bench.py --config 1 --arith fast --steps 5 --warmup 3 --no-big --no-oneshot \
      --no-cpu-baseline --no-secondary > $out/r${rep}_${mb}.json 2> $out/r${rep}_${mb}.err
  python - $out/r${rep}_${mb}.json $rep $mb >> $out/summary.txt <<'PY'
import json, sys
try:
    d = json.loads(open(sys.argv[1]).read().strip().splitlines()[-1])
    r = d["roofline"]
    print(f"rep {sys.argv[2]} res {sys.argv[3]:>7s}: {d['value']:9.1f} it/s  e2e {d['e2e']['value']:9.1f}  A.D {r['ad_ms_per_launch']*1e3:8.2f} us")
except Exception as e:
    print(f"rep {sys.argv[2]} {sys.argv[3]}: failed {e}")
PY
done; done
