#!/bin/bash
# A/B of library build variants (tools/variants.sh) on the GPU box:
#   VARIANTS="old la4" CFGS="1 2 3" ARITH=exact bash tools/ab_variants.sh
out=gpurun_out/ab
mkdir -p $out
for v in ${VARIANTS:-old}; do
  lib=$PWD/paper_1204_0069_b200/_lib/variants/$v/libcoopcg_gpu.so
  if [ -n "$PARITY" ]; then
    COOPCG_LIB_PATH=$lib timeout 600 python -m pytest tests/test_gpu_parity.py tests/test_gpu_multi.py tests/test_gpu_fast.py tests/test_gpu_launch_modes.py tests/test_gpu_mccg.py -x -q > $out/parity_$v.log 2>&1
    echo "$v parity rc=$? $(tail -1 $out/parity_$v.log)" >> $out/summary.txt
  fi
  for c in ${CFGS:-1 2}; do for a in ${ARITH:-exact}; do
    COOPCG_LIB_PATH=$lib timeout 600 python bench.py --config $c --arith $a --steps ${STEPS:-3} --warmup 3 --no-big --no-oneshot \
        --no-cpu-baseline --no-secondary > $out/${v}_cfg${c}_$a.json 2> $out/${v}_cfg${c}_$a.err
    python - $out/${v}_cfg${c}_$a.json $v $c $a >> $out/summary.txt <<'PY'
import json, sys
try:
    d = json.loads(open(sys.argv[1]).read().strip().splitlines()[-1])
    r = d["roofline"]
    print(f"{sys.argv[2]:10s} cfg{sys.argv[3]} {sys.argv[4]:5s}: {d['value']:9.1f} it/s  A.D {r['ad_ms_per_launch']*1e3:9.2f} us  frac {r['frac']:.3f}  clocks {d.get('clocks', {}).get('sm_mhz')} {d.get('clocks', {}).get('reasons')}")
except Exception as e:
    print(f"{sys.argv[2]} cfg{sys.argv[3]} {sys.argv[4]}: failed {e}")
PY
  done; done
done
