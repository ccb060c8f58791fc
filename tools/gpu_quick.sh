#!/bin/bash
# Quick check on the GPU box after a fast-mode change: the fast / launch-mode /
# multi-shard parity tests, then one bench line per config in CFGS (fast mode).
out=gpurun_out/quick
mkdir -p $out
timeout 900 python -m pytest tests/test_gpu_fast.py tests/test_gpu_launch_modes.py tests/test_gpu_multi.py tests/test_gpu_p2p.py -x -q > $out/tests.log 2>&1
echo "tests rc=$? $(tail -1 $out/tests.log)" > $out/summary.txt
for c in ${CFGS:-0 1 2}; do for a in ${ARITH:-fast}; do
  timeout 600 python bench.py --config $c --arith $a --steps ${STEPS:-3} --warmup 3 --no-big --no-oneshot \
      --no-cpu-baseline --no-secondary > $out/cfg${c}_$a.json 2> $out/cfg${c}_$a.err
  python - $out/cfg${c}_$a.json $c $a >> $out/summary.txt <<'PY'
import json, sys
try:
    d = json.loads(open(sys.argv[1]).read().strip().splitlines()[-1])
    r = d["roofline"]
    print(f"cfg{sys.argv[2]} {sys.argv[3]:5s}: {d['value']:9.1f} it/s  A.D {r['ad_ms_per_launch']*1e3:9.2f} us  frac {r['frac']:.3f}  clocks {d.get('clocks', {}).get('sm_mhz')} {d.get('clocks', {}).get('reasons')}")
except Exception as e:
    print(f"cfg{sys.argv[2]} {sys.argv[3]}: failed {e}")
PY
done; done
