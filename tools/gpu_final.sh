#!/bin/bash
# Round-end refresh on the GPU box: the -m gpu suite (timed), smoke(), the
# default bench line with the driver's flags, and the per-config sweep.
out=gpurun_out/final
mkdir -p $out
t0=$(date +%s)
timeout 1500 python -m pytest tests -m gpu -x -q --durations=12 > $out/gpu_tests.log 2>&1
echo "gpu_tests rc=$? s=$(( $(date +%s) - t0 ))" >> $out/status.txt
cp gpurun_out/full_config_parity.json $out/ 2>/dev/null
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > $out/smoke.log 2>&1
echo "smoke rc=$?" >> $out/status.txt
t0=$(date +%s)
timeout 900 python bench.py --gpus 1 --steps 20 --warmup 5 > $out/bench.json 2> $out/bench.err
echo "bench rc=$? s=$(( $(date +%s) - t0 ))" >> $out/status.txt
timeout 900 python bench.py --impl reference --gpus 1 --steps 20 --warmup 5 > $out/bench_reference.json 2> $out/bench_reference.err
echo "bench_reference rc=$?" >> $out/status.txt
bash tools/sweep_configs.sh final/sweep
echo done >> $out/status.txt
