#!/bin/bash
# Round-end style verification on the GPU box: the -m gpu suite (timed, with
# per-test durations), smoke(), the default bench line as the driver runs it.
out=gpurun_out/verify
mkdir -p $out
t0=$(date +%s)
timeout 1500 python -m pytest tests -m gpu -x -q --durations=25 > $out/gpu_tests.log 2>&1
echo "gpu_tests rc=$? s=$(( $(date +%s) - t0 ))" >> $out/status.txt
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > $out/smoke.log 2>&1
echo "smoke rc=$?" >> $out/status.txt
t0=$(date +%s)
timeout 900 python bench.py --gpus 1 --steps 20 --warmup 5 > $out/bench.json 2> $out/bench.err
echo "bench rc=$? s=$(( $(date +%s) - t0 ))" >> $out/status.txt
