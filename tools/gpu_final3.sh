#!/bin/bash
# Last refresh of round 2: the GPU suite, smoke(), the default bench line (all
# configs), the reference arm, and the torchrun rank path with one rank.
out=gpurun_out/final3
mkdir -p $out
t0=$(date +%s)
timeout 1500 python -m pytest tests -m gpu -x -q --durations=15 > $out/gpu_tests.log 2>&1
echo "gpu_tests rc=$? s=$(( $(date +%s) - t0 ))" >> $out/status.txt
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > $out/smoke.log 2>&1
echo "smoke rc=$?" >> $out/status.txt
t0=$(date +%s)
timeout 900 python bench.py --gpus 1 --steps 20 --warmup 5 > $out/bench.json 2> $out/bench.err
echo "bench rc=$? s=$(( $(date +%s) - t0 ))" >> $out/status.txt
timeout 900 python bench.py --impl reference --gpus 1 --steps 20 --warmup 5 > $out/bench_reference.json 2> $out/bench_reference.err
echo "bench_reference rc=$?" >> $out/status.txt
timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node 1 --master-addr 127.0.0.1 --master-port 29533 \
    bench.py --rank-path --no-big --steps 2 --warmup 3 --no-cpu-baseline > $out/rank_path.json 2> $out/rank_path.err
echo "rank_path rc=$?" >> $out/status.txt
timeout 120 python bench.py --gpus 2 --steps 1 --warmup 1 > $out/gpus2_on_one.json 2> $out/gpus2_on_one.err
echo "gpus2_on_one_gpu rc=$? ($(tail -1 $out/gpus2_on_one.err | cut -c1-120))" >> $out/status.txt
echo done >> $out/status.txt
