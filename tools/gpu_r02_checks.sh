#!/bin/bash
# Round-2 path checks + ncu captures (runs on the GPU box).
out=gpurun_out/r02chk
mkdir -p $out
# the torchrun (one process per GPU) path with one rank: NCCL rank context, gloo control plane
timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node 1 --master-addr 127.0.0.1 --master-port 29533 \
    bench.py --rank-path --no-big --steps 2 --warmup 3 --no-cpu-baseline > $out/rank_path.json 2> $out/rank_path.err
echo "rank_path rc=$?" >> $out/status.txt
# --gpus 2 on a one-GPU box must fail clearly
timeout 120 python bench.py --gpus 2 --no-big --steps 1 --warmup 3 > $out/gpus2.out 2>&1
echo "gpus2 rc=$?" >> $out/status.txt
# ncu: launch lists + full captures of the top kernels at cfg 2 and cfg 4
B="python bench.py --steps 1 --warmup 3 --no-cpu-baseline --no-big --no-oneshot --no-secondary"
for a in exact fast; do
  ncu --metrics gpu__time_duration.sum --clock-control none -s 400 -c 120 --csv \
      --log-file $out/launches_${a}_cfg2.csv $B --arith $a > /dev/null 2>&1
  python tools/launches.py $out/launches_${a}_cfg2.csv > $out/launches_${a}_cfg2.txt 2>&1
done
ncu --set full --clock-control none --import-source on -k regex:"ad_exact_pipe|chain_kernel" -s 20 -c 3 \
    -o $out/exact_cfg2 -f $B --arith exact > $out/ncu_exact.log 2>&1
ncu --set full --clock-control none --import-source on -k regex:"ad_fast|fast_iter" -s 20 -c 2 \
    -o $out/fast_cfg2 -f $B --arith fast > $out/ncu_fast.log 2>&1
echo done >> $out/status.txt
