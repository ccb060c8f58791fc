mkdir -p gpurun_out/it4
python -m pytest tests/test_gpu_fast.py tests/test_gpu_launch_modes.py tests/test_gpu_multi.py tests/test_gpu_mccg.py -q -x -p no:cacheprovider > gpurun_out/it4/tests.log 2>&1; echo rc=$? >> gpurun_out/it4/tests.log
B="python bench.py --steps 3 --warmup 3 --no-cpu-baseline --no-big --no-oneshot --no-secondary --arith fast"
for c in 2 1 0 3; do timeout 300 $B --config $c > gpurun_out/it4/bench_fast_cfg$c.json 2>&1; done
ncu --set full --clock-control none --import-source on -k regex:fast_iter_kernel -s 20 -c 1 -o gpurun_out/it4/fused -f $B > gpurun_out/it4/ncu.log 2>&1
echo done
