mkdir -p gpurun_out/it3
python -m pytest tests/test_gpu_fast.py tests/test_gpu_launch_modes.py tests/test_gpu_multi.py tests/test_gpu_mccg.py -q -x -p no:cacheprovider > gpurun_out/it3/tests.log 2>&1; echo rc=$? >> gpurun_out/it3/tests.log
B="python bench.py --steps 3 --warmup 3 --no-cpu-baseline --no-big --no-oneshot --no-secondary --arith fast"
timeout 300 $B > gpurun_out/it3/bench_fast_cfg2.json 2>&1
timeout 300 $B --config 1 > gpurun_out/it3/bench_fast_cfg1.json 2>&1
COOPCG_NO_FUSE=1 timeout 300 $B > gpurun_out/it3/bench_fast_cfg2_nofuse.json 2>&1
COOPCG_NO_FUSE=1 timeout 300 $B --config 1 > gpurun_out/it3/bench_fast_cfg1_nofuse.json 2>&1
ncu --set full --clock-control none --import-source on -k regex:fast_iter_kernel -s 20 -c 1 -o gpurun_out/it3/fused -f $B > gpurun_out/it3/ncu.log 2>&1
echo done
