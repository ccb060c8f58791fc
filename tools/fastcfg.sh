timeout 800 python -m pytest tests -q -m gpu > gpurun_out/gpu_tests.log 2>&1; echo rc=$? >> gpurun_out/gpu_tests.log
for c in 2 3 4; do timeout 600 python bench.py --config $c --steps 2 --warmup 1 --arith fast --no-secondary --no-cpu-baseline > gpurun_out/fast_cfg$c.log 2>&1; done
