#!/bin/bash
# GPU tests + exact and fast bench lines + launch lists for both (one gpurun call).
# usage: tools/gpu_cycle2.sh TAG
TAG=${1:-cycle2}
cd /root/repo
timeout 2400 /usr/local/graft/bin/gpurun --timeout 1500 -- "timeout 900 python -m pytest tests -x -q -m gpu > gpurun_out/gpu_tests.log 2>&1; echo \"pytest rc=\$?\" >> gpurun_out/gpu_tests.log; for a in exact fast; do timeout 600 python bench.py --steps 3 --warmup 2 --no-cpu-baseline --no-secondary --arith \$a > gpurun_out/bench_\$a.log 2>&1 && ncu --metrics gpu__time_duration.sum --clock-control none -s 300 -c 60 --csv --log-file gpurun_out/launches_\$a.csv python bench.py --steps 1 --warmup 1 --no-cpu-baseline --no-secondary --arith \$a > gpurun_out/ncu_\$a.log 2>&1; done; echo rc=\$?" > gpurun_out/$TAG.log 2>&1
tail -1 gpurun_out/$TAG.log
tail -2 gpurun_out/gpu_tests.log
for a in exact fast; do
python3 -c "import json,sys; d=json.loads(open('gpurun_out/bench_$a.log').readlines()[-1]); print('$a value', round(d['value'],1), 'e2e', round(d['e2e']['value'],1), 'ad_ms', round(d['roofline']['ad_ms_per_launch'],4), 'frac', round(d['roofline']['frac'],3), 'ms/step', round(d['ms_per_step'],2))" || tail -5 gpurun_out/bench_$a.log
python3 tools/launches.py gpurun_out/launches_$a.csv | head -9
done
