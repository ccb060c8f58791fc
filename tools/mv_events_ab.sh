cd /root/repo
for arith in exact fast; do
 for ev in 1 0 8; do
  COOPCG_MV_EVERY=$ev timeout 300 python bench.py --steps 3 --warmup 2 --no-cpu-baseline --no-secondary --arith $arith > gpurun_out/mv_${arith}_$ev.log 2>&1
 done
 COOPCG_NO_PDL=1 timeout 300 python bench.py --steps 3 --warmup 2 --no-cpu-baseline --no-secondary --arith $arith > gpurun_out/mv_${arith}_nopdl.log 2>&1
done
