#!/bin/bash
# Does the evict-last k-range of A (COOPCG_L2_RES_MB) really stay in L2 between
# iterations?  DRAM bytes and duration of in-solve fast A.D launches at cfg 1,
# caches NOT flushed between ncu passes.  Runs ON the GPU box.
out=gpurun_out/l2res_ncu
mkdir -p $out
B="python bench.py --config 1 --arith fast --steps 1 --warmup 1 --no-cpu-baseline --no-secondary --no-big --no-oneshot"
for mb in ${MBS:-0 64 96}; do
  COOPCG_L2_RES_MB=$mb ncu --cache-control none --clock-control none \
      --metrics gpu__time_duration.sum,dram__bytes_read.sum,lts__t_sector_hit_rate.pct,lts__t_sectors_srcunit_tex_op_read.sum \
      -k regex:"ad_fast" -s 300 -c 6 --csv --log-file $out/res_${mb}.csv $B > $out/res_${mb}.log 2>&1
done
echo done > $out/status.txt
