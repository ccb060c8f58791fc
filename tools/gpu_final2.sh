#!/bin/bash
# Round-2 end refresh, session 4: gpu_final.sh (suite, smoke, default bench,
# reference arm, per-config sweep), then the launch lists of HEAD at cfg 1 / 2
# in both modes and a warm-cache ncu capture of the cfg 1 fast A.D (L2-resident
# share of A: caches NOT flushed between passes).  Runs ON the GPU box.
bash tools/gpu_final.sh
out=gpurun_out/final
unset COOPCG_LIB_PATH
for c in 1 2; do for a in exact fast; do
  B="python bench.py --config $c --arith $a --steps 1 --warmup 1 --no-cpu-baseline --no-secondary --no-big --no-oneshot"
  ncu --metrics gpu__time_duration.sum --clock-control none -s 300 -c 60 --csv \
      --log-file $out/launches_${a}_cfg$c.csv $B > /dev/null 2>&1
  python tools/launches.py $out/launches_${a}_cfg$c.csv > $out/launches_${a}_cfg$c.txt 2>&1
done; done
B="python bench.py --config 1 --arith fast --steps 1 --warmup 1 --no-cpu-baseline --no-secondary --no-big --no-oneshot"
for mb in 0 default; do
  if [ $mb = 0 ]; then export COOPCG_L2_RES_MB=0; else unset COOPCG_L2_RES_MB; fi
  ncu --cache-control none --clock-control none \
      --metrics gpu__time_duration.sum,dram__bytes_read.sum,lts__t_sector_hit_rate.pct,lts__t_sectors_srcunit_tex_op_read.sum \
      -k regex:"ad_fast" -s 300 -c 6 --csv --log-file $out/ncu_warm_fast_cfg1_res_$mb.csv $B > /dev/null 2>&1
done
unset COOPCG_L2_RES_MB
ncu --set full --clock-control none --import-source on -k regex:"ad_fast" -s 60 -c 1 \
    -o $out/ncu_full_fast_cfg1 -f $B > $out/ncu_full_fast_cfg1.log 2>&1
echo done2 >> $out/status.txt
