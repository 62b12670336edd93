#!/bin/bash
# Super-block size sweep of the uniform 2U kernel: throughput (A/B tool) and
# DRAM bytes per launch (ncu) at the C2 shape, k = 500 and 200.
OUT=gpurun_out/${1:-usb}
mkdir -p $OUT
for sb in ${SBS:-2048 3072 4096 6144 8192 16384}; do
  AB_KS=500,200 AB_REPS=4 AB_ARMS="[{\"uniform_2u\":2,\"uniform_sb_docs\":$sb}]" python tools/ab_uniform.py >> $OUT/ab.jsonl 2>&1
  for k in 500 200; do
    BBMH_OPT_UNIFORM_SB_DOCS=$sb BBMH_OPT_UNIFORM_2U=2 ONCE_K=$k ONCE_DOCS=350000 ncu --metrics dram__bytes_read.sum,gpu__time_duration.sum,lts__t_sector_hit_rate.pct \
      --clock-control none -k regex:sketch_uniform -s 1 -c 1 --csv python tools/uniform_once.py 2>/dev/null | grep -E "dram__|gpu__time|lts__" | sed "s/^/sb=$sb k=$k /" >> $OUT/ncu.txt
  done
done
