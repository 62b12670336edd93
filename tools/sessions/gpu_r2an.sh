#!/bin/bash
# Session AN: uniform 2U super-block size around the L2 cliff at C2 (k = 500):
# speed (A/B, forced sizes) and DRAM bytes of one full launch per size.
OUT=gpurun_out/r2an
mkdir -p $OUT
python -c "import __graft_entry__ as g; g.build()" > $OUT/build.log 2>&1
AB_KS=500 AB_REPS=5 AB_ARMS='[{"uniform_2u":2,"uniform_sb_docs":3600},{"uniform_2u":2,"uniform_sb_docs":4080},{"uniform_2u":2,"uniform_sb_docs":4300},{"uniform_2u":2,"uniform_sb_docs":4500},{"uniform_2u":2,"uniform_sb_docs":0}]' timeout 900 python tools/ab_uniform.py > $OUT/sb.jsonl 2> $OUT/sb.err
for sb in 3600 4080 4300 4500; do
  BBMH_OPT_UNIFORM_SB_DOCS=$sb ONCE_UNIFORM=2 ONCE_K=500 ONCE_DOCS=350000 timeout 600 ncu --metrics dram__bytes_read.sum,gpu__time_duration.sum \
    --clock-control none -k regex:sketch_uniform -s 1 -c 1 --csv python tools/uniform_once.py 2>/dev/null | grep -E "dram__|gpu__time" | sed "s/^/sb=$sb /" >> $OUT/ncu.txt
done
echo done > $OUT/DONE
