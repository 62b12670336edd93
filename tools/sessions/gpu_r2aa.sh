#!/bin/bash
# Session AA: uniform 2U super-blocks of 58 MB (traffic, speed); persistent 4U-bit kernel shapes at k = 500 (C2): J x threads per
# CTA through the shape_j / shape_tpb options (codes compared to the default).
OUT=gpurun_out/r2aa
mkdir -p $OUT
python -c "import __graft_entry__ as g; g.build()" > $OUT/build.log 2>&1
AB_SCHEME=4u-bit AB_DOCS=150000 AB_KS=500 AB_REPS=2 AB_ARMS='[{"uniform_4u":0,"shape_j":4,"shape_tpb":128},{"uniform_4u":0,"shape_j":8,"shape_tpb":64},{"uniform_4u":0,"shape_j":1,"shape_tpb":256},{"uniform_4u":0,"shape_j":2,"shape_tpb":128},{"uniform_4u":0,"shape_j":4,"shape_tpb":64},{"uniform_4u":0,"shape_j":7,"shape_tpb":32}]' timeout 1200 python tools/ab_uniform.py > $OUT/shapes_4u.jsonl 2> $OUT/shapes_4u.err
# the uniform 2U kernel with the 58 MB super-blocks: DRAM bytes of one full C2
# launch, and the bench line
ONCE_UNIFORM=2 ONCE_K=500 ONCE_DOCS=350000 timeout 600 ncu --metrics dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum,lts__t_sector_hit_rate.pct \
  --clock-control none -k regex:sketch_uniform -s 1 -c 1 --csv python tools/uniform_once.py > $OUT/ncu_sb58.csv 2> $OUT/ncu_sb58.err
timeout 900 python bench.py --no-cpu --schemes 2u > $OUT/bench_2u.json 2> $OUT/bench_2u.err
SANITIZE_ONLY=rest timeout 1200 compute-sanitizer --tool racecheck --error-exitcode 9 --print-limit 20 \
    python tools/sanitize_driver.py > $OUT/racecheck_rest.log 2>&1
echo "exit $?" >> $OUT/racecheck_rest.log
echo done > $OUT/DONE
