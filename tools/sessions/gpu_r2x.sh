#!/bin/bash
# Session X: end-of-round evidence with the final code -- smoke, the default
# bench line (C2) and its reference arm, the C4 bench line and its reference
# arm, and a 4U-bit k = 300 full-size run (the uniform 4U kernel).
OUT=gpurun_out/r2x
mkdir -p $OUT
python -c "import __graft_entry__ as g; g.build()" > $OUT/build.log 2>&1
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > $OUT/smoke.log 2>&1; echo "smoke exit $?" >> $OUT/smoke.log
timeout 900 python bench.py > $OUT/bench.json 2> $OUT/bench.err; echo "bench exit $?" >> $OUT/bench.err
timeout 600 python bench.py --impl reference > $OUT/bench_ref.json 2> $OUT/bench_ref.err; echo "ref exit $?" >> $OUT/bench_ref.err
timeout 1500 python bench.py --config c4 > $OUT/bench_c4.json 2> $OUT/bench_c4.err; echo "c4 exit $?" >> $OUT/bench_c4.err
timeout 600 python bench.py --config c4 --impl reference > $OUT/bench_c4_ref.json 2> $OUT/bench_c4_ref.err; echo "c4 ref exit $?" >> $OUT/bench_c4_ref.err
AB_SCHEME=4u-bit AB_KS=300,500 AB_REPS=3 AB_ARMS='[{"uniform_4u":1}]' timeout 900 python tools/ab_uniform.py > $OUT/u4_fullsize.jsonl 2> $OUT/u4_fullsize.err
echo done > $OUT/DONE
