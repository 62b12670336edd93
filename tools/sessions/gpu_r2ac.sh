#!/bin/bash
# Session AC: the C4 bench line and its reference arm with the final build.
OUT=gpurun_out/r2ac
mkdir -p $OUT
python -c "import __graft_entry__ as g; g.build()" > $OUT/build.log 2>&1
timeout 1500 python bench.py --config c4 > $OUT/bench_c4.json 2> $OUT/bench_c4.err; echo "c4 exit $?" >> $OUT/bench_c4.err
timeout 600 python bench.py --config c4 --impl reference > $OUT/bench_c4_ref.json 2> $OUT/bench_c4_ref.err; echo "c4 ref exit $?" >> $OUT/bench_c4_ref.err
echo done > $OUT/DONE
