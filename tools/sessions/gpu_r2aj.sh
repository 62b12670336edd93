#!/bin/bash
# Session AJ: where the C5 small-batch latency goes (2U and 4U-bit, k = 500).
OUT=gpurun_out/r2aj
mkdir -p $OUT
python -c "import __graft_entry__ as g; g.build()" > $OUT/build.log 2>&1
C5_SCHEME=2u timeout 300 python tools/c5_breakdown.py > $OUT/c5_2u.jsonl 2> $OUT/c5_2u.err
C5_SCHEME=4u-bit timeout 300 python tools/c5_breakdown.py > $OUT/c5_4u.jsonl 2> $OUT/c5_4u.err
echo done > $OUT/DONE
