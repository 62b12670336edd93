#!/bin/bash
# ncu captures of the small-k split kernel (2U k=1: HBM-bound) and the LibSVM parser kernels.
OUT=gpurun_out/${1:-nx}
mkdir -p $OUT
python -c "import __graft_entry__ as g; g.build()" > $OUT/build.log 2>&1
SCHEME=2u K=1 timeout 600 ncu --set full --clock-control none --import-source on -k regex:sketch_split -s 2 -c 1 \
    -o $OUT/prof_split_2u_k1 python tools/run_one_sketch.py > $OUT/ncu_split.log 2>&1
TRACE_DOCS=4000 timeout 600 ncu --set full --clock-control none -k regex:seg_emit -s 3 -c 1 \
    -o $OUT/prof_seg_emit python tools/trace_loader.py > $OUT/ncu_parse.log 2>&1
echo done > $OUT/DONE
