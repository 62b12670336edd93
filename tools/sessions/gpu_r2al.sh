#!/bin/bash
# Session AL: C5 4U-bit latency with thinner persistent shapes (more CTAs per
# document for small batches).
OUT=gpurun_out/r2al
mkdir -p $OUT
python -c "import __graft_entry__ as g; g.build()" > $OUT/build.log 2>&1
C5_SCHEMES=4u-bit C5_ARMS='[{"shape_j":0,"shape_tpb":0},{"shape_j":1,"shape_tpb":256},{"shape_j":1,"shape_tpb":128},{"shape_j":2,"shape_tpb":128},{"shape_j":1,"shape_tpb":64},{"shape_j":2,"shape_tpb":64}]' timeout 900 python tools/c5_chunks_ab.py > $OUT/c5_shapes.jsonl 2> $OUT/c5_shapes.err
echo done > $OUT/DONE
