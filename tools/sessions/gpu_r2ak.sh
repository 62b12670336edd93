#!/bin/bash
# Session AK: C5 latency, zero-copy against smaller pipelined chunks.
OUT=gpurun_out/r2ak
mkdir -p $OUT
python -c "import __graft_entry__ as g; g.build()" > $OUT/build.log 2>&1
timeout 600 python tools/c5_chunks_ab.py > $OUT/c5_chunks.jsonl 2> $OUT/c5_chunks.err
echo done > $OUT/DONE
