#!/bin/bash
# Session AM: C5 latency with the 4U saturation figure (default shapes), the
# 4U k sweep (big batches must keep their shapes), and the 4U GPU tests.
OUT=gpurun_out/r2am
mkdir -p $OUT
python -c "import __graft_entry__ as g; g.build()" > $OUT/build.log 2>&1
C5_ARMS='[{"zero_copy":1}]' timeout 600 python tools/c5_chunks_ab.py > $OUT/c5.jsonl 2> $OUT/c5.err
timeout 900 python tools/bench_configs.py --only ksweep --out $OUT/ksweep.jsonl > $OUT/ksweep.log 2>&1
timeout 900 python -m pytest tests -q -m gpu -k "4u or parity or uniform4 or fullsize" > $OUT/pytest.log 2>&1; echo "pytest exit $?" >> $OUT/pytest.log
echo done > $OUT/DONE
