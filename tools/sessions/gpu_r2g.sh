#!/bin/bash
# Round-2 session G: N=2 bench path test, C4 pipeline A/B (parser priority,
# sketch grid room), GPU tests.
OUT=gpurun_out/r2g
mkdir -p $OUT
python -c "import __graft_entry__ as g; g.build()" > $OUT/build.log 2>&1
timeout 900 python tools/c4_pipeline_ab.py > $OUT/c4_ab.jsonl 2> $OUT/c4_ab.err
timeout 900 python -m pytest tests -q -m gpu > $OUT/pytest_gpu.log 2>&1; echo "pytest gpu exit $?" >> $OUT/pytest_gpu.log
echo done > $OUT/DONE
