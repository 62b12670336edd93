#!/bin/bash
# Parity suite + online small-batch (C5) latency after an engine change.
TAG=${1:-c5}
OUT=gpurun_out/$TAG
mkdir -p $OUT
timeout 900 python -m pytest tests -x -q -m gpu > $OUT/pytest_gpu.log 2>&1; echo "pytest gpu exit $?" >> $OUT/pytest_gpu.log
timeout 600 python tools/bench_configs.py --only c5 --out $OUT/c5.jsonl > $OUT/c5.log 2>&1; echo "c5 exit $?" >> $OUT/c5.log
echo done > $OUT/DONE
