#!/bin/bash
# Round-2 session F: compute-sanitizer over every kernel (incl. tickets, ranges,
# replay), the k sweep with the small-k tickets, C5 online latency.
OUT=gpurun_out/r2f
mkdir -p $OUT
bash tools/gpu_sanitize.sh r2f/san
timeout 900 python tools/bench_configs.py --only ksweep --out $OUT/ksweep.jsonl > $OUT/ksweep.log 2>&1
timeout 900 python tools/bench_configs.py --only c5 --out $OUT/c5.jsonl > $OUT/c5.log 2>&1
echo done > $OUT/DONE
