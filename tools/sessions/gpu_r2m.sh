#!/bin/bash
# Session M: e2e mixing sweep (delta_raw_every) at the full C2 shape; bench
# with the new uniform crossover (k = 500 webspam rows take the uniform kernel).
OUT=gpurun_out/r2m
mkdir -p $OUT
E2E_DOCS=350000 E2E_MODES=auto E2E_RAWS=0,6,4,3,2 E2E_PINNED=1 timeout 900 python tools/e2e_probe.py > $OUT/e2e_mix.jsonl 2> $OUT/e2e_mix.err
timeout 900 python bench.py --no-cpu --schemes 2u > $OUT/bench.json 2> $OUT/bench.err; echo "bench exit $?" >> $OUT/bench.err
echo done > $OUT/DONE
