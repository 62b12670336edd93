#!/bin/bash
# Kernel-variant sweep: int-pipe microbenchmarks + sketch launch-knob grid (TUNE_GRID json file).
TAG=${1:-t}
GRID=${2:-}
OUT=gpurun_out/$TAG
mkdir -p $OUT
python -c "import __graft_entry__ as g; g.build()" > $OUT/build.log 2>&1
timeout 200 python tools/intpeak.py $OUT/int_peaks.json > $OUT/intpeak.log 2>&1
if [ -n "$GRID" ]; then
  TUNE_GRID="$(cat $GRID)" TUNE_DOCS=${TUNE_DOCS:-200000} TUNE_SCHEMES=${TUNE_SCHEMES:-2u} timeout 600 python tools/tune.py > $OUT/tune.jsonl 2> $OUT/tune.err
fi
echo done > $OUT/DONE
