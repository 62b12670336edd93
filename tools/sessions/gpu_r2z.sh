#!/bin/bash
# Session Z: where the full-driver racecheck spends its time (progress marks
# on stderr), with a longer limit.
OUT=gpurun_out/r2z
mkdir -p $OUT
python -c "import __graft_entry__ as g; g.build()" > $OUT/build.log 2>&1
SANITIZE_ONLY=rest timeout 2400 compute-sanitizer --tool racecheck --error-exitcode 9 --print-limit 20 \
    python tools/sanitize_driver.py > $OUT/racecheck.log 2>&1
echo "exit $?" >> $OUT/racecheck.log
echo done > $OUT/DONE
