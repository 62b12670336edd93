#!/bin/bash
# compute-sanitizer (memcheck, racecheck, synccheck, initcheck) over every kernel.
OUT=gpurun_out/${1:-san}
mkdir -p $OUT
python -c "import __graft_entry__ as g; g.build()" > $OUT/build.log 2>&1
timeout 300 python tools/sanitize_driver.py > $OUT/plain.log 2>&1; echo "exit $?" >> $OUT/plain.log
for tool in memcheck racecheck synccheck initcheck; do
  timeout 900 compute-sanitizer --tool $tool --error-exitcode 9 --print-limit 20 \
      python tools/sanitize_driver.py > $OUT/$tool.log 2>&1
  echo "exit $?" >> $OUT/$tool.log
done
echo done > $OUT/DONE
