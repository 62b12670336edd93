#!/bin/bash
# Session V: GPU tests with the uniform 4U-bit kernel (chosen by the
# persistent shape) and the uniform 2U kernel at 16 < k < 32; the k sweep
# with those defaults; racecheck / initcheck over the smaller sanitizer driver.
OUT=gpurun_out/r2v
mkdir -p $OUT
python -c "import __graft_entry__ as g; g.build()" > $OUT/build.log 2>&1
timeout 1200 python -m pytest tests -q -m gpu > $OUT/pytest_gpu.log 2>&1; echo "pytest gpu exit $?" >> $OUT/pytest_gpu.log
timeout 900 python tools/bench_configs.py --only ksweep --out $OUT/ksweep.jsonl > $OUT/ksweep.log 2>&1
for tool in racecheck initcheck memcheck; do
  timeout 1200 compute-sanitizer --tool $tool --error-exitcode 9 --print-limit 20 \
      python tools/sanitize_driver.py > $OUT/san_$tool.log 2>&1
  echo "exit $?" >> $OUT/san_$tool.log
done
echo done > $OUT/DONE
