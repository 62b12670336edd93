#!/bin/bash
# compute-sanitizer (memcheck, racecheck, synccheck, initcheck) over every kernel.
OUT=gpurun_out/${1:-san}
mkdir -p $OUT
python -c "import __graft_entry__ as g; g.build()" > $OUT/build.log 2>&1
timeout 300 python tools/sanitize_driver.py > $OUT/plain.log 2>&1; echo "exit $?" >> $OUT/plain.log
for tool in memcheck racecheck synccheck initcheck; do
  # racecheck instruments every shared-memory access: the uniform kernels
  # (thousands of documents) and the VW sort run in separate passes
  # (and with blocking launches: racecheck serialises kernels across host
  # threads, and the multi-threaded pipelines stalled under it otherwise)
  only=""; blocking=0; [ $tool = racecheck ] && only=rest && blocking=1
  CUDA_LAUNCH_BLOCKING=$blocking SANITIZE_ONLY=$only timeout 900 compute-sanitizer --tool $tool --error-exitcode 9 --print-limit 20 \
      python tools/sanitize_driver.py > $OUT/$tool.log 2>&1
  echo "exit $?" >> $OUT/$tool.log
done
SANITIZE_ONLY=uniform timeout 900 compute-sanitizer --tool racecheck --error-exitcode 9 --print-limit 20 \
    python tools/sanitize_driver.py > $OUT/racecheck_uniform.log 2>&1
echo "exit $?" >> $OUT/racecheck_uniform.log
# the VW row kernel's shared-memory sort, on the VW parity tests
timeout 900 compute-sanitizer --tool racecheck --error-exitcode 9 python -m pytest tests/test_gpu_vw.py -q -k "matches" \
    > $OUT/racecheck_vw.log 2>&1
echo "exit $?" >> $OUT/racecheck_vw.log
echo done > $OUT/DONE
