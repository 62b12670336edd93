#!/bin/bash
# Round-2 session H: the VW row kernel (tests, sanitizer, timing vs the reference).
OUT=gpurun_out/r2h
mkdir -p $OUT
python -c "import __graft_entry__ as g; g.build()" > $OUT/build.log 2>&1
timeout 600 python -m pytest tests/test_gpu_vw.py -q > $OUT/pytest_vw.log 2>&1; echo "exit $?" >> $OUT/pytest_vw.log
timeout 900 compute-sanitizer --tool memcheck --error-exitcode 9 python -m pytest tests/test_gpu_vw.py -q -k long > $OUT/memcheck_vw.log 2>&1; echo "exit $?" >> $OUT/memcheck_vw.log
timeout 900 compute-sanitizer --tool racecheck --error-exitcode 9 python -m pytest tests/test_gpu_vw.py -q -k "matches" > $OUT/racecheck_vw.log 2>&1; echo "exit $?" >> $OUT/racecheck_vw.log
timeout 900 python tools/bench_configs.py --only next --out $OUT/next.jsonl > $OUT/next.log 2>&1
timeout 900 python -m pytest tests -q -m gpu > $OUT/pytest_gpu.log 2>&1; echo "pytest gpu exit $?" >> $OUT/pytest_gpu.log
echo done > $OUT/DONE
