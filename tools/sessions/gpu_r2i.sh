#!/bin/bash
# Round-2 session I: GPU tests with 4 text lanes by default, C4 bench again.
OUT=gpurun_out/r2i
mkdir -p $OUT
python -c "import __graft_entry__ as g; g.build()" > $OUT/build.log 2>&1
timeout 900 python -m pytest tests -q -m gpu > $OUT/pytest_gpu.log 2>&1; echo "pytest gpu exit $?" >> $OUT/pytest_gpu.log
timeout 1500 python bench.py --config c4 > $OUT/bench_c4.json 2> $OUT/bench_c4.err; echo "bench c4 exit $?" >> $OUT/bench_c4.err
echo done > $OUT/DONE
