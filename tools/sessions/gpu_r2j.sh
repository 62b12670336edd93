#!/bin/bash
# Round-2 session J: smoke, full GPU tests, compute-sanitizer over every kernel
# (4 text lanes by default, VW row kernel), the default bench.
OUT=gpurun_out/r2j
mkdir -p $OUT
python -c "import __graft_entry__ as g; g.build()" > $OUT/build.log 2>&1
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > $OUT/smoke.log 2>&1; echo "smoke exit $?" >> $OUT/smoke.log
timeout 900 python -m pytest tests -q -m gpu > $OUT/pytest_gpu.log 2>&1; echo "pytest gpu exit $?" >> $OUT/pytest_gpu.log
bash tools/gpu_sanitize.sh r2j/san
timeout 900 python bench.py > $OUT/bench.json 2> $OUT/bench.err; echo "bench exit $?" >> $OUT/bench.err
timeout 600 python bench.py --impl reference > $OUT/bench_ref.json 2> $OUT/bench_ref.err; echo "ref exit $?" >> $OUT/bench_ref.err
echo done > $OUT/DONE
