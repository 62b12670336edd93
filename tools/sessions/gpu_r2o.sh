#!/bin/bash
# Session O: GPU tests, the 2U bench line with the host-budget transfer mix,
# mixed-transfer sweep for reference.
OUT=gpurun_out/r2o
mkdir -p $OUT
python -c "import __graft_entry__ as g; g.build()" > $OUT/build.log 2>&1
timeout 900 python -m pytest tests -q -m gpu > $OUT/pytest_gpu.log 2>&1; echo "pytest gpu exit $?" >> $OUT/pytest_gpu.log
timeout 900 python bench.py --no-cpu --schemes 2u > $OUT/bench.json 2> $OUT/bench.err; echo "bench exit $?" >> $OUT/bench.err
python -c "
from paper_1205_2958_b200 import bbmh; import json
print(json.dumps(bbmh.host_budget(1)))" > $OUT/budget.json 2>&1
echo done > $OUT/DONE
