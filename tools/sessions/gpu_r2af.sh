#!/bin/bash
# Session AF: the default bench line after the host-mix tie rule; the delta /
# uniform GPU tests.
OUT=gpurun_out/r2af
mkdir -p $OUT
python -c "import __graft_entry__ as g; g.build()" > $OUT/build.log 2>&1
timeout 900 python -m pytest tests/test_gpu_delta.py tests/test_gpu_uniform.py tests/test_gpu_uniform4.py -q > $OUT/pytest.log 2>&1; echo "pytest exit $?" >> $OUT/pytest.log
timeout 900 python bench.py > $OUT/bench.json 2> $OUT/bench.err; echo "bench exit $?" >> $OUT/bench.err
echo done > $OUT/DONE
