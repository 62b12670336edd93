#!/bin/bash
# GPU LibSVM parser: parity tests, the file-path tests, and the loader throughput with and without it.
OUT=gpurun_out/${1:-gp}
mkdir -p $OUT
python -c "import __graft_entry__ as g; g.build()" > $OUT/build.log 2>&1
timeout 900 python -m pytest tests/test_gpu_parse.py tests/test_gpu_parity.py -x -q -m gpu > $OUT/pytest.log 2>&1; echo "exit $?" >> $OUT/pytest.log
timeout 600 python tools/bench_configs.py --only loader --out $OUT/loader_gpu.jsonl > $OUT/loader_gpu.log 2>&1
BBMH_OPT_GPU_PARSE=0 timeout 600 python tools/bench_configs.py --only loader --out $OUT/loader_cpu.jsonl > $OUT/loader_cpu.log 2>&1
echo done > $OUT/DONE
