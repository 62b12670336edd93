#!/bin/bash
# Round-2 session B: GPU tests (range-sharded loader, options), residency probe,
# the default bench (C2 + perm leg) and the C4 bench.
OUT=gpurun_out/r2b
mkdir -p $OUT
python -c "import __graft_entry__ as g; g.build()" > $OUT/build.log 2>&1
timeout 900 python -m pytest tests -q -m gpu > $OUT/pytest_gpu.log 2>&1; echo "pytest gpu exit $?" >> $OUT/pytest_gpu.log
nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++20 -I paper_1205_2958_b200/csrc tools/residency_probe.cu \
  paper_1205_2958_b200/csrc/perm.cu paper_1205_2958_b200/csrc/options.cpp -o /tmp/residency_probe > $OUT/probe_build.log 2>&1
timeout 120 /tmp/residency_probe 50000 > $OUT/residency.jsonl 2>&1
timeout 120 /tmp/residency_probe 350000 >> $OUT/residency.jsonl 2>&1
timeout 900 python bench.py > $OUT/bench.json 2> $OUT/bench.err; echo "bench exit $?" >> $OUT/bench.err
timeout 1200 python bench.py --config c4 > $OUT/bench_c4.json 2> $OUT/bench_c4.err; echo "bench c4 exit $?" >> $OUT/bench_c4.err
echo done > $OUT/DONE
