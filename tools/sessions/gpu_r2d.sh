#!/bin/bash
# Round-2 session D: GPU tests (replay, first-block batch budget), small-k
# dynamic tickets A/B, the C4 bench with epoch replay, the default bench.
OUT=gpurun_out/r2d
mkdir -p $OUT
python -c "import __graft_entry__ as g; g.build()" > $OUT/build.log 2>&1
timeout 900 python -m pytest tests -q -m gpu > $OUT/pytest_gpu.log 2>&1; echo "pytest gpu exit $?" >> $OUT/pytest_gpu.log
G='[{"J":0,"TILE":0,"DYN":0},{"J":0,"TILE":0,"DYN":1},{"J":0,"TILE":0,"DYN":0},{"J":0,"TILE":0,"DYN":1}]'
for K in 1 8 16 32; do
  TUNE_K=$K TUNE_GRID="$G" TUNE_DOCS=200000 TUNE_SCHEMES=2u timeout 300 python tools/tune.py >> $OUT/dyn_smallk.jsonl 2>> $OUT/dyn.err
  TUNE_K=$K TUNE_GRID="$G" TUNE_DOCS=200000 TUNE_SCHEMES=4u-bit timeout 300 python tools/tune.py >> $OUT/dyn_smallk.jsonl 2>> $OUT/dyn.err
done
timeout 1500 python bench.py --config c4 > $OUT/bench_c4.json 2> $OUT/bench_c4.err; echo "bench c4 exit $?" >> $OUT/bench_c4.err
timeout 900 python bench.py > $OUT/bench.json 2> $OUT/bench.err; echo "bench exit $?" >> $OUT/bench.err
echo done > $OUT/DONE
