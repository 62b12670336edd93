#!/bin/bash
# Session L: uniform kernel with the shared-memory transpose -- crossover
# against the persistent kernel by row length and k, GPU tests, bench.
OUT=gpurun_out/r2l
mkdir -p $OUT
python -c "import __graft_entry__ as g; g.build()" > $OUT/build.log 2>&1
for nnz in 1500 2600 3728 6000 12000; do
  docs=$(( 1300000000 / nnz ))
  AB_NNZ=$nnz AB_DOCS=$docs AB_KS=300,400,500,544 AB_REPS=3 AB_ARMS='[{"uniform_2u":2}]' timeout 600 python tools/ab_uniform.py >> $OUT/crossover.jsonl 2>> $OUT/crossover.err
done
timeout 900 python -m pytest tests -x -q -m gpu > $OUT/pytest_gpu.log 2>&1; echo "pytest gpu exit $?" >> $OUT/pytest_gpu.log
timeout 900 python bench.py > $OUT/bench.json 2> $OUT/bench.err; echo "bench exit $?" >> $OUT/bench.err
echo done > $OUT/DONE
