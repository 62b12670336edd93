#!/bin/bash
# Session N: uniform kernel 16- vs 32-function groups (A/B over k and row
# length), the mixed-transfer tests, the 2U bench line with its e2e leg.
OUT=gpurun_out/r2n
mkdir -p $OUT
python -c "import __graft_entry__ as g; g.build()" > $OUT/build.log 2>&1
for nnz in 3728 12000; do
  docs=$(( 1300000000 / nnz ))
  AB_NNZ=$nnz AB_DOCS=$docs AB_KS=500,200,64 AB_REPS=3 AB_ARMS='[{"uniform_2u":2,"uniform_group":32},{"uniform_2u":2,"uniform_group":16}]' timeout 600 python tools/ab_uniform.py >> $OUT/group_ab.jsonl 2>> $OUT/group_ab.err
done
timeout 900 python -m pytest tests -x -q -m gpu > $OUT/pytest_gpu.log 2>&1; echo "pytest gpu exit $?" >> $OUT/pytest_gpu.log
timeout 900 python bench.py --no-cpu --schemes 2u > $OUT/bench.json 2> $OUT/bench.err; echo "bench exit $?" >> $OUT/bench.err
echo done > $OUT/DONE
