#!/bin/bash
# Session P: uniform kernel, one loop for every group (uniform-indexed
# coefficient loads) vs per-group compiled loops; host budget with the 1 GiB
# DRAM probe; the 2U bench line.
OUT=gpurun_out/r2p
mkdir -p $OUT
python -c "import __graft_entry__ as g; g.build()" > $OUT/build.log 2>&1
python -c "
from paper_1205_2958_b200 import bbmh; import json
print(json.dumps(bbmh.host_budget(1)))" > $OUT/budget.json 2>&1
for nnz in 3728 12000; do
  docs=$(( 1300000000 / nnz ))
  AB_NNZ=$nnz AB_DOCS=$docs AB_KS=500,200,64 AB_REPS=3 AB_ARMS='[{"uniform_2u":2,"uniform_variant":0},{"uniform_2u":2,"uniform_variant":1}]' timeout 600 python tools/ab_uniform.py >> $OUT/gen_ab.jsonl 2>> $OUT/gen_ab.err
done
timeout 900 python bench.py --no-cpu --schemes 2u > $OUT/bench.json 2> $OUT/bench.err; echo "bench exit $?" >> $OUT/bench.err
echo done > $OUT/DONE
