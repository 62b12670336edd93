#!/bin/bash
# Session T: the coefficient-uniform 4U-bit kernel against the persistent one
# (A/B, codes compared); uniform 2U kernel for 16 < k <= 32 against the lane-split kernel
# (A/B); the k sweep with the round-2 kernels; C5 online latencies.
OUT=gpurun_out/r2t
mkdir -p $OUT
python -c "import __graft_entry__ as g; g.build()" > $OUT/build.log 2>&1
AB_SCHEME=4u-bit AB_DOCS=100000 AB_KS=500,200,64 AB_BS=8,1 AB_REPS=2 timeout 900 python tools/ab_uniform.py > $OUT/u4_ab.jsonl 2> $OUT/u4_ab.err
AB_SCHEME=4u-bit AB_DIM=1048576 AB_DOCS=100000 AB_KS=500 AB_REPS=2 timeout 600 python tools/ab_uniform.py >> $OUT/u4_ab.jsonl 2>> $OUT/u4_ab.err
AB_KS=20,24,28,32 AB_REPS=4 AB_ARMS='[{"uniform_2u":2}]' timeout 600 python tools/ab_uniform.py > $OUT/smallk_ab.jsonl 2> $OUT/smallk_ab.err
AB_NNZ=12000 AB_DOCS=108000 AB_KS=24,32 AB_REPS=4 AB_ARMS='[{"uniform_2u":2}]' timeout 600 python tools/ab_uniform.py >> $OUT/smallk_ab.jsonl 2>> $OUT/smallk_ab.err
timeout 900 python tools/bench_configs.py --only ksweep,c5 --out $OUT/configs.jsonl > $OUT/configs.log 2>&1
echo done > $OUT/DONE
