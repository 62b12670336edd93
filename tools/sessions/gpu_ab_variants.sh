#!/bin/bash
# A/B of uniform-kernel body variants (option uniform_variant) against the
# persistent kernel, then an ncu capture of the uniform kernel at k = 500.
OUT=gpurun_out/${1:-ab1}
mkdir -p $OUT
AB_KS=${AB_KS:-500,200,64} AB_REPS=4 AB_ARMS=${AB_ARMS:-'[{"uniform_2u":2,"uniform_variant":0},{"uniform_2u":2,"uniform_variant":2},{"uniform_2u":2,"uniform_variant":5},{"uniform_2u":2,"uniform_variant":7}]'} \
  timeout 900 python tools/ab_uniform.py > $OUT/ab.jsonl 2> $OUT/ab.err
[ "${NCU:-1}" = "1" ] && NCU_KS="500" bash tools/sessions/gpu_ncu_uni_stalls.sh ${1:-ab1}/ncu
echo done > $OUT/DONE
