#!/bin/bash
# Round-2 ncu evidence for the 2U headline kernel (the coefficient-uniform
# kernel, uniform.cu): one full-size C2 launch under --set full, and the
# launch list of a short bench run (kernel shares of the step).
TAG=${1:-ncu_r2}
OUT=gpurun_out/$TAG
mkdir -p $OUT
python -c "import __graft_entry__ as g; g.build()" > $OUT/build.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:sketch_uniform -s 3 -c 1 \
    -o $OUT/prof_2u_uniform_full python bench.py --steps 1 --warmup 3 --schemes 2u --e2e-steps 1 --no-cpu > $OUT/ncu_2u.log 2>&1
python tools/ncu_summary.py $OUT/prof_2u_uniform_full.ncu-rep > $OUT/ncu_2u_uniform_full_size.txt 2>&1
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $OUT/launches.csv \
    python bench.py --steps 3 --warmup 3 --e2e-steps 1 --no-cpu > $OUT/launches.log 2>&1
echo done > $OUT/DONE
