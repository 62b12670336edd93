#!/bin/bash
# Full-size ncu captures of the headline kernels (one launch each, C2 size).
TAG=${1:-ncu}
OUT=gpurun_out/$TAG
mkdir -p $OUT
python -c "import __graft_entry__ as g; g.build()" > $OUT/build.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:sketch_kernel -s 3 -c 1 \
    -o $OUT/prof_2u_full python bench.py --steps 1 --warmup 3 --schemes 2u --e2e-steps 1 --no-cpu > $OUT/ncu_2u.log 2>&1
timeout 1200 ncu --set full --clock-control none --import-source on -k regex:sketch_kernel -s 3 -c 1 \
    -o $OUT/prof_4u_full python bench.py --steps 1 --warmup 3 --schemes 4u-bit --e2e-steps 1 --no-cpu > $OUT/ncu_4u.log 2>&1
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $OUT/launches.csv \
    python bench.py --steps 3 --warmup 3 --e2e-steps 1 --no-cpu > $OUT/launches.log 2>&1
echo done > $OUT/DONE
