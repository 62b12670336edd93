#!/bin/bash
# Round-2 session A: GPU tests after the options refactor, the shared-memory
# carveout A/B of the persistent sketch kernel (occupancy), and ncu of the
# permutation-mode kernels.
OUT=gpurun_out/r2a
mkdir -p $OUT
nproc > $OUT/nproc.txt; lscpu > $OUT/lscpu.txt; free -g > $OUT/free.txt; df -h /tmp . > $OUT/df.txt
python -c "import __graft_entry__ as g; g.build()" > $OUT/build.log 2>&1
timeout 600 python -m pytest tests -x -q -m gpu > $OUT/pytest_gpu.log 2>&1; echo "pytest gpu exit $?" >> $OUT/pytest_gpu.log
# carveout A/B: library shapes at k = 500 / 300 / 200, default (-1) vs max shared (100), twice
G='[{"J":0,"TILE":0,"CARVEOUT":-1},{"J":0,"TILE":0,"CARVEOUT":100},{"J":0,"TILE":0,"CARVEOUT":-1},{"J":0,"TILE":0,"CARVEOUT":100}]'
for K in 500 300 200; do
  TUNE_K=$K TUNE_GRID="$G" TUNE_DOCS=200000 TUNE_SCHEMES=2u timeout 300 python tools/tune.py >> $OUT/carveout.jsonl 2>> $OUT/carveout.err
  TUNE_K=$K TUNE_GRID="$G" TUNE_DOCS=50000 TUNE_SCHEMES=4u-bit timeout 300 python tools/tune.py >> $OUT/carveout.jsonl 2>> $OUT/carveout.err
done
# occupancy counters of the 2U k=500 launch under both settings
for C in -1 100; do
  BBMH_OPT_CARVEOUT=$C timeout 600 ncu --section Occupancy --section LaunchStats --section SpeedOfLight \
    --metrics sm__warps_active.avg.pct_of_peak_sustained_active,sm__pipe_fmaheavy_cycles_active.avg.pct_of_peak_sustained_active,sm__ctas_launched.sum,smsp__warps_launched.sum \
    --clock-control none -k regex:sketch_kernel -s 2 -c 1 --csv \
    python bench.py --docs 50000 --steps 1 --warmup 2 --schemes 2u --e2e-steps 1 --no-cpu > $OUT/ncu_occ_c$C.csv 2> $OUT/ncu_occ_c$C.err
done
# permutation mode: build kernel (k = 16 tables of 2^24) and one table-outer pass at C3 (k = 500)
timeout 300 ncu --set full --clock-control none --import-source on -k regex:perm_shuffle -c 1 \
  -o $OUT/prof_permgen python tools/run_perm.py --docs 2000 --k 16 > $OUT/ncu_permgen.log 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:perm_pass -s 3 -c 1 \
  -o $OUT/prof_permpass python tools/run_perm.py --docs 100000 --k 500 > $OUT/ncu_permpass.log 2>&1
timeout 300 python tools/run_perm.py --docs 350000 --k 500 --reps 3 > $OUT/perm_c3_350k.json 2> $OUT/perm_c3_350k.err
echo done > $OUT/DONE
