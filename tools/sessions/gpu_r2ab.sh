#!/bin/bash
# Session AB: final validation -- GPU tests, smoke, the default bench line and
# its reference arm with the final build; racecheck of the rest of the driver
# with launches made blocking (CUDA_LAUNCH_BLOCKING=1).
OUT=gpurun_out/r2ab
mkdir -p $OUT
python -c "import __graft_entry__ as g; g.build()" > $OUT/build.log 2>&1
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > $OUT/smoke.log 2>&1; echo "smoke exit $?" >> $OUT/smoke.log
timeout 1200 python -m pytest tests -q -m gpu > $OUT/pytest_gpu.log 2>&1; echo "pytest gpu exit $?" >> $OUT/pytest_gpu.log
timeout 900 python bench.py > $OUT/bench.json 2> $OUT/bench.err; echo "bench exit $?" >> $OUT/bench.err
timeout 600 python bench.py --impl reference > $OUT/bench_ref.json 2> $OUT/bench_ref.err; echo "ref exit $?" >> $OUT/bench_ref.err
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $OUT/launches.csv \
    python bench.py --steps 3 --warmup 3 --e2e-steps 1 --no-cpu > $OUT/launches.log 2>&1
CUDA_LAUNCH_BLOCKING=1 SANITIZE_ONLY=rest timeout 900 compute-sanitizer --tool racecheck --error-exitcode 9 --print-limit 20 \
    python tools/sanitize_driver.py > $OUT/racecheck_rest.log 2>&1
echo "exit $?" >> $OUT/racecheck_rest.log
echo done > $OUT/DONE
