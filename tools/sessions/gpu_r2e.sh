#!/bin/bash
# Round-2 session E: range-sharded lanes on the C4 text (host-side scaling of
# the loader) and the launch list of the bench command.
OUT=gpurun_out/r2e
mkdir -p $OUT
python -c "import __graft_entry__ as g; g.build()" > $OUT/build.log 2>&1
timeout 900 python tools/c4_lanes.py --scheme 2u > $OUT/c4_lanes_2u.jsonl 2> $OUT/c4_lanes.err
timeout 900 python tools/c4_lanes.py --scheme 4u-bit > $OUT/c4_lanes_4u.jsonl 2>> $OUT/c4_lanes.err
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 600 --csv --log-file $OUT/launches_bench.csv \
    python bench.py --docs 50000 --steps 2 --warmup 1 --e2e-steps 1 --perm-steps 1 --no-cpu > $OUT/ncu_bench.log 2>&1
timeout 600 python -m pytest tests/test_gpu_vw.py -q > $OUT/pytest_vw.log 2>&1; echo "exit $?" >> $OUT/pytest_vw.log
echo done > $OUT/DONE
