#!/bin/bash
# ncu capture of the prototype kernel (developer experiment)
mkdir -p gpurun_out/pn
TUNE_DOCS=20000 timeout 600 ncu --set full --clock-control none --import-source on -k regex:wproto -c 1 -o gpurun_out/pn/wproto python tools/proto/run_proto2u.py > gpurun_out/pn/log.txt 2>&1
echo done > gpurun_out/pn/DONE
