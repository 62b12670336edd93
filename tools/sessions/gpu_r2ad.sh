#!/bin/bash
# Session AD: ncu --set full of the uniform 4U-bit kernel (k = 300, C2 docs)
# and of the persistent 4U-bit kernel at the same k, for the record.
OUT=gpurun_out/r2ad
mkdir -p $OUT
python -c "import __graft_entry__ as g; g.build()" > $OUT/build.log 2>&1
cat > /tmp/once4.py <<'PY'
import os, sys
sys.path.insert(0, os.getcwd())
import torch, bench
from paper_1205_2958_b200 import bbmh
n, k = 60000, 300
bbmh.set_option("uniform_4u", int(os.environ.get("U4", "1")))
d_rp, d_idx = bench.make_corpus_device(torch, n, bench.NNZ, bench.D_WEBSPAM, 1, torch.device("cuda", 0))
f = bbmh.Family(3, bench.D_WEBSPAM, k, bench.SEED)
codes = torch.zeros(n * k, dtype=torch.uint8, device="cuda")
for _ in range(2):
    f.sketch_csr_device(d_rp.data_ptr(), d_idx.data_ptr(), n, 8, codes.data_ptr(), stream=torch.cuda.current_stream().cuda_stream)
torch.cuda.synchronize()
PY
U4=1 timeout 900 ncu --set full --clock-control none --import-source on -k regex:sketch_uniform4 -s 1 -c 1 -o $OUT/u4_k300 python /tmp/once4.py > $OUT/u4.log 2>&1
U4=0 timeout 900 ncu --set full --clock-control none --import-source on -k regex:sketch_kernel -s 1 -c 1 -o $OUT/p4_k300 python /tmp/once4.py > $OUT/p4.log 2>&1
echo done > $OUT/DONE
