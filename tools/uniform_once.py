"""One 2U sketch of an HBM-resident webspam-shaped corpus (for ncu captures of
the uniform kernel). ONCE_K, ONCE_DOCS, ONCE_UNIFORM (option uniform_2u)."""
import os
import sys

ROOT = os.path.abspath(os.path.join(os.path.dirname(__file__), ".."))
sys.path.insert(0, ROOT)
import torch  # noqa: E402

import bench  # noqa: E402
from paper_1205_2958_b200 import bbmh  # noqa: E402

n = int(os.environ.get("ONCE_DOCS", "100000"))
k = int(os.environ.get("ONCE_K", "500"))
bbmh.set_option("uniform_2u", int(os.environ.get("ONCE_UNIFORM", "1")))
dev = torch.device("cuda", 0)
d_rp, d_idx = bench.make_corpus_device(torch, n, bench.NNZ, bench.D_2U, 1, dev)
fam = bbmh.Family(1, bench.D_2U, k, bench.SEED)
codes = torch.zeros(n * k, dtype=torch.uint8, device=dev)
st = torch.cuda.current_stream()
for _ in range(2):
    fam.sketch_csr_device(d_rp.data_ptr(), d_idx.data_ptr(), n, 8, codes.data_ptr(), stream=st.cuda_stream)
torch.cuda.synchronize()
