"""e2e pipeline probe for cfg2: HostPipeline step time with the current
operator settings (env: HBP_PACKED_X etc.), K steps."""
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402

import bench  # noqa: E402
import paper_2504_08860_b200 as H  # noqa: E402

cfgname = sys.argv[1] if len(sys.argv) > 1 else "cfg2"
K = int(sys.argv[2]) if len(sys.argv) > 2 else 20
dev = torch.device("cuda", 0)
desc, rows, cols, rp, col, val, C, vdt = bench.make_matrix_gpu(cfgname, 0, dev)
cfg = H.PartitionConfig(col_width=C)
csr = H.CsrMatrix(rows, cols, rp, col, val)
grid = H.make_grid(csr, cfg)
hbp = H.build_hbp(csr, grid, H.hash_permutations(grid, H.sample_hash_params(grid, cfg)),
                  with_add_sign=False, with_zero_row=False)
del csr, grid, col, val
pipe = H.HostPipeline(hbp, depth=3)
xh = torch.empty(cols, dtype=vdt, pin_memory=True)
xh.uniform_(-1, 1)
yhs = [torch.empty(rows, dtype=vdt, pin_memory=True) for _ in range(3)]
pipe.run([xh] * 5, [yhs[i % 3] for i in range(5)])
torch.cuda.synchronize()
for rep in range(3):
    s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    s.record()
    pipe.run([xh] * K, [yhs[i % 3] for i in range(K)])
    e.record()
    torch.cuda.synchronize()
    print(f"{cfgname} packed={pipe.op.hot.packed if pipe.op.hot is not None else None} "
          f"e2e ms/step {s.elapsed_time(e) / K:.4f}", flush=True)
