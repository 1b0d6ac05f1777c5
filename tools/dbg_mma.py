import sys, os
sys.path.insert(0, os.getcwd())
import torch
from paper_2311_18677_b200 import kernels as K
torch.manual_seed(0)
for M in (16, 8, 2):
    x = torch.randn(M, 4096, device="cuda").bfloat16()
    w = torch.randn(4096, 4096, device="cuda").bfloat16()
    base = K.gemv(x, w, K.EPI_F32).clone()
    bad = 0
    for i in range(200):
        o = K.gemv(x, w, K.EPI_F32)
        d = (o != base)
        if d.any():
            bad += 1
            if bad <= 3:
                idx = d.nonzero()
                print("M", M, "iter", i, "ndiff", idx.shape[0], "rows", sorted(set(idx[:, 0].tolist()))[:8],
                      "cols", idx[:8, 1].tolist(), "maxdiff", (o - base).abs().max().item(), flush=True)
    print("M", M, "bad", bad, "/ 200", flush=True)
