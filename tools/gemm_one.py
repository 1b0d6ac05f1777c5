import sys, os
sys.path.insert(0, os.getcwd())
import torch
from paper_2311_18677_b200 import kernels as K
M, N, Kd = 1024, 22016, 4096
a = torch.randn(M, Kd, device="cuda").bfloat16(); w = torch.randn(N, Kd, device="cuda").bfloat16()
K.gemm(a, w, K.EPI_SWIGLU); torch.cuda.synchronize()
w2 = torch.randn(12288, 4096, device="cuda").bfloat16()
K.gemm(a, w2, K.EPI_BF16); torch.cuda.synchronize()
print("ok")
