"""One launch of each prefill GEMM flavour at the 7B 1024-token shapes (for ncu)."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from paper_2311_18677_b200 import kernels as K
M = 1024
a = torch.randn(M, 4096, device="cuda").bfloat16()
w = torch.randn(22016, 4096, device="cuda").bfloat16()
K.gemm(a, w, K.EPI_SWIGLU); torch.cuda.synchronize()
wq = torch.randn(12288, 4096, device="cuda").bfloat16()
qkv = torch.empty(M, 12288, device="cuda").bfloat16()
pos = torch.arange(M, device="cuda", dtype=torch.int32)
kp = torch.zeros(M // 16 + 1, 32, 16, 128, device="cuda").bfloat16(); vp = torch.zeros_like(kp)
K.gemm_qkv_rope(a, wq, qkv, pos, 32, 32, 10000.0, k_layer=kp.data_ptr(), v_layer=vp.data_ptr(),
                slots=pos, rope_table=K.rope_table(10000.0, 4096))
torch.cuda.synchronize()
print("ok")
