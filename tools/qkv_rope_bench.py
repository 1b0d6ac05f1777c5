"""Fused QKV-GEMM + RoPE/KV-write epilogue vs GEMM then swb_rope_kv_write (7B prefill shape)."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from paper_2311_18677_b200 import kernels as K
M, d, H, Hkv = 1024, 4096, 32, 32
N = (H + 2 * Hkv) * 128
a = torch.randn(M, d, device="cuda").bfloat16()
w = torch.randn(N, d, device="cuda").bfloat16()
pos = torch.arange(M, device="cuda", dtype=torch.int32)
kp = torch.zeros(M // 16 + 1, Hkv, 16, 128, device="cuda").bfloat16(); vp = torch.zeros_like(kp)
slots = torch.arange(M, device="cuda", dtype=torch.int32)
qkv = torch.empty(M, N, device="cuda").bfloat16()
tab = K.rope_table(10000.0, 16384)
def t(f, n=20):
    for _ in range(3): f()
    torch.cuda.synchronize(); s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    s.record()
    for _ in range(n): f()
    e.record(); torch.cuda.synchronize(); return s.elapsed_time(e) / n * 1e3
fused = t(lambda: K.gemm_qkv_rope(a, w, qkv, pos, H, Hkv, 10000.0, k_layer=kp.data_ptr(), v_layer=vp.data_ptr(), slots=slots, rope_table=tab))
sep = t(lambda: (K.gemm(a, w, K.EPI_BF16, out=qkv), K.rope_kv_write(qkv, pos, H, Hkv, 128, 10000.0, kp.data_ptr(), vp.data_ptr(), slots, 16)))
plain = t(lambda: K.gemm(a, w, K.EPI_BF16, out=qkv))
print(f"fused {fused:.1f} us  gemm+rope {sep:.1f} us  gemm alone {plain:.1f} us")
