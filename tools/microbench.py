"""CUDA-event micro-benchmarks of the hot kernels at the bench shapes."""
import json, math, os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from paper_2311_18677_b200 import kernels as K

def timeit(fn, iters=20, warm=3):
    """Device time per call: `iters` calls captured in one CUDA graph (no
    host launch overhead), replayed after warm-up, timed with events."""
    for _ in range(warm): fn()
    torch.cuda.synchronize()
    g = torch.cuda.CUDAGraph()
    with torch.cuda.graph(g):
        for _ in range(iters): fn()
    g.replay(); torch.cuda.synchronize()
    s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    s.record(); g.replay(); e.record(); torch.cuda.synchronize()
    return s.elapsed_time(e) / iters

res = {}
d, f, V = 4096, 11008, 32000
shapes = {"qkv": (3 * d, d), "o": (d, d), "gu": (2 * f, d), "down": (d, f), "lm": (V, d)}
# several weight copies so consecutive launches don't hit L2
for name, (N, Kd) in shapes.items():
    ws = [torch.randn(N, Kd, device="cuda").bfloat16() for _ in range(4)]
    for M in (1, 2, 4, 8):
        x = torch.randn(M, Kd, device="cuda").bfloat16()
        epi = K.EPI_SWIGLU if name == "gu" else K.EPI_BF16
        out = torch.empty(M, N // 2 if name == "gu" else N, device="cuda", dtype=torch.bfloat16)
        i = [0]
        def fn():
            K.gemv(x, ws[i[0] % 4], epi, out=out); i[0] += 1
        ms = timeit(fn)
        res[f"gemv_{name}_M{M}"] = {"us": ms * 1e3, "GBps": N * Kd * 2 / ms / 1e6}
for name, (N, Kd) in shapes.items():
    M = 1024
    a = torch.randn(M, Kd, device="cuda").bfloat16()
    wt = torch.randn(N, Kd, device="cuda").bfloat16()
    epi = K.EPI_SWIGLU if name == "gu" else K.EPI_BF16
    ms = timeit(lambda: K.gemm(a, wt, epi))
    res[f"gemm_{name}_M{M}"] = {"us": ms * 1e3, "TFLOPs": 2 * M * N * Kd / ms / 1e9}
M, N, Kd = 8192, 8192, 8192
a = torch.randn(M, Kd, device="cuda").bfloat16(); wt = torch.randn(N, Kd, device="cuda").bfloat16()
ms = timeit(lambda: K.gemm(a, wt, K.EPI_BF16), iters=10)
res["gemm_8192^3"] = {"us": ms * 1e3, "TFLOPs": 2 * M * N * Kd / ms / 1e9}
ms = timeit(lambda: torch.matmul(a, wt.t()), iters=10)
res["cublas_8192^3"] = {"us": ms * 1e3, "TFLOPs": 2 * M * N * Kd / ms / 1e9}
# decode attention, 7B shape ctx 1100
H = Hkv = 32; dh = 128; bs = 16; B = 1
nblk = 2000
kp = torch.randn(nblk, Hkv, bs, dh, device="cuda").bfloat16(); vp = torch.randn_like(kp)
tables = torch.arange(80, device="cuda", dtype=torch.int32).view(1, 80)
qkv = torch.randn(B, 3 * H * dh, device="cuda").bfloat16()
lens = torch.tensor([1100], device="cuda", dtype=torch.int32)
for part in (64, 128, 256):
    ws = torch.zeros(K.attn_decode_workspace_bytes(B, H, 1152, part, dh), dtype=torch.uint8, device="cuda")
    ms = timeit(lambda: K.attn_decode(qkv, kp.data_ptr(), vp.data_ptr(), tables, lens, B, H, Hkv, dh, bs, 0.088, 1152, part, ws))
    res[f"attn_decode_ctx1100_part{part}"] = {"us": ms * 1e3, "GBps": 1100 * Hkv * dh * 4 / ms / 1e6}
qkv = torch.randn(1024, 3 * H * dh, device="cuda").bfloat16()
cu = torch.tensor([0, 1024], device="cuda", dtype=torch.int32)
ms = timeit(lambda: K.attn_prefill(qkv, cu, 1, 1024, H, Hkv, dh, 0.088))
res["attn_prefill_1024"] = {"us": ms * 1e3, "TFLOPs": 2 * 1024 * 1024 * H * dh / ms / 1e9}
print(json.dumps(res, indent=1))
