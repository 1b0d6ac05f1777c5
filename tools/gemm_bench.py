"""Prefill GEMM throughput at the bench shapes (CUDA-graph timed, weights
rotated so each launch streams its W from HBM).  SWB_GEMM_PAIR=0/1 A/B."""
import json, os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from paper_2311_18677_b200 import kernels as K


def timeit(fn, iters=20, warm=3):
    for _ in range(warm):
        fn()
    torch.cuda.synchronize()
    g = torch.cuda.CUDAGraph()
    with torch.cuda.graph(g):
        for _ in range(iters):
            fn()
    g.replay()
    torch.cuda.synchronize()
    s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    s.record(); g.replay(); e.record(); torch.cuda.synchronize()
    return s.elapsed_time(e) / iters


SHAPES = {  # name: (M, N, K, epilogue)
    "7b.qkv": (1024, 12288, 4096, K.EPI_BF16), "7b.o": (1024, 4096, 4096, K.EPI_RESID_F32),
    "7b.gu": (1024, 22016, 4096, K.EPI_SWIGLU), "7b.down": (1024, 4096, 11008, K.EPI_RESID_F32),
    "7b.qkv2k": (2048, 12288, 4096, K.EPI_BF16),
    "70b-tp2.qkv": (1024, 5120, 8192, K.EPI_BF16), "70b-tp2.gu": (1024, 28672, 8192, K.EPI_SWIGLU),
    "70b-tp2.down": (1024, 8192, 14336, K.EPI_F32),
    "sq8192": (8192, 8192, 8192, K.EPI_BF16),
}
res = {"pair": os.environ.get("SWB_GEMM_PAIR", "1")}
for name, (M, N, Kd, epi) in SHAPES.items():
    a = torch.randn(M, Kd, device="cuda").bfloat16()
    ws = [torch.randn(N, Kd, device="cuda").bfloat16() for _ in range(2)]
    nout = N // 2 if epi == K.EPI_SWIGLU else N
    dt = torch.float32 if epi in (K.EPI_RESID_F32, K.EPI_F32) else torch.bfloat16
    out = torch.zeros(M, nout, dtype=dt, device="cuda")
    resid = out if epi == K.EPI_RESID_F32 else None
    i = [0]

    def fn():
        K.gemm(a, ws[i[0] % 2], epi, out=out, resid=resid)
        i[0] += 1
    ms = timeit(fn, iters=10 if M >= 8192 else 20)
    res[name] = round(2 * M * N * Kd / ms / 1e9, 1)
    if name == "sq8192":
        res["cublas_sq8192"] = round(2 * M * N * Kd / timeit(lambda: torch.matmul(a, ws[0].t()), iters=10) / 1e9, 1)
print(json.dumps(res), flush=True)
