"""Copy-engine peer copies vs a concurrent prefill GEMM (one process, 2
GPUs): can a bf16 partial travel to the peer by DMA while the tensor cores
run, without slowing either?  Prints us for GEMM alone, copy alone, both."""
import json, os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from paper_2311_18677_b200 import kernels as K

M, N, Kd = int(os.environ.get("M", "1024")), int(os.environ.get("N", "28672")), 8192
MB = float(os.environ.get("MB", "16"))
torch.cuda.set_device(0)
a = torch.randn(M, Kd, device="cuda:0").bfloat16()
w = torch.randn(N, Kd, device="cuda:0").bfloat16()
out = torch.empty(M, N, device="cuda:0", dtype=torch.bfloat16)
src = torch.empty(int(MB * 2**20) // 2, device="cuda:0", dtype=torch.bfloat16)
dst = torch.empty_like(src, device="cuda:1")
s_cp = torch.cuda.Stream(device=0)


def gemm():
    K.gemm(a, w, K.EPI_BF16, out=out)


def copy():
    with torch.cuda.stream(s_cp):
        dst.copy_(src, non_blocking=True)


def timed(fn, n=10):
    torch.cuda.synchronize(0); torch.cuda.synchronize(1)
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(n):
        fn()
    s_cp.wait_stream(torch.cuda.current_stream()) if False else None
    torch.cuda.current_stream().wait_stream(s_cp)
    e1.record()
    torch.cuda.synchronize(0)
    return e0.elapsed_time(e1) * 1e3 / n


def both():
    ev = torch.cuda.Event()
    ev.record()
    s_cp.wait_event(ev)
    copy()
    gemm()


for f in (gemm, copy, both):
    timed(f, 3)
r = {"M": M, "N": N, "K": Kd, "copy_MB": MB, "gemm_us": timed(gemm), "copy_us": timed(copy),
     "both_us": timed(both)}
r["copy_GBps"] = MB * 2**20 / r["copy_us"] / 1e3
print(json.dumps({k: round(v, 2) if isinstance(v, float) else v for k, v in r.items()}))
