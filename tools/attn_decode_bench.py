"""Decode attention (swb_attn_decode_step) alone: KV bytes / time over batch
and context (CUDA-graph timed, pool > L2)."""
import json, os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from paper_2311_18677_b200 import kernels as K


def timeit(fn, iters=20):
    for _ in range(3):
        fn()
    torch.cuda.synchronize()
    g = torch.cuda.CUDAGraph()
    with torch.cuda.graph(g):
        for _ in range(iters):
            fn()
    g.replay(); torch.cuda.synchronize()
    s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    s.record(); g.replay(); e.record(); torch.cuda.synchronize()
    return s.elapsed_time(e) / iters


res = {}
dh, bs = 128, 16
# SHAPES="name:H:Hkv,..." and CASES="B:ctx,..." override the defaults
shapes = [(n, int(h), int(k)) for n, h, k in
          (x.split(":") for x in os.environ.get("SHAPES", "7b:32:32,70b-tp2:32:4").split(","))]
cases = [tuple(int(v) for v in x.split(":")) for x in
         os.environ.get("CASES", "1:1100,8:1100,32:1100,1:8000,8:4000").split(",")]
for name, H, Hkv in shapes:
    for B, ctx in cases:
        nblk = B * (ctx // bs + 8) + 16
        kp = torch.randn(nblk, Hkv, bs, dh, device="cuda").bfloat16()
        vp = torch.randn_like(kp)
        maxb = ctx // bs + 8
        tables = torch.randperm(nblk, device="cuda").int()[:B * maxb].view(B, maxb).contiguous()
        qkv = torch.randn(B, (H + 2 * Hkv) * dh, device="cuda").bfloat16()
        ctxs = torch.full((B,), ctx, dtype=torch.int32, device="cuda")
        part = int(os.environ.get("PART", "128"))
        max_ctx = ((ctx + 64 + part - 1) // part) * part
        ws = torch.zeros(K.attn_decode_workspace_bytes(B, H, max_ctx, part, dh), dtype=torch.uint8,
                         device="cuda")
        out = torch.empty(B, H * dh, dtype=torch.bfloat16, device="cuda")
        f = lambda: K.attn_decode_step(qkv, kp.data_ptr(), vp.data_ptr(), tables, ctxs, B, H, Hkv,  # noqa: E731
                                       dh, bs, 0.088, max_ctx, part, ws, out)
        ms = timeit(f)
        byts = B * ctx * Hkv * dh * 2 * 2
        res[f"{name}_B{B}_ctx{ctx}"] = {"us": round(ms * 1e3, 1), "GBps": round(byts / ms / 1e6)}
        del kp, vp
print(json.dumps(res))
