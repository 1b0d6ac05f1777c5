"""Per-CTA globaltimer timeline of one decode-attention launch (tensor-core
GQA kernel, cluster form) — needs the probe build of libswb200: `make
probe-lib`, then on the GPU box `cp build/var/libswb200_probe.so
paper_2311_18677_b200/libswb200.so` before running this.  SHAPE=H:Hkv, CTX,
B.  (70B TP4, ctx 1500: pages land ~3.5 us after launch, the CTA's 64 KB of
K/V being the bound; the warp combine and the cluster merge were 1.5-2.3 us
each before they were reworked.)"""
import json, os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from paper_2311_18677_b200 import kernels as K

H, Hkv = (int(v) for v in os.environ.get("SHAPE", "16:2").split(":"))
ctx, B = int(os.environ.get("CTX", "1500")), int(os.environ.get("B", "1"))
dh, bs, part = 128, 16, 128
nblk = B * (ctx // bs + 8) + 16
kp = torch.randn(nblk, Hkv, bs, dh, device="cuda").bfloat16()
vp = torch.randn_like(kp)
maxb = ctx // bs + 8
tables = torch.randperm(nblk, device="cuda").int()[:B * maxb].view(B, maxb).contiguous()
qkv = torch.randn(B, (H + 2 * Hkv) * dh, device="cuda").bfloat16()
ctxs = torch.full((B,), ctx, dtype=torch.int32, device="cuda")
max_ctx = ((ctx + 64 + part - 1) // part) * part
ws = torch.zeros(K.attn_decode_workspace_bytes(B, H, max_ctx, part, dh), dtype=torch.uint8,
                 device="cuda")
out = torch.empty(B, H * dh, dtype=torch.bfloat16, device="cuda")
f = lambda: K.attn_decode_step(qkv, kp.data_ptr(), vp.data_ptr(), tables, ctxs, B, H, Hkv,  # noqa: E731
                               dh, bs, 0.088, max_ctx, part, ws, out)
for _ in range(5):
    f()
torch.cuda.synchronize()
NP = max_ctx // part
# the cluster launches use 8 or 16 partitions per (b, kv head): size for 16
ncta = max(NP, 16) * Hkv * B
probe = torch.zeros(ncta * 16, dtype=torch.int64, device="cuda")
os.environ["SWB_ATTN_PROBE_ADDR"] = str(probe.data_ptr())
res = []
for rep in range(3):
    probe.zero_()
    torch.cuda.synchronize()
    f()
    torch.cuda.synchronize()
    p = probe.view(ncta, 16).double()
    t0 = p[:, 0][p[:, 0] > 0].min()
    names = (["start", "pdl_wait", "q_staged", "k_landed", "v_landed", "pv_done", "combined",
              "pushed/merge_wait", "out_written"] if H // Hkv > 2 else
             ["start", "pdl_wait", "q_ready", "first_page", "pages_done", "combine_start",
              "pushed", "merge_wait", "out_written"])
    row = {}
    for k, n in enumerate(names):
        col = p[:, k]
        col = col[col > 0]
        if col.numel():
            c = (col - t0) / 1e3
            row[n] = [round(c.min().item(), 2), round(c.median().item(), 2), round(c.max().item(), 2)]
    res.append(row)
del os.environ["SWB_ATTN_PROBE_ADDR"]
print(json.dumps({"H": H, "Hkv": Hkv, "ctx": ctx, "B": B, "ctas": ncta,
                  "timeline_us [min, median, max]": res[-1]}))
