"""Marginal in-step cost of each kernel family of the 7B decode step (CUDA
graph, B=1, ctx ~1100): the step is captured with one family replaced by
nothing and timed against the full step.  Timing-only (the numerics of an
ablated step are wrong).  MODEL / B / CTX from the environment."""
import json, os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from paper_2311_18677_b200 import kernels as K
from paper_2311_18677_b200.model import get_config, init_weights
from paper_2311_18677_b200.runner import ModelRunner
from paper_2311_18677_b200.kvcache import KVCacheManager

cfg = get_config(os.environ.get("MODEL", "llama2-7b"))
w = init_weights(cfg)
B, CTX = int(os.environ.get("B", "1")), int(os.environ.get("CTX", "1100"))
kv = KVCacheManager(cfg.n_layers, B * ((CTX + 200) // 16 + 2) + 16, cfg.n_kv_heads, cfg.head_dim, 16, max(4, B), (CTX + 200) // 16 + 2)
r = ModelRunner(w, kv)
seqs = [kv.allocate(CTX + 100) for _ in range(B)]
orig = {n: getattr(K, n) for n in ("attn_decode_step", "gemv_rmsnorm", "linear", "argmax")}
wo = {id(l.wo) for l in w.layers}
wd = {id(l.wd) for l in w.layers}
wqkv = {id(l.wqkv) for l in w.layers}
wgu = {id(l.wgu) for l in w.layers}


def skip_linear(ids):
    def f(x, wt, *a, **k):
        if id(wt) in ids:
            return k.get("out")
        return orig["linear"](x, wt, *a, **k)
    return f


def skip_norm_gemv(ids):
    def f(x, nw, eps, wt, *a, **k):
        if id(wt) in ids:
            return k.get("out")
        return orig["gemv_rmsnorm"](x, nw, eps, wt, *a, **k)
    return f


variants = {
    "full": {},
    "no_attention": {"attn_decode_step": lambda *a, **k: k.get("out")},
    "no_o_proj": {"linear": skip_linear(wo)},
    "no_down_proj": {"linear": skip_linear(wd)},
    "no_qkv": {"gemv_rmsnorm": skip_norm_gemv(wqkv)},
    "no_gate_up": {"gemv_rmsnorm": skip_norm_gemv(wgu)},
}


def step_ms():
    r.graphs.clear()
    g = r.decode_graph(B, CTX + 100, 64)
    g.load(seqs, [1] * B, [CTX] * B)
    g.capture()
    res = []
    for _ in range(5):
        g.load(seqs, [1] * B, [CTX] * B)
        s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        torch.cuda.synchronize(); s.record()
        for _ in range(20):
            g.replay()
        e.record(); torch.cuda.synchronize()
        res.append(s.elapsed_time(e) / 20)
    return min(res), g.launches_per_step


out = {"model": cfg.name, "B": B, "ctx": CTX}
for name, patch in variants.items():
    for n, f in orig.items():
        setattr(K, n, f)
    for n, f in patch.items():
        setattr(K, n, f)
    ms, launches = step_ms()
    out[name] = {"step_ms": round(ms, 4), "launches": launches}
for n, f in orig.items():
    setattr(K, n, f)
full = out["full"]["step_ms"]
out["marginal_us_per_layer"] = {k[3:]: round((full - v["step_ms"]) * 1e3 / cfg.n_layers, 2)
                                for k, v in out.items() if isinstance(v, dict) and k.startswith("no_")}
print(json.dumps(out))
