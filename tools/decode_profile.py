"""Decode steps (CUDA graph) of a model at batch B and context ~ctx, for ncu
launch lists and A/B timing.  Prints device ms/step over `reps` replays."""
import argparse, json, os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from paper_2311_18677_b200.model import get_config, init_weights
from paper_2311_18677_b200.runner import ModelRunner
from paper_2311_18677_b200.kvcache import KVCacheManager

ap = argparse.ArgumentParser()
ap.add_argument("--model", default="llama2-7b")
ap.add_argument("--B", type=int, nargs="+", default=[1])
ap.add_argument("--ctx", type=int, default=1100)
ap.add_argument("--reps", type=int, default=30)
a = ap.parse_args()
cfg = get_config(a.model)
w = init_weights(cfg)
maxb = max(a.B)
nblk = maxb * ((a.ctx + 200) // 16 + 1)
kv = KVCacheManager(cfg.n_layers, nblk, cfg.n_kv_heads, cfg.head_dim, 16, maxb, (a.ctx + 200) // 16 + 1)
r = ModelRunner(w, kv)
seqs = [kv.allocate(a.ctx + 100) for _ in range(maxb)]
for B in a.B:
    g = r.decode_graph(B, a.ctx + 100, 64)
    g.load(seqs[:B], [1] * B, [a.ctx] * B)
    g.capture()
    res = []
    for rep in range(3):
        g.load(seqs[:B], [1] * B, [a.ctx] * B)
        s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        torch.cuda.synchronize(); s.record()
        for _ in range(a.reps): g.replay()
        e.record(); torch.cuda.synchronize()
        res.append(s.elapsed_time(e) / a.reps)
    byts = cfg.decode_bytes([a.ctx] * B)
    ms = min(res)
    print(json.dumps({"model": cfg.name, "B": B, "ctx": a.ctx, "step_ms": ms,
                      "GBps": byts / ms / 1e6, "launches_per_step": g.launches_per_step}), flush=True)
