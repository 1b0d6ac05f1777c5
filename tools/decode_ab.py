"""Device time of one decode step (CUDA graph, B=1, ctx~1100) of the 7B model
for the current environment (A/B switches: SWB_PDL, SWB_FUSED_NORM)."""
import os, sys, json
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from paper_2311_18677_b200.model import get_config, init_weights
from paper_2311_18677_b200.runner import ModelRunner
from paper_2311_18677_b200.kvcache import KVCacheManager
cfg = get_config(os.environ.get("MODEL", "llama2-7b"))
w = init_weights(cfg)
kv = KVCacheManager(cfg.n_layers, 512, cfg.n_kv_heads, cfg.head_dim, 16, 4, 128)
r = ModelRunner(w, kv)
B = int(os.environ.get("B", "1"))
seqs = [kv.allocate(1200) for _ in range(B)]
g = r.decode_graph(B, 1200, 64)
g.load(seqs, [1] * B, [1100] * B)
g.capture()
res = []
for rep in range(5):
    g.load(seqs, [1] * B, [1100] * B)
    s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    torch.cuda.synchronize(); s.record()
    for _ in range(20): g.replay()
    e.record(); torch.cuda.synchronize()
    res.append(s.elapsed_time(e) / 20)
print(json.dumps({"env": {k: os.environ.get(k) for k in ("SWB_PDL", "SWB_FUSED_NORM", "B")},
                  "step_ms": min(res), "launches_per_step": g.launches_per_step}))
