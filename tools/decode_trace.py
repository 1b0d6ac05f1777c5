"""Phase timeline of the one-launch decode step (CTA 0 timestamps at every
grid barrier: arrive / release), 7B B=1 ctx~1100."""
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
for _ in range(3):
    g.replay()
torch.cuda.synchronize()
import numpy as np
tr = np.frombuffer(g.mega_ws[:2048 * 8].cpu().numpy().tobytes(), dtype=np.uint64)
n = 5 * cfg.n_layers + 2
ts = tr[1:2 * n]
t0 = int(tr[1])
names = ["P0"] + [f"L{l}{ph}" for l in range(cfg.n_layers) for ph in "ABCDE"] + ["F"]
# phase k runs from release of barrier k (index 2k-1) to arrival at barrier k+1 (index 2k)
dur = {}
for k in range(1, n):
    start = int(tr[2 * k - 1]); arrive = int(tr[2 * k]); rel = int(tr[2 * k + 1]) if 2 * k + 1 < len(tr) else arrive
    ph = names[k] if k < len(names) else f"x{k}"
    dur[ph] = ((arrive - start) / 1e3, (rel - arrive) / 1e3)
tot = {p: 0.0 for p in "ABCDE"}
bw = {p: 0.0 for p in "ABCDE"}
for k, (work, wait) in dur.items():
    if k.startswith("L"):
        tot[k[-1]] += work; bw[k[-1]] += wait
att = [[(int(tr[1024 + l * 8 + k]) - int(tr[1024 + l * 8])) / 1e3 for k in range(8)] for l in range(3)]
print("attention CTA0 marks (us from phase start: issued, landed, computed, pre-merge, done, after-rope, item-start):", att)
print(json.dumps({"phase_work_us_total": tot, "barrier_wait_us_total": bw,
                  "layer0": {k: v for k, v in dur.items() if k.startswith("L0")},
                  "F": dur.get("F"), "step_us": (int(tr[2 * n - 1]) - int(tr[1])) / 1e3 if len(tr) > 2 * n else None}, indent=1))
