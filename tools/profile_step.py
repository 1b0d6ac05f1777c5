"""One prefill + a few decode steps of the bench workload, for ncu launch
lists (kept short so ncu's per-kernel replay stays bounded)."""
import argparse, os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from paper_2311_18677_b200 import kernels as K
from paper_2311_18677_b200.model import get_config, init_weights
from paper_2311_18677_b200.runner import ModelRunner
from paper_2311_18677_b200.kvcache import KVCacheManager

ap = argparse.ArgumentParser()
ap.add_argument("--model", default="llama2-7b")
ap.add_argument("--prompt", type=int, default=1024)
ap.add_argument("--steps", type=int, default=3)
ap.add_argument("--graph", type=int, default=1)
a = ap.parse_args()
cfg = get_config(a.model)
w = init_weights(cfg)
kv = KVCacheManager(cfg.n_layers, 1024, cfg.n_kv_heads, cfg.head_dim, 16, 4, 128)
r = ModelRunner(w, kv)
P, O = a.prompt, a.steps + 1
seq = kv.allocate(P + O)
toks = torch.randint(0, cfg.vocab, (P,), dtype=torch.int32, device="cuda")
meta = ModelRunner.pack_meta([P]).cuda()
slots = torch.empty(P, dtype=torch.int32, device="cuda")
K.slots_from_table(kv.table_row_ptr(seq), 0, P, 16, slots)
first = r.prefill(toks, [P], meta, local_slots=slots)
g = r.decode_graph(1, P + O, O)
g.load([seq], first[:1], [P])
if a.graph:
    g.capture()
for _ in range(a.steps):
    g.replay()
torch.cuda.synchronize()
print("ok", g.out_ring[0, :a.steps].tolist())
