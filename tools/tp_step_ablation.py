"""Marginal in-step cost of each part of a tensor-parallel decode step (run
under torchrun): the B=1 CUDA-graph step captured with one part removed —
attention, the O / down reductions (projection kept, no exchange), or one
projection — timed against the full step, max over ranks.  Timing only."""
import json, os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import torch.distributed as dist
from paper_2311_18677_b200 import kernels as K
from paper_2311_18677_b200.kvcache import KVCacheManager
from paper_2311_18677_b200.model import get_config, init_weights
from paper_2311_18677_b200.runner import ModelRunner

rank, world = int(os.environ["RANK"]), int(os.environ["WORLD_SIZE"])
torch.cuda.set_device(int(os.environ.get("LOCAL_RANK", rank)))
dist.init_process_group("nccl", device_id=torch.device("cuda", torch.cuda.current_device()))
cfg = get_config(os.environ.get("MODEL", "llama2-70b"))
CTX = int(os.environ.get("CTX", "1500"))
w = init_weights(cfg, seed=0, tp=world, rank=rank)
kv = KVCacheManager(cfg.n_layers, (CTX + 200) // 16 + 16, cfg.n_kv_heads // world, cfg.head_dim,
                    16, 4, (CTX + 200) // 16 + 2)
r = ModelRunner(w, kv, tp_group=dist.group.WORLD)
seq = kv.allocate(CTX + 100)
orig_attn, orig_proj = K.attn_decode_step, r._proj_reduce
wo = {id(l.wo) for l in w.layers}
wd = {id(l.wd) for l in w.layers}


def no_reduce(inp, wt, x, bias=None):
    K.linear(inp, wt, K.EPI_RESID_F32, out=x, resid=x)


def skip(ids):
    def f(inp, wt, x, bias=None):
        if id(wt) in ids:
            return
        orig_proj(inp, wt, x, bias)
    return f


variants = {"full": {}, "no_attention": {"attn": lambda *a, **k: k.get("out")},
            "no_reductions": {"proj": no_reduce}, "no_o_proj": {"proj": skip(wo)},
            "no_down_proj": {"proj": skip(wd)}}


def step_ms():
    r.graphs.clear()
    g = r.decode_graph(1, CTX + 100, 64)
    g.load([seq], [1], [CTX])
    g.capture()
    res = []
    for _ in range(5):
        g.load([seq], [1], [CTX])
        dist.barrier()
        s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        torch.cuda.synchronize(); s.record()
        for _ in range(20):
            g.replay()
        e.record(); torch.cuda.synchronize()
        res.append(s.elapsed_time(e) / 20)
    t = torch.tensor([min(res)], device="cuda")
    dist.all_reduce(t, op=dist.ReduceOp.MAX)
    return t.item()


out = {"model": cfg.name, "tp": world, "ctx": CTX}
for name, patch in variants.items():
    K.attn_decode_step = patch.get("attn", orig_attn)
    r._proj_reduce = patch.get("proj", orig_proj)
    out[name] = round(step_ms(), 4)
K.attn_decode_step, r._proj_reduce = orig_attn, orig_proj
out["marginal_us_per_layer"] = {k[3:]: round((out["full"] - v) * 1e3 / cfg.n_layers, 2)
                                for k, v in out.items() if k.startswith("no_")}
if rank == 0:
    print(json.dumps(out), flush=True)
dist.barrier()
dist.destroy_process_group()
