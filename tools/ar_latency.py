"""Latency of the decode-size TP all-reduce and its share of a TP decode step
(run under torchrun, 2 or 4 ranks):

  1. a CUDA graph of 100 back-to-back swb_tp_allreduce_f32 calls at decode
     message sizes (B * d fp32) -> us per all-reduce;
  2. the decode-graph step of a reduced-depth Llama-2-70B TP shard (16 layers,
     B=1) with the all-reduces as shipped vs replaced by the local projection
     alone (numerically wrong, timing only) -> the all-reduces' cost in the step.
"""
import dataclasses
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import torch.distributed as dist

from paper_2311_18677_b200 import kernels as K
from paper_2311_18677_b200.kvcache import KVCacheManager, blocks_for
from paper_2311_18677_b200.model import get_config, init_weights
from paper_2311_18677_b200.runner import ModelRunner
from paper_2311_18677_b200.tpcomm import TPComm

rank, world = int(os.environ["RANK"]), int(os.environ["WORLD_SIZE"])
torch.cuda.set_device(rank)
dist.init_process_group("nccl", device_id=torch.device("cuda", rank))
res = {"world": world}
ev = lambda: torch.cuda.Event(enable_timing=True)  # noqa: E731

c = TPComm(dist.group.WORLD, 64 * 16384 * 4)
for n in (8192, 14336, 8 * 8192, 32 * 8192):
    x = torch.empty(n, device="cuda")
    s = torch.cuda.Stream()
    g = torch.cuda.CUDAGraph()
    for p in (0, 1):
        c.slot(p, (n,)).fill_(1.0)
    torch.cuda.synchronize()
    with torch.cuda.stream(s):
        c.reset()
        for _ in range(4):
            c.allreduce(c.next_slot(), x)
        torch.cuda.synchronize()
        c.reset()
        with torch.cuda.graph(g, stream=s):
            for _ in range(100):
                c.allreduce(c.next_slot(), x)
    torch.cuda.synchronize()
    g.replay()
    torch.cuda.synchronize()
    dist.barrier()
    a, b = ev(), ev()
    a.record()
    for _ in range(5):
        g.replay()
    b.record()
    torch.cuda.synchronize()
    res[f"ar_chain_n{n}_us"] = round(a.elapsed_time(b) / 500 * 1e3, 2)
    if world == 2 or n < (1 << 18):   # the two-shot form rewrites the slots
        assert float(x[0]) == world, float(x[0])

cfg = dataclasses.replace(get_config(os.environ.get("MODEL", "llama2-70b")), n_layers=16)
w = init_weights(cfg, seed=0, tp=world, rank=rank)
ctx = 1100
kv = KVCacheManager(cfg.n_layers, 2 * blocks_for(ctx + 200, 16) + 64, cfg.n_kv_heads // world,
                    cfg.head_dim, 16, 4, blocks_for(ctx + 200, 16))
runner = ModelRunner(w, kv, tp_group=dist.group.WORLD)
seq = kv.allocate(ctx + 100)


def step_ms():
    g = runner.decode_graph(1, ctx + 100, 64)
    g.load([seq], [1], [ctx])
    g.capture()
    out = []
    for _ in range(3):
        g.load([seq], [1], [ctx])
        torch.cuda.synchronize()
        dist.barrier()
        a, b = ev(), ev()
        a.record()
        for _ in range(20):
            g.replay()
        b.record()
        torch.cuda.synchronize()
        out.append(a.elapsed_time(b) / 20)
    return min(out)


res["step16_ms"] = round(step_ms(), 4)
orig = ModelRunner._proj_reduce


def no_ar(self, inp, w, x, bias=None):
    K.linear(inp, w, K.EPI_RESID_F32, out=x, resid=x, bias=bias)


ModelRunner._proj_reduce = no_ar
res["step16_no_ar_ms"] = round(step_ms(), 4)
ModelRunner._proj_reduce = orig
res["ar_cost_per_call_us"] = round((res["step16_ms"] - res["step16_no_ar_ms"]) * 1e3 / 32, 2)
if rank == 0:
    print(json.dumps(res), flush=True)
dist.barrier()
os._exit(0)
