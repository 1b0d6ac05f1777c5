"""TP all-reduce at prefill / decode sizes: peer-memory kernel (tpcomm) vs
NCCL, fp32 sum, CUDA-event timed (run under torchrun, 2 or 4 ranks)."""
import json, os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import torch.distributed as dist
from paper_2311_18677_b200.tpcomm import TPComm

rank, world = int(os.environ["RANK"]), int(os.environ["WORLD_SIZE"])
torch.cuda.set_device(rank)
dist.init_process_group("nccl", device_id=torch.device("cuda", rank))
res = {}
c = TPComm(dist.group.WORLD, 2048 * 8192 * 4)
for rows in (1, 8, 1024, 1500, 2048):
    n = rows * 8192
    x = torch.empty(n, device="cuda")
    ev = lambda: torch.cuda.Event(enable_timing=True)  # noqa: E731
    for name in ("peer", "nccl"):
        def f():
            if name == "peer":
                s = c.next_slot()
                c.slot(s, (n,)).fill_(1.0)
                c.allreduce(s, x)
            else:
                x.fill_(1.0)
                dist.all_reduce(x)
        for _ in range(3):
            f()
        torch.cuda.synchronize(); dist.barrier()
        a, b = ev(), ev()
        a.record()
        for _ in range(20):
            f()
        b.record(); torch.cuda.synchronize()
        us = a.elapsed_time(b) / 20 * 1e3
        res[f"{name}_rows{rows}_us"] = round(us, 1)
if rank == 0:
    print(json.dumps({"world": world, **res}))
dist.barrier()
os._exit(0)
