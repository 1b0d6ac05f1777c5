"""Fused projection + all-reduce push vs the two-kernel form (decode, one
row), CUDA-graph timed: (a) GEMV into the TP slot + push all-reduce kernel,
(b) swb_gemv_bf16_tp + receive kernel, (c)/(d) each GEMV alone.  Run under
torchrun with 2 or 4 ranks."""
import json, os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import torch.distributed as dist
from paper_2311_18677_b200 import kernels as K
from paper_2311_18677_b200.tpcomm import TPComm

rank, world = int(os.environ["RANK"]), int(os.environ["WORLD_SIZE"])
torch.cuda.set_device(rank)
dist.init_process_group("nccl", device_id=torch.device("cuda", rank))
comm = TPComm(dist.group.WORLD, 64 * 8192 * 4)
N, Kd = int(os.environ.get("N", "8192")), int(os.environ.get("KD", "2048"))
w = (torch.randn(N, Kd, device="cuda") * 0.02).bfloat16()
x = torch.randn(1, Kd, device="cuda").bfloat16()
out = torch.empty(1, N, device="cuda")
epi = K.EPI_F32


def plain():
    s = comm.next_slot()
    K.linear(x, w, epi, out=comm.slot(s, (1, N)))
    comm.allreduce(s, out)


def fused():
    s = comm.next_slot()
    K.gemv_tp(x, w, epi, comm._h, s)
    comm.allreduce_recv(s, out)


def gemv_tp_only():
    s = comm.next_slot()
    K.gemv_tp(x, w, epi, comm._h, s)


def gemv_only():
    K.linear(x, w, epi, out=out)


def timeit(body, reps=50):
    comm.reset()
    body(); body()
    torch.cuda.synchronize(); dist.barrier()
    g = torch.cuda.CUDAGraph()
    with torch.cuda.graph(g):
        comm.reset()
        for _ in range(reps):
            body()
    res = []
    for _ in range(5):
        dist.barrier()
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record(); g.replay(); b.record(); torch.cuda.synchronize()
        res.append(a.elapsed_time(b) * 1e3 / reps)
    t = torch.tensor([min(res)], device="cuda")
    dist.all_reduce(t, op=dist.ReduceOp.MAX)
    return round(t.item(), 2)


r = {"world": world, "N": N, "K": Kd, "plain_us": timeit(plain), "fused_us": timeit(fused),
     "gemv_only_us": timeit(gemv_only), "gemv_tp_only_us": timeit(gemv_tp_only)}
if rank == 0:
    print(json.dumps(r), flush=True)
dist.barrier()
dist.destroy_process_group()
