"""NVLink peer-memory TP all-reduce (tpcomm.py / swb_tp_allreduce_f32) on
>= 2 GPUs, one process per GPU: the result equals the rank-ordered fp32 sum
bit for bit on every rank, across alternating slots, sizes from one decode
row to a prefill batch, and inside a replayed CUDA graph; and a TP=2 tiny
model generates the same tokens as TP=1 (tools/tp_check.py semantics)."""

import os
import socket
import sys

import pytest
import torch
import torch.multiprocessing as mp

pytestmark = pytest.mark.gpu
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, q):
    sys.path.insert(0, ROOT)
    import torch.distributed as dist
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    torch.cuda.set_device(rank)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        from paper_2311_18677_b200.tpcomm import TPComm
        comm = TPComm(dist.group.WORLD, 1024 * 8192 * 4)
        errs = []
        for it, n in enumerate([8192, 4 * 8192, 1000 * 8192, 4, 8192 * 1024]):
            s = comm.next_slot()
            parts = [torch.randn(n, generator=torch.Generator().manual_seed(100 * it + r))
                     for r in range(world)]
            ref = parts[0].clone()
            for r in range(1, world):
                ref += parts[r]
            comm.slot(s, (n,)).copy_(parts[rank].cuda())
            out = torch.empty(n, device="cuda")
            comm.allreduce(s, out)
            torch.cuda.synchronize()
            if not torch.equal(out.cpu(), ref):
                errs.append(("eager", n, (out.cpu() - ref).abs().max().item()))
        # graph replay: two reductions per replay, inputs refreshed in between
        n = 4 * 8192
        src = torch.empty(2, n, device="cuda")
        outs = torch.empty(2, n, device="cuda")

        def body():
            comm.reset()
            for k in range(2):
                s = comm.next_slot()
                comm.slot(s, (n,)).copy_(src[k])
                comm.allreduce(s, outs[k])
        body()
        torch.cuda.synchronize()
        g = torch.cuda.CUDAGraph()
        with torch.cuda.graph(g):
            body()
        for rep in range(5):
            parts = [torch.randn(2, n, generator=torch.Generator().manual_seed(7 * rep + r))
                     for r in range(world)]
            ref = parts[0].clone()
            for r in range(1, world):
                ref += parts[r]
            src.copy_(parts[rank].cuda())
            dist.barrier()
            g.replay()
            torch.cuda.synchronize()
            if not torch.equal(outs.cpu(), ref):
                errs.append(("graph", rep, (outs.cpu() - ref).abs().max().item()))
        comm.close()
        q.put((rank, errs))
    finally:
        dist.destroy_process_group()


@pytest.mark.skipif(torch.cuda.device_count() < 2, reason="needs >= 2 GPUs")
def test_tp_allreduce_p2p_exact():
    world = min(4, torch.cuda.device_count())
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, q)) for r in range(world)]
    for p in procs:
        p.start()
    res = [q.get(timeout=300) for _ in range(world)]
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    for rank, errs in res:
        assert errs == [], (rank, errs)


@pytest.mark.skipif(torch.cuda.device_count() < 2, reason="needs >= 2 GPUs")
def test_tp2_tiny_matches_tp1():
    import subprocess
    port = _free_port()
    r = subprocess.run([sys.executable, "-m", "torch.distributed.run", "--nproc-per-node", "2",
                        "--master-addr", "127.0.0.1", "--master-port", str(port),
                        os.path.join(ROOT, "tools", "tp_check.py")],
                       capture_output=True, text=True, timeout=600, cwd=ROOT)
    assert r.returncode == 0, r.stdout[-2000:] + r.stderr[-2000:]
    assert '"ok": true' in r.stdout
