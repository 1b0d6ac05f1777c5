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


def _fused_worker(rank, world, port, q):
    """Fused projection + all-reduce (swb_gemv_bf16_tp pushes the partial from
    its epilogue; swb_tp_allreduce_recv_f32 waits and sums) equals the
    two-kernel form bit for bit, eagerly and inside replayed CUDA graphs, with
    the slots alternating between fused and unfused uses.  Both forms on the
    same streaming GEMV (one-row GEMVs outside the fused push would
    otherwise go to the mma.sync kernel, whose sums round differently)."""
    sys.path.insert(0, ROOT)
    os.environ["SWB_GEMV_M1_MMA"] = "0"
    import torch.distributed as dist
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    torch.cuda.set_device(rank)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        from paper_2311_18677_b200 import kernels as K
        from paper_2311_18677_b200.tpcomm import TPComm
        comm = TPComm(dist.group.WORLD, 64 * 8192 * 4)
        N, Kd = 8192, 2048
        g = torch.Generator(device="cuda").manual_seed(11 + rank)
        w = (torch.randn(N, Kd, device="cuda", generator=g) * 0.02).bfloat16()
        x = torch.randn(1, Kd, device="cuda", generator=g).bfloat16()
        resid = torch.randn(1, N, device="cuda", generator=torch.Generator(device="cuda")
                            .manual_seed(999))
        epi = K.EPI_RESID_F32 if rank == 0 else K.EPI_F32
        errs = []

        def fused(out):
            s = comm.next_slot()
            K.gemv_tp(x, w, epi, comm._h, s, resid=resid if rank == 0 else None)
            comm.allreduce_recv(s, out)

        def plain(out):
            s = comm.next_slot()
            K.linear(x, w, epi, out=comm.slot(s, (1, N)), resid=resid)
            comm.allreduce(s, out)
        for it in range(6):
            a, b = torch.empty(1, N, device="cuda"), torch.empty(1, N, device="cuda")
            fused(a)
            plain(b)
            torch.cuda.synchronize()
            if not torch.equal(a, b):
                errs.append(("eager", it, (a - b).abs().max().item()))
        ref = b.clone()
        outs = torch.empty(2, 1, N, device="cuda")

        def body():
            comm.reset()
            fused(outs[0])
            fused(outs[1])
        body()
        torch.cuda.synchronize()
        gr = torch.cuda.CUDAGraph()
        with torch.cuda.graph(gr):
            body()
        for rep in range(5):
            outs.zero_()
            dist.barrier()
            gr.replay()
            torch.cuda.synchronize()
            if not (torch.equal(outs[0], ref) and torch.equal(outs[1], ref)):
                errs.append(("graph", rep))
        comm.close()
        q.put((rank, errs))
    finally:
        dist.destroy_process_group()


@pytest.mark.skipif(torch.cuda.device_count() < 2, reason="needs >= 2 GPUs")
def test_fused_projection_allreduce_exact():
    world = min(4, torch.cuda.device_count())
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_fused_worker, args=(r, world, port, q)) for r in range(world)]
    for p in procs:
        p.start()
    res = [q.get(timeout=300) for _ in range(world)]
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    for rank, errs in res:
        assert errs == [], (rank, errs)


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


_BIG = {"SWB_TP_AR_NCCL_BYTES": "65536"}


@pytest.mark.skipif(torch.cuda.device_count() < 2, reason="needs >= 2 GPUs")
@pytest.mark.parametrize("model,env,args", [
    ("tiny", {}, []), ("tiny", _BIG, []),
    ("tiny", {**_BIG, "SWB_TP_STAGE_CHUNKS": "1"}, ["--prompt", "600"]),
    ("tiny", {**_BIG, "SWB_TP_STAGE": "0"}, []), ("bloom-tiny", _BIG, [])])
def test_tp2_tiny_matches_tp1(model, env, args):
    """TP=2 pool == TP=1 tokens; with a 64 KB threshold the tiny prefill's
    reductions take the production prefill path — bf16 partials exchanged
    by the copy engines (projections in 2 row chunks, or 1) and added to the fp32
    residual inside the next norm, or with SWB_TP_STAGE=0 all-reduced by
    NCCL — while decode keeps the peer all-reduce, as at full size."""
    import subprocess
    port = _free_port()
    r = subprocess.run([sys.executable, "-m", "torch.distributed.run", "--nproc-per-node", "2",
                        "--master-addr", "127.0.0.1", "--master-port", str(port),
                        os.path.join(ROOT, "tools", "tp_check.py"), "--model", model, *args],
                       capture_output=True, text=True, timeout=600, cwd=ROOT,
                       env={**os.environ, **env})
    assert r.returncode == 0, r.stdout[-2000:] + r.stderr[-2000:]
    assert '"ok": true' in r.stdout


@pytest.mark.skipif(torch.cuda.device_count() < 4, reason="needs >= 4 GPUs")
@pytest.mark.parametrize("model,env,args", [
    ("tiny-tp4", {}, []), ("bloom-tiny-tp4", {**_BIG, "SWB_TP_STAGE": "1"}, []),
    ("tiny-tp4", {**_BIG, "SWB_TP_STAGE": "1", "SWB_TP_STAGE_CHUNKS": "2"}, ["--prompt", "600"]),
    ("tiny-tp4", _BIG, [])])
def test_tp4_pool_matches_tp1(model, env, args):
    """A TP=4 pool (push all-reduce for decode; prefill sizes through NCCL's
    bf16 all-reduce, or the copy-engine exchange forced with SWB_TP_STAGE=1)
    generates the TP=1 tokens, logits within tolerance."""
    import subprocess
    port = _free_port()
    r = subprocess.run([sys.executable, "-m", "torch.distributed.run", "--nproc-per-node", "4",
                        "--master-addr", "127.0.0.1", "--master-port", str(port),
                        os.path.join(ROOT, "tools", "tp_check.py"), "--model", model, *args],
                       capture_output=True, text=True, timeout=600, cwd=ROOT,
                       env={**os.environ, **env})
    assert r.returncode == 0, r.stdout[-2000:] + r.stderr[-2000:]
    assert '"ok": true' in r.stdout


@pytest.mark.skipif(torch.cuda.device_count() < 2, reason="needs >= 2 GPUs")
def test_realtime_trace_serving_one_pair(tmp_path):
    """bench.py --trace: a Splitwise pair (2 processes) serves a short
    reference-preset trace in real time; every request completes, the JSON
    line carries TTFT / TBT percentiles, and the tokens generated through
    the cross-process push + device hand-off + continuous batching are the
    fp32 oracle's greedy tokens wherever its top-2 margin is decisive."""
    import json
    import subprocess
    port = _free_port()
    dump = str(tmp_path / "tokens.json")
    r = subprocess.run([sys.executable, "-m", "torch.distributed.run", "--nproc-per-node", "2",
                        "--master-addr", "127.0.0.1", "--master-port", str(port),
                        os.path.join(ROOT, "bench.py"), "--gpus", "2", "--model", "tiny",
                        "--warmup", "1", "--prompt", "128", "--out", "8", "--trace",
                        "conversation", "--rate", "20", "--duration", "2", "--max-output", "24",
                        "--dump-tokens", dump],
                       capture_output=True, text=True, timeout=600, cwd=ROOT)
    assert r.returncode == 0, r.stdout[-2000:] + r.stderr[-2000:]
    line = json.loads([ln for ln in r.stdout.splitlines() if ln.startswith("{")][-1])
    assert line["requests"] > 10 and line["ttft_ms"]["p50"] > 0 and line["tbt_ms"]["p99"] > 0
    assert line["output_tokens"] >= line["requests"]
    # the same trace and prompts bench.py built (reference generator, seed 77 prompts)
    sys.path.insert(0, os.path.join(ROOT, "tools"))
    from oracle.decoder import OracleDecoder
    from paper_2311_18677_b200.model import get_config, init_weights
    from reftrace import preset_trace
    reqs = preset_trace("conversation", 20.0, 2.0, 0)
    cfg = get_config("tiny")
    g = torch.Generator().manual_seed(77)
    prompts = {q.id: torch.randint(0, cfg.vocab, (q.prompt_tokens,), generator=g,
                                   dtype=torch.int32) for q in reqs}
    got = {int(k): v for k, v in json.load(open(dump)).items()}
    assert len(got) == len(reqs)
    orc = OracleDecoder.from_weights(init_weights(cfg, seed=0))
    for q in sorted(reqs, key=lambda q: q.prompt_tokens)[:4]:
        toks = got[q.id]
        assert len(toks) == min(q.output_tokens, 24)
        ref_toks, ref_logits = orc.generate(prompts[q.id].tolist(), len(toks), forced=toks[:-1])
        top2 = ref_logits.topk(2, -1).values
        for i, dec in enumerate(((top2[:, 0] - top2[:, 1]) > 0.02).tolist()):
            if dec:
                assert toks[i] == ref_toks[i], (q.id, i)


@pytest.mark.skipif(torch.cuda.device_count() < 4, reason="needs >= 4 GPUs")
def test_realtime_trace_serving_two_pairs_jsq():
    """bench.py --trace on two Splitwise pairs with live JSQ routing
    (control.RouteBoard): every request is routed once and completes."""
    import json
    import subprocess
    port = _free_port()
    r = subprocess.run([sys.executable, "-m", "torch.distributed.run", "--nproc-per-node", "4",
                        "--master-addr", "127.0.0.1", "--master-port", str(port),
                        os.path.join(ROOT, "bench.py"), "--gpus", "4", "--model", "tiny",
                        "--warmup", "1", "--prompt", "128", "--out", "8", "--trace",
                        "conversation", "--rate", "40", "--duration", "2", "--max-output", "24",
                        "--route", "jsq"],
                       capture_output=True, text=True, timeout=600, cwd=ROOT)
    assert r.returncode == 0, r.stdout[-2000:] + r.stderr[-2000:]
    line = json.loads([ln for ln in r.stdout.splitlines() if ln.startswith("{")][-1])
    assert line["config"]["routing"] == "jsq"
    assert line["requests"] > 20 and line["output_tokens"] >= line["requests"]


def test_vocab_parallel_pick_equals_full_argmax():
    """swb_argmax_shard over TP vocabulary shards + a summed candidate table +
    swb_argmax_pick == swb_argmax over the full vocabulary (ties included)."""
    from paper_2311_18677_b200 import kernels as K
    rows, V, tp = 5, 32000, 4
    logits = torch.randn(rows, V, device="cuda")
    logits[1, 7] = logits[1, 16007] = 100.0          # tie across shards: lowest index wins
    Vs = V // tp
    total = torch.zeros(rows, tp, 2, device="cuda")
    for r in range(tp):
        cand = torch.full((rows, tp, 2), float("nan"), device="cuda")
        K.argmax_shard(logits[:, r * Vs:(r + 1) * Vs].contiguous(), r * Vs, r, tp, cand)
        total += cand
    got = torch.empty(rows, dtype=torch.int32, device="cuda")
    K.argmax_pick(total, rows, tp, got)
    want = torch.empty(rows, dtype=torch.int32, device="cuda")
    K.argmax(logits, out=want)
    assert got.tolist() == want.tolist()
    assert got[1].item() == 7
