"""Worker of tests/test_ipc_pair_gpu.py: a Splitwise pair as TWO processes on
ONE GPU — the real cross-process path (CUDA-IPC mapping of the token pool,
hand-off records written by the prompt GPU into the token host's shared
table) without needing a second GPU.  Nothing here waits on the device for
another process: the token host polls host memory.

rank 1 = token machine (owns the pool), rank 0 = prompt machine.
Phase 1: single requests of the lengths in CASES, pushed into reserved
         pages; the token side checks the block table against the CPU
         lowest-free-first allocator, the pushed K/V bit-for-bit against a
         co-located prefill of the same prompt, and decodes from the pushed
         KV: tokens equal the co-located run's; for the tiny model the
         teacher-forced logits are checked against the fp32 oracle.
Phase 2: PromptServer.serve_burst / TokenServer.serve_burst (the bench's
         path) on three requests; generated tokens equal co-located runs.
"""

from __future__ import annotations

import dataclasses
import json
import os
import sys
import time

import torch
import torch.distributed as dist

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def _cfg(model):
    from paper_2311_18677_b200.model import get_config
    if model == "tiny":
        return get_config("tiny")
    return dataclasses.replace(get_config(model), n_layers=2, name=f"{model}-2L")


def colocated(w, prompt, n_out, want_logits=False):
    """Reference run on a private pool of this process: (tokens, K pages,
    V pages, logits)."""
    from paper_2311_18677_b200 import kernels as K
    from paper_2311_18677_b200.kvcache import KVCacheManager
    from paper_2311_18677_b200.runner import ModelRunner
    cfg = w.cfg
    P = len(prompt)
    nb = (P + n_out + 15) // 16 + 2
    kv = KVCacheManager(cfg.n_layers, nb, cfg.n_kv_heads, cfg.head_dim, 16, 2, nb)
    r = ModelRunner(w, kv)
    seq = kv.allocate(P + n_out)
    toks = torch.tensor(prompt, dtype=torch.int32, device="cuda")
    slots = torch.empty(P, dtype=torch.int32, device="cuda")
    K.slots_from_table(kv.table_row_ptr(seq), 0, P, 16, slots)
    first = r.prefill(toks, [P], ModelRunner.pack_meta([P]).cuda(), local_slots=slots)
    torch.cuda.synchronize()
    pages = gather(kv, seq, P)
    out, logits = decode(r, kv, seq, int(first[0]), P, n_out, want_logits)
    if want_logits:
        logits.insert(0, r.plogits[0].clone().cpu())
    return out, pages, logits


def colocated_batch(w, prompts, n_out):
    """The burst as ONE co-located prefill batch + one B=len(prompts) decode
    graph — the schedule the pair runs (the prompt machine batches all three,
    the token machine admits the landed group together)."""
    from paper_2311_18677_b200 import kernels as K
    from paper_2311_18677_b200.kvcache import KVCacheManager
    from paper_2311_18677_b200.runner import ModelRunner
    cfg = w.cfg
    lens = [len(p) for p in prompts]
    nb = sum((n + n_out + 15) // 16 for n in lens) + 4
    kv = KVCacheManager(cfg.n_layers, nb, cfg.n_kv_heads, cfg.head_dim, 16, len(prompts), nb)
    r = ModelRunner(w, kv)
    seqs = [kv.allocate(n + n_out) for n in lens]
    toks = torch.tensor(sum(prompts, []), dtype=torch.int32, device="cuda")
    slots = torch.empty(sum(lens), dtype=torch.int32, device="cuda")
    off = 0
    for sq, n in zip(seqs, lens):
        K.slots_from_table(kv.table_row_ptr(sq), 0, n, 16, slots[off:off + n])
        off += n
    first = r.prefill(toks, lens, ModelRunner.pack_meta(lens).cuda(), local_slots=slots)
    # the token server's context bucket (TokenServer._graph_for): same
    # attention partitioning, so the same split-K merge order
    need = max(lens) + n_out
    g = r.decode_graph(len(prompts), 2048 * ((need + 2047) // 2048), n_out)
    g.load(seqs, first[:len(prompts)], lens)
    g.capture()
    for _ in range(n_out - 1):
        g.replay()
    torch.cuda.synchronize()
    return [[int(first[b])] + g.out_ring[b, :n_out - 1].tolist() for b in range(len(prompts))]


def gather(kv, seq, P):
    tb = kv.tables()[seq].long()
    p = torch.arange(P, device="cuda")
    return [(kv.k_view(li)[tb[p // 16], :, p % 16].clone(),
             kv.v_view(li)[tb[p // 16], :, p % 16].clone()) for li in range(kv.num_layers)]


def decode(runner, kv, seq, first, P, n_out, want_logits=False):
    g = runner.decode_graph(1, P + n_out, n_out)
    g.load([seq], [first], [P])
    g.capture()
    logits = []
    for _ in range(n_out - 1):
        g.replay()
        if want_logits:
            logits.append(g.logits[0].clone().cpu())
    torch.cuda.synchronize()
    return [first] + g.out_ring[0, :n_out - 1].tolist(), logits


def main(rank, port, model, out_path, cases):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=2)
    torch.cuda.set_device(0)
    from oracle.decoder import LowestFreeAllocator
    from paper_2311_18677_b200.control import recv_reservations, send_reservations
    from paper_2311_18677_b200.kvcache import KVCacheManager
    from paper_2311_18677_b200.model import init_weights
    from paper_2311_18677_b200.runner import ModelRunner
    from paper_2311_18677_b200.splitwise import PromptServer, TokenServer
    from paper_2311_18677_b200.workers import SchedulerConfig
    cfg = _cfg(model)
    w = init_weights(cfg, seed=0)
    n_out = 12
    gen = torch.Generator().manual_seed(3)
    prompts = [torch.randint(0, cfg.vocab, (n,), generator=gen).tolist() for n in cases]
    burst = [torch.randint(0, cfg.vocab, (n,), generator=gen).tolist()
             for n in (min(cases[-1], 200), 45, 97)]
    NB = 1024
    if rank == 1:
        kv = KVCacheManager(cfg.n_layers, NB, cfg.n_kv_heads, cfg.head_dim, 16, 8, 128)
        runner = ModelRunner(w, kv)
        server = TokenServer(runner, None, 0, SchedulerConfig(), machine_id=0, prompt_machines=1)
        cpu = LowestFreeAllocator(NB)
        pad = kv.allocate(100)              # non-trivial tables
        cpu.alloc(7)
        dist.send_object_list([kv.ipc_handle(), server.table.name, server.res_boxes[0].name],
                              dst=0)
        res = {"cases": []}
        for P, prompt in zip(cases, prompts):
            seq, ep = server._reserve(P + n_out)
            want_table = cpu.alloc((P + n_out + 15) // 16)
            torch.cuda.synchronize()
            send_reservations([seq], 0, None, [ep])
            server.watch.expect(0, seq, ep, P, n_out)
            t0 = time.perf_counter()
            rows = []
            while not rows:
                rows = server.watch.poll()
                if time.perf_counter() - t0 > 120:
                    raise TimeoutError("hand-off never landed")
            (_rid, _seq, _plen, first, _n), = rows
            table = kv.tables()[seq, :len(want_table)].tolist()
            pushed = gather(kv, seq, P)
            ref_toks, ref_pages, ref_logits = colocated(w, prompt, n_out,
                                                        want_logits=(model == "tiny"))
            kv_exact = all(torch.equal(a.view(torch.int16), b.view(torch.int16))
                           for (ka, va), (kb, vb) in zip(pushed, ref_pages)
                           for a, b in ((ka, kb), (va, vb)))
            toks, logits = decode(runner, kv, seq, first, P, n_out, want_logits=(model == "tiny"))
            case = {"P": P, "table_ok": table == want_table, "kv_exact": kv_exact,
                    "first": first, "tokens": toks, "colocated_tokens": ref_toks}
            if model == "tiny":
                from oracle.decoder import OracleDecoder
                orc = OracleDecoder.from_weights(w)
                _, ol = orc.generate(prompt, n_out, forced=toks[:-1])
                logits.insert(0, ref_logits[0])
                case["max_dlogit_vs_oracle"] = float((torch.stack(logits) - ol).abs().max())
                case["max_logit"] = float(ol.abs().max())
            kv.release(seq)
            cpu.free(want_table)
            res["cases"].append(case)
        dist.barrier()
        # phase 2: the bench's serve_burst path
        reqs = [(100 + i, torch.tensor(p, dtype=torch.int32), n_out) for i, p in enumerate(burst)]
        emit, tokens, first_seen = server.serve_burst(reqs, time.perf_counter())
        ref = colocated_batch(w, burst, n_out)
        res["burst"] = [{"rid": rid, "tokens": tokens[rid], "colocated": ref[i],
                         "emitted": len(emit[rid]), "first_seen": rid in first_seen}
                        for i, (rid, _, _) in enumerate(reqs)]
        res["burst_steps"] = [b for b, _, _ in server.step_log]
        kv.release(pad)
        server.close()
        with open(out_path, "w") as f:
            json.dump(res, f)
    else:
        handle = [None, None, None]
        dist.recv_object_list(handle, src=1)
        peer = KVCacheManager.open_peer(handle[0])
        runner = ModelRunner(w, None)
        server = PromptServer(runner, {0: peer}, None, 1, SchedulerConfig(), {0: handle[1]},
                              machine_id=0, res_boxes={0: handle[2]})
        modes = []
        for P, prompt in zip(cases, prompts):
            (seq,), (ep,) = recv_reservations(1, 1, None, with_epochs=True)
            toks = torch.tensor(prompt, dtype=torch.int32, device="cuda")
            server._run_batch([(0, prompt, n_out)], {0: (0, seq, ep)}, toks)
            modes.append(server.push_log[-1].mode)
        runner.finish_push_stats(block=True)
        dist.barrier()
        reqs = [(100 + i, torch.tensor(p, dtype=torch.int32), n_out) for i, p in enumerate(burst)]
        server.serve_burst(reqs, time.perf_counter())
        server.close()
        with open(out_path + ".prompt", "w") as f:
            json.dump({"modes": modes}, f)
    dist.barrier()
    dist.destroy_process_group()


if __name__ == "__main__":
    main(int(sys.argv[1]), int(sys.argv[2]), sys.argv[3], sys.argv[4],
         [int(x) for x in sys.argv[5].split(",")])
