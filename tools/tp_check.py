"""Tensor-parallel pool check (run with torchrun, 2 or 4 GPUs):

  python -m torch.distributed.run --nproc-per-node 2 --master-addr 127.0.0.1 \
      --master-port 29533 tools/tp_check.py [--model tiny] [--prompt 300 --out 16]

Every rank holds one TP shard (heads and FFN columns split, NCCL all-reduce
after the O and down projections).  Rank 0 gathers the shards, rebuilds the
logical single-GPU model and checks that the TP pool's greedy tokens equal
the TP=1 run and that logits agree within the bf16 tolerance; with --time it
also reports per-GPU prefill and decode-step times (e.g. llama2-70b TP2)."""

import argparse
import json
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import torch
import torch.distributed as dist

from paper_2311_18677_b200 import kernels as K
from paper_2311_18677_b200.kvcache import KVCacheManager
from paper_2311_18677_b200.model import LayerWeights, Weights, get_config, init_weights
from paper_2311_18677_b200.runner import ModelRunner


def run(runner, kv, prompt, n_out):
    P = len(prompt)
    seq = kv.allocate(P + n_out)
    toks = torch.tensor(prompt, dtype=torch.int32, device="cuda")
    slots = torch.empty(P, dtype=torch.int32, device="cuda")
    K.slots_from_table(kv.table_row_ptr(seq), 0, P, kv.block_size, slots)
    first = runner.prefill(toks, [P], ModelRunner.pack_meta([P]).cuda(), local_slots=slots)
    logits = [runner.plogits[0].clone()]
    g = runner.decode_graph(1, P + n_out, n_out)
    g.load([seq], first[:1], [P])
    g.capture()
    for _ in range(n_out - 1):
        g.replay()
        logits.append(g.logits[0].clone())
    torch.cuda.synchronize()
    toks_out = [int(first[0])] + g.out_ring[0, :n_out - 1].tolist()
    kv.release(seq)
    return toks_out, torch.stack(logits)


def time_phases(runner, kv, P, reps=5, batch=1):
    cfg = runner.cfg
    seq = kv.allocate(P + 64)
    extra = [kv.allocate(P + 64) for _ in range(batch - 1)]
    toks = torch.randint(0, cfg.vocab, (P,), dtype=torch.int32, device="cuda")
    slots = torch.empty(P, dtype=torch.int32, device="cuda")
    K.slots_from_table(kv.table_row_ptr(seq), 0, P, kv.block_size, slots)
    meta = ModelRunner.pack_meta([P]).cuda()
    ev = lambda: torch.cuda.Event(enable_timing=True)  # noqa: E731
    pre = []
    for _ in range(reps):
        a, b = ev(), ev()
        dist.barrier()
        a.record()
        first = runner.prefill(toks, [P], meta, local_slots=slots)
        b.record()
        torch.cuda.synchronize()
        pre.append(a.elapsed_time(b))
    g = runner.decode_graph(batch, P + 64, 64)
    g.load([seq] + extra, [int(first[0])] * batch, [P] * batch)
    g.capture()
    a, b = ev(), ev()
    dist.barrier()
    a.record()
    for _ in range(32):
        g.replay()
    b.record()
    torch.cuda.synchronize()
    kv.release(seq)
    for s_ in extra:
        kv.release(s_)
    return min(pre), a.elapsed_time(b) / 32


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--model", default="tiny")
    ap.add_argument("--prompt", type=int, default=300)
    ap.add_argument("--out", type=int, default=16)
    ap.add_argument("--time", action="store_true")
    ap.add_argument("--batch", type=int, default=1)
    ap.add_argument("--no-ar", action="store_true",
                    help="timing only: skip the TP all-reduces (wrong numerics)")
    a = ap.parse_args()
    rank, world = int(os.environ["RANK"]), int(os.environ["WORLD_SIZE"])
    torch.cuda.set_device(int(os.environ.get("LOCAL_RANK", rank)))
    dist.init_process_group("nccl", device_id=torch.device("cuda", torch.cuda.current_device()))
    cfg = get_config(a.model)
    w = init_weights(cfg, seed=0, tp=world, rank=rank)
    kv = KVCacheManager(cfg.n_layers, 1024, cfg.n_kv_heads // world, cfg.head_dim, 16, max(4, a.batch),
                        (a.prompt + 128) // 16 + 2)
    runner = ModelRunner(w, kv, tp_group=dist.group.WORLD)
    if a.no_ar:
        runner._allreduce = lambda x: None
    prompt = torch.randint(0, cfg.vocab, (a.prompt,), generator=torch.Generator().manual_seed(3)).tolist()
    if a.time:
        pre, dec = time_phases(runner, kv, a.prompt, batch=a.batch)
        t = torch.tensor([pre, dec], device="cuda")
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        if rank == 0:
            print(json.dumps({"model": cfg.name, "tp": world, "prompt": a.prompt,
                              "batch": a.batch, "allreduce": not a.no_ar,
                              "prefill_ms": t[0].item(), "decode_step_ms": t[1].item(),
                              "prefill_tflops_per_gpu": cfg.prefill_flops(a.prompt, world) /
                              t[0].item() / 1e9,
                              "decode_GBps_per_gpu": cfg.decode_bytes([a.prompt + 32] * a.batch, world) /
                              t[1].item() / 1e6}))
        dist.destroy_process_group()
        return
    toks_tp, logits_tp = run(runner, kv, prompt, a.out)
    # gather shards and rebuild the logical TP=1 model on rank 0
    hq, hkv, dh = cfg.n_heads // world, cfg.n_kv_heads // world, cfg.head_dim
    layers = []
    names = ("wqkv", "wo", "wgu", "wd") + (("bqkv", "bup") if cfg.is_bloom else ())

    def unshard_qkv(parts):
        q = torch.cat([p[:hq * dh] for p in parts])
        k = torch.cat([p[hq * dh:(hq + hkv) * dh] for p in parts])
        v = torch.cat([p[(hq + hkv) * dh:] for p in parts])
        return torch.cat([q, k, v]).contiguous()
    for lw in w.layers:
        parts = {}
        for name in names:
            t = getattr(lw, name).contiguous()
            lst = [torch.empty_like(t) for _ in range(world)]
            dist.all_gather(lst, t)
            parts[name] = lst
        if rank == 0:
            full_lw = LayerWeights(lw.attn_norm, unshard_qkv(parts["wqkv"]),
                                   torch.cat(parts["wo"], 1).contiguous(), lw.mlp_norm,
                                   torch.cat(parts["wgu"]).contiguous(),
                                   torch.cat(parts["wd"], 1).contiguous())
            if cfg.is_bloom:
                full_lw.attn_norm_b, full_lw.mlp_norm_b = lw.attn_norm_b, lw.mlp_norm_b
                full_lw.bqkv = unshard_qkv(parts["bqkv"])
                full_lw.bup = torch.cat(parts["bup"]).contiguous()
                full_lw.bo, full_lw.bd = lw.bo, lw.bd
            layers.append(full_lw)
    if rank == 0:
        extra = {}
        if cfg.is_bloom:
            from paper_2311_18677_b200.model import alibi_slopes
            extra = dict(final_norm_b=w.final_norm_b, emb_norm=w.emb_norm,
                         emb_norm_b=w.emb_norm_b,
                         alibi=torch.tensor(alibi_slopes(cfg.n_heads), device="cuda"))
        full = Weights(cfg, 1, 0, w.embed, w.lm_head, w.final_norm, layers, **extra)
        kv1 = KVCacheManager(cfg.n_layers, 1024, cfg.n_kv_heads, cfg.head_dim, 16, 4,
                             (a.prompt + 128) // 16 + 2)
        toks_1, logits_1 = run(ModelRunner(full, kv1), kv1, prompt, a.out)
        if logits_tp.shape[-1] != logits_1.shape[-1]:   # vocab-parallel head: rank 0's shard
            logits_1 = logits_1[..., :logits_tp.shape[-1]]
        d = (logits_tp - logits_1).abs().max().item()
        scale = logits_1.abs().max().item()
        ok = toks_tp == toks_1 and d <= 0.03 + 0.02 * scale
        print(json.dumps({"model": cfg.name, "tp": world, "tokens_equal": toks_tp == toks_1,
                          "max_dlogit": d, "logit_scale": scale, "ok": ok}))
        if not ok:
            sys.exit(1)
    dist.barrier()
    dist.destroy_process_group()
    _ = time


if __name__ == "__main__":
    main()
