"""Layer-wise KV-push overhead on the prompt phase (verdict r1 item 4; the
paper reports the transfer overhead as < 7 % of prompt compute,
PAPER.md:884-888): for the SAME prompt, TTFT when the token phase is
co-located (the prefill writes the local pool) vs split (every layer's K/V is
pushed over NVLink into another GPU's paged pool while the next layers
compute; TTFT ends when the last push landed).

    overhead = TTFT(split) / TTFT(co-located) - 1

Run: python tools/push_overhead.py --model llama2-7b --prompt 1024   (2 GPUs,
     one process: pool on GPU 1)
     torchrun --nproc-per-node 4 tools/push_overhead.py --model llama2-70b
     --tp 4 --prompt 1500   (TP4 prompt pool on GPUs 0-3; rank i pushes its
     KV head slice into rank (i+1)%4's pool — the 4+4 split emulated on 4
     GPUs, the receiving GPU also computing)
Timing: CUDA events on the prompt GPU, median of --trials, max over TP ranks.
--ncu-only: two split prefills and nothing else (for an ncu NVLink-counter
capture of kv_push_kernel: nvltx__bytes.sum / nvlrx__bytes.sum per launch).
"""
import argparse
import json
import os
import statistics
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402
import torch.distributed as dist  # noqa: E402

from paper_2311_18677_b200 import _abi  # noqa: E402
from paper_2311_18677_b200 import kernels as K  # noqa: E402
from paper_2311_18677_b200.kvcache import KVCacheManager, blocks_for  # noqa: E402
from paper_2311_18677_b200.model import get_config, init_weights  # noqa: E402
from paper_2311_18677_b200.runner import ModelRunner, PushSegment, PushStats  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--model", default="llama2-7b")
    ap.add_argument("--tp", type=int, default=1)
    ap.add_argument("--prompt", type=int, default=1024)
    ap.add_argument("--trials", type=int, default=10)
    ap.add_argument("--push-ctas", type=int, default=64)
    ap.add_argument("--ncu-only", action="store_true")
    a = ap.parse_args()
    tp = a.tp
    rank = int(os.environ.get("RANK", "0"))
    if tp > 1:
        torch.cuda.set_device(rank)
        dist.init_process_group("nccl", device_id=torch.device("cuda", rank))
        group = dist.new_group(list(range(tp)))
        ctrl = dist.new_group(backend="gloo")
    else:
        torch.cuda.set_device(0)
        group = ctrl = None
    cfg = get_config(a.model)
    P = a.prompt
    hkv = cfg.n_kv_heads // tp
    nb = blocks_for(P, 16) + 8
    w = init_weights(cfg, seed=0, tp=tp, rank=rank)
    local_kv = KVCacheManager(cfg.n_layers, nb, hkv, cfg.head_dim, 16, 2, nb)
    if tp == 1:
        with torch.cuda.device(1):
            dst_kv = KVCacheManager(cfg.n_layers, nb, hkv, cfg.head_dim, 16, 2, nb)
            dseq = dst_kv.allocate(P)
            torch.cuda.synchronize()
        _abi.call("swb_enable_peer", 1)
        dst_dev = 1
    else:
        # rank i's pool receives rank (i-1)'s pushes
        own = KVCacheManager(cfg.n_layers, nb, hkv, cfg.head_dim, 16, 2, nb)
        dseq_own = own.allocate(P)
        torch.cuda.synchronize()
        hs = [None] * tp
        dist.all_gather_object(hs, (own.ipc_handle(), dseq_own), group=ctrl)
        h, dseq = hs[(rank + 1) % tp]
        dst_kv = KVCacheManager.open_peer(h)
        dst_dev = (rank + 1) % tp
    runner = ModelRunner(w, local_kv, tp_group=group, push_ctas=a.push_ctas)
    gen = torch.Generator().manual_seed(5)
    toks = torch.randint(0, cfg.vocab, (P,), generator=gen, dtype=torch.int32).cuda()
    meta = ModelRunner.pack_meta([P]).cuda()
    lseq = local_kv.allocate(P)
    slots = torch.empty(P, dtype=torch.int32, device="cuda")
    K.slots_from_table(local_kv.table_row_ptr(lseq), 0, P, 16, slots)
    ev = lambda: torch.cuda.Event(enable_timing=True)  # noqa: E731

    def colocated():
        e0, e1 = ev(), ev()
        e0.record()
        runner.prefill(toks, [P], meta, local_slots=slots)
        e1.record()
        torch.cuda.synchronize()
        return e0.elapsed_time(e1)

    def split():
        st = PushStats(bytes_per_layer=P * 2 * hkv * cfg.head_dim * 2)
        runner.prefill(toks, [P], meta, push=[PushSegment(0, P, dst_kv, dseq)], push_stats=st)
        torch.cuda.synchronize()
        runner.finish_push_stats()
        return st

    if a.ncu_only:
        split()
        split()
        return
    for _ in range(3):
        colocated()
        split()
    co, sp, comp, tail, layer_gbs = [], [], [], [], []
    for _ in range(a.trials):           # interleaved, so clocks / thermals hit both alike
        co.append(colocated())
        st = split()
        sp.append(st.compute_ms + st.tail_ms)
        comp.append(st.compute_ms)
        tail.append(st.tail_ms)
        layer_gbs.append(statistics.mean(st.bytes_per_layer / (m * 1e6) for m in st.layer_ms))
    # push kernel alone: one layer, no concurrent compute
    qkv = torch.randn(P, runner.qkv_cols, device="cuda").bfloat16()
    dslots = torch.empty(P, dtype=torch.int32, device="cuda")
    K.slots_from_table(dst_kv.table_row_ptr(dseq), 0, P, 16, dslots)
    for _ in range(3):
        K.kv_push_layer(qkv, P, runner.hq, hkv, cfg.head_dim, dst_kv.k_layer_ptr(0),
                        dst_kv.v_layer_ptr(0), dslots, 16, a.push_ctas)
    e0, e1 = ev(), ev()
    e0.record()
    for _ in range(20):
        K.kv_push_layer(qkv, P, runner.hq, hkv, cfg.head_dim, dst_kv.k_layer_ptr(0),
                        dst_kv.v_layer_ptr(0), dslots, 16, a.push_ctas)
    e1.record()
    torch.cuda.synchronize()
    alone_gbs = P * 2 * hkv * cfg.head_dim * 2 / (e0.elapsed_time(e1) / 20 * 1e6)
    vals = torch.tensor([statistics.median(co), statistics.median(sp), statistics.median(comp),
                         statistics.median(tail), -statistics.mean(layer_gbs), -alone_gbs],
                        dtype=torch.float64)
    if tp > 1:
        dist.all_reduce(vals, op=dist.ReduceOp.MAX, group=ctrl)   # slowest rank (GB/s: min)
    co_ms, sp_ms, comp_ms, tail_ms, gbs, alone = vals.tolist()
    if rank == 0:
        print(json.dumps({
            "model": cfg.name, "tp": tp, "prompt_tokens": P, "trials": a.trials,
            "push_ctas": a.push_ctas, "dst_device": dst_dev,
            "ttft_colocated_ms": co_ms, "ttft_split_ms": sp_ms,
            "overhead_frac": sp_ms / co_ms - 1.0,
            "split_compute_ms": comp_ms, "split_visible_tail_ms": tail_ms,
            "compute_slowdown_frac": comp_ms / co_ms - 1.0,
            "push_in_flight_GBps": -gbs, "push_alone_GBps": -alone,
            "push_bytes_per_layer_per_gpu": P * 2 * hkv * cfg.head_dim * 2,
            "nvlink_peak_GBps": 770.0,
            "note": "TTFT = prompt compute (CUDA events on the prompt GPU); split adds the "
                    "tail until the last layer's push landed; medians over interleaved "
                    "trials, max over TP ranks"}), flush=True)
    if tp > 1:
        dist.barrier(group=ctrl)
        dist.destroy_process_group()


if __name__ == "__main__":
    main()
