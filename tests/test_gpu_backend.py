"""Measured trace replay: the reference's lifecycle / scheduler with every
iteration executed on the GPU (gpu_backend.GpuBackend)."""
import pytest
import torch

from paper_2311_18677_b200.cluster import ClusterConfig
from paper_2311_18677_b200.driver import Driver, Request
from reftrace import preset_trace

pytestmark = pytest.mark.gpu


def _trace(n_out_cap=12):
    reqs = preset_trace("conversation", 20.0, 1.0, 5)[:12]
    return [Request(r.id, r.arrival, min(r.prompt_tokens, 700), min(r.output_tokens, n_out_cap))
            for r in reqs]


@pytest.mark.parametrize("design,p,t", [("Splitwise-BB", 1, 1), ("Baseline-B200", 1, 0),
                                        ("Splitwise-BB", 2, 1)])
def test_trace_replay_on_gpu(design, p, t):
    from paper_2311_18677_b200.gpu_backend import GpuBackend
    reqs = _trace()
    be = GpuBackend("tiny", max_seqs=32)
    drv = Driver(ClusterConfig(design, p, t, llm="tiny"), be.perf_models(), reqs, backend=be,
                 record_log=False)
    free0 = {mid: r.kv.free_blocks for mid, r in be.runners.items()}
    res = drv.run()
    for r in res.report.records:
        assert len(r.emissions) == r.output_tokens
        assert r.ttft_ms > 0 and r.completion >= r.first_token_time
        if design.startswith("Splitwise") and r.output_tokens > 1:
            assert r.token_machine != r.prompt_machine
            assert r.transfer_visible_ms >= 0.0 and r.transfer_raw_ms > 0.0
    torch.cuda.synchronize()
    assert {mid: r.kv.free_blocks for mid, r in be.runners.items()} == free0   # all released
    kinds = {k for _, k, _, _ in be.iter_log}
    assert kinds == {"prompt", "token"}
    s = res.report.summary()
    assert s["requests"] == len(reqs) and s["tokens_per_s"] > 0


def test_split_and_colocated_generate_same_tokens():
    """Token ids through the Splitwise path (layer-wise push into the token
    machine's pool) equal the co-located path's at batch 1 (arrivals far
    apart, so both decode every request alone)."""
    from paper_2311_18677_b200.gpu_backend import GpuBackend
    reqs = [Request(i, 10.0 * i, 100 + 37 * i, 9) for i in range(3)]
    toks = {}
    for design, p, t in (("Splitwise-BB", 1, 1), ("Baseline-B200", 1, 0)):
        be = GpuBackend("tiny", max_seqs=8)
        seen = {}
        orig = be._decode

        def spy(mid, tasks, orig=orig, be=be, seen=seen):
            ms = orig(mid, tasks)
            for tk in tasks:
                seen.setdefault(tk.request_id, []).append(be.state[tk.request_id].cur)
            return ms
        be._decode = spy
        Driver(ClusterConfig(design, p, t, llm="tiny"), be.perf_models(), reqs, backend=be,
               record_log=False).run()
        toks[design] = seen
    assert toks["Splitwise-BB"] == toks["Baseline-B200"]


def test_mixed_iteration_matches_separate_phases():
    """ModelRunner.mixed (prompt rows + decode rows through the same GEMMs)
    produces the same first tokens and decode tokens as a prefill followed by
    a decode step, and writes the prompt's KV like the prefill does."""
    from paper_2311_18677_b200 import kernels as K
    from paper_2311_18677_b200.kvcache import KVCacheManager
    from paper_2311_18677_b200.model import get_config, init_weights
    from paper_2311_18677_b200.runner import ModelRunner
    cfg = get_config("tiny")
    w = init_weights(cfg, seed=0)
    g = torch.Generator().manual_seed(9)
    old = [torch.randint(0, cfg.vocab, (n,), generator=g, dtype=torch.int32) for n in (40, 70)]
    new = torch.randint(0, cfg.vocab, (50,), generator=g, dtype=torch.int32)
    out = {}
    for mode in ("mixed", "separate"):
        kv = KVCacheManager(cfg.n_layers, 128, cfg.n_kv_heads, cfg.head_dim, 16, 8, 16)
        r = ModelRunner(w, kv)
        seqs, firsts = [], []
        for p in old:
            s = kv.allocate(len(p) + 8)
            sl = torch.empty(len(p), dtype=torch.int32, device="cuda")
            K.slots_from_table(kv.table_row_ptr(s), 0, len(p), 16, sl)
            firsts.append(int(r.prefill(p.cuda(), [len(p)], ModelRunner.pack_meta([len(p)]).cuda(),
                                        local_slots=sl)[0]))
            seqs.append(s)
        sn = kv.allocate(len(new) + 8)
        sl = torch.empty(len(new), dtype=torch.int32, device="cuda")
        K.slots_from_table(kv.table_row_ptr(sn), 0, len(new), 16, sl)
        meta = ModelRunner.pack_meta([len(new)]).cuda()
        if mode == "mixed":
            tables = kv.tables()[torch.tensor(seqs, device="cuda")].contiguous()
            ctx = torch.tensor([len(p) for p in old], dtype=torch.int32, device="cuda")
            nxt = r.mixed(new.cuda(), [len(new)], meta, sl, tables,
                          torch.tensor(firsts, dtype=torch.int32, device="cuda"), ctx, 256)
            out[mode] = nxt.tolist()
            assert ctx.tolist() == [41, 71]
        else:
            f = int(r.prefill(new.cuda(), [len(new)], meta, local_slots=sl)[0])
            gr = r.decode_graph(2, 256, 4)
            gr.load(seqs, firsts, [len(p) for p in old])
            gr.replay()
            out[mode] = [f] + gr.next_tok.tolist()
        torch.cuda.synchronize()
        tb = kv.tables()[sn].long()
        p = torch.arange(len(new), device="cuda")
        out[mode + "_kv"] = kv.k_view(1)[tb[p // 16], :, p % 16].float().clone()
    assert out["mixed"] == out["separate"]
    assert (out["mixed_kv"] - out["separate_kv"]).abs().max().item() < 0.05


def test_parked_token_tasks_decode_the_oracle_tokens():
    """A mixed (Baseline) machine with max_token_batch = 2: prompts arriving
    while two token tasks decode take a slot, so a resident token task is
    PARKED for that iteration (reference machine.py:207-231; PAPER.md:625-628
    preemption with aging).  Parking must not disturb its KV or context:
    every request's tokens equal the fp32 oracle's greedy tokens wherever the
    oracle's top-2 margin is decisive (> 0.02, ~6x the tiny model's observed
    bf16 logit error)."""
    import dataclasses
    from oracle.decoder import OracleDecoder
    from paper_2311_18677_b200.gpu_backend import GpuBackend
    reqs = [Request(0, 0.0, 200, 16), Request(1, 0.00005, 150, 16), Request(2, 0.0003, 300, 8),
            Request(3, 0.0005, 100, 8), Request(4, 0.0007, 120, 6)]
    be = GpuBackend("tiny", max_seqs=16, clock="modeled")
    drv = Driver(ClusterConfig("Baseline-B200", 1, 0, llm="tiny"), be.perf_models(), reqs,
                 backend=be, record_log=False)
    for m in drv.cluster.machines.values():
        m.perf = dataclasses.replace(m.perf, max_token_batch=2)
    res = drv.run()
    assert max(r.preempt_count for r in res.report.records) >= 1      # parking happened
    assert {k for _, k, _, _ in be.iter_log} >= {"mixed", "token"}
    orc = OracleDecoder.from_weights(be.runners[0].w)
    for r in reqs:
        got = be.tokens[r.id]
        assert len(got) == r.output_tokens
        prompt = be._prompt_ids(r.id, r.prompt_tokens).tolist()
        ref_toks, ref_logits = orc.generate(prompt, r.output_tokens, forced=got[:-1])
        top2 = ref_logits.topk(2, -1).values
        decisive = (top2[:, 0] - top2[:, 1]) > 0.02
        for i in range(r.output_tokens):
            if decisive[i]:
                assert got[i] == ref_toks[i], (r.id, i)


def test_chunked_prefill_decodes_the_oracle_tokens():
    """Chunked prefill on an always-mixed machine (SchedulerConfig.
    prefill_chunk_tokens = 64): every iteration runs the running sequences'
    decode rows plus a chunk of the head prompt (swb_attn_chunk over the
    pages of the earlier chunks); nobody is parked, and every request's tokens
    equal the fp32 oracle's wherever its top-2 margin is decisive."""
    from oracle.decoder import OracleDecoder
    from paper_2311_18677_b200.gpu_backend import GpuBackend
    from paper_2311_18677_b200.workers import SchedulerConfig
    reqs = [Request(0, 0.0, 200, 12), Request(1, 0.00005, 150, 12), Request(2, 0.0003, 300, 8),
            Request(3, 0.0005, 100, 8), Request(4, 0.0007, 37, 6)]
    be = GpuBackend("tiny", max_seqs=16, clock="modeled")
    cc = ClusterConfig("Baseline-B200", 1, 0, llm="tiny")
    cc.sched = SchedulerConfig(prefill_chunk_tokens=64)
    drv = Driver(cc, be.perf_models(), reqs, backend=be, record_log=False)
    res = drv.run()
    kinds = [k for _, k, _, _ in be.iter_log]
    assert "chunk" in kinds and "prompt" not in kinds and "mixed" not in kinds
    assert max(r.preempt_count for r in res.report.records) == 0
    orc = OracleDecoder.from_weights(be.runners[0].w)
    for r in reqs:
        got = be.tokens[r.id]
        assert len(got) == r.output_tokens
        prompt = be._prompt_ids(r.id, r.prompt_tokens).tolist()
        ref_toks, ref_logits = orc.generate(prompt, r.output_tokens, forced=got[:-1])
        top2 = ref_logits.topk(2, -1).values
        decisive = (top2[:, 0] - top2[:, 1]) > 0.02
        for i in range(r.output_tokens):
            if decisive[i]:
                assert got[i] == ref_toks[i], (r.id, i)
    torch.cuda.synchronize()
