"""Driver backend whose iterations run on B200s (measured trace replay).

``driver.Driver`` reproduces the reference engine's request lifecycle
(reference engine.py:202-336) on a virtual millisecond clock; with
``ModeledBackend`` every duration comes from a PerfModel lookup, i.e. the
reference's ``prompt_time`` / ``token_iter_time`` / ``plan_transfer``
(perf.py:119-132, transfer.py:79-99).  ``GpuBackend`` replaces each lookup
with the real work on the machine's GPU and returns its measured device time:

* a prompt iteration prefills the batch's prompts (libswb200 tcgen05 GEMMs,
  attention, ...) and — when a request's token machine is another GPU —
  pushes every finished layer's K/V straight into that GPU's paged blocks
  (P2P stores over NVLink, peer access inside this process), overlapping the
  next layers; the iteration lasts until the last layer's compute ends and
  the request's TRANSFER event follows after the measured push tail
  (``transfer_visible_ms``);
* a token iteration runs one CUDA-graph decode step for exactly the batch
  the token machine formed (Machine.form_batch: slots, memory, FCFS), with
  the requests' real tokens and contexts, and returns its device time;
* a mixed iteration (Baseline designs) runs both and takes their sum (the
  reference's default mixing rule, machine.py:238-243).

So the scheduling semantics are the reference's, exactly as pinned by the
golden tests, while every latency on the clock is a B200 measurement for the
actual batch composition.  Machines map onto GPUs of this process (one GPU
per machine; several machines may share a GPU for small tests).  The
concurrent multi-process serving path is ``splitwise.py``.
"""

from __future__ import annotations

import os

import torch

from . import _abi
from . import kernels as K
from .errors import CapacityError
from .kvcache import KVCacheManager, blocks_for
from .model import get_config, init_weights
from .runner import ModelRunner, PushSegment, PushStats
from .serving import pool_blocks_for_memory
from .splitwise import estimated_perf_model
from .workers import PROMPT

CTX_BUCKET = 2048          # decode graphs are captured per (batch, context bucket)


class PoolExhausted(RuntimeError):
    """A token machine's physical KV pool cannot hold another routed request:
    the offered load exceeds what the pool ratio sustains (the reference's
    provisioning treats a RuntimeError as 'fails at this load',
    provision.py:138-143)."""


class _Seq:
    __slots__ = ("machine", "seq", "cur", "ctx")

    def __init__(self, machine, seq, cur, ctx):
        self.machine, self.seq, self.cur, self.ctx = machine, seq, cur, ctx


class GpuBackend:
    def __init__(self, model: str, devices: dict | None = None, seed: int = 0,
                 block_size: int = 16, max_seqs: int = 256, max_ctx: int = 8192 + 4096,
                 kv_share: float | None = None, prompt_seed: int = 1234,
                 clock: str = "measured", mixed: bool = True):
        """clock="measured": the virtual clock advances by the measured device
        times (the product).  clock="modeled": the work still runs on the GPU
        but the clock advances by the PerfModel estimates, which makes the
        schedule independent of timing noise (reproducible debugging).
        mixed=True runs an iteration holding both prompt and token tasks as one
        fused step (ModelRunner.mixed); False runs prefill then decode."""
        self.cfg = get_config(model)
        self.clock = clock
        self.mixed = mixed
        self.devices = devices
        self.seed = seed
        self.block_size = block_size
        self.max_seqs = max_seqs
        self.max_ctx = max_ctx
        self.kv_share = kv_share
        self.prompt_seed = prompt_seed
        self.runners: dict[int, ModelRunner] = {}
        self.dev: dict[int, int] = {}
        self.state: dict[int, _Seq] = {}
        self.visible: dict[int, tuple[float, float]] = {}
        self.iter_log: list[tuple] = []     # (machine, kind, batch tokens/rows, ms)
        self.tokens: dict[int, list] = {}   # rid -> generated token ids (first, then decode)
        self.driver = None

    # ------------------------------------------------------------ set-up
    def perf_models(self, machine_type: str = "B200") -> dict:
        """Roofline-estimated PerfModel for batch formation / admission; the
        capacity is the device pool actually allocated (set in attach)."""
        return {machine_type: estimated_perf_model(self.cfg, None, self.cfg.weight_bytes(1))}

    def attach(self, driver) -> None:
        self.driver = driver
        ms = driver.cluster.machines
        ngpu = torch.cuda.device_count()
        devs = self.devices or {mid: i % ngpu for i, mid in enumerate(sorted(ms))}
        per_dev: dict[int, int] = {}
        for mid in sorted(ms):
            per_dev[devs[mid]] = per_dev.get(devs[mid], 0) + 1
        weights = {}
        for mid in sorted(ms):
            d = devs[mid]
            self.dev[mid] = d
            with torch.cuda.device(d):
                if d not in weights:
                    weights[d] = init_weights(self.cfg, seed=self.seed)
                share = self.kv_share or 1.0 / per_dev[d]
                nb = pool_blocks_for_memory(self.cfg, 1, self.block_size, reserve_bytes=3 << 30,
                                            frac=0.85 * share)
                nb = min(nb, self.max_seqs * blocks_for(self.max_ctx, self.block_size))
                kv = KVCacheManager(self.cfg.n_layers, nb, self.cfg.n_kv_heads,
                                    self.cfg.head_dim, self.block_size, self.max_seqs,
                                    blocks_for(self.max_ctx, self.block_size))
                self.runners[mid] = ModelRunner(weights[d], kv)
            # admission capacity = weights + this machine's physical pool
            m = ms[mid]
            m.perf = estimated_perf_model(self.cfg, kv, weights[d].nbytes())
        for a in set(devs.values()):
            with torch.cuda.device(a):
                for b in set(devs.values()):
                    if a != b:
                        _abi.call("swb_enable_peer", b)

    def _prompt_ids(self, rid: int, n: int) -> torch.Tensor:
        g = torch.Generator().manual_seed(self.prompt_seed + rid)
        return torch.randint(0, self.cfg.vocab, (n,), generator=g, dtype=torch.int32)

    # ------------------------------------------------------------ iterations
    def _dbg(self, what):
        mode = os.environ.get("SWB_DEBUG_SYNC", "")
        if mode and (mode == "1" or what.split()[-1 if what in ("prefill", "decode") else 1]
                     .startswith(mode)):
            for d in set(self.dev.values()):
                torch.cuda.synchronize(d)
            print("ok:", what, flush=True)

    def iteration_ms(self, machine, batch) -> float:
        if getattr(batch, "prompt_chunk", None) is not None:
            ms = self._mixed_chunk(machine.id, batch)
            return ms if self.clock == "measured" else batch.iteration_time
        ms = 0.0
        if (batch.prompt_tasks and batch.token_tasks and self.mixed and
                all(self.driver.records[t.request_id].token_machine == machine.id
                    for t in batch.prompt_tasks)):
            # mixed batch: prompt rows and decode rows share every weight pass
            ms = self._mixed(machine.id, batch.prompt_tasks, batch.token_tasks)
            return ms if self.clock == "measured" else batch.iteration_time
        if batch.prompt_tasks:
            self._dbg(f"before prefill m{machine.id} lens={[t.tokens for t in batch.prompt_tasks]}")
            ms += self._prefill(machine.id, batch.prompt_tasks)
            self._dbg("prefill")
        if batch.token_tasks:
            self._dbg(f"before decode m{machine.id} B={len(batch.token_tasks)} ctx="
                      f"{[self.state[t.request_id].ctx for t in batch.token_tasks]}")
            ms += self._decode(machine.id, batch.token_tasks)
            self._dbg("decode")
        return ms if self.clock == "measured" else batch.iteration_time

    def _prefill(self, mid: int, tasks) -> float:
        recs = [self.driver.records[t.request_id] for t in tasks]
        local = [r for r in recs if r.token_machine == mid]
        remote = [r for r in recs if r.token_machine != mid]
        ms = 0.0
        for group, push in ((local, False), (remote, True)):
            if group:
                ms += self._prefill_group(mid, group, push)
        return ms

    def _prefill_group(self, mid: int, recs, push: bool) -> float:
        runner, dev = self.runners[mid], self.dev[mid]
        seqs = []
        for r in recs:   # reserve the final context in the token machine's pool
            tm = r.token_machine
            with torch.cuda.device(self.dev[tm]):
                try:
                    seqs.append(self.runners[tm].kv.allocate(r.prompt_tokens + r.output_tokens))
                except CapacityError as e:
                    raise PoolExhausted(f"machine {tm}: {e} ({len(self.state)} requests hold "
                                        "KV)") from e
        for tm in {r.token_machine for r in recs}:
            torch.cuda.synchronize(self.dev[tm])       # table rows written before peers read
        lens = [r.prompt_tokens for r in recs]
        with torch.cuda.device(dev):
            toks = torch.cat([self._prompt_ids(r.request_id, r.prompt_tokens) for r in recs])
            toks = toks.pin_memory().to(f"cuda:{dev}", non_blocking=True)
            meta = ModelRunner.pack_meta(lens).pin_memory().to(f"cuda:{dev}", non_blocking=True)
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            stats = None
            if push:
                segs, off = [], 0
                for r, s, n in zip(recs, seqs, lens):
                    segs.append(PushSegment(off, n, self.runners[r.token_machine].kv, s))
                    off += n
                stats = PushStats(bytes_per_layer=off * 2 * runner.hkv * runner.dh * 2)
                e0.record()
                first = runner.prefill(toks, lens, meta, push=segs, push_stats=stats)
            else:
                kv = runner.kv
                slots = torch.empty(sum(lens), dtype=torch.int32, device=f"cuda:{dev}")
                off = 0
                for s, n in zip(seqs, lens):
                    K.slots_from_table(kv.table_row_ptr(s), 0, n, kv.block_size,
                                       slots[off:off + n])
                    off += n
                e0.record()
                first = runner.prefill(toks, lens, meta, local_slots=slots)
            e1.record()
            first_h = first.cpu()                   # synchronises the prompt GPU
            if push:
                runner.finish_push_stats()
                ms = stats.compute_ms
                for r in recs:
                    self.visible[r.request_id] = (stats.tail_ms, sum(stats.layer_ms))
            else:
                ms = e0.elapsed_time(e1)
        for r, s, f in zip(recs, seqs, first_h.tolist()):
            self.state[r.request_id] = _Seq(r.token_machine, s, int(f), r.prompt_tokens)
            self.tokens[r.request_id] = [int(f)]
        self.iter_log.append((mid, "prompt", sum(lens), ms))
        return ms

    def _decode(self, mid: int, tasks) -> float:
        runner, dev = self.runners[mid], self.dev[mid]
        sts = [self.state[t.request_id] for t in tasks]
        B = len(sts)
        bucket = CTX_BUCKET * ((max(s.ctx for s in sts) + 2 + CTX_BUCKET - 1) // CTX_BUCKET)
        with torch.cuda.device(dev):
            g = runner.decode_graph(B, bucket, 1)
            g.load([s.seq for s in sts], [s.cur for s in sts], [s.ctx for s in sts])
            if g.graph is None:
                g.capture()
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record()
            g.replay()
            e1.record()
            nxt = g.next_tok.cpu().tolist()         # synchronises
            ms = e0.elapsed_time(e1)
        for tk, s, t in zip(tasks, sts, nxt):
            s.cur = int(t)
            self.tokens[tk.request_id].append(int(t))
            s.ctx += 1
        self.iter_log.append((mid, "token", B, ms))
        return ms

    def _mixed(self, mid: int, ptasks, ttasks) -> float:
        runner, dev = self.runners[mid], self.dev[mid]
        kv = runner.kv
        recs = [self.driver.records[t.request_id] for t in ptasks]
        sts = [self.state[t.request_id] for t in ttasks]
        with torch.cuda.device(dev):
            seqs = [kv.allocate(r.prompt_tokens + r.output_tokens) for r in recs]
            lens = [r.prompt_tokens for r in recs]
            toks = torch.cat([self._prompt_ids(r.request_id, r.prompt_tokens) for r in recs])
            toks = toks.pin_memory().to(f"cuda:{dev}", non_blocking=True)
            meta = ModelRunner.pack_meta(lens).pin_memory().to(f"cuda:{dev}", non_blocking=True)
            slots = torch.empty(sum(lens), dtype=torch.int32, device=f"cuda:{dev}")
            off = 0
            for s, n in zip(seqs, lens):
                K.slots_from_table(kv.table_row_ptr(s), 0, n, kv.block_size, slots[off:off + n])
                off += n
            idx = torch.tensor([s.seq for s in sts], dtype=torch.long, device=f"cuda:{dev}")
            tables = torch.index_select(kv.tables(), 0, idx)
            dtok = torch.tensor([s.cur for s in sts], dtype=torch.int32, device=f"cuda:{dev}")
            dctx = torch.tensor([s.ctx for s in sts], dtype=torch.int32, device=f"cuda:{dev}")
            bucket = CTX_BUCKET * ((max(s.ctx for s in sts) + 2 + CTX_BUCKET - 1) // CTX_BUCKET)
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record()
            nxt = runner.mixed(toks, lens, meta, slots, tables, dtok, dctx, bucket)
            e1.record()
            nxt_h = nxt.cpu().tolist()
            ms = e0.elapsed_time(e1)
        R = len(recs)
        for r, s, f in zip(recs, seqs, nxt_h[:R]):
            self.state[r.request_id] = _Seq(mid, s, int(f), r.prompt_tokens)
            self.tokens[r.request_id] = [int(f)]
        for tk, s, t in zip(ttasks, sts, nxt_h[R:]):
            s.cur = int(t)
            self.tokens[tk.request_id].append(int(t))
            s.ctx += 1
        self.iter_log.append((mid, "mixed", sum(lens) + len(sts), ms))
        return ms

    def _mixed_chunk(self, mid: int, batch) -> float:
        """Chunked-prefill iteration of an always-mixed machine: a chunk of
        the head prompt plus one decode token of every scheduled sequence."""
        runner, dev = self.runners[mid], self.dev[mid]
        kv = runner.kv
        task = batch.prompt_tasks[0]
        start, n = batch.prompt_chunk
        rec = self.driver.records[task.request_id]
        sts = [self.state[t.request_id] for t in batch.token_tasks]
        with torch.cuda.device(dev):
            if start == 0:          # first chunk: reserve the final context
                seq = kv.allocate(rec.prompt_tokens + rec.output_tokens)
                self._chunking = getattr(self, "_chunking", {})
                self._chunking[rec.request_id] = seq
            seq = self._chunking[rec.request_id]
            ids = self._prompt_ids(rec.request_id, rec.prompt_tokens)[start:start + n]
            toks = ids.pin_memory().to(f"cuda:{dev}", non_blocking=True)
            args = {}
            if sts:
                idx = torch.tensor([s.seq for s in sts], dtype=torch.long, device=f"cuda:{dev}")
                args = dict(
                    dec_tables=torch.index_select(kv.tables(), 0, idx),
                    dec_tok=torch.tensor([s.cur for s in sts], dtype=torch.int32,
                                         device=f"cuda:{dev}"),
                    dec_ctx=torch.tensor([s.ctx for s in sts], dtype=torch.int32,
                                         device=f"cuda:{dev}"),
                    dec_max_ctx=CTX_BUCKET * ((max(s.ctx for s in sts) + 2 + CTX_BUCKET - 1)
                                              // CTX_BUCKET))
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record()
            nxt = runner.mixed_chunk(toks, seq, start, **args)
            e1.record()
            nxt_h = nxt.cpu().tolist()
            ms = e0.elapsed_time(e1)
        if start + n == rec.prompt_tokens:       # last chunk: the first token
            self._chunking.pop(rec.request_id)
            self.state[rec.request_id] = _Seq(mid, seq, int(nxt_h[0]), rec.prompt_tokens)
            self.tokens[rec.request_id] = [int(nxt_h[0])]
        for tk, s, t in zip(batch.token_tasks, sts, nxt_h[1:]):
            s.cur = int(t)
            self.tokens[tk.request_id].append(int(t))
            s.ctx += 1
        self.iter_log.append((mid, "chunk", n + len(sts), ms))
        return ms

    # ------------------------------------------------------------ hand-off
    def transfer_visible_ms(self, driver, rec, prompt_ms: float) -> float:
        tail, raw = self.visible.pop(rec.request_id, (0.0, 0.0))
        rec.transfer_raw_ms = raw
        return tail

    def release(self, rec) -> None:
        s = self.state.pop(rec.request_id, None)
        if s is not None:
            with torch.cuda.device(self.dev[s.machine]):
                self.runners[s.machine].kv.release(s.seq)
                if os.environ.get("SWB_DEBUG_SYNC") == "release":
                    torch.cuda.synchronize()


__all__ = ["GpuBackend", "PoolExhausted", "PROMPT"]
