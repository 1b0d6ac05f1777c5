"""User-facing single-GPU engine: both phases on one GPU (the reference's
Baseline design — an always-mixed machine, cluster.py:22-24, :98-103).

``ColocatedEngine.generate`` is the end-to-end call a user makes: prompts come
from host memory (pinned), are copied to the device inside the call, the
prompt phase emits each request's first token, and every token-phase
iteration streams its new tokens back to the host.  Emission times are host
monotonic-clock observations of the device events, so TTFT / TBT are what a
client would see (RequestRecord semantics, reference engine.py:71-91).
"""

from __future__ import annotations

import time
from dataclasses import dataclass, field

import torch

from . import kernels as K
from .kvcache import KVCacheManager, blocks_for
from .model import ModelConfig, Weights
from .runner import ModelRunner


@dataclass
class GenRequest:
    id: int
    prompt: torch.Tensor          # int32 host tensor (pinned preferred)
    n_out: int
    arrival: float = 0.0          # host monotonic seconds


@dataclass
class GenResult:
    id: int
    tokens: list = field(default_factory=list)
    emissions: list = field(default_factory=list)  # host seconds per token
    arrival: float = 0.0

    @property
    def ttft_ms(self):
        return (self.emissions[0] - self.arrival) * 1e3

    def tbt_ms(self):
        e = self.emissions
        return [(b - a) * 1e3 for a, b in zip(e, e[1:])]


def pool_blocks_for_memory(cfg: ModelConfig, tp: int, block_size: int, reserve_bytes: int,
                           frac: float = 0.85) -> int:
    """Blocks that fit in the device memory left after weights (capacity =
    free HBM after weights)."""
    free, _total = torch.cuda.mem_get_info()
    budget = max(0, int(free * frac) - reserve_bytes)
    per_block = block_size * cfg.kv_bytes_per_token(tp)
    return max(1, budget // per_block)


class ColocatedEngine:
    def __init__(self, weights: Weights, num_blocks: int | None = None, block_size: int = 16,
                 max_seqs: int = 64, max_ctx: int = 8192 + 4096):
        self.cfg = weights.cfg
        self.w = weights
        if num_blocks is None:
            num_blocks = min(pool_blocks_for_memory(self.cfg, weights.tp, block_size,
                                                    reserve_bytes=2 << 30),
                             max_seqs * blocks_for(max_ctx, block_size))
        self.kv = KVCacheManager(self.cfg.n_layers, num_blocks, self.cfg.n_kv_heads // weights.tp,
                                 self.cfg.head_dim, block_size, max_seqs,
                                 blocks_for(max_ctx, block_size))
        self.runner = ModelRunner(weights, self.kv)
        self.host_tok = torch.empty(1 << 16, dtype=torch.int32).pin_memory()

    # ------------------------------------------------------------------
    def generate(self, requests: list[GenRequest], prompt_token_cap: int = 2048) -> list[GenResult]:
        """Serve ``requests`` end to end (static batch: prefill in chunks of at
        most ``prompt_token_cap`` tokens, head prompt always admitted — the
        reference's prompt batching rule, machine.py:186-203 — then batched
        decode until every request has its outputs)."""
        dev = self.runner.dev
        kv = self.kv
        res = {r.id: GenResult(r.id, arrival=r.arrival) for r in requests}
        seqs = {r.id: kv.allocate(len(r.prompt) + r.n_out) for r in requests}
        first_host = {}
        # ---- prompt phase, FCFS chunks
        i = 0
        while i < len(requests):
            chunk, total = [], 0
            while i < len(requests):
                n = len(requests[i].prompt)
                if chunk and total + n > prompt_token_cap:
                    break
                chunk.append(requests[i])
                total += n
                i += 1
            lens = [len(r.prompt) for r in chunk]
            toks_h = torch.cat([r.prompt for r in chunk]).pin_memory()
            meta_h = ModelRunner.pack_meta(lens).pin_memory()
            toks = toks_h.to(dev, non_blocking=True)
            meta = meta_h.to(dev, non_blocking=True)
            slots = torch.empty(total, dtype=torch.int32, device=dev)
            off = 0
            for r, n in zip(chunk, lens):
                K.slots_from_table(kv.table_row_ptr(seqs[r.id]), 0, n, kv.block_size,
                                   slots[off:off + n])
                off += n
            first = self.runner.prefill(toks, lens, meta, local_slots=slots)
            fh = torch.empty(len(chunk), dtype=torch.int32).pin_memory()
            fh.copy_(first, non_blocking=True)
            ev = torch.cuda.Event()
            ev.record()
            ev.synchronize()
            now = time.perf_counter()
            for j, r in enumerate(chunk):
                first_host[r.id] = int(fh[j])
                res[r.id].tokens.append(int(fh[j]))
                res[r.id].emissions.append(now)
        # ---- token phase: one graph for the whole batch
        live = [r for r in requests if r.n_out > 1]
        if live:
            B = len(live)
            steps = max(r.n_out for r in live) - 1
            max_ctx = max(len(r.prompt) + r.n_out for r in live)
            g = self.runner.decode_graph(B, max_ctx, steps)
            g.load([seqs[r.id] for r in live], [first_host[r.id] for r in live],
                   [len(r.prompt) for r in live])
            if g.graph is None:
                g.capture()
            ring_h = torch.empty(steps + 1, B, dtype=torch.int32).pin_memory()
            evs = [torch.cuda.Event() for _ in range(steps)]
            for s in range(steps):
                g.replay()
                ring_h[s].copy_(g.next_tok, non_blocking=True)
                evs[s].record()
                if s > 0:
                    self._emit(evs[s - 1], ring_h[s - 1], live, res, s)
            self._emit(evs[steps - 1], ring_h[steps - 1], live, res, steps)
        for r in requests:
            kv.release(seqs[r.id])
        return [res[r.id] for r in requests]

    @staticmethod
    def _emit(ev, row, live, res, step_no):
        ev.synchronize()
        now = time.perf_counter()
        for b, r in enumerate(live):
            if step_no < r.n_out:
                res[r.id].tokens.append(int(row[b]))
                res[r.id].emissions.append(now)
