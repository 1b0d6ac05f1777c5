"""PerfModel-compatible cost model measured on B200 — the seam through which
B200 measurements re-enter the reference's scheduler and simulator
(SURVEY §8(f) rank 1).

``PerfModel`` keeps the reference's duck type (reference perf.py:91-141):
``prompt_time(tokens)``, ``token_iter_time(batch)`` (CapacityError above
``max_token_batch``), ``kv_cache_bytes``, ``memory_in_use``,
``kv_bytes_per_token``, ``weight_memory``, ``memory_capacity``,
``max_token_batch``, ``machine_type``; piecewise-linear between knots with
edge-slope extrapolation (perf.py:77-88).  The machines' batch formation
(workers.py) calls it for its iteration estimates.

``measure_perf_model`` fills the knots by timing real prefills and decode
steps of a ``ModelRunner`` with CUDA events, and ``export_profile_csv``
writes them in the reference's profile CSV format (perf.py:353-365) so
``splitsim fit-model`` / ``simulate --profile`` can consume B200 numbers.
"""

from __future__ import annotations

import io
from dataclasses import dataclass

import numpy as np

from .errors import CapacityError, ValidationError

PROFILE_HEADER = "machine_type,llm,phase,prompt_tokens,batch_size,time_ms,memory_bytes"


def piecewise_eval(x, xs, ys) -> float:
    """Linear between knots, exact at knots, edge slopes beyond the ends."""
    x = float(x)
    n = len(xs)
    if n == 1:
        return float(ys[0])
    if x >= xs[-1]:
        lo, hi = n - 2, n - 1
    elif x <= xs[0]:
        lo, hi = 0, 1
    else:
        return float(np.interp(x, xs, ys))
    slope = (ys[hi] - ys[lo]) / (xs[hi] - xs[lo])
    anchor = hi if x >= xs[-1] else lo
    return float(ys[anchor] + slope * (x - xs[anchor]))


@dataclass
class PerfModel:
    machine_type: str
    llm: str
    prompt_knots: tuple
    token_knots: tuple
    kv_bytes_per_token: float
    weight_memory: float
    memory_capacity: float
    max_token_batch: int

    def __post_init__(self):
        knots = []
        for xs, ys in (self.prompt_knots, self.token_knots):
            xs, ys = np.asarray(xs, dtype=float), np.asarray(ys, dtype=float)
            if np.any(np.diff(xs) <= 0):
                raise ValidationError("knot abscissas must be strictly increasing")
            if np.any(ys <= 0):
                raise ValidationError("predicted times must be strictly positive")
            knots.append((xs, ys))
        self.prompt_knots, self.token_knots = knots
        if self.kv_bytes_per_token <= 0:
            raise ValidationError("kv_bytes_per_token must be positive")

    def prompt_time(self, total_prompt_tokens: int) -> float:
        if total_prompt_tokens < 1:
            raise ValidationError("prompt tokens must be >= 1")
        return piecewise_eval(total_prompt_tokens, *self.prompt_knots)

    def token_iter_time(self, batch_size: int) -> float:
        if batch_size < 1:
            raise ValidationError("batch size must be >= 1")
        if batch_size > self.max_token_batch:
            raise CapacityError(
                f"batch {batch_size} exceeds max_token_batch {self.max_token_batch}")
        return piecewise_eval(batch_size, *self.token_knots)

    def kv_cache_bytes(self, context_tokens: int) -> float:
        if context_tokens < 0:
            raise ValidationError("context tokens must be >= 0")
        return context_tokens * self.kv_bytes_per_token

    def memory_in_use(self, active_contexts) -> float:
        return self.weight_memory + sum(self.kv_cache_bytes(c) for c in active_contexts)


def export_profile_csv(model: PerfModel) -> str:
    """Knots as profile rows (reference format, perf.py:353-365)."""
    buf = io.StringIO()
    buf.write(PROFILE_HEADER + "\n")
    for x, y in zip(*model.prompt_knots):
        mem = model.weight_memory + x * model.kv_bytes_per_token
        buf.write(f"{model.machine_type},{model.llm},prompt,{int(x)},0,{y:.6f},{mem:.0f}\n")
    for x, y in zip(*model.token_knots):
        buf.write(f"{model.machine_type},{model.llm},token,0,{int(x)},{y:.6f},0\n")
    return buf.getvalue()


def measure_perf_model(runner, machine_type: str = "B200",
                       prompt_points=(128, 256, 512, 1024, 1500, 2048),
                       batch_points=(1, 2, 4, 8, 16), context: int = 1024,
                       reps: int = 3) -> PerfModel:
    """Time real prefills / decode steps on ``runner``'s GPU and build the
    knots (median of ``reps`` CUDA-event timings per point)."""
    import torch

    from . import kernels as K
    from .runner import ModelRunner
    cfg, kv = runner.cfg, runner.kv
    ev = lambda: torch.cuda.Event(enable_timing=True)  # noqa: E731
    p_ms = []
    for P in prompt_points:
        seq = kv.allocate(P + 1)
        toks = torch.randint(0, cfg.vocab, (P,), dtype=torch.int32, device=runner.dev)
        meta = ModelRunner.pack_meta([P]).to(runner.dev)
        slots = torch.empty(P, dtype=torch.int32, device=runner.dev)
        K.slots_from_table(kv.table_row_ptr(seq), 0, P, kv.block_size, slots)
        ts = []
        for _ in range(reps + 1):
            a, b = ev(), ev()
            a.record()
            runner.prefill(toks, [P], meta, local_slots=slots)
            b.record()
            torch.cuda.synchronize()
            ts.append(a.elapsed_time(b))
        p_ms.append(float(np.median(ts[1:])))
        kv.release(seq)
    t_ms = []
    for B in batch_points:
        seqs = [kv.allocate(context + 8) for _ in range(B)]
        g = runner.decode_graph(B, context + 8, 8)
        g.load(seqs, [1] * B, [context] * B)
        g.capture()
        ts = []
        for _ in range(reps + 1):
            g.load(seqs, [1] * B, [context] * B)
            a, b = ev(), ev()
            a.record()
            g.replay()
            b.record()
            torch.cuda.synchronize()
            ts.append(a.elapsed_time(b))
        t_ms.append(float(np.median(ts[1:])))
        for s in seqs:
            kv.release(s)
    kvb = cfg.kv_bytes_per_token(runner.tp)
    cap = runner.w.nbytes() + kv.num_blocks * kv.block_size * kvb
    return PerfModel(machine_type, cfg.name, (list(prompt_points), p_ms),
                     (list(batch_points), t_ms), float(kvb), float(runner.w.nbytes()),
                     float(cap), cfg.max_token_batch)
