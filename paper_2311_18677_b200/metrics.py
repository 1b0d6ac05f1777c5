"""Request-level metrics with the reference's definitions (reference
engine.py:35-113): TTFT = first emission - arrival, E2E = completion -
arrival, TBT = gaps between successive emissions (the first gap carries the
KV transfer's visible latency), nearest-rank percentiles, throughput =
requests / makespan.  Added for the B200 path: output tokens / makespan.
Times here are host monotonic-clock milliseconds observed when the device
work completed (not modelled)."""

from __future__ import annotations

import math
from dataclasses import dataclass, field

from .errors import ValidationError


def percentile(samples, p: float):
    """Nearest-rank: element ceil(p*n)-1 of the sorted samples."""
    if len(samples) == 0:
        raise ValidationError("percentile of empty sample set")
    if not 0.0 < p <= 1.0:
        raise ValidationError("p must be in (0, 1]")
    ordered = sorted(samples)
    return ordered[max(0, math.ceil(p * len(ordered)) - 1)]


@dataclass
class RequestRecord:
    request_id: int
    arrival_ms: float
    prompt_tokens: int
    output_tokens: int
    prompt_machine: int = -1
    token_machine: int = -1
    first_token_time: float | None = None
    emissions: list = field(default_factory=list)
    completion: float | None = None
    transfer_visible_ms: float = 0.0
    transfer_raw_ms: float = 0.0
    preempt_count: int = 0
    tokens: list = field(default_factory=list)
    arrival_s: float | None = None      # the trace's arrival (CSV output)

    @property
    def ttft_ms(self) -> float:
        return self.first_token_time - self.arrival_ms

    @property
    def e2e_ms(self) -> float:
        return self.completion - self.arrival_ms

    def tbt_ms(self) -> list:
        e = self.emissions
        return [b - a for a, b in zip(e, e[1:])]


@dataclass
class MetricsReport:
    records: list
    makespan_ms: float
    utilization: dict = field(default_factory=dict)

    @property
    def throughput_rps(self) -> float:
        return len(self.records) / (self.makespan_ms / 1e3) if self.makespan_ms > 0 else 0.0

    @property
    def tokens_per_s(self) -> float:
        n = sum(len(r.emissions) for r in self.records)
        return n / (self.makespan_ms / 1e3) if self.makespan_ms > 0 else 0.0

    def summary(self) -> dict:
        out = {"requests": len(self.records), "throughput_rps": self.throughput_rps,
               "tokens_per_s": self.tokens_per_s}
        if not self.records:
            return out
        series = {"ttft_ms": [r.ttft_ms for r in self.records],
                  "e2e_ms": [r.e2e_ms for r in self.records],
                  "tbt_ms": [g for r in self.records for g in r.tbt_ms()]}
        for name, vals in series.items():
            if not vals:
                continue
            for p in (0.5, 0.9, 0.99):
                out[f"{name}_p{int(p * 100)}"] = percentile(vals, p)
        return out


REQUEST_CSV_HEADER = ("request_id,arrival_s,ttft_ms,e2e_ms,prompt_machine,"
                      "token_machine,transfer_visible_ms,preempt_count")


def requests_csv(records) -> str:
    """Per-request CSV, byte-compatible with the reference's requests_csv
    (engine.py:369-379)."""
    out = [REQUEST_CSV_HEADER]
    for r in records:
        arr = r.arrival_s if r.arrival_s is not None else r.arrival_ms / 1e3
        out.append(f"{r.request_id},{arr:.6f},{r.ttft_ms:.6f},{r.e2e_ms:.6f},"
                   f"{r.prompt_machine},{r.token_machine},{r.transfer_visible_ms:.6f},"
                   f"{r.preempt_count}")
    return "\n".join(out) + "\n"


def tbt_csv(records) -> str:
    """Per-gap TBT CSV (reference engine.py:382-388)."""
    out = ["request_id,gap_index,tbt_ms"]
    for r in records:
        for i, gap in enumerate(r.tbt_ms()):
            out.append(f"{r.request_id},{i},{gap:.6f}")
    return "\n".join(out) + "\n"
