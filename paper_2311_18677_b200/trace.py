"""Synthetic request traces with the reference's workload presets.

Restates the reference generator (reference trace.py:69-153, :156-157,
:215-243) so the GPU serving runs use the same request shapes as the
reference simulator without importing it on the GPU box:

* arrivals: Poisson — i.i.d. exponential gaps with mean 1/rate, drawn in
  chunks of max(256, int(0.2 * rate * duration) + 1) from a Philox(seed)
  generator until the cumulative time passes ``duration``;
* sizes: drawn after all arrivals — first every prompt size, then every
  output size — each rounded to an integer and clamped to its support
  (the clamped draws are counted, not resampled);
* presets (medians of the production traces the paper characterises):
  coding prompt lognormal(ln 1500, 1.1) in [512, 8192], output
  lognormal(ln 13, 0.8) in [1, 1000]; conversation prompt
  lognormal(ln 1020, 1.1) in [256, 8192], output a two-component lognormal
  mixture, component 2 (ln 320, 0.7) with probability 0.55 else (ln 20, 0.8),
  in [1, 4096].

The draw order is what pins a seed to a trace; tests/test_trace.py checks this
module request-for-request against traces the real reference produced
(tests/golden/engine.json).
"""

from __future__ import annotations

import math
from dataclasses import dataclass

import numpy as np

from .driver import Request
from .errors import ValidationError


@dataclass(frozen=True)
class SizeDistribution:
    kind: str                 # "lognormal" | "bimodal-lognormal"
    params: tuple
    min_tokens: int = 1
    max_tokens: int = 1 << 20

    def sample(self, rng: np.random.Generator, n: int) -> tuple[np.ndarray, int]:
        if n == 0:
            return np.zeros(0, dtype=np.int64), 0
        if self.kind == "lognormal":
            mu, sigma = self.params
            raw = rng.lognormal(mu, sigma, n)
        elif self.kind == "bimodal-lognormal":
            w2, mu1, s1, mu2, s2 = self.params
            second = rng.random(n) < w2
            c2 = rng.lognormal(mu2, s2, n)        # both components are drawn,
            c1 = rng.lognormal(mu1, s1, n)        # component 2 first
            raw = np.where(second, c2, c1)
        else:
            raise ValidationError(f"unknown size distribution {self.kind!r}")
        vals = np.rint(raw).astype(np.int64)
        clamped = int(np.count_nonzero((vals < self.min_tokens) | (vals > self.max_tokens)))
        return np.clip(vals, self.min_tokens, self.max_tokens), clamped


PRESETS = {
    "coding": {
        "prompt": SizeDistribution("lognormal", (math.log(1500), 1.1), 512, 8192),
        "output": SizeDistribution("lognormal", (math.log(13), 0.8), 1, 1000),
    },
    "conversation": {
        "prompt": SizeDistribution("lognormal", (math.log(1020), 1.1), 256, 8192),
        "output": SizeDistribution("bimodal-lognormal",
                                   (0.55, math.log(20), 0.8, math.log(320), 0.7), 1, 4096),
    },
}


def generate_trace(prompt_dist: SizeDistribution, output_dist: SizeDistribution, rate: float,
                   duration: float, seed: int) -> list[Request]:
    """Poisson-arrival requests over ``duration`` seconds (ids in arrival order)."""
    if rate < 0:
        raise ValidationError("rate must be >= 0")
    if duration <= 0:
        raise ValidationError("duration must be > 0")
    rng = np.random.Generator(np.random.Philox(seed))
    arrivals: list[float] = []
    if rate > 0:
        t = 0.0
        chunk_n = max(256, int(rate * duration * 0.2) + 1)
        while True:
            cum = t + np.cumsum(rng.exponential(1.0 / rate, size=chunk_n))
            inside = cum[cum <= duration]
            arrivals.extend(inside.tolist())
            if len(inside) < len(cum):
                break
            t = cum[-1]
    n = len(arrivals)
    prompts, _ = prompt_dist.sample(rng, n)
    outputs, _ = output_dist.sample(rng, n)
    return [Request(i, arrivals[i], int(prompts[i]), int(outputs[i])) for i in range(n)]


TRACE_HEADER = "arrival_s,prompt_tokens,output_tokens"


def serialize_trace(requests: list[Request]) -> str:
    """The reference's three-column trace CSV (trace.py:206-212)."""
    lines = [TRACE_HEADER] + [f"{r.arrival:.6f},{r.prompt_tokens},{r.output_tokens}"
                              for r in requests]
    return "\n".join(lines) + "\n"


def parse_trace(text: str) -> list[Request]:
    """Parse the trace CSV (reference trace.py:160-203): header checked, blank
    lines skipped, counts >= 1, arrivals >= 0, stable-sorted by arrival and
    re-numbered in that order."""
    lines = text.strip().splitlines()
    if not lines:
        raise ValidationError("empty trace")
    if lines[0].strip() != TRACE_HEADER:
        raise ValidationError(f"line 1: expected header {TRACE_HEADER!r}, got {lines[0]!r}")
    rows = []
    for i, line in enumerate(lines[1:], start=2):
        if not line.strip():
            continue
        parts = line.split(",")
        if len(parts) != 3:
            raise ValidationError(f"line {i}: expected 3 fields, got {len(parts)}")
        try:
            arrival, prompt, output = float(parts[0]), int(parts[1]), int(parts[2])
        except ValueError as exc:
            raise ValidationError(f"line {i}: {exc}") from None
        if prompt < 1 or output < 1:
            raise ValidationError(f"line {i}: non-positive token count")
        if arrival < 0:
            raise ValidationError(f"line {i}: negative arrival")
        rows.append((arrival, prompt, output))
    if not rows:
        raise ValidationError("empty trace")
    order = sorted(range(len(rows)), key=lambda k: rows[k][0])
    return [Request(rid, *rows[k]) for rid, k in enumerate(order)]


def preset_trace(preset: str, rate: float, duration: float, seed: int) -> list[Request]:
    if preset not in PRESETS:
        raise ValidationError(f"unknown preset {preset!r} (have {sorted(PRESETS)})")
    p = PRESETS[preset]
    return generate_trace(p["prompt"], p["output"], rate, duration, seed)


__all__ = ["SizeDistribution", "PRESETS", "TRACE_HEADER", "generate_trace", "preset_trace",
           "serialize_trace", "parse_trace"]
