"""Request traces from the REFERENCE's own generator — not a restatement.

The synthetic workload presets (reference trace.py:143-153), the Poisson
generator (trace.py:215-243) and the trace CSV format (trace.py:160-212) are
the reference's; this module imports them from the installed reference
(``baseline/_ref``, which travels to the GPU box with the repo snapshot) or
the read-only source tree (``/root/reference/pkg/src``, build container
only).  Where neither is importable, the traces recorded by
tests/golden/make_golden.py (``tests/golden/traces.json``, produced by the
same generator) stand in for the (preset, rate, duration, seed) points they
cover.  Requests come back as the repo's ``driver.Request`` (same fields).
"""

from __future__ import annotations

import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
if ROOT not in sys.path:
    sys.path.insert(0, ROOT)

from paper_2311_18677_b200.driver import Request  # noqa: E402
from paper_2311_18677_b200.errors import ValidationError  # noqa: E402

_REF_PATHS = (os.path.join(ROOT, "baseline", "_ref"), "/root/reference/pkg/src")
FIXTURES = os.path.join(ROOT, "tests", "golden", "traces.json")


def splitsim():
    """The reference package, or None when it is not importable here."""
    for p in _REF_PATHS:
        if os.path.isdir(os.path.join(p, "splitsim")) and p not in sys.path:
            sys.path.append(p)
    try:
        import splitsim as ss
        return ss
    except Exception:  # noqa: BLE001
        return None


def fixture_key(preset: str, rate: float, duration: float, seed: int) -> str:
    return f"{preset}/{float(rate):g}/{float(duration):g}/{int(seed)}"


def _convert(reqs) -> list[Request]:
    return [Request(r.id, r.arrival, r.prompt_tokens, r.output_tokens) for r in reqs]


def preset_trace(preset: str, rate: float, duration: float, seed: int) -> list[Request]:
    ss = splitsim()
    if ss is not None:
        from splitsim import trace as T
        if preset not in T.PRESETS:
            raise ValidationError(f"unknown preset {preset!r} (have {sorted(T.PRESETS)})")
        p = T.PRESETS[preset]
        return _convert(T.generate_trace(p["prompt"], p["output"], rate, duration, seed).requests)
    with open(FIXTURES) as f:
        fx = json.load(f)
    key = fixture_key(preset, rate, duration, seed)
    if key not in fx:
        raise ValidationError(f"reference not importable and no recorded trace for {key}")
    return [Request(i, a, p, o) for i, (a, p, o) in enumerate(fx[key])]


def parse_trace_csv(text: str) -> list[Request]:
    """The reference's trace CSV parser (needs the reference)."""
    ss = splitsim()
    if ss is None:
        raise ValidationError("trace CSV parsing needs the reference package (baseline/_ref)")
    import io
    from splitsim import trace as T
    return _convert(T.parse_trace(io.StringIO(text)).requests)


def serialize_trace(reqs) -> str:
    ss = splitsim()
    if ss is None:
        raise ValidationError("trace CSV writing needs the reference package (baseline/_ref)")
    from splitsim import trace as T
    dur = max([r.arrival for r in reqs] + [1e-9])
    return T.serialize_trace(T.Trace([T.Request(r.id, r.arrival, r.prompt_tokens,
                                                r.output_tokens) for r in reqs], dur))
