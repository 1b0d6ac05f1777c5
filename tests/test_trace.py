"""The trace generator reproduces the reference's traces request-for-request
(tests/golden/engine.json was produced by the real splitsim.generate_trace,
reference trace.py:215-243, with the seeds / rates below)."""
import json
import os

import pytest

from paper_2311_18677_b200.trace import PRESETS, generate_trace, preset_trace

HERE = os.path.dirname(os.path.abspath(__file__))
LAYOUTS = 6   # make_golden.gen_engine: seed = 7 + layout index, 20 s traces


def _golden_runs():
    with open(os.path.join(HERE, "golden", "engine.json")) as f:
        runs = json.load(f)
    return [r for r in runs if r["preset"] in PRESETS]


def test_matches_reference_traces():
    runs = _golden_runs()
    assert len(runs) == 2 * LAYOUTS
    for i, run in enumerate(runs):
        seed = 7 + i // 2
        got = preset_trace(run["preset"], run["rate"], 20.0, seed)
        want = sorted(run["records"], key=lambda r: r["id"])
        assert len(got) == len(want), (run["preset"], seed)
        for g, w in zip(got, want):
            assert g.id == w["id"]
            assert g.arrival == pytest.approx(w["arrival"], abs=1e-12)
            assert (g.prompt_tokens, g.output_tokens) == (w["prompt_tokens"], w["output_tokens"])


def test_support_clamps_and_rate():
    tr = preset_trace("coding", 50.0, 20.0, 3)
    assert all(512 <= r.prompt_tokens <= 8192 and 1 <= r.output_tokens <= 1000 for r in tr)
    assert 800 < len(tr) < 1200
    tr = preset_trace("conversation", 50.0, 20.0, 3)
    assert all(256 <= r.prompt_tokens <= 8192 and 1 <= r.output_tokens <= 4096 for r in tr)
    assert [r.arrival for r in tr] == sorted(r.arrival for r in tr)
    assert generate_trace(PRESETS["coding"]["prompt"], PRESETS["coding"]["output"], 0.0, 5.0, 1) == []
