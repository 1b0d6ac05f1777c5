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


def _csv_runs():
    with open(os.path.join(HERE, "golden", "csv.json")) as f:
        return json.load(f)


def test_trace_csv_round_trip_matches_reference():
    from paper_2311_18677_b200.trace import parse_trace, serialize_trace
    for run in _csv_runs():
        tr = preset_trace(run["preset"], run["rate"], run["duration"], run["seed"])
        assert serialize_trace(tr) == run["trace_csv"]
        parsed = parse_trace(run["trace_csv"])      # arrivals carry the CSV's 6 decimals
        assert parsed == [type(r)(r.id, float(f"{r.arrival:.6f}"), r.prompt_tokens,
                                  r.output_tokens) for r in tr]


def test_request_and_tbt_csv_match_reference():
    """The driver (reference lifecycle, H100 calibration) emits the same
    requests / TBT CSV text as the reference simulator (engine.py:369-388)."""
    from paper_2311_18677_b200.cluster import ClusterConfig
    from paper_2311_18677_b200.driver import Driver
    from paper_2311_18677_b200.metrics import requests_csv, tbt_csv
    from paper_2311_18677_b200.perf import PerfModel
    with open(os.path.join(HERE, "golden", "perf.json")) as f:
        perf = {row["machine_type"]: PerfModel(row["machine_type"], row["llm"],
                                               tuple(row["prompt_knots"]),
                                               tuple(row["token_knots"]), row["kv"],
                                               row["weights"], row["capacity"], row["max_batch"])
                for row in json.load(f) if row["llm"] == "llama2-70b"}
    for run in _csv_runs():
        tr = preset_trace(run["preset"], run["rate"], run["duration"], run["seed"])
        cc = ClusterConfig(run["design"], run["prompt_machines"], run["token_machines"])
        res = Driver(cc, perf, tr, duration_s=run["duration"]).run()
        recs = [res.records[r.id] for r in tr]
        assert requests_csv(recs) == run["requests_csv"]
        assert tbt_csv(recs) == run["tbt_csv"]


def test_parse_trace_rejects_bad_input():
    from paper_2311_18677_b200.errors import ValidationError
    from paper_2311_18677_b200.trace import parse_trace
    for bad in ("", "a,b,c\n1,2,3", "arrival_s,prompt_tokens,output_tokens\n1,0,3",
                "arrival_s,prompt_tokens,output_tokens\n-1,2,3",
                "arrival_s,prompt_tokens,output_tokens\n1,2"):
        with pytest.raises(ValidationError):
            parse_trace(bad)
    tr = parse_trace("arrival_s,prompt_tokens,output_tokens\n2.0,5,6\n\n1.0,7,8\n")
    assert [(r.id, r.arrival, r.prompt_tokens) for r in tr] == [(0, 1.0, 7), (1, 2.0, 5)]
