"""Host-side parity with the REAL reference, through golden fixtures recorded
from it (tests/golden/make_golden.py imports /root/reference read-only).

Pinned here: the transfer planner (transfer.py:66-99), the piecewise cost
evaluation (perf.py:77-132), the machine-level scheduler (machine.py:118-275:
prompt cap, head-of-line admission, memory admission, token slots, aged
priority, preemption/parking, iteration mixing rule, completion events) and
the whole request lifecycle + JSQ routing + metrics (engine.py / cluster.py)
replayed request-for-request on the reference's own calibration presets.
"""

import json
import os

import pytest

from paper_2311_18677_b200 import transfer as T
from paper_2311_18677_b200.perf import PerfModel, piecewise_eval
from paper_2311_18677_b200.workers import Machine, SchedulerConfig, Task

GOLD = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden")


def _load(name):
    with open(os.path.join(GOLD, f"{name}.json")) as f:
        return json.load(f)


def test_transfer_plans_match_reference():
    rows = _load("transfer")
    assert len(rows) >= 100
    for r in rows:
        cfg = T.TransferConfig(**r["config"])
        plan = T.plan_transfer(r["prompt_tokens"], r["kv_bytes"], r["prompt_ms"], cfg,
                               mode=r["mode_arg"])
        assert plan.mode == r["mode"]
        assert plan.raw_time == pytest.approx(r["raw"], rel=1e-12, abs=1e-12)
        assert plan.visible_latency == pytest.approx(r["visible"], rel=1e-12, abs=1e-12)
        assert plan.overlap_hidden == pytest.approx(r["hidden"], rel=1e-12, abs=1e-9)
        assert T.select_mode(r["prompt_tokens"], cfg) == r["select"]


def test_transfer_reference_known_answers():
    # reference tests/test_transfer.py:21-25, :56-63 (H100 pair, 80 layers)
    cfg = T.TransferConfig(num_layers=80, **T.H100_PAIR)
    kv = 1500 * 2_621_440
    assert T.raw_transfer_time(kv, cfg) == pytest.approx(78.6432)
    plan = T.plan_transfer(1500, kv, 95.0, cfg)
    assert plan.mode == T.LAYERWISE and plan.visible_latency == pytest.approx(5.0)
    assert plan.overlap_hidden == pytest.approx(73.6432)
    assert T.select_mode(511, cfg) == T.SERIALIZED and T.select_mode(512, cfg) == T.LAYERWISE


def test_piecewise_cost_model_matches_reference():
    for p in _load("perf"):
        m = PerfModel(p["machine_type"], p["llm"], tuple(p["prompt_knots"]),
                      tuple(p["token_knots"]), p["kv"], p["weights"], p["capacity"],
                      p["max_batch"])
        for x, y in p["prompt_eval"]:
            assert m.prompt_time(x) == pytest.approx(y, rel=1e-12)
        for b, y in p["token_eval"]:
            assert m.token_iter_time(b) == pytest.approx(y, rel=1e-12)
        assert piecewise_eval(p["prompt_knots"][0][0], *p["prompt_knots"]) == \
            pytest.approx(p["prompt_knots"][1][0])


def _snap(m, batch):
    s = {"pending_token_count": m.pending_token_count, "memory_used": m.memory_used(),
         "resident": [[t.request_id, t.tokens, t.remaining_output, t.parked, t.preempt_count]
                      for t in m.resident],
         "pending_prompts": [t.request_id for t in m.pending_prompts],
         "pending_tokens": [t.request_id for t in m.pending_tokens_q]}
    if batch is not None:
        s["batch"] = {"prompts": [t.request_id for t in batch.prompt_tasks],
                      "tokens": [t.request_id for t in batch.token_tasks],
                      "iteration_time": batch.iteration_time, "kind": batch.kind}
    return s


def _close(a, b):
    if isinstance(a, float) or isinstance(b, float):
        return a == pytest.approx(b, rel=1e-12, abs=1e-9)
    if isinstance(a, list):
        return len(a) == len(b) and all(_close(x, y) for x, y in zip(a, b))
    if isinstance(a, dict):
        return a.keys() == b.keys() and all(_close(a[k], b[k]) for k in a)
    return a == b


@pytest.mark.parametrize("idx", range(24))
def test_machine_scheduler_replays_reference(idx):
    sc = _load("machine")[idx]
    p = sc["perf"]
    perf = PerfModel("H100", sc["llm"], tuple(p["prompt_knots"]), tuple(p["token_knots"]),
                     p["kv"], p["weights"], p["capacity"], p["max_batch"])
    sched = SchedulerConfig(**sc["sched"])
    role = sc["role"]
    m = Machine(0, None, perf, role if role != "mixed" else "prompt", sched,
                always_mixed=(role == "mixed"))
    batch = None
    for op in sc["ops"]:
        if op["op"] == "enqueue":
            m.enqueue(Task(op["request_id"], op["kind"], op["tokens"], op["now"],
                           op["output_tokens"], op["remaining_output"]), op["now"])
        elif op["op"] == "form_batch":
            batch = m.form_batch(op["now"])
            m.running = batch
            got = _snap(m, batch)
            assert _close(got, op["expect"]), (op["now"], got, op["expect"])
        else:
            ev = m.complete_iteration(batch, op["now"])
            assert [[k, t.request_id] for k, t in ev] == op["events"]
            assert _close(_snap(m, None), op["expect"])


def test_engine_lifecycle_replays_reference():
    """Full request lifecycle on the reference's calibration: every request's
    routing, TTFT, E2E, TBT gaps and visible transfer latency match."""
    from paper_2311_18677_b200.cluster import ClusterConfig
    from paper_2311_18677_b200.driver import Driver, Request
    perf = {row["machine_type"]: PerfModel(row["machine_type"], row["llm"],
                                           tuple(row["prompt_knots"]), tuple(row["token_knots"]),
                                           row["kv"], row["weights"], row["capacity"],
                                           row["max_batch"])
            for row in _load("perf") if row["llm"] == "llama2-70b"}
    runs = _load("engine")
    assert len(runs) >= 10
    for run in runs:
        reqs = [Request(r["id"], r["arrival"], r["prompt_tokens"], r["output_tokens"])
                for r in run["records"]]
        cc = ClusterConfig(run["design"], run["prompt_machines"], run["token_machines"])
        res = Driver(cc, perf, reqs, duration_s=20.0).run()
        for r in run["records"]:
            got = res.records[r["id"]]
            assert (got.prompt_machine, got.token_machine) == (r["prompt_machine"],
                                                               r["token_machine"])
            assert got.ttft_ms == pytest.approx(r["ttft_ms"], abs=1e-6)
            assert got.e2e_ms == pytest.approx(r["e2e_ms"], abs=1e-6)
            assert got.tbt_ms() == pytest.approx(r["tbt_ms"], abs=1e-6)
            assert got.transfer_visible_ms == pytest.approx(r["transfer_visible_ms"], abs=1e-9)
            assert got.preempt_count == r["preempt_count"]
        s = res.report.summary()
        for k in ("ttft_ms_p50", "ttft_ms_p99", "e2e_ms_p50", "tbt_ms_p50", "tbt_ms_p99"):
            if k in run["summary"]:
                assert s[k] == pytest.approx(run["summary"][k], abs=1e-6), k
