"""Generate golden fixtures from the REAL reference (splitsim), imported
read-only from /root/reference/pkg/src in the build container.

The reference cannot travel to the GPU box, so its observable behaviour on
the hot path's scheduling/transfer semantics is recorded here as JSON and
replayed by tests/test_reference_parity.py against this repo's host code:

  transfer.json  plan_transfer / select_mode / raw_transfer_time over a grid
                 (reference transfer.py:66-99)
  perf.json      calibration knots + _piecewise_eval at interior/edge/
                 extrapolated points (perf.py:77-88, :297-350)
  machine.json   randomized enqueue / form_batch / complete_iteration scripts
                 on prompt, token and mixed machines (machine.py:118-275)
  engine.json    full Simulator runs (engine.py:160-358) on small traces:
                 per-request TTFT/E2E/TBT, routing, transfer visible latency
  csv.json       the reference's trace CSV / requests_csv / tbt_csv text for
                 two runs (engine.py:369-391, trace.py:206-212)
  traces.json    the reference generator's preset traces (trace.py:143-153,
                 :215-243) at the (preset, rate, duration, seed) points the GPU
                 tests and bench --trace use, for boxes where the installed
                 reference (baseline/_ref) is absent (tools/reftrace.py)

Run:  python tests/golden/make_golden.py [name ...]   (needs /root/reference)
"""

from __future__ import annotations

import json
import os
import random
import sys

REF = "/root/reference/pkg/src"
HERE = os.path.dirname(os.path.abspath(__file__))


def load_ref():
    if REF not in sys.path:
        sys.path.insert(0, REF)
    import splitsim  # noqa: F401
    from splitsim import cluster, engine, machine, perf, trace, transfer
    return cluster, engine, machine, perf, trace, transfer


def gen_transfer(transfer):
    out = []
    rng = random.Random(1)
    cfgs = [dict(transfer.H100_PAIR, num_layers=80), dict(transfer.A100_PAIR, num_layers=70),
            dict(bandwidth=6.16e12, mode_threshold_tokens=33, layerwise_constant_ms=0.05,
                 num_layers=32)]
    for c in cfgs:
        tc = transfer.TransferConfig(**c)
        for _ in range(60):
            p = rng.choice([1, 2, 31, 32, 33, 511, 512, 513, 1023, 1024, 1500, 4096, 8192,
                            rng.randint(1, 9000)])
            kv = p * rng.choice([2621440.0, 327680.0, 524288.0, 4014080.0])
            pm = rng.choice([0.0, 5.0, 84.0, 95.0, 250.0, rng.uniform(0, 400)])
            mode = rng.choice([None, None, "serialized", "layerwise"])
            plan = transfer.plan_transfer(p, kv, pm, tc, mode=mode)
            out.append({"config": c, "prompt_tokens": p, "kv_bytes": kv, "prompt_ms": pm,
                        "mode_arg": mode, "mode": plan.mode, "raw": plan.raw_time,
                        "visible": plan.visible_latency, "hidden": plan.overlap_hidden,
                        "select": transfer.select_mode(p, tc)})
    return out


def gen_perf(perf):
    out = []
    for llm in perf.LLMS:
        for mt in ("A100", "H100", "H100cap"):
            m = perf.get_calibration(llm, mt)
            pts_p = [1, 2, 64, 128, 700, 1020, 1500, 2048, 3000, 8192, 10000]
            pts_t = sorted({1, 2, 3, 17, min(32, m.max_token_batch), m.max_token_batch})
            out.append({
                "llm": llm, "machine_type": mt,
                "prompt_knots": [list(map(float, m.prompt_knots[0])), list(map(float, m.prompt_knots[1]))],
                "token_knots": [list(map(float, m.token_knots[0])), list(map(float, m.token_knots[1]))],
                "kv": m.kv_bytes_per_token, "weights": m.weight_memory,
                "capacity": m.memory_capacity, "max_batch": m.max_token_batch,
                "prompt_eval": [[x, m.prompt_time(x)] for x in pts_p],
                "token_eval": [[b, m.token_iter_time(b)] for b in pts_t],
            })
    return out


def _snap_machine(m, batch):
    snap = {"pending_token_count": m.pending_token_count,
            "memory_used": m.memory_used(),
            "resident": [[t.request_id, t.tokens, t.remaining_output, t.parked, t.preempt_count]
                         for t in m.resident],
            "pending_prompts": [t.request_id for t in m.pending_prompts],
            "pending_tokens": [t.request_id for t in m.pending_tokens_q]}
    if batch is not None:
        snap["batch"] = {"prompts": [t.request_id for t in batch.prompt_tasks],
                         "tokens": [t.request_id for t in batch.token_tasks],
                         "iteration_time": batch.iteration_time, "kind": batch.kind}
    return snap


def gen_machine(machine, perf):
    scripts = []
    for seed in range(24):
        rng = random.Random(100 + seed)
        role = ["prompt", "token", "mixed"][seed % 3]
        llm = "llama2-70b" if seed % 2 == 0 else "bloom-176b"
        pm = perf.get_calibration(llm, "H100")
        cap_scale = rng.choice([1.0, 0.5, 0.47])   # squeeze memory to hit admission limits
        pm = perf.PerfModel(pm.machine_type, pm.llm, pm.prompt_knots, pm.token_knots,
                            pm.kv_bytes_per_token, pm.weight_memory,
                            pm.weight_memory + (pm.memory_capacity - pm.weight_memory) * cap_scale,
                            pm.max_token_batch)
        sched = machine.SchedulerConfig(prompt_token_cap=rng.choice([2048, 1024, 4096]),
                                        max_preemptions=rng.choice([1, 2, 4]),
                                        mixing_rule=rng.choice(["sum", "max"]))
        m = machine.Machine(0, perf.MACHINE_SPECS["H100"], pm,
                            home_role=role if role != "mixed" else "prompt", sched=sched,
                            always_mixed=(role == "mixed"))
        ops, now, rid = [], 0.0, 0
        for step in range(60):
            now += rng.choice([0.0, 1.0, 5.0, 31.0])
            for _ in range(rng.choice([0, 0, 1, 2, 3])):
                kind = "prompt" if (role == "prompt" or (role == "mixed" and rng.random() < 0.5)) \
                    else "token"
                out_tok = rng.choice([1, 2, 5, 13, 129, 400])
                if kind == "prompt":
                    t = machine.Task(rid, "prompt", rng.choice([64, 512, 1020, 1500, 2048, 3000,
                                                                rng.randint(1, 8192)]),
                                     now, out_tok, out_tok)
                else:
                    p = rng.choice([100, 1020, 1500, 4000, rng.randint(1, 8192)])
                    t = machine.Task(rid, "token", p + 1, now, out_tok, max(1, out_tok - 1))
                m.enqueue(t, now)
                ops.append({"op": "enqueue", "now": now, "request_id": rid, "kind": kind,
                            "tokens": t.tokens, "output_tokens": t.output_tokens,
                            "remaining_output": t.remaining_output})
                rid += 1
            if m.running is None and m.has_work():
                b = m.form_batch(now)
                m.running = b
                ops.append({"op": "form_batch", "now": now, "expect": _snap_machine(m, b)})
                if b is not None:
                    now += b.iteration_time
                    ev = m.complete_iteration(b, now)
                    ops.append({"op": "complete", "now": now,
                                "events": [[k, t.request_id] for k, t in ev],
                                "expect": _snap_machine(m, None)})
        scripts.append({"seed": seed, "role": role, "llm": llm, "cap_scale": cap_scale,
                        "perf": {"prompt_knots": [list(map(float, pm.prompt_knots[0])),
                                                  list(map(float, pm.prompt_knots[1]))],
                                 "token_knots": [list(map(float, pm.token_knots[0])),
                                                 list(map(float, pm.token_knots[1]))],
                                 "kv": pm.kv_bytes_per_token, "weights": pm.weight_memory,
                                 "capacity": pm.memory_capacity, "max_batch": pm.max_token_batch},
                        "sched": {"prompt_token_cap": sched.prompt_token_cap,
                                  "max_preemptions": sched.max_preemptions,
                                  "mixing_rule": sched.mixing_rule},
                        "ops": ops})
    return scripts


def gen_engine(engine, cluster, perf, trace):
    runs = []
    perfs = {"H100": perf.get_calibration("llama2-70b", "H100"),
             "A100": perf.get_calibration("llama2-70b", "A100")}
    layouts = [("Baseline-H100", 1, 0), ("Splitwise-HH", 1, 1), ("Splitwise-HH", 2, 2),
               ("Splitwise-AA", 2, 1), ("Baseline-H100", 4, 0), ("Splitwise-HA", 3, 2)]
    for i, (design, p, t) in enumerate(layouts):
        for preset, rate in (("coding", 2.0), ("conversation", 1.0)):
            pd, od = trace.PRESETS[preset]["prompt"], trace.PRESETS[preset]["output"]
            tr = trace.generate_trace(pd, od, rate, 20.0, seed=7 + i)
            cc = cluster.ClusterConfig(design, p, t)
            res = engine.Simulator(cc, perfs, tr).run()
            recs = []
            for r in res.report.records:
                recs.append({"id": r.request.id, "arrival": r.request.arrival,
                             "prompt_tokens": r.request.prompt_tokens,
                             "output_tokens": r.request.output_tokens,
                             "prompt_machine": r.prompt_machine, "token_machine": r.token_machine,
                             "ttft_ms": r.ttft_ms, "e2e_ms": r.e2e_ms, "tbt_ms": r.tbt_ms(),
                             "transfer_visible_ms": r.transfer_visible_ms,
                             "preempt_count": r.preempt_count})
            runs.append({"design": design, "prompt_machines": p, "token_machines": t,
                         "preset": preset, "rate": rate, "records": recs,
                         "summary": res.report.summary()})
    # the reference's single-request oracle (tests/test_acceptance.py:89-97)
    tr = trace.Trace([trace.Request(0, 0.0, 1500, 13)], 1.0)
    res = engine.Simulator(cluster.ClusterConfig("Baseline-H100", 1, 0), perfs, tr).run()
    r = res.report.records[0]
    runs.append({"design": "Baseline-H100", "prompt_machines": 1, "token_machines": 0,
                 "preset": "single-1500-13", "rate": 0, "records": [
                     {"id": 0, "arrival": 0.0, "prompt_tokens": 1500, "output_tokens": 13,
                      "prompt_machine": 0, "token_machine": 0, "ttft_ms": r.ttft_ms,
                      "e2e_ms": r.e2e_ms, "tbt_ms": r.tbt_ms(), "transfer_visible_ms": 0.0,
                      "preempt_count": 0}], "summary": res.report.summary()})
    return runs


def gen_csv(engine, cluster, perf, trace):
    """Reference CSV outputs (trace CSV, requests_csv, tbt_csv, engine.py:369-391;
    trace.py:206-212) for two runs, compared as exact strings."""
    perfs = {"H100": perf.get_calibration("llama2-70b", "H100"),
             "A100": perf.get_calibration("llama2-70b", "A100")}
    out = []
    for design, p, t, preset, rate, seed in (("Splitwise-HH", 2, 2, "coding", 2.0, 21),
                                             ("Baseline-H100", 2, 0, "conversation", 1.0, 22)):
        pd, od = trace.PRESETS[preset]["prompt"], trace.PRESETS[preset]["output"]
        tr = trace.generate_trace(pd, od, rate, 15.0, seed=seed)
        res = engine.Simulator(cluster.ClusterConfig(design, p, t), perfs, tr).run()
        out.append({"design": design, "prompt_machines": p, "token_machines": t,
                    "preset": preset, "rate": rate, "seed": seed, "duration": 15.0,
                    "trace_csv": trace.serialize_trace(tr),
                    "requests_csv": engine.requests_csv(res), "tbt_csv": engine.tbt_csv(res)})
    return out


TRACE_POINTS = ([(pr, rate, dur, 0) for pr in ("conversation", "coding")
                 for rate in (1.0, 2.0, 4.0, 8.0, 16.0, 24.0) for dur in (15.0, 20.0, 60.0)]
                + [("conversation", 20.0, 1.0, 5), ("conversation", 20.0, 2.0, 0),
                   ("conversation", 40.0, 2.0, 0)])


def gen_traces(trace):
    out = {}
    for preset, rate, dur, seed in TRACE_POINTS:
        pd, od = trace.PRESETS[preset]["prompt"], trace.PRESETS[preset]["output"]
        tr = trace.generate_trace(pd, od, rate, dur, seed=seed)
        out[f"{preset}/{rate:g}/{dur:g}/{seed}"] = [[r.arrival, r.prompt_tokens, r.output_tokens]
                                                    for r in tr.requests]
    return out


def main():
    cluster, engine, machine, perf, trace, transfer = load_ref()
    gens = {"transfer": lambda: gen_transfer(transfer), "perf": lambda: gen_perf(perf),
            "machine": lambda: gen_machine(machine, perf),
            "engine": lambda: gen_engine(engine, cluster, perf, trace),
            "csv": lambda: gen_csv(engine, cluster, perf, trace),
            "traces": lambda: gen_traces(trace)}
    names = sys.argv[1:] or list(gens)
    fixtures = {n: gens[n]() for n in names}
    for name, data in fixtures.items():
        with open(os.path.join(HERE, f"{name}.json"), "w") as f:
            json.dump(data, f, separators=(",", ":"))
        print(name, len(data))


if __name__ == "__main__":
    main()
