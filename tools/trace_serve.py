"""Trace-driven serving on B200s: the reference's request lifecycle and
scheduler (driver.Driver, pinned to splitsim by the golden tests) with every
prompt / token iteration and KV push executed on the GPUs of this process
(gpu_backend.GpuBackend), over a synthetic trace of the reference's presets
(trace.py: conversation / coding, Poisson arrivals).  Prints one JSON line:
TTFT / TBT / E2E p50-p99, tokens/s, machine utilisation, KV-transfer visible
latency, and the same trace priced by the PerfModel lookups (ModeledBackend
with the B200 roofline estimates) and by the reference simulator's H100
calibration for comparison.

  python tools/trace_serve.py --design Splitwise-BB --prompt-machines 1 \\
      --token-machines 1 --preset conversation --rate 2 --duration 20
"""
import argparse, json, os, statistics, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402
from paper_2311_18677_b200.cluster import ClusterConfig  # noqa: E402
from paper_2311_18677_b200.driver import Driver  # noqa: E402
from paper_2311_18677_b200.gpu_backend import GpuBackend  # noqa: E402
from reftrace import preset_trace  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--model", default="llama2-7b")
    ap.add_argument("--design", default="Splitwise-BB")
    ap.add_argument("--prompt-machines", type=int, default=1)
    ap.add_argument("--token-machines", type=int, default=1)
    ap.add_argument("--preset", default="conversation")
    ap.add_argument("--rate", type=float, default=2.0)
    ap.add_argument("--duration", type=float, default=20.0)
    ap.add_argument("--seed", type=int, default=0)
    ap.add_argument("--clock", default="measured", choices=["measured", "modeled"])
    ap.add_argument("--no-mixed", action="store_true",
                    help="run mixed batches as prefill then decode (no fused step)")
    ap.add_argument("--trace-csv", default="", help="replay this trace CSV instead of a preset")
    ap.add_argument("--out-dir", default="", help="write requests.csv / tbt.csv / trace.csv here")
    ap.add_argument("--max-output", type=int, default=0,
                    help="clamp output lengths (0 = preset support)")
    a = ap.parse_args()
    if a.trace_csv:
        from reftrace import parse_trace_csv as parse_trace
        with open(a.trace_csv) as f:
            reqs = parse_trace(f.read())
        a.preset, a.duration = os.path.basename(a.trace_csv), max(r.arrival for r in reqs) or 1.0
    else:
        reqs = preset_trace(a.preset, a.rate, a.duration, a.seed)
    if a.max_output:
        from paper_2311_18677_b200.driver import Request
        reqs = [Request(r.id, r.arrival, r.prompt_tokens, min(r.output_tokens, a.max_output))
                for r in reqs]
    backend = GpuBackend(a.model, clock=a.clock, mixed=not a.no_mixed)
    cc = ClusterConfig(a.design, a.prompt_machines, a.token_machines, llm=a.model)
    t0 = time.perf_counter()
    drv = Driver(cc, backend.perf_models(), reqs, backend=backend, record_log=False,
                 horizon_s=a.duration + 3600)
    setup = time.perf_counter() - t0
    t0 = time.perf_counter()
    from paper_2311_18677_b200.gpu_backend import PoolExhausted
    try:
        res = drv.run()
    except PoolExhausted as e:
        done = [r for r in drv.records.values() if r.completion is not None]
        print(json.dumps({"tool": "trace_serve", "model": a.model, "design": cc.design,
                          "machines": {"prompt": a.prompt_machines, "token": a.token_machines},
                          "trace": {"preset": a.preset, "rate": a.rate, "duration_s": a.duration,
                                    "seed": a.seed, "requests": len(reqs)},
                          "sustainable": False, "reason": str(e),
                          "completed_before": len(done)}), flush=True)
        return
    wall = time.perf_counter() - t0
    s = res.report.summary()
    if a.out_dir:
        from paper_2311_18677_b200.metrics import requests_csv, tbt_csv
        from reftrace import serialize_trace
        os.makedirs(a.out_dir, exist_ok=True)
        recs_sorted = [res.records[r.id] for r in reqs]
        for name, text in (("requests.csv", requests_csv(recs_sorted)),
                           ("tbt.csv", tbt_csv(recs_sorted)), ("trace.csv", serialize_trace(reqs))):
            with open(os.path.join(a.out_dir, name), "w") as f:
                f.write(text)
    recs = res.report.records
    vis = [r.transfer_visible_ms for r in recs if r.token_machine != r.prompt_machine
           and r.output_tokens > 1]
    raw = [r.transfer_raw_ms for r in recs if r.token_machine != r.prompt_machine
           and r.output_tokens > 1]
    pl = [x for x in backend.iter_log if x[1] in ("prompt", "mixed")]
    tl = [x for x in backend.iter_log if x[1] == "token"]
    out = {"tool": "trace_serve", "model": a.model, "design": cc.design,
           "machines": {"prompt": a.prompt_machines, "token": a.token_machines},
           "gpus": torch.cuda.device_count(), "trace": {"preset": a.preset, "rate": a.rate,
           "duration_s": a.duration, "seed": a.seed, "requests": len(reqs),
           "max_output": a.max_output or None},
           "sustainable": True, "summary": s, "utilization": res.report.utilization,
           "kv_transfer": {"visible_ms_p50": statistics.median(vis) if vis else None,
                           "raw_ms_p50": statistics.median(raw) if raw else None},
           "iterations": {"prompt": len(pl), "token": len(tl),
                          "mixed": sum(1 for x in backend.iter_log if x[1] == "mixed"),
                          "prompt_tokens_mean": statistics.mean(x[2] for x in pl) if pl else 0,
                          "decode_batch_mean": statistics.mean(x[2] for x in tl) if tl else 0,
                          "decode_ms_mean": statistics.mean(x[3] for x in tl) if tl else 0},
           "clock": "virtual ms clock advanced by measured device times (CUDA events)",
           "wall_s": wall, "setup_s": setup}
    print(json.dumps(out), flush=True)


if __name__ == "__main__":
    main()
