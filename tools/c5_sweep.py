"""C5-style scheduler sweep on B200 calibrations.

Phase 1 (GPU, torchrun --nproc-per-node TP): measure a PerfModel of one TP
machine of MODEL (real prefills at several prompt lengths and CUDA-graph
decode steps at several batch sizes, measure_perf_model) and write it in the
reference's profile-CSV format (rank 0).

Phase 2 (CPU, --sweep PROFILE): drive the reference request lifecycle
(driver.Driver, pinned to splitsim by the golden tests) with that PerfModel
for the Splitwise design (1 prompt + 1 token machine = 2 TP machines) and the
co-located Baseline design on the same GPU count, over a request-rate sweep
of the reference's trace preset; print TTFT / TBT / E2E percentiles and
throughput per (design, rate).  The Baseline runs are cross-checked against
the reference simulator itself fed the same profile (splitsim.Simulator).

  torchrun --nproc-per-node 4 tools/c5_sweep.py --model bloom-176b --out prof.csv
  python tools/c5_sweep.py --sweep prof.csv --preset conversation
"""
import argparse
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def measure(a):
    import torch
    import torch.distributed as dist
    from paper_2311_18677_b200.kvcache import KVCacheManager, blocks_for
    from paper_2311_18677_b200.model import get_config, init_weights
    from paper_2311_18677_b200.perf import export_profile_csv, measure_perf_model
    from paper_2311_18677_b200.runner import ModelRunner
    rank, world = int(os.environ.get("RANK", 0)), int(os.environ.get("WORLD_SIZE", 1))
    torch.cuda.set_device(int(os.environ.get("LOCAL_RANK", rank)))
    group = None
    if world > 1:
        dist.init_process_group("nccl", device_id=torch.device("cuda", torch.cuda.current_device()))
        group = dist.group.WORLD
    cfg = get_config(a.model)
    w = init_weights(cfg, seed=0, tp=world, rank=rank)
    bmax = min(cfg.max_token_batch, 32)
    kv = KVCacheManager(cfg.n_layers, bmax * blocks_for(a.context + 16, 16) + 8192 // 16 + 64,
                        cfg.n_kv_heads // world, cfg.head_dim, 16, bmax + 4,
                        blocks_for(max(8192, a.context) + 16, 16))
    runner = ModelRunner(w, kv, tp_group=group)
    batches = tuple(b for b in (1, 2, 4, 8, 16, 32) if b <= bmax)
    if bmax not in batches:
        batches += (bmax,)
    model = measure_perf_model(runner, prompt_points=(128, 512, 1024, 2048, 4096, 8192),
                               batch_points=batches, context=a.context, reps=3)
    if rank == 0:
        with open(a.out, "w") as f:
            f.write(export_profile_csv(model))
        print(json.dumps({"model": cfg.name, "tp": world, "prompt_knots": model.prompt_knots,
                          "token_knots": model.token_knots, "profile": a.out}), flush=True)
    if world > 1:
        dist.barrier()
        torch.cuda.synchronize()
        os._exit(0)        # NCCL / TP-comm teardown at exit is not needed (and can stall)


def sweep(a):
    from paper_2311_18677_b200.cluster import ClusterConfig
    from paper_2311_18677_b200.driver import Driver
    from paper_2311_18677_b200.perf import PerfModel
    from reftrace import preset_trace
    text = open(a.sweep).read()
    samples = []     # (machine_type, llm, phase, prompt_tokens, batch_size, time_ms, memory)
    for line in text.strip().splitlines()[1:]:
        f = line.split(",")
        samples.append((f[0], f[1], f[2], int(f[3]), int(f[4]), float(f[5]), float(f[6])))
    pm = [s for s in samples if s[2] == "prompt"]
    tk = [s for s in samples if s[2] == "token"]
    mtype, llm = samples[0][0], samples[0][1]
    kvb = (pm[-1][6] - pm[0][6]) / (pm[-1][3] - pm[0][3])
    weights = pm[0][6] - pm[0][3] * kvb
    model = PerfModel("B200", llm, ([s[3] for s in pm], [s[5] for s in pm]),
                      ([s[4] for s in tk], [s[5] for s in tk]), kvb, weights,
                      a.capacity_gb * 1e9, max(s[4] for s in tk))
    perf = {"B200": model}
    rows = []
    for rate in [float(r) for r in a.rates.split(",")]:
        reqs = preset_trace(a.preset, rate, a.duration, a.seed)
        for design, p, t in (("Splitwise-BB", 1, 1), ("Baseline-B200", 2, 0)):
            try:
                res = Driver(ClusterConfig(design, p, t, llm=llm), perf, reqs, record_log=False,
                             horizon_s=a.duration + 3600).run()
                s = res.report.summary()
                rows.append({"design": design, "rate": rate, "requests": len(reqs),
                             "ttft_p50": s.get("ttft_ms_p50"), "ttft_p99": s.get("ttft_ms_p99"),
                             "tbt_p50": s.get("tbt_ms_p50"), "tbt_p99": s.get("tbt_ms_p99"),
                             "e2e_p50": s.get("e2e_ms_p50"), "tokens_per_s": s["tokens_per_s"]})
            except RuntimeError as e:
                rows.append({"design": design, "rate": rate, "requests": len(reqs),
                             "unsustainable": str(e)[:80]})
    # cross-check: the reference simulator on the same profile (Baseline design)
    check = None
    try:
        sys.path.insert(0, os.path.join(ROOT, "baseline", "_ref"))
        import splitsim as ss
        rmodel, _ = ss.fit_piecewise_linear(ss.parse_profile_csv(text.replace(mtype, "H100")),
                                            memory_capacity=a.capacity_gb * 1e9)
        rate = float(a.rates.split(",")[0])
        reqs = preset_trace(a.preset, rate, a.duration, a.seed)
        tr = ss.Trace([ss.Request(r.id, r.arrival, r.prompt_tokens, r.output_tokens)
                       for r in reqs], a.duration)
        ref = ss.Simulator(ss.ClusterConfig("Baseline-H100", 2, 0), {"H100": rmodel}, tr).run()
        ours = [r for r in rows if r["design"] == "Baseline-B200" and r["rate"] == rate][0]
        rs = ref.report.summary()
        check = {"rate": rate, "reference_ttft_p50": rs.get("ttft_ms_p50"),
                 "ours_ttft_p50": ours.get("ttft_p50"),
                 "reference_tbt_p50": rs.get("tbt_ms_p50"), "ours_tbt_p50": ours.get("tbt_p50")}
    except Exception as e:  # noqa: BLE001
        check = {"unavailable": str(e)[:120]}
    print(json.dumps({"tool": "c5_sweep", "profile": a.sweep, "preset": a.preset,
                      "duration_s": a.duration, "rows": rows, "reference_check": check}))


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--model", default="bloom-176b")
    ap.add_argument("--out", default="gpurun_out/b200_profile.csv")
    ap.add_argument("--context", type=int, default=1024)
    ap.add_argument("--sweep", default="")
    ap.add_argument("--preset", default="conversation")
    ap.add_argument("--rates", default="0.5,1,2,4,6,8")
    ap.add_argument("--duration", type=float, default=120.0)
    ap.add_argument("--seed", type=int, default=0)
    ap.add_argument("--capacity-gb", type=float, default=4 * 180.0)
    a = ap.parse_args()
    if a.sweep:
        sweep(a)
    else:
        measure(a)


if __name__ == "__main__":
    main()
