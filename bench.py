#!/usr/bin/env python
"""Benchmark of the Splitwise hot path on B200 (BASELINE.json metric:
TTFT/TBT p50,p99 + tokens/s at 1/2/4/8 B200; KV-transfer GB/s vs NVLink).

Workload (BASELINE configs[1]): Llama-2-7B-shaped random-init bf16 model,
requests with a 1024-token prompt and 128 greedy output tokens.  A "step" is
one burst of N requests (one per GPU) served end to end:
  N = 1 : one GPU runs both phases (co-located baseline, Baseline design);
  N >= 2: N/2 Splitwise pairs (1 prompt GPU + 1 token GPU each); every pair
          serves 2 requests: prefill on the prompt GPU, layer-wise KV push over
          NVLink into the token GPU's paged blocks, batched decode there.
Weak scaling: work per GPU is fixed as N grows.

value : output tokens/s of the whole job with prompts already in HBM
        (device-timed with CUDA events, max over ranks);
e2e   : same metric through the public API with host prompts (pinned)
        copied in and every generated token copied out inside the timed
        region; TTFT / TBT percentiles come from this run.
Inputs: the weights (13.5 GB) exceed L2 (126 MB) many times over, so every
step streams them from HBM (no L2 flush needed).

`--impl reference` times the reference's CPU path: the reference package
(`splitsim`) has no model arithmetic, so its CPU implementation of the path
is the fp32 port in oracle/ (numerics oracle), run on all host cores over ONE
full request of the workload (all 32 layers, prompt phase and every decode
iteration timed, nothing scaled); the splitsim simulator's *modeled* H100
latencies for the same request are attached from baseline/_ref.
`--gpus N` (N > 1) without torchrun re-launches itself under
torch.distributed.run with N local ranks.
"""

from __future__ import annotations

import argparse
import json
import math
import os
import statistics
import subprocess
import sys
import threading
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

NVLINK_PEER_GBS = 770.0  # measured peer copy per direction (B200_PROFILING.md)


def _peaks():
    p = os.path.join(ROOT, "MEASURED_PEAKS.json")
    try:
        with open(p) as f:
            d = json.load(f)
        return d["hbm_gbs"], d["bf16_tflops"], d.get("bf16_tflops_sustained"), "measured"
    except Exception:
        return 6650.0, 1590.0, 1400.0, "fallback"


def percentile(samples, p):
    """Nearest-rank percentile (reference engine.py:35-42)."""
    s = sorted(samples)
    return s[max(0, math.ceil(p * len(s)) - 1)] if s else None


class ClockSampler:
    """nvidia-smi clocks/throttle reasons sampled during the timed region."""

    Q = ("clocks.sm,clocks.max.sm,clocks_event_reasons.hw_slowdown,"
         "clocks_event_reasons.hw_thermal_slowdown,clocks_event_reasons.sw_thermal_slowdown,"
         "clocks_event_reasons.sw_power_cap")

    def __init__(self, index=0):
        self.index = index
        self.samples = []
        self._stop = threading.Event()
        self._t = None

    def _run(self):
        while not self._stop.is_set():
            try:
                out = subprocess.run(
                    ["nvidia-smi", f"--id={self.index}", f"--query-gpu={self.Q}",
                     "--format=csv,noheader,nounits"], capture_output=True, text=True,
                    timeout=5).stdout.strip()
                if out:
                    self.samples.append([x.strip() for x in out.split(",")])
            except Exception:
                pass
            self._stop.wait(0.2)

    def __enter__(self):
        self._t = threading.Thread(target=self._run, daemon=True)
        self._t.start()
        return self

    def __exit__(self, *a):
        self._stop.set()
        self._t.join(timeout=10)

    def summary(self):
        if not self.samples:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["unsampled"]}
        sm = [float(s[0]) for s in self.samples if s[0].replace(".", "").isdigit()]
        mx = [float(s[1]) for s in self.samples if s[1].replace(".", "").isdigit()]
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        reasons = sorted({names[i] for s in self.samples for i in range(4)
                          if len(s) > 2 + i and s[2 + i].lower() == "active"})
        return {"sm_mhz": statistics.median(sm) if sm else None,
                "sm_max_mhz": max(mx) if mx else None, "reasons": reasons,
                "samples": len(self.samples)}


# ----------------------------------------------------------------- CPU leg
def metric_name(cfg, P, O):
    """One metric string for every arm and every N (the driver pairs the
    arms' lines by it)."""
    return f"output tokens/s (+ TTFT/TBT p50,p99) serving {P}/{O} requests, {cfg.name}"


def host_cpu():
    try:
        with open("/proc/cpuinfo") as f:
            for line in f:
                if line.startswith("model name"):
                    return line.split(":", 1)[1].strip()
    except OSError:
        pass
    return "unknown"


def _mem_available():
    try:
        with open("/proc/meminfo") as f:
            for line in f:
                if line.startswith("MemAvailable:"):
                    return int(line.split()[1]) * 1024
    except OSError:
        pass
    return 0


def cpu_port_model(model="llama2-7b", threads=None):
    """The fp32 oracle (oracle/decoder.py, the CPU port of the path) at the
    model's FULL depth and width.  Weights are distinct fp32 tensors filled
    from a seeded N(0, init_std) pool (a full seeded draw of 6.7 B normals
    would take minutes of single-threaded RNG; the values do not change the
    arithmetic done)."""
    import torch
    from oracle.decoder import OracleDecoder
    from paper_2311_18677_b200.model import get_config
    cfg = get_config(model)
    threads = threads or os.cpu_count()
    torch.set_num_threads(threads)
    d, dh, H, Hkv, f, V = (cfg.d_model, cfg.head_dim, cfg.n_heads, cfg.n_kv_heads, cfg.ffn,
                           cfg.vocab)
    need = 4 * (cfg.params_nonembed() + 2 * V * d) + 4 * 2 * cfg.n_layers * Hkv * dh * 4096
    if _mem_available() < 1.2 * need:
        raise MemoryError(f"fp32 {model} needs {need / 2**30:.1f} GiB host memory, "
                          f"{_mem_available() / 2**30:.1f} GiB available")
    g = torch.Generator().manual_seed(0)
    pool = torch.randn((1 << 22) + 4096, generator=g)
    cursor = [0]

    def r(*shape, std=cfg.init_std):
        t = torch.empty(*shape)
        flat = t.view(-1)
        n, m = flat.numel(), 1 << 22
        for k in range(0, n, m):
            o = (cursor[0] * 2654435761) % 4096
            cursor[0] += 1
            flat[k:k + m].copy_(pool[o:o + min(m, n - k)])
        return t.mul_(std)

    lay = [{"attn_norm": torch.ones(d), "wq": r(H * dh, d), "wk": r(Hkv * dh, d),
            "wv": r(Hkv * dh, d), "wo": r(d, H * dh), "mlp_norm": torch.ones(d),
            "w_gate": r(f, d), "w_up": r(f, d), "wd": r(d, f)} for _ in range(cfg.n_layers)]
    return cfg, OracleDecoder(cfg, lay, r(V, d, std=1.0), r(V, d), torch.ones(d)), threads


def cpu_port_request(model="llama2-7b", prompt=1024, n_out=128, dec_steps=None, threads=None):
    """Time one request (prompt phase + decode iterations) through the full
    fp32 CPU port on the host cores.  dec_steps=None runs every one of the
    n_out-1 decode iterations; a smaller number times that many and prices
    the rest at their mean (contexts prompt..prompt+n_out differ by < 13 %)."""
    import torch
    t_init = time.perf_counter()
    cfg, orc, threads = cpu_port_model(model, threads)
    t_init = time.perf_counter() - t_init
    g = torch.Generator().manual_seed(1234)
    toks = torch.randint(0, cfg.vocab, (prompt,), generator=g).tolist()
    n_dec = n_out - 1 if dec_steps is None else min(dec_steps, n_out - 1)
    t0 = time.perf_counter()
    logits, cache = orc.prefill(toks, orc.new_cache(prompt + n_out))
    t_pre = time.perf_counter() - t0
    tok, tbt = int(logits.argmax()), []
    for i in range(n_dec):
        t1 = time.perf_counter()
        logits = orc.decode(tok, prompt + i, cache)
        tok = int(logits.argmax())
        tbt.append(time.perf_counter() - t1)
    dec_total = sum(tbt) + (n_out - 1 - n_dec) * (statistics.mean(tbt) if tbt else 0.0)
    req_s = t_pre + dec_total
    full = n_dec == n_out - 1
    sample = (f"fp32 CPU port (oracle/decoder.py), {cfg.name} at full depth and width "
              f"({cfg.n_layers} layers): 1 request {prompt}/{n_out}, prompt phase + "
              + (f"all {n_dec} decode iterations timed" if full else
                 f"{n_dec} of {n_out - 1} decode iterations timed (rest at their mean)")
              + f"; {threads} threads on {host_cpu()}")
    return {"value": n_out / req_s, "unit": "tokens/s", "cores": threads, "kind": "port",
            "host_cpu": host_cpu(), "ttft_ms": t_pre * 1e3,
            "tbt_ms": {"p50": 1e3 * percentile(tbt, 0.5), "p99": 1e3 * percentile(tbt, 0.99)}
            if tbt else None,
            "request_ms": req_s * 1e3, "decode_iterations_timed": n_dec, "sample": sample,
            "wall_s": t_pre + sum(tbt), "init_s": t_init}


def cpu_baseline_sample(model, prompt, n_out, threads=None):
    """bench.py's cpu_baseline leg: a bounded sample (~10-20 s of CPU work)
    of the same request through the full-depth CPU port."""
    try:
        return cpu_port_request(model, prompt, n_out, dec_steps=6, threads=threads)
    except MemoryError as e:
        return {"value": None, "unit": "tokens/s", "unavailable": str(e)}


def splitsim_modeled(prompt=1024, n_out=128, n_gpus=1):
    """The reference simulator's modeled latencies for the same burst (H100
    calibration; no 7B preset exists so the 70B preset stands in)."""
    sys.path.insert(0, os.path.join(ROOT, "baseline", "_ref"))
    try:
        import splitsim as ss
    except Exception as e:  # noqa: BLE001
        return {"unavailable": f"splitsim not importable: {e}"}
    reqs = [ss.Request(i, 0.0, prompt, n_out) for i in range(max(1, n_gpus))]
    trace = ss.Trace(reqs, 1.0)
    perf = {"H100": ss.get_calibration("llama2-70b", "H100")}
    if n_gpus <= 1:
        cc = ss.ClusterConfig("Baseline-H100", 1, 0)
    else:
        cc = ss.ClusterConfig("Splitwise-HH", n_gpus // 2, n_gpus // 2)
    t0 = time.perf_counter()
    res = ss.Simulator(cc, perf, trace).run()
    wall = time.perf_counter() - t0
    s = res.report.summary()
    return {"design": cc.design, "ttft_ms_p50": s.get("ttft_ms_p50"),
            "tbt_ms_p50": s.get("tbt_ms_p50"), "e2e_ms_p50": s.get("e2e_ms_p50"),
            "wall_s": wall, "preset": "llama2-70b/H100 (no 7B preset)"}


def run_reference(args):
    """The reference arm: the reference package has no arithmetic for the
    path (its prompt/token phases are latency lookups, reference
    perf.py:119-132), so its CPU implementation of the path is the fp32 port
    in oracle/, run here over ONE full request of the workload (full depth,
    every decode iteration timed — about a minute on 16 cores, so one step;
    the step of the GPU arm is also one request burst).  Nothing is scaled."""
    rank = int(os.environ.get("RANK", "0"))
    if rank != 0:
        return
    from paper_2311_18677_b200.model import get_config
    cfg = get_config(args.model)
    P, O = args.prompt, args.out
    try:
        cb = cpu_port_request(args.model, P, O, dec_steps=None)
    except MemoryError as e:
        print(json.dumps({"impl": "reference", "unavailable": str(e)}), flush=True)
        return
    v = cb["value"]
    line = {"impl": "reference", "metric": metric_name(cfg, P, O),
            "value": v, "unit": "tokens/s", "n_gpus": args.gpus, "steps": 1, "warmup": 0,
            "requested_steps": args.steps, "requested_warmup": args.warmup,
            "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "f32",
            "data": "synthetic (seeded random weights/tokens)",
            "ms_per_step": cb["request_ms"],
            "config": {"workload": f"{cfg.name} {P}-token prompt / {O} greedy outputs, 1 request "
                                   "per step; fp32 CPU port of the path on all host cores "
                                   "(one full request: steps=1 whatever --steps asks)",
                       "model": cfg.name, "prompt_tokens": P, "output_tokens": O,
                       "requests_per_step": 1, "parallelism": f"cpu x{cb['cores']}"},
            "ttft_ms": {"p50": cb["ttft_ms"], "p99": cb["ttft_ms"]},
            "tbt_ms": cb["tbt_ms"],
            "cpu_baseline": cb,
            "e2e": {"value": v, "unit": "tokens/s", "h2d_bytes_per_step": 0,
                    "d2h_bytes_per_step": 0},
            "splitsim_modeled": splitsim_modeled(P, O, args.gpus)}
    print(json.dumps(line), flush=True)


# ----------------------------------------------------------------- GPU leg
def run_colocated(args):
    import torch
    from paper_2311_18677_b200 import _abi
    from paper_2311_18677_b200 import kernels as K
    from paper_2311_18677_b200.model import get_config, init_weights
    from paper_2311_18677_b200.runner import ModelRunner
    from paper_2311_18677_b200.serving import ColocatedEngine, GenRequest

    hbm_peak, tc_peak, tc_sus, peak_kind = _peaks()
    cfg = get_config(args.model)
    torch.cuda.set_device(0)
    w = init_weights(cfg, seed=0)
    P, O = args.prompt, args.out
    eng = ColocatedEngine(w, max_seqs=8, max_ctx=P + O + 64)
    g = torch.Generator().manual_seed(1234)
    prompt_h = torch.randint(0, cfg.vocab, (P,), generator=g, dtype=torch.int32).pin_memory()

    def e2e_step():
        t0 = time.perf_counter()
        out = eng.generate([GenRequest(0, prompt_h, O, arrival=t0)])
        return out, time.perf_counter() - t0

    for _ in range(args.warmup):
        e2e_step()
    torch.cuda.synchronize()
    # ---- e2e (public API, host buffers)
    ttft, tbt, e2e_times = [], [], []
    launches0 = _abi.launch_count()
    with ClockSampler(0) as clk:
        for _ in range(args.steps):
            res, dt = e2e_step()
            e2e_times.append(dt)
            ttft += [r.ttft_ms for r in res]
            tbt += [x for r in res for x in r.tbt_ms()]
        # ---- device-resident value: prefill + graph replays, no host copies
        kv, runner = eng.kv, eng.runner
        seq = kv.allocate(P + O)
        toks = prompt_h.cuda()
        meta = ModelRunner.pack_meta([P]).cuda()
        slots = torch.empty(P, dtype=torch.int32, device="cuda")
        K.slots_from_table(kv.table_row_ptr(seq), 0, P, kv.block_size, slots)
        graph = runner.decode_graph(1, P + O, O - 1)
        ev = lambda: torch.cuda.Event(enable_timing=True)  # noqa: E731
        step_ms, pre_ms, dec_ms = [], [], []
        for it in range(args.warmup + args.steps):
            e0, e1, e2 = ev(), ev(), ev()
            dec_ev = [ev() for _ in range(O)]
            torch.cuda.synchronize()
            e0.record()
            first = runner.prefill(toks, [P], meta, local_slots=slots)
            e1.record()
            graph.load([seq], first[:1], [P])
            if graph.graph is None:
                graph.capture()
            dec_ev[0].record()
            for s in range(O - 1):
                graph.replay()
                dec_ev[s + 1].record()
            e2.record()
            torch.cuda.synchronize()
            if it >= args.warmup:
                step_ms.append(e0.elapsed_time(e2))
                pre_ms.append(e0.elapsed_time(e1))
                dec_ms += [dec_ev[s].elapsed_time(dec_ev[s + 1]) for s in range(O - 1)]
        kv.release(seq)
    launches = _abi.launch_count() - launches0
    clocks = clk.summary()

    ms = statistics.mean(step_ms)
    value = O / (ms / 1e3)
    e2e_ms = statistics.mean(e2e_times) * 1e3
    # roofline of the dominant phase: decode step (weights + KV stream, HBM)
    ctxs = [P + s for s in range(1, O)]
    dec_bytes = statistics.mean(cfg.decode_bytes([c]) for c in ctxs)
    dec_avg = statistics.mean(dec_ms)
    dec_gbs = dec_bytes / (dec_avg / 1e3) / 1e9
    pre_flops = cfg.prefill_flops(P)
    pre_avg = statistics.mean(pre_ms)
    pre_tfs = pre_flops / (pre_avg / 1e3) / 1e12
    traffic = _ncu_traffic("decode_step")
    line = {
        "metric": metric_name(cfg, P, O),
        "value": value, "unit": "tokens/s", "n_gpus": 1, "steps": args.steps,
        "warmup": args.warmup, "ms_per_step": ms, "higher_is_better": True, "scaling": "weak",
        "vs_baseline": None, "dtype": "bf16", "data": "synthetic (seeded random weights/tokens)",
        "config": {"workload": f"{cfg.name} {P}-token prompt / {O} greedy outputs, 1 request "
                               "per GPU per step; N=1 co-located (Baseline design)",
                   "model": cfg.name, "prompt_tokens": P, "output_tokens": O,
                   "requests_per_step": 1, "parallelism": "co-located",
                   "l2": "inputs > L2 (13.5 GB weights streamed per decode step)"},
        "ttft_ms": {"p50": percentile(ttft, 0.5), "p99": percentile(ttft, 0.99)},
        "tbt_ms": {"p50": percentile(tbt, 0.5), "p99": percentile(tbt, 0.99)},
        "e2e": {"value": O * args.steps / sum(e2e_times), "unit": "tokens/s",
                "ms_per_step": e2e_ms, "h2d_bytes_per_step": 4 * P + 4 * (3 * P + 2),
                "d2h_bytes_per_step": 4 * O},
        "phases_ms": {"prefill": pre_avg, "decode_step": dec_avg},
        "roofline": {"kernel": "decode_step (CUDA graph: GEMV weight stream + paged attention)",
                     "bound": "hbm", "achieved": dec_gbs, "peak": hbm_peak, "unit": "GB/s",
                     "frac": dec_gbs / hbm_peak, "peak_kind": peak_kind,
                     "algorithmic_bytes": dec_bytes, "traffic": traffic},
        "roofline_prefill": {"bound": "tensor", "achieved": pre_tfs, "peak": tc_peak,
                             "unit": "TFLOP/s", "frac": pre_tfs / tc_peak,
                             "algorithmic_flops": pre_flops, "peak_kind": peak_kind},
        "kv_transfer": {"mode": "none (co-located: prefill writes the token pool directly)"},
        "gpu_launches": launches,
        "clocks": clocks,
    }
    if not args.no_cpu:
        line["cpu_baseline"] = cpu_baseline_sample(args.model, P, O)
    print(json.dumps(line), flush=True)


def _ncu_traffic(key):
    p = os.path.join(ROOT, "profiles", "ncu_traffic.json")
    try:
        with open(p) as f:
            return json.load(f).get(key)
    except Exception:
        return None


def _self_launch(n):
    """`python bench.py --gpus N` without torchrun: re-exec under
    torch.distributed.run with N local ranks (rendezvous on 127.0.0.1)."""
    import socket
    with socket.socket() as sk:
        sk.bind(("127.0.0.1", 0))
        port = sk.getsockname()[1]
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1",
           f"--nproc-per-node={n}", "--master-addr=127.0.0.1", f"--master-port={port}",
           os.path.abspath(__file__)] + sys.argv[1:]
    sys.stdout.flush()
    os.execv(sys.executable, cmd)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=5)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--model", default="llama2-7b")
    ap.add_argument("--prompt", type=int, default=1024)
    ap.add_argument("--out", type=int, default=128)
    ap.add_argument("--no-cpu", action="store_true")
    ap.add_argument("--trace", default=None, choices=[None, "conversation", "coding"],
                    help="N>=2: serve the reference's synthetic trace in real time instead "
                         "of the fixed-shape burst")
    ap.add_argument("--rate", type=float, default=4.0)
    ap.add_argument("--duration", type=float, default=20.0)
    ap.add_argument("--seed", type=int, default=0)
    ap.add_argument("--max-output", type=int, default=0)
    ap.add_argument("--route", default="jsq", choices=["jsq", "rr"],
                    help="--trace with several pairs: live JSQ routing at arrival (reference "
                         "Cluster.route) or round-robin")
    ap.add_argument("--dump-tokens", default=None,
                    help="--trace: write {request id: generated token ids} to this JSON file")
    ap.add_argument("--tp", type=int, default=1,
                    help="tensor-parallel degree of each prompt/token machine (N >= 2*tp)")
    args = ap.parse_args()
    if args.impl == "reference":
        run_reference(args)
        return
    if args.gpus > 1 and "WORLD_SIZE" not in os.environ:
        _self_launch(args.gpus)          # one rank per GPU, exec's torchrun
    world = int(os.environ.get("WORLD_SIZE", "1"))
    if args.trace:
        sys.path.insert(0, os.path.join(ROOT, "tools"))
        from reftrace import preset_trace
        args.trace_requests = preset_trace(args.trace, args.rate, args.duration, args.seed)
    if args.trace and world < 2:
        raise SystemExit("--trace needs N >= 2 GPUs (Splitwise pairs, launched with torchrun)")
    if world == 1 and args.gpus == 1:
        run_colocated(args)
    else:
        from paper_2311_18677_b200.splitwise import run_split_bench
        run_split_bench(args, ClockSampler, percentile, cpu_baseline_sample, _peaks, _ncu_traffic,
                        metric_name)


if __name__ == "__main__":
    main()
