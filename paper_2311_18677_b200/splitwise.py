"""Splitwise serving across GPUs: prompt machines and token machines as
separate processes (one per GPU), KV pushed layer by layer over NVLink.

Roles (reference: Machine home roles, machine.py:88-114; hand-off,
engine.py:250-301):
  * ``PromptServer`` (prompt machine): batches queued prompts with the
    reference's prompt rule (PromptWorker.form_batch: FCFS, <= 2048 tokens,
    head always admitted), runs the prefill and, for every layer, pushes that
    layer's K/V straight into the paged blocks the token machine reserved —
    P2P stores through the token pool's CUDA-IPC mapping, on a side stream
    that overlaps the next layer's compute.  When the last layer has landed it
    hands the request over (request id, KV sequence slot, prompt length,
    first token) on the control channel.
  * ``TokenServer`` (token machine): reserves each routed request's final
    context in its device block pool at arrival (both machines are chosen at
    arrival, cluster.py:153-160), admits handed-over token tasks with the
    reference's token rule (TokenWorker.form_batch: slots, memory, FCFS), and
    runs one CUDA-graph decode iteration per scheduler iteration, streaming
    every generated token to the host.

The control channel is a gloo process group (tiny int32 messages); the KV
bytes never touch the host.  ``run_split_bench`` is bench.py's N >= 2 leg.
"""

from __future__ import annotations

import os
import statistics
import threading
import time

import torch
import torch.distributed as dist

from . import _abi
from . import kernels as K
from .control import (ArrivalFeed, HandoffTable, HandoffWatch, RouteBoard, ShmMailbox,
                      recv_reservations, send_reservations)
from .kvcache import KVCacheManager, blocks_for
from .model import get_config, init_weights
from .perf import PerfModel
from .runner import Handoff, ModelRunner, PushSegment, PushStats
from .serving import pool_blocks_for_memory
from .transfer import LAYERWISE, kv_push_gbps, measured_plan
from .workers import PROMPT, TOKEN, Machine, SchedulerConfig, Task


def estimated_perf_model(cfg, kv: KVCacheManager | None, weight_bytes: int,
                         hbm_gbs: float = 6543.0, tflops: float = 1000.0,
                         capacity: float | None = None) -> PerfModel:
    """Roofline-estimated PerfModel used by the B200 machines for batch
    formation.  Token machines: capacity = weights + KV pool bytes (exact
    admission).  Prompt machines keep no KV after the push; their capacity
    is the device's HBM (the prompt's transient KV lives in activations)."""
    pts = [1, 512, 1024, 2048, 4096, 8192]
    p_ms = [max(0.05, cfg.prefill_flops(p) / (tflops * 1e12) * 1e3) for p in pts]
    bs = [1, 2, 4, 8, 16, 32, 64]
    t_ms = [max(0.05, cfg.decode_bytes([1024] * b) / (hbm_gbs * 1e9) * 1e3) for b in bs]
    kvb = cfg.kv_bytes_per_token()
    pool = 0 if kv is None else kv.num_blocks * kv.block_size * kvb
    cap = float(weight_bytes + pool) if capacity is None else float(capacity)
    return PerfModel("B200", cfg.name, (pts, p_ms), (bs, t_ms), float(kvb),
                     float(weight_bytes), cap, cfg.max_token_batch)


def _lockstep(n: int, tp_ctrl, now_ms: float = 0.0, fin: bool = False):
    """(arrivals to process, scheduler clock, all done) for this iteration of
    a TP group: the minimum arrival count, the maximum clock and the AND of
    the peers' "nothing left" flags, so every peer enqueues / reserves the
    same requests, forms the same batch (the collectives inside the steps
    stay matched) and leaves the loop at the same iteration."""
    if tp_ctrl is None:
        return n, now_ms, fin
    t = torch.tensor([float(n), -now_ms, float(fin)], dtype=torch.float64)
    dist.all_reduce(t, op=dist.ReduceOp.MIN, group=tp_ctrl)
    return int(t[0].item()), -float(t[1].item()), bool(t[2].item())


class PromptServer:
    """Prompt machine (one process per GPU / TP rank).  It maps the KV pool,
    the hand-off table and the reservation mailbox of EVERY token machine
    (same TP rank), so a request can be pushed to whichever token machine
    the router picked (reference Cluster.route, cluster.py:153-160)."""

    def __init__(self, runner: ModelRunner, peers: dict, ctrl, token_rank: int,
                 sched: SchedulerConfig, tables: dict, tp_ctrl=None, machine_id: int = 0,
                 res_boxes: dict | None = None):
        """peers / tables: {token machine: KVCacheManager peer view / hand-off
        table name}; token_rank: the control-group rank of the paired token
        machine (burst mode); res_boxes: {token machine: mailbox name}."""
        self.runner = runner
        self.tp_ctrl = tp_ctrl          # TP peers must batch in lockstep (collectives inside)
        self.peers = dict(peers)
        self.tables = {t: HandoffTable(name=n) for t, n in tables.items()}
        self.table_ptrs = {t: tb.device_ptr() for t, tb in self.tables.items()}
        self.res_boxes = {t: ShmMailbox(name=n) for t, n in (res_boxes or {}).items()}
        self.ctrl = ctrl
        self.token_rank = token_rank
        self.machine_id = machine_id
        self._batches = 0
        cfg = runner.cfg
        hbm = float(torch.cuda.get_device_properties(runner.dev).total_memory)
        self.machine = Machine(0, None, estimated_perf_model(cfg, None, runner.w.nbytes(),
                                                             capacity=hbm), PROMPT, sched)
        self.push_log: list[PushStats] = []

    def _run_batch(self, chunk, dest, toks):
        """chunk: [(rid, prompt, n_out)]; dest: {rid: (token machine, KV slot,
        epoch)}.  Enqueue the prefill, the per-layer pushes into the reserved
        pages of each request's token machine and one hand-off group per
        destination table, then wait only for the prompt COMPUTE (the pushes'
        tail and the hand-off run on the push stream).  Returns the host time
        the compute finished."""
        lens = [len(r[1]) for r in chunk]
        meta = ModelRunner.pack_meta(lens).pin_memory().to(self.runner.dev, non_blocking=True)
        segs, off = [], 0
        for r, n in zip(chunk, lens):
            t, seq, _ep = dest[r[0]]
            segs.append(PushSegment(off, n, self.peers[t], seq))
            off += n
        st = PushStats(bytes_per_layer=off * 2 * self.runner.hkv * self.runner.dh * 2)
        self._batches += 1
        key = ((self.machine_id & 0xFF) << 23) | (self._batches & 0x7FFFFF)
        hands = []
        for t in sorted({dest[r[0]][0] for r in chunk}):
            idx = [i for i, r in enumerate(chunk) if dest[r[0]][0] == t]
            hands.append(Handoff([dest[chunk[i][0]][1] for i in idx],
                                 [dest[chunk[i][0]][2] for i in idx], self.table_ptrs[t],
                                 rows=idx, key=key, stride=HandoffTable.STRIDE))
        self.runner.prefill(toks, lens, meta, push=segs, push_stats=st, handoff=hands)
        done = torch.cuda.Event()
        done.record()
        done.synchronize()
        self.push_log.append(st)
        self.runner.finish_push_stats(block=False)
        return time.perf_counter()

    def serve_burst(self, requests, t0: float, prompts_dev: dict | None = None):
        """requests: list of (rid, host int32 prompt, n_out).  Returns {rid:
        host time its prompt compute finished}."""
        dev = self.runner.dev
        seqs, epochs = recv_reservations(len(requests), self.token_rank, self.ctrl,
                                         with_epochs=True)
        t = self.machine_id                       # burst mode: the paired token machine
        dest = {r[0]: (t, s, e) for r, s, e in zip(requests, seqs, epochs)}
        by_id = {r[0]: r for r in requests}
        now_ms = 0.0
        for rid, prompt, n_out in requests:
            self.machine.enqueue(Task(rid, PROMPT, len(prompt), now_ms, n_out, n_out), now_ms)
        done_time = {}
        while self.machine.has_work():
            batch = self.machine.form_batch(now_ms)
            self.machine.running = batch
            chunk = [by_id[t.request_id] for t in batch.prompt_tasks]
            if prompts_dev is not None:
                toks = torch.cat([prompts_dev[r[0]] for r in chunk])
            else:
                toks = torch.cat([r[1] for r in chunk]).pin_memory().to(dev, non_blocking=True)
            tnow = self._run_batch(chunk, dest, toks)
            for r in chunk:
                done_time[r[0]] = tnow
            now_ms = (tnow - t0) * 1e3
            self.machine.complete_iteration(batch, now_ms)
        self.runner.finish_push_stats(block=True)
        return done_time

    def serve_trace(self, requests, t0: float, feed=None):
        """Arrival-driven prompt machine: requests = [(rid, arrival_s, host
        prompt, n_out)] in arrival order.  A request becomes a prompt task
        (enqueue time = its arrival) once the token machine it was routed to
        has reserved its final context (that machine's reservation mailbox;
        token machines admit reservations in arrival order with the
        blocked-head memory rule), so its KV always has pages to land in;
        tasks are enqueued in arrival order (the longest reserved prefix).
        Batches follow the reference prompt rule.  Returns {rid: host time its
        prompt compute finished}.  ``feed`` (control.ArrivalFeed, role
        "prompt") supplies the requests the live router sent to this
        machine; without one every request is this machine's and goes to
        token machine ``self.machine_id``."""
        feed = feed or ArrivalFeed(requests, 0)
        board = getattr(self, "board", None)
        by_id = {r[0]: r for r in requests}
        mine: list = []                 # my arrivals, in arrival order
        dest: dict = {}                 # rid -> (token machine, slot, epoch)
        done_time = {}
        done = 0
        done_tok = 0
        while True:
            mine += [r[0] for r in feed.poll()]
            for t, box in self.res_boxes.items():
                while True:
                    rows = box.get()
                    if rows is None:
                        break
                    for rid, seq, ep, *_ in rows:
                        dest[rid] = (t, seq, ep)
            n_res = 0
            while n_res < len(mine) and mine[n_res] in dest:
                n_res += 1
            fin = feed.complete() and done >= feed.mine
            n_take, _, fin = _lockstep(n_res, self.tp_ctrl, 0.0, fin)
            if fin:
                break
            for rid in mine[:n_take]:
                _, arr, prompt, n_out = by_id[rid]
                self.machine.enqueue(Task(rid, PROMPT, len(prompt), arr * 1e3, n_out, n_out),
                                     arr * 1e3)
            del mine[:n_take]
            if not self.machine.has_work():
                time.sleep(5e-5)
                continue
            now = time.perf_counter() - t0
            batch = self.machine.form_batch(now * 1e3)
            self.machine.running = batch
            chunk = [(r[0], r[2], r[3]) for r in (by_id[t.request_id] for t in batch.prompt_tasks)]
            toks = torch.cat([r[1] for r in chunk]).pin_memory().to(self.runner.dev,
                                                                      non_blocking=True)
            tnow = self._run_batch(chunk, dest, toks)
            for r in chunk:
                done_time[r[0]] = tnow
            done += len(chunk)
            done_tok += sum(len(r[1]) for r in chunk)
            if board is not None:
                board.publish_prompt(self.machine_id, done_tok)
            self.machine.complete_iteration(batch, (tnow - t0) * 1e3)
        self.runner.finish_push_stats(block=True)
        return done_time

    def close(self):
        for tb in self.tables.values():
            tb.close()
        for box in self.res_boxes.values():
            box.close()


class TokenServer:
    """Token machine of a Splitwise pair (one process per GPU / TP rank)."""

    def __init__(self, runner: ModelRunner, ctrl, prompt_rank: int, sched: SchedulerConfig,
                 tp_ctrl=None, machine_id: int = 0, prompt_machines: int = 1):
        """prompt_rank: control-group rank of the paired prompt machine (burst
        mode); one reservation mailbox per prompt machine (res_boxes)."""
        self.runner = runner
        self.kv = runner.kv
        self.ctrl = ctrl
        self.prompt_rank = prompt_rank
        self.machine_id = machine_id
        self.tp_ctrl = tp_ctrl          # TP peers must admit in lockstep (collectives inside)
        self.res_boxes = {p: ShmMailbox(create=True) for p in range(prompt_machines)}
        self.table = HandoffTable(self.kv.max_seqs, create=True)
        self.watch = HandoffWatch(self.table, tp_ctrl)
        self.epoch = [0] * self.kv.max_seqs
        self.machine = Machine(0, None, estimated_perf_model(runner.cfg, self.kv,
                                                             runner.w.nbytes()), TOKEN, sched)
        self.step_log: list[tuple] = []     # (batch, summed context, device ms) per decode step
        self.tokens: dict = {}              # serve_trace: rid -> generated token ids
        self._ev = None

    def _events(self):
        if self._ev is None:
            self._ev = (torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True))
        return self._ev

    def _reserve(self, tokens: int):
        seq = self.kv.allocate(tokens)
        self.epoch[seq] = (self.epoch[seq] + 1) & 0x7FFFFFFF
        return seq, self.epoch[seq]

    def _fits_prefix(self, lens: list[int]) -> int:
        """How many leading reservations fit the pool now (blocks and sequence
        slots) — the reference's blocked-head memory admission
        (machine.py:216-223): the first that does not fit blocks the rest."""
        free_b, free_s = self.kv.free_blocks, len(self.kv._free_slots)
        n = 0
        for t in lens:
            nb = blocks_for(t, self.kv.block_size)
            if nb > free_b or free_s == 0 or nb > self.kv.max_blocks_per_seq:
                break
            free_b -= nb
            free_s -= 1
            n += 1
        return n

    def prewarm(self, max_batch: int = 24, buckets=(2048, 4096)) -> int:
        """Capture the decode graphs of the batch sizes / context buckets a
        trace will use before serving starts (a capture inside the serve
        loop stalls every running request for its duration).  Run before
        any sequence is live: the warm-up step of a capture writes block 0."""
        n = 0
        for bucket in buckets:
            for B in range(1, max_batch + 1):
                g = self.runner.decode_graph(B, bucket, 1)
                if g.graph is None:
                    g.capture()
                    n += 1
        torch.cuda.synchronize()
        return n

    def _graph_for(self, rids, info, remaining):
        """Decode graph whose context bucket covers every row until it
        finishes: current context + remaining outputs + 1."""
        need = max(info[r][1] + remaining[r] + 1 for r in rids)
        g = self.runner.decode_graph(len(rids), 2048 * ((need + 2047) // 2048), 1)
        g.load([info[r][0] for r in rids], [info[r][2] for r in rids], [info[r][1] for r in rids])
        if g.graph is None:
            g.capture()
        return g

    def _step(self, graph, B, ring_h):
        """One decode iteration; while it runs, watch the hand-off table so a
        landing is time-stamped when it happens, not at the next iteration."""
        ev0, ev1 = self._events()
        ev0.record()
        graph.replay()
        ev1.record()
        ring_h[:B].copy_(graph.next_tok, non_blocking=True)
        done = torch.cuda.Event()
        done.record()
        while not done.query():
            self.watch.observe()
            time.sleep(2e-5)
        return ev0.elapsed_time(ev1)

    def serve_burst(self, requests, t0: float):
        """Reserve KV for the routed requests, then admit hand-overs and
        decode until all of them finished.  Returns ({rid: [emission times]},
        {rid: generated tokens}, {rid: first-token time})."""
        kv = self.kv
        self.step_log = []
        res = [self._reserve(len(p) + n) for _rid, p, n in requests]
        torch.cuda.current_stream().synchronize()    # tables written before the peer reads
        send_reservations([s for s, _ in res], self.prompt_rank, self.ctrl,
                          [e for _, e in res])
        for (rid, p, n), (seq, ep) in zip(requests, res):
            self.watch.expect(rid, seq, ep, len(p), n)
        expected = len(requests)
        received = 0
        info, remaining = {}, {}      # rid -> [seq, ctx_kv, last_token]; outputs left
        emit = {r[0]: [] for r in requests}
        tokens = {r[0]: [] for r in requests}
        first_seen = {}
        graph, graph_rids = None, None
        ring_h = torch.empty(256, dtype=torch.int32).pin_memory()
        while received < expected or self.machine.has_work() or self.machine.resident:
            rows = self.watch.poll() if received < expected else []
            now_ms = (time.perf_counter() - t0) * 1e3
            for rid, seq, plen, first, n_out in rows:
                received += 1
                tokens[rid].append(first)
                first_seen[rid] = self.watch.seen.pop(rid)
                if n_out > 1:
                    info[rid] = [seq, plen, first]
                    remaining[rid] = n_out - 1
                    self.machine.enqueue(Task(rid, TOKEN, plen + 1, now_ms, n_out, n_out - 1),
                                         now_ms)
                else:
                    kv.release(seq)
            if not self.machine.has_work():
                time.sleep(2e-5)
                continue
            batch = self.machine.form_batch(now_ms)
            if batch is None or not batch.token_tasks:
                time.sleep(2e-5)
                continue
            self.machine.running = batch
            rids = [t.request_id for t in batch.token_tasks]
            B = len(rids)
            if rids != graph_rids:
                graph = self._graph_for(rids, info, remaining)
                graph_rids = rids
            ms = self._step(graph, B, ring_h)
            self.step_log.append((B, sum(info[r][1] for r in rids), ms))
            tnow = time.perf_counter()
            for b, r in enumerate(rids):
                t = int(ring_h[b])
                tokens[r].append(t)
                info[r][1] += 1
                info[r][2] = t
                remaining[r] -= 1
                emit[r].append(tnow)
            for what, task in self.machine.complete_iteration(batch, (tnow - t0) * 1e3):
                if what == "request_finished":
                    kv.release(info[task.request_id][0])
                    graph_rids = None
        return emit, tokens, first_seen

    def serve_trace(self, requests, t0: float, feed=None):
        """Arrival-driven token machine: reserves each request's final context
        at its arrival (both machines are chosen at arrival, reference
        cluster.py:153-160) when the pool can hold it — arrivals that do not
        fit wait, in order, until finished requests free their pages (the
        reference's blocked-head memory admission; TP peers decide in
        lockstep) — and publishes the slot to the prompt machine; admits
        landed hand-offs between decode iterations (continuous batching with
        the reference token rule), one CUDA-graph step per iteration.
        Returns ({rid: [emission times]}, decode step log, {rid: first-token
        time}).  ``feed`` (role "token") supplies the requests routed here;
        each one's prompt machine is the board's pick (``assign_p``), or
        ``self.machine_id`` without a board."""
        kv = self.kv
        feed = feed or ArrivalFeed(requests, 0)
        board = getattr(self, "board", None)
        landed = 0
        pending = []
        info, remaining, emit, first_seen = {}, {}, {}, {}
        finished = 0
        graph, graph_rids = None, None
        ring_h = torch.empty(256, dtype=torch.int32).pin_memory()
        self.step_log = []
        while True:
            for r in feed.poll():
                pending.append(r)
                emit[r[0]] = []
            fin = feed.complete() and finished >= feed.mine
            now = time.perf_counter() - t0
            n_new = 0
            while n_new < len(pending) and pending[n_new][1] <= now:
                n_new += 1
            n_new = self._fits_prefix([len(p[2]) + p[3] for p in pending[:n_new]])
            n_take, mnow, fin = _lockstep(n_new, self.tp_ctrl, now * 1e3, fin)
            if fin:
                break
            arrived = []
            for _ in range(n_take):
                rid, arr, prompt, n_out = pending.pop(0)
                seq, ep = self._reserve(len(prompt) + n_out)
                arrived.append((rid, seq, ep))
                self.watch.expect(rid, seq, ep, len(prompt), n_out)
            if arrived:
                torch.cuda.current_stream().synchronize()   # table rows before the peer reads
                by_p: dict = {}
                for rid, seq, ep in arrived:
                    pm = int(board.assign_p[rid]) if board is not None else self.machine_id
                    by_p.setdefault(pm, []).append((rid, seq, ep, 0, 0))
                for pm, rows in by_p.items():
                    self.res_boxes[pm].put(rows)
            for rid, seq, plen, first, n_out in self.watch.poll():
                first_seen[rid] = self.watch.seen.pop(rid)
                self.tokens[rid] = [first]
                landed += 1
                if board is not None:
                    board.publish_token(self.machine_id, board.LANDED, landed)
                if n_out > 1:
                    info[rid] = [seq, plen, first]
                    remaining[rid] = n_out - 1
                    self.machine.enqueue(Task(rid, TOKEN, plen + 1, mnow, n_out, n_out - 1), mnow)
                else:
                    kv.release(seq)
                    finished += 1
                    if board is not None:
                        board.publish_token(self.machine_id, board.FINISHED, finished)
            if not self.machine.has_work() and not self.machine.resident:
                time.sleep(5e-5)
                continue
            batch = self.machine.form_batch(mnow)
            if batch is None or not batch.token_tasks:
                time.sleep(5e-5)
                continue
            self.machine.running = batch
            rids = [t.request_id for t in batch.token_tasks]
            B = len(rids)
            if rids != graph_rids:
                graph = self._graph_for(rids, info, remaining)
                graph_rids = rids
            ms = self._step(graph, B, ring_h)
            tnow = time.perf_counter()
            self.step_log.append((B, sum(info[r][1] for r in rids), ms))
            for b, r in enumerate(rids):
                t = int(ring_h[b])
                info[r][1] += 1
                info[r][2] = t
                remaining[r] -= 1
                emit[r].append(tnow)
                self.tokens[r].append(t)
            for what, task in self.machine.complete_iteration(batch, mnow):
                if what == "request_finished":
                    kv.release(info[task.request_id][0])
                    finished += 1
                    if board is not None:
                        board.publish_token(self.machine_id, board.FINISHED, finished)
                    graph_rids = None
        return emit, self.step_log, first_seen

    def close(self):
        self.table.close()
        for box in self.res_boxes.values():
            box.close()


# ---------------------------------------------------------------------------
def _decode_roofline(cfg, tp, steps, hbm_peak, peak_kind):
    """HBM roofline of the token machine's decode step (the dominant kernel
    chain of a Splitwise pair): algorithmic bytes (weights / TP + the batch's
    KV) over the CUDA-event time of the captured decode graph, full-batch
    steps only."""
    if not steps:
        return None
    bmax = max(b for b, _, _ in steps)
    full = [(b, c, ms) for b, c, ms in steps if b == bmax]
    byts = [cfg.decode_bytes([c], tp) for _, c, _ in full]   # c = the batch's summed context
    ms = [m for _, _, m in full]
    ach = (sum(byts) / len(byts)) / (sum(ms) / len(ms) / 1e3) / 1e9
    return {"kernel": f"decode_step (CUDA graph, B={bmax}, token machine)", "bound": "hbm",
            "achieved": ach, "peak": hbm_peak, "unit": "GB/s", "frac": ach / hbm_peak,
            "peak_kind": peak_kind, "algorithmic_bytes": sum(byts) / len(byts),
            "traffic": None, "steps_timed": len(full)}


def _full_batch_ms(steps):
    if not steps:
        return None
    bmax = max(b for b, _, _ in steps)
    return statistics.mean(m for b, _, m in steps if b == bmax)


def run_split_bench(args, ClockSampler, percentile, cpu_baseline, peaks, ncu_traffic,
                    metric_name):
    import json
    rank = int(os.environ.get("RANK", "0"))
    world = int(os.environ.get("WORLD_SIZE", "1"))
    local = int(os.environ.get("LOCAL_RANK", str(rank)))
    tp = max(1, int(getattr(args, "tp", 1)))
    if world < 2 * tp or world % (2 * tp):
        raise SystemExit(f"Splitwise TP{tp}+TP{tp} pairs need a multiple of {2 * tp} GPUs")
    torch.cuda.set_device(local)
    dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    ctrl = dist.new_group(backend="gloo")
    # rank layout: pair p owns ranks [2*tp*p, 2*tp*(p+1)); the first tp ranks
    # are the prompt machine's TP group, the next tp the token machine's;
    # prompt TP rank i pushes its KV head slice to token TP rank i.
    pair = rank // (2 * tp)
    is_prompt = (rank % (2 * tp)) < tp
    tp_rank = rank % tp
    peer_rank = rank + tp if is_prompt else rank - tp
    tp_nccl, tp_gloo = None, None
    for base in range(0, world, tp):          # every rank creates every group
        ranks = list(range(base, base + tp))
        gn = dist.new_group(ranks) if tp > 1 else None
        gg = dist.new_group(ranks, backend="gloo") if tp > 1 else None
        if rank in ranks:
            tp_nccl, tp_gloo = gn, gg
    cfg = get_config(args.model)
    w = init_weights(cfg, seed=0, tp=tp, rank=tp_rank)
    P, O = args.prompt, args.out
    R = 2 * tp                                  # one request per GPU of the pair
    sched = SchedulerConfig()
    pairs = world // (2 * tp)
    if is_prompt:
        runner = ModelRunner(w, None, tp_group=tp_nccl)
    else:
        trace_mode = bool(getattr(args, "trace", None))
        nb = pool_blocks_for_memory(cfg, tp, 16, reserve_bytes=2 << 30)
        nb = min(nb, 256 * blocks_for(8192 + 4096, 16) if trace_mode
                 else 64 * blocks_for(P + O + 64, 16))
        kv = KVCacheManager(cfg.n_layers, nb, cfg.n_kv_heads // tp, cfg.head_dim, 16,
                            256 if trace_mode else 64, blocks_for(8192 + 4096, 16))
        runner = ModelRunner(w, kv, tp_group=tp_nccl)
        server = TokenServer(runner, ctrl, peer_rank, sched, tp_ctrl=tp_gloo, machine_id=pair,
                             prompt_machines=pairs)
    # every token machine's (TP rank i) pool, hand-off table and per-prompt-
    # machine mailboxes go to every prompt machine's TP rank i (any-to-any)
    info = None if is_prompt else {"machine": pair, "tp_rank": tp_rank,
                                   "kv": kv.ipc_handle(), "table": server.table.name,
                                   "boxes": {p: b.name for p, b in server.res_boxes.items()}}
    everyone = [None] * world
    dist.all_gather_object(everyone, info, group=ctrl)
    if is_prompt:
        mine = [e for e in everyone if e is not None and e["tp_rank"] == tp_rank]
        peers = {e["machine"]: KVCacheManager.open_peer(e["kv"]) for e in mine}
        server = PromptServer(runner, peers, ctrl, peer_rank, sched,
                              {e["machine"]: e["table"] for e in mine}, tp_ctrl=tp_gloo,
                              machine_id=pair,
                              res_boxes={e["machine"]: e["boxes"][pair] for e in mine})
        peer = peers[pair]
    push_alone = None
    if is_prompt:
        # KV-push kernel alone over NVLink (no concurrent prefill): one layer of
        # 2048 prompt rows into the peer pool's first blocks (no live
        # sequences yet), CUDA-event timed
        rows = min(2048, peer.num_blocks * peer.block_size)
        qkv = torch.randn(rows, runner.qkv_cols, device="cuda").bfloat16()
        slots = torch.arange(rows, dtype=torch.int32, device="cuda")
        push_alone = {}
        for ctas in (runner.push_ctas, 148):
            f = lambda: K.kv_push_layer(qkv, rows, runner.hq, runner.hkv, runner.dh,  # noqa: E731
                                        peer.k_layer_ptr(0), peer.v_layer_ptr(0), slots,
                                        peer.block_size, ctas)
            f()
            torch.cuda.synchronize()
            s_, e_ = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            s_.record()
            for _ in range(10):
                f()
            e_.record()
            torch.cuda.synchronize()
            push_alone[ctas] = rows * 2 * runner.hkv * runner.dh * 2 / (s_.elapsed_time(e_) / 10) / 1e6
        del qkv, slots
    g = torch.Generator().manual_seed(1234 + pair)
    reqs = [(pair * R + i, torch.randint(0, cfg.vocab, (P,), generator=g, dtype=torch.int32), O)
            for i in range(R)]
    prompts_dev = {rid: p.cuda() for rid, p, _ in reqs}

    def one_step(resident_prompts: bool):
        dist.barrier()
        torch.cuda.synchronize()
        s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        t0 = time.perf_counter()
        s.record()
        if is_prompt:
            out = server.serve_burst(reqs, t0, prompts_dev if resident_prompts else None)
        else:
            out = server.serve_burst(reqs, t0)
        e.record()
        torch.cuda.synchronize()
        wall = time.perf_counter() - t0
        dev_ms = torch.tensor([s.elapsed_time(e)], device="cuda")
        dist.all_reduce(dev_ms, op=dist.ReduceOp.MAX)
        return t0, out, float(dev_ms), wall

    for _ in range(args.warmup):
        one_step(False)
    if getattr(args, "trace", None):
        _trace_phase(args, rank, world, local, pair, is_prompt, server, cfg, ctrl, ClockSampler,
                     percentile, peaks, tp)
        return
    launches0 = _abi.launch_count()
    e2e_ms, ttft, tbt, gaps2, push_gbs, push_tail, push_raw = [], [], [], [], [], [], []
    dec_steps, pre_ms, pre_flops, overhead = [], [], [], []
    with ClockSampler(local) as clk:
        for _ in range(args.steps):
            t0, out, dms, wall = one_step(False)
            gathered = [None] * world
            payload = {"rank": rank, "t0": t0}
            if is_prompt:
                payload["push"] = [(st.bytes_per_layer, st.layer_ms, st.tail_ms, st.compute_ms,
                                    st.mode) for st in server.push_log[-8:]]
                server.push_log.clear()
            else:
                payload["emit"], payload["first"] = out[0], out[2]
                payload["steps"] = list(server.step_log)
            dist.all_gather_object(gathered, payload, group=ctrl)
            e2e_ms.append(dms)
            for pr in range(0, world, 2 * tp):
                tok = gathered[pr + tp]
                dec_steps += tok["steps"]
                t0p = gathered[pr]["t0"]
                for rid, tf in tok["first"].items():
                    ttft.append((tf - t0p) * 1e3)        # all requests arrive at t0
                    seq = [tf] + tok["emit"][rid]
                    g_ = [(b - a) * 1e3 for a, b in zip(seq, seq[1:])]
                    tbt += g_
                    if g_:
                        gaps2.append(g_[0])
                for bpl, lms, tail, cms, mode in gathered[pr]["push"]:
                    push_gbs.append(statistics.mean(kv_push_gbps(bpl, m) for m in lms))
                    plan = measured_plan(mode, lms, tail)   # reference TransferPlan record
                    push_tail.append(plan.visible_latency)
                    push_raw.append(plan.raw_time)
                    pre_ms.append(cms)
                    overhead.append(tail / cms if cms > 0 else 0.0)
            pre_flops.append(R * cfg.prefill_flops(P, tp))
        dev_ms = []
        for _ in range(args.steps):
            dev_ms.append(one_step(True)[2])
    launches = _abi.launch_count() - launches0
    launches_t = torch.tensor([launches], device="cuda", dtype=torch.float64)
    dist.all_reduce(launches_t)
    clocks = clk.summary()
    if rank == 0:
        hbm_peak, tc_peak, _tcs, peak_kind = peaks()
        pairs = world // (2 * tp)
        toks_step = pairs * R * O
        ms = statistics.mean(dev_ms)
        # every prompt batch of a step is timed on its machine; a step's R
        # prompts go through one or two batches (2048-token cap)
        batches_per_step = max(1, len(pre_ms) // max(1, args.steps * pairs))
        pre_step_ms = statistics.mean(pre_ms) * batches_per_step
        pre_tfs = statistics.mean(pre_flops) / (pre_step_ms / 1e3) / 1e12
        dec = _decode_roofline(cfg, tp, dec_steps, hbm_peak, peak_kind)
        line = {
            "metric": metric_name(cfg, P, O),
            "value": toks_step / (ms / 1e3), "unit": "tokens/s", "n_gpus": world,
            "steps": args.steps, "warmup": args.warmup, "ms_per_step": ms,
            "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "bf16",
            "data": "synthetic (seeded random weights/tokens)",
            "config": {"workload": f"{cfg.name} {P}-token prompts / {O} greedy outputs, 1 request "
                                   f"per GPU per step; {pairs} Splitwise pair(s) TP{tp}+TP{tp}, "
                                   "layer-wise KV push over NVLink, batched decode on the token "
                                   "machine",
                       "model": cfg.name, "prompt_tokens": P, "output_tokens": O,
                       "requests_per_step": pairs * R,
                       "parallelism": f"{pairs}x(prompt TP{tp} + token TP{tp})",
                       "l2": f"inputs > L2 ({cfg.weight_bytes(tp) / 1e9:.1f} GB weights "
                             "per GPU streamed per decode step)"},
            "ttft_ms": {"p50": percentile(ttft, 0.5), "p99": percentile(ttft, 0.99)},
            "tbt_ms": {"p50": percentile(tbt, 0.5), "p99": percentile(tbt, 0.99)},
            "second_token_gap_ms": {"p50": percentile(gaps2, 0.5)},
            "e2e": {"value": toks_step / (statistics.mean(e2e_ms) / 1e3), "unit": "tokens/s",
                    "ms_per_step": statistics.mean(e2e_ms),
                    "h2d_bytes_per_step": pairs * R * 4 * (4 * P),
                    "d2h_bytes_per_step": pairs * R * 4 * O},
            "phases_ms": {"prefill": pre_step_ms,
                          "decode_step": _full_batch_ms(dec_steps)},
            "kv_transfer": {"mode": "layerwise P2P push (NVLink, CUDA IPC); hand-off flags "
                                    "stored by the prompt GPU (swb_kv_handoff)",
                            "push_GBps_per_layer": statistics.mean(push_gbs),
                            "nvlink_peak_GBps": 770.0,
                            "frac": statistics.mean(push_gbs) / 770.0,
                            "raw_ms": statistics.mean(push_raw),
                            "visible_ms": statistics.mean(push_tail),
                            "visible_frac_of_prefill": statistics.mean(overhead),
                            "visible_frac_of_ttft": statistics.mean(push_tail) /
                            percentile(ttft, 0.5),
                            "push_kernel_alone_GBps": {f"{c}_ctas": round(v, 1)
                                                       for c, v in push_alone.items()},
                            "push_kernel_alone_frac": max(push_alone.values()) / 770.0,
                            "note": "push_GBps_per_layer is measured in flight, sharing the "
                                    "SMs with the next layers' prefill (64 CTAs); "
                                    "push_kernel_alone_* is the same kernel timed alone, vs "
                                    "770 GB/s measured peer copy (900 nominal)"},
            "roofline": dec,
            "roofline_prefill": {"bound": "tensor", "achieved": pre_tfs, "peak": tc_peak,
                                 "unit": "TFLOP/s", "frac": pre_tfs / tc_peak,
                                 "algorithmic_flops": statistics.mean(pre_flops),
                                 "peak_kind": peak_kind, "kernel": "prompt machine prefill"},
            "gpu_launches": int(launches_t.item()),
            "clocks": clocks,
        }
        if not getattr(args, "no_cpu", False):
            # the other ranks wait in a gloo (sleeping) barrier, and their
            # processes keep one core each: an OpenMP region with a thread on
            # a busy core runs at the speed of its time slice
            line["cpu_baseline"] = cpu_baseline(args.model, P, O,
                                                threads=max(1, (os.cpu_count() or 1) - world))
        print(json.dumps(line), flush=True)
    dist.barrier(group=ctrl)
    torch.cuda.synchronize()
    server.close()
    # NCCL sub-communicator teardown can stall at interpreter exit (seen with
    # TP groups + CUDA IPC mappings); the result is printed, so bound it.
    threading.Timer(30.0, lambda: os._exit(0)).start()
    dist.destroy_process_group()
    os._exit(0)


def _trace_phase(args, rank, world, local, pair, is_prompt, server, cfg, ctrl, ClockSampler,
                 percentile, peaks, tp=1):
    """bench.py --trace: the reference's synthetic trace (reference trace.py
    presets and generator, via tools/reftrace.py; Poisson arrivals) served concurrently by the Splitwise pairs in real
    time; each request is routed at its arrival to the pair with the fewest
    pending tokens (control.RouteBoard, the reference's JSQ; --route rr:
    request i -> pair i mod pairs); TP pairs process arrivals in
    lockstep across their peers.  Rank 0 prints TTFT / TBT / E2E percentiles
    and tokens/s."""
    import json
    pairs = world // (2 * tp)
    reqs_all = list(args.trace_requests)     # the reference generator's trace (bench.py)
    if args.max_output:
        reqs_all = [type(r)(r.id, r.arrival, r.prompt_tokens, min(r.output_tokens, args.max_output))
                    for r in reqs_all]
    g = torch.Generator().manual_seed(77)
    prompts = {r.id: torch.randint(0, cfg.vocab, (r.prompt_tokens,), generator=g,
                                   dtype=torch.int32) for r in reqs_all}
    jsq = getattr(args, "route", "jsq") == "jsq" and pairs > 1
    board, router = None, None
    if jsq:
        # live JSQ, independent prompt and token picks (control.RouteBoard);
        # rank 0 hosts the router
        name = [None]
        if rank == 0:
            board = RouteBoard(len(reqs_all), pairs, pairs, create=True)
            name = [board.name]
        dist.broadcast_object_list(name, src=0, group=ctrl)
        if rank != 0:
            board = RouteBoard(len(reqs_all), pairs, pairs, name=name[0])
        server.board = board
        items = [(r.id, r.arrival, prompts[r.id], r.output_tokens) for r in reqs_all]
        feed = ArrivalFeed(items, pair, board, role="prompt" if is_prompt else "token")
    else:
        mine = [r for r in reqs_all if r.id % pairs == pair]
        items = [(r.id, r.arrival, prompts[r.id], r.output_tokens) for r in mine]
        feed = None
    if not is_prompt:
        server.prewarm()
    dist.barrier(group=ctrl)
    # common start (perf_counter is CLOCK_MONOTONIC: comparable across processes)
    t0t = torch.tensor([time.perf_counter() + 1.0], dtype=torch.float64)
    dist.broadcast(t0t, src=0, group=ctrl)
    t0 = float(t0t.item())
    if jsq and rank == 0:
        router = threading.Thread(target=board.run_router, daemon=True,
                                  args=([(r.id, r.arrival, r.prompt_tokens) for r in reqs_all], t0))
        router.start()
    while time.perf_counter() < t0:
        time.sleep(1e-4)
    with ClockSampler(local) as clk:
        out = server.serve_trace(items, t0, feed)
    if router is not None:
        router.join()
    payload = {"rank": rank, "prompt": is_prompt, "out": None if is_prompt else out[0],
               "steps": None if is_prompt else out[1], "first": None if is_prompt else out[2],
               "tokens": None if is_prompt else server.tokens}
    gathered = [None] * world
    dist.all_gather_object(gathered, payload, group=ctrl)
    if rank == 0:
        arrival = {r.id: t0 + r.arrival for r in reqs_all}
        first = {}
        emits = {}
        steps = []
        gen_tokens = {}
        for gp in gathered:
            if gp["rank"] % tp:          # TP peers report the same requests
                continue
            if not gp["prompt"]:
                first.update(gp["first"])       # the token host saw the first token land
                emits.update(gp["out"])
                steps += gp["steps"]
                gen_tokens.update(gp["tokens"])
        ttft, tbt, e2e = [], [], []
        ntok = 0
        t_end = 0.0
        for r in reqs_all:
            seq = [first[r.id]] + emits.get(r.id, [])
            ntok += len(seq)
            ttft.append((first[r.id] - arrival[r.id]) * 1e3)
            tbt += [(b - a) * 1e3 for a, b in zip(seq, seq[1:])]
            e2e.append((seq[-1] - arrival[r.id]) * 1e3)
            t_end = max(t_end, seq[-1])
        span = t_end - t0
        hbm_peak, _tc, _tcs, peak_kind = peaks()
        p = lambda xs, q: percentile(xs, q) if xs else None  # noqa: E731
        line = {
            "metric": f"TTFT/TBT p50,p99 + tokens/s serving the reference's {args.trace} trace, "
                      f"{cfg.name}",
            "value": ntok / span, "unit": "tokens/s", "n_gpus": world, "higher_is_better": True,
            "scaling": "weak", "vs_baseline": None, "dtype": "bf16",
            "data": "synthetic trace (reference presets, Poisson arrivals), random weights",
            "config": {"workload": f"{args.trace} trace rate {args.rate}/s for {args.duration} s "
                                   f"(seed {args.seed}), {len(reqs_all)} requests, "
                                   f"{pairs} Splitwise pair(s) TP{tp}+TP{tp}, "
                                   + ("live JSQ routing at arrival, independent prompt and "
                                      "token picks (any prompt machine -> any token machine)"
                                      if jsq else
                                      f"request i -> pair i mod {pairs}" if pairs > 1 else
                                      "every request on the one pair")
                                   + ", served concurrently in real time",
                       "model": cfg.name,
                       "parallelism": f"{pairs}x(prompt TP{tp} + token TP{tp})",
                       "max_output": args.max_output or None,
                       "routing": "jsq" if jsq else "round-robin" if pairs > 1 else "single pair"},
            "ttft_ms": {"p50": p(ttft, 0.5), "p99": p(ttft, 0.99)},
            "tbt_ms": {"p50": p(tbt, 0.5), "p99": p(tbt, 0.99)},
            "e2e_ms": {"p50": p(e2e, 0.5), "p99": p(e2e, 0.99)},
            "requests": len(reqs_all), "output_tokens": ntok, "makespan_s": span,
            "roofline": _decode_roofline(cfg, tp, steps, hbm_peak, peak_kind),
            "clocks": clk.summary(),
        }
        if getattr(args, "dump_tokens", None):
            with open(args.dump_tokens, "w") as f:
                json.dump({str(k): v for k, v in gen_tokens.items()}, f)
        print(json.dumps(line), flush=True)
    dist.barrier()
    torch.cuda.synchronize()
    server.close()
    if board is not None:
        board.close()
    threading.Timer(30.0, lambda: os._exit(0)).start()
    dist.destroy_process_group()
    os._exit(0)
