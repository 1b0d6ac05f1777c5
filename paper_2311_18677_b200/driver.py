"""Request-lifecycle driver: arrival -> JSQ route (both machines at arrival)
-> prompt iterations -> KV hand-off -> token iterations -> completion.

The hand-off rules are the reference engine's (reference engine.py:202-336):
* on arrival, route and enqueue the prompt task (tokens = prompt size,
  remaining = outputs) on the prompt machine (engine.py:230-248);
* when a prompt finishes its first token is emitted; if more tokens are
  due, the token task (tokens = prompt + 1, remaining = outputs - 1,
  engine.py:292-297) is enqueued on the token machine — immediately when it
  is the same machine, otherwise once the KV transfer's visible latency has
  elapsed, the transfer being planned over the batch's prompt compute time
  (engine.py:253, :275-290, :325-327);
* after every event the pools are maintained and every touched idle machine
  with work forms its next batch, in machine-id order (engine.py:206-228,
  :311-336); memory never exceeds capacity (engine.py:338-342).

Iteration and transfer durations come from a *backend*.  ``ModeledBackend``
prices them with the machines' PerfModel (virtual clock) — with the
reference's calibration presets it reproduces the reference simulator
request-for-request (tests/test_reference_parity.py), and with B200-measured
PerfModels (perf.measure_perf_model) it is the C5-style scheduler sweep.
The GPU serving paths (serving.py / splitwise.py) drive the same Machine /
Cluster objects with durations measured on the device.
"""

from __future__ import annotations

import heapq
import math
from dataclasses import dataclass, field

from .cluster import Cluster, ClusterConfig
from .metrics import MetricsReport, RequestRecord
from .transfer import plan_transfer
from .workers import PROMPT, TOKEN, Task

ARRIVAL, ITERATION, TRANSFER, MAINTENANCE = (
    "request_arrival", "iteration_complete", "transfer_complete", "pool_maintenance")


@dataclass(frozen=True)
class Request:
    id: int
    arrival: float        # seconds
    prompt_tokens: int
    output_tokens: int


class ModeledBackend:
    """Durations from the PerfModels (the reference's timing model)."""

    def iteration_ms(self, machine, batch) -> float:
        return batch.iteration_time

    def transfer_visible_ms(self, driver, rec: RequestRecord, prompt_ms: float) -> float:
        perf = driver.cluster.machines[rec.prompt_machine].perf
        kv = perf.kv_cache_bytes(rec.prompt_tokens)
        plan = plan_transfer(rec.prompt_tokens, kv, prompt_ms, driver.config.transfer)
        rec.transfer_raw_ms = plan.raw_time
        return plan.visible_latency


@dataclass
class DriverResult:
    report: MetricsReport
    records: dict
    event_log: list = field(default_factory=list)
    cluster: Cluster | None = None


class Driver:
    def __init__(self, config: ClusterConfig, perf_models: dict, requests: list,
                 backend=None, horizon_s: float | None = None, record_log: bool = True,
                 duration_s: float | None = None):
        self.config = config
        self.cluster = Cluster(config, perf_models)
        self.requests = list(requests)
        self.backend = backend or ModeledBackend()
        span = duration_s if duration_s is not None else max(
            (r.arrival for r in self.requests), default=0.0)
        self.horizon_ms = 1e3 * (horizon_s if horizon_s is not None else span + 600.0)
        self.record_log = record_log
        self.records: dict[int, RequestRecord] = {}
        self._queue: list = []
        self._counter = 0
        self._log: list = []
        self._touched: set[int] = set()
        self._prompt_ms: dict[int, float] = {}
        self._done = 0
        if hasattr(self.backend, "attach"):     # measured backends bind machines to GPUs
            self.backend.attach(self)

    # ---- plumbing ----------------------------------------------------------
    def _schedule(self, t_ms: float, kind: str, payload) -> None:
        heapq.heappush(self._queue, (t_ms, self._counter, kind, payload))
        self._counter += 1

    def _note(self, t_ms: float, kind: str, text: str) -> None:
        if self.record_log:
            self._log.append((t_ms, len(self._log), kind, text))

    def _moves(self, moves) -> None:
        for t, mid, old, new in moves:
            self._note(t, "pool_transition", f"machine={mid} from={old} to={new}")
            self._touched.add(mid)

    # ---- main loop -----------------------------------------------------------
    def run(self) -> DriverResult:
        for r in self.requests:
            self.records[r.id] = RequestRecord(r.id, r.arrival * 1e3, r.prompt_tokens,
                                               r.output_tokens, arrival_s=r.arrival)
            self._schedule(r.arrival * 1e3, ARRIVAL, r.id)
        win = self.config.repurpose_window_s
        if self.config.repurpose_enabled and math.isfinite(win):
            self._schedule(win * 1e3, MAINTENANCE, None)
        handlers = {ARRIVAL: self._arrival, ITERATION: self._iteration_done,
                    TRANSFER: self._transfer_done, MAINTENANCE: self._maintenance}
        total = len(self.requests)
        while self._queue and self._done < total:
            t, _, kind, payload = heapq.heappop(self._queue)
            if t > self.horizon_ms:
                raise RuntimeError(f"run exceeded horizon with {total - self._done} unfinished")
            handlers[kind](t, payload)
            self._moves(self.cluster.update_pools(t))
            self._dispatch(t)
        if self._done < total:
            raise RuntimeError("event queue drained with unfinished requests")
        recs = [self.records[r.id] for r in self.requests]
        makespan = max((r.completion for r in recs), default=0.0)
        util = {m.id: (m.busy_time / makespan if makespan > 0 else 0.0)
                for m in self.cluster.machines.values()}
        return DriverResult(MetricsReport(recs, makespan, util), self.records, self._log,
                            self.cluster)

    # ---- handlers --------------------------------------------------------------
    def _enqueue(self, t_ms, mid, task: Task) -> None:
        m = self.cluster.machines[mid]
        m.enqueue(task, t_ms)
        self._note(t_ms, "task_enqueued",
                   f"machine={mid} request={task.request_id} kind={task.kind} tokens={task.tokens}")
        self._moves(self.cluster.note_enqueue(m, task.kind, t_ms))
        self._touched.add(mid)

    def _arrival(self, t_ms, rid) -> None:
        rec = self.records[rid]
        d = self.cluster.route(rid, t_ms)
        rec.prompt_machine, rec.token_machine = d.prompt_machine, d.token_machine
        self._note(t_ms, ARRIVAL, f"request={rid} prompt_machine={d.prompt_machine} "
                                  f"token_machine={d.token_machine}")
        self._enqueue(t_ms, d.prompt_machine,
                      Task(rid, PROMPT, rec.prompt_tokens, t_ms, rec.output_tokens,
                           rec.output_tokens))

    def _iteration_done(self, t_ms, mid) -> None:
        m = self.cluster.machines[mid]
        batch = m.running
        prompt_ms = self._prompt_ms.pop(id(batch), 0.0)
        self._note(t_ms, ITERATION, f"machine={mid}")
        for what, task in m.complete_iteration(batch, t_ms):
            rec = self.records[task.request_id]
            if what == "prompt_finished":
                rec.first_token_time = t_ms
                rec.emissions.append(t_ms)
                if rec.output_tokens > 1:
                    self._hand_off(t_ms, rec, prompt_ms)
            elif what == "token_emitted":
                rec.emissions.append(t_ms)
            elif what == "request_finished":
                rec.completion = t_ms
                rec.preempt_count = task.preempt_count
                self._done += 1
                if hasattr(self.backend, "release"):
                    self.backend.release(rec)
        self._touched.add(mid)

    def _hand_off(self, t_ms, rec: RequestRecord, prompt_ms: float) -> None:
        if rec.token_machine == rec.prompt_machine:
            self._token_task(t_ms, rec)
            return
        visible = self.backend.transfer_visible_ms(self, rec, prompt_ms)
        rec.transfer_visible_ms = visible
        self._schedule(t_ms + visible, TRANSFER, rec.request_id)

    def _transfer_done(self, t_ms, rid) -> None:
        rec = self.records[rid]
        self._note(t_ms, TRANSFER, f"request={rid} visible_ms={rec.transfer_visible_ms:.6f}")
        self._token_task(t_ms, rec)

    def _token_task(self, t_ms, rec: RequestRecord) -> None:
        self._enqueue(t_ms, rec.token_machine,
                      Task(rec.request_id, TOKEN, rec.prompt_tokens + 1, t_ms,
                           rec.output_tokens, rec.output_tokens - 1))

    def _maintenance(self, t_ms, _payload) -> None:
        win_ms = self.config.repurpose_window_s * 1e3
        for t, mid, old, new in self.cluster.repurpose(t_ms, win_ms):
            self._note(t, MAINTENANCE, f"machine={mid} repurposed {old}->{new}")
            self._touched.add(mid)
        if self._done < len(self.requests):
            self._schedule(t_ms + win_ms, MAINTENANCE, None)

    def _dispatch(self, t_ms) -> None:
        for mid in sorted(self._touched):
            m = self.cluster.machines[mid]
            if not (m.is_idle() and m.has_work()):
                continue
            batch = m.form_batch(t_ms)
            if batch is None:
                continue
            m.running = batch
            dur = self.backend.iteration_ms(m, batch)
            m.busy_until = t_ms + dur
            m.busy_time += dur
            if batch.prompt_tasks:
                self._prompt_ms[id(batch)] = m.perf.prompt_time(
                    sum(t.tokens for t in batch.prompt_tasks))
            if m.memory_used() > m.perf.memory_capacity + 1e-6:
                raise RuntimeError(f"machine {mid} over memory capacity")
            self._schedule(t_ms + dur, ITERATION, mid)
            self._note(t_ms, "batch_started",
                       f"machine={mid} kind={batch.kind} iter_ms={batch.iteration_time:.6f}")
        self._touched.clear()
