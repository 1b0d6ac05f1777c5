"""Control channel between a prompt machine and its token machine.

Only tiny int32 messages cross it (the KV bytes go GPU-to-GPU over NVLink):

  * reservation  token -> prompt : the KV sequence slots the token machine
    reserved (final context = prompt + outputs) for the routed requests, so
    the prompt machine can push each layer straight into those blocks
    (both machines are chosen at arrival, reference cluster.py:153-160);
  * hand-off     prompt -> token : one row per request whose prompt phase
    finished and whose KV landed: (request id, KV slot, prompt length, first
    token, output tokens) — the reference's TRANSFER event + token-task
    enqueue (engine.py:286-297).

Hand-offs travel through a single-producer/single-consumer mailbox in host
shared memory (``ShmMailbox``; the pair always shares a node because the KV
moves over NVLink), because a decode loop must be able to *poll* for them
between iterations: a gloo ``irecv`` only reports completion once waited on.
``HandoffReceiver`` polls it; when the token machine is a tensor-parallel
group, every TP peer admits a hand-off at the same scheduler iteration (a MIN
all-reduce of "received" flags over the TP group), so the peers' batches —
and the NCCL all-reduces inside their decode steps — stay identical.
"""

from __future__ import annotations

import time
from multiprocessing import shared_memory

import numpy as np
import torch
import torch.distributed as dist

HANDOFF_FIELDS = ("request_id", "kv_slot", "prompt_tokens", "first_token", "output_tokens")


def send_reservations(slots, dst: int, group) -> None:
    dist.send(torch.tensor(list(slots), dtype=torch.int32), dst=dst, group=group)


def recv_reservations(n: int, src: int, group) -> list:
    buf = torch.empty(n, dtype=torch.int32)
    dist.recv(buf, src=src, group=group)
    return buf.tolist()


class ShmMailbox:
    """SPSC ring of int64 records in /dev/shm: header [write_seq, read_seq],
    then NSLOT slots of [n_rows, rows(MAXROWS x 5)].  The producer writes the
    slot, then publishes write_seq (an aligned 8-byte store, ordered after the
    slot writes on x86-TSO); the consumer reads it, then bumps read_seq."""

    NSLOT, MAXROWS = 64, 64
    SLOT = 1 + MAXROWS * 5

    def __init__(self, name: str | None = None, create: bool = False):
        size = 8 * (2 + self.NSLOT * self.SLOT)
        if create:
            self.shm = shared_memory.SharedMemory(create=True, size=size)
        else:
            self.shm = shared_memory.SharedMemory(name=name)
            try:  # the creator owns (and unlinks) the segment, not the attacher
                from multiprocessing import resource_tracker
                resource_tracker.unregister(self.shm._name, "shared_memory")
            except Exception:
                pass
        self.owner = create
        self.a = np.ndarray((2 + self.NSLOT * self.SLOT,), dtype=np.int64, buffer=self.shm.buf)
        if create:
            self.a[:] = 0

    @property
    def name(self) -> str:
        return self.shm.name

    def put(self, rows) -> None:
        rows = [list(r) for r in rows]
        for i in range(0, len(rows), self.MAXROWS):
            chunk = rows[i:i + self.MAXROWS]
            seq = int(self.a[0])
            while seq - int(self.a[1]) >= self.NSLOT:   # ring full: consumer lags
                time.sleep(1e-4)
            base = 2 + (seq % self.NSLOT) * self.SLOT
            self.a[base] = len(chunk)
            self.a[base + 1:base + 1 + 5 * len(chunk)] = np.asarray(chunk, dtype=np.int64).ravel()
            self.a[0] = seq + 1

    def ready(self) -> bool:
        return int(self.a[0]) > int(self.a[1])

    def get(self):
        seq = int(self.a[1])
        if int(self.a[0]) <= seq:
            return None
        base = 2 + (seq % self.NSLOT) * self.SLOT
        n = int(self.a[base])
        rows = [tuple(int(v) for v in self.a[base + 1 + 5 * i:base + 6 + 5 * i]) for i in range(n)]
        self.a[1] = seq + 1
        return rows

    def close(self) -> None:
        try:
            self.shm.close()
            if self.owner:
                self.shm.unlink()
        except Exception:
            pass


class RouteBoard:
    """Live JSQ routing across Splitwise pairs served concurrently in real
    time (bench.py --trace).  One /dev/shm segment per run:

      * ``assign[rid]`` — the pair a request was routed to (-1 = not yet
        arrived), written once by the router at the request's arrival;
      * per pair, cumulative counters the servers publish (absolute values, so
        every TP peer may write them): prompt tokens / requests whose prompt
        phase finished (prompt machine), requests finished (token machine).

    The router keeps the cumulative routed prompt tokens and requests per
    pair, so pending(pair) = queued prompt tokens (routed − prompt-done) +
    one per live token task (prompt-done − finished): the reference's
    ``pending_tokens`` (cluster.py:82-84) of the pair's prompt machine plus
    that of its token machine.  The pick is the reference's ``_argmin``
    (cluster.py:129-134): lowest (pending, id).  The prompt → token pairing
    is fixed (each prompt machine pushes to its own token machine), so the
    two JSQ picks of ``Cluster.route`` (cluster.py:153-160) collapse into
    one pick over pairs."""

    PROMPT_TOK, PROMPT_REQ, FINISHED = 0, 1, 2

    def __init__(self, n_requests: int, pairs: int, name: str | None = None,
                 create: bool = False):
        self.n, self.pairs = n_requests, pairs
        size = 8 * (n_requests + 3 * pairs + 1)
        if create:
            self.shm = shared_memory.SharedMemory(create=True, size=size)
        else:
            self.shm = shared_memory.SharedMemory(name=name)
            try:
                from multiprocessing import resource_tracker
                resource_tracker.unregister(self.shm._name, "shared_memory")
            except Exception:
                pass
        self.owner = create
        a = np.ndarray((n_requests + 3 * pairs + 1,), dtype=np.int64, buffer=self.shm.buf)
        self.assign = a[:n_requests]
        self.load = a[n_requests:n_requests + 3 * pairs].reshape(pairs, 3)
        if create:
            self.assign[:] = -1
            self.load[:] = 0
        self.routed_tok = [0] * pairs
        self.routed_req = [0] * pairs

    @property
    def name(self) -> str:
        return self.shm.name

    # -- servers --------------------------------------------------------
    def publish(self, pair: int, field: int, value: int) -> None:
        self.load[pair, field] = value

    # -- router ---------------------------------------------------------
    def pending(self, pair: int) -> int:
        tok, req, fin = (int(v) for v in self.load[pair])
        return (self.routed_tok[pair] - tok) + (req - fin)

    def route(self, rid: int, prompt_tokens: int) -> int:
        best = min(range(self.pairs), key=lambda p: (self.pending(p), p))
        self.routed_tok[best] += prompt_tokens
        self.routed_req[best] += 1
        self.assign[rid] = best     # publish last: servers poll assign
        return best

    def run_router(self, requests, t0: float) -> None:
        """Route each request at its arrival (wall clock from t0); requests =
        [(rid, arrival_s, prompt_tokens)] in arrival order."""
        for rid, arr, ptok in requests:
            while True:
                d = t0 + arr - time.perf_counter()
                if d <= 0:
                    break
                time.sleep(min(d, 1e-3))
            self.route(rid, ptok)

    def close(self) -> None:
        try:
            self.shm.close()
            if self.owner:
                self.shm.unlink()
        except Exception:
            pass


class ArrivalFeed:
    """Server side of the live routing: yields, in arrival order, the
    requests routed to ``pair`` whose routing is already published.  With no
    board it is the static list (request i -> pair i mod pairs)."""

    def __init__(self, requests, pair: int, board: RouteBoard | None = None):
        self.all = list(requests)
        self.pair = pair
        self.board = board
        self.cursor = 0
        self.mine = 0

    def poll(self) -> list:
        out = []
        if self.board is None:
            out, self.all = self.all, []
            self.mine += len(out)
            return out
        while self.cursor < len(self.all):
            r = self.all[self.cursor]
            p = int(self.board.assign[r[0]])
            if p < 0:
                break
            if p == self.pair:
                out.append(r)
            self.cursor += 1
        self.mine += len(out)
        return out

    def complete(self) -> bool:
        """Every request has been routed (so ``mine`` is final)."""
        if self.board is None:
            return not self.all
        return self.cursor == len(self.all)


class HandoffReceiver:
    """Token-side end: owns the mailbox (its name goes to the prompt side at
    start-up) and polls it between decode iterations."""

    def __init__(self, tp_group=None):
        self.box = ShmMailbox(create=True)
        self.tp_group = tp_group

    @property
    def name(self) -> str:
        return self.box.name

    def poll(self, block: bool = False):
        """Rows of the next hand-off, or None if it has not arrived on every TP
        peer yet.  ``block`` waits for it."""
        while True:
            ready = 1 if self.box.ready() else 0
            if self.tp_group is not None:
                flag = torch.tensor([ready], dtype=torch.int32)
                dist.all_reduce(flag, op=dist.ReduceOp.MIN, group=self.tp_group)
                ready = int(flag.item())
            if ready:
                return self.box.get()
            if not block:
                return None
            time.sleep(2e-5)

    def close(self) -> None:
        self.box.close()


class HandoffSender:
    """Prompt-side end: attaches to the token machine's mailbox by name."""

    def __init__(self, name: str):
        self.box = ShmMailbox(name=name)

    def send(self, rows) -> None:
        self.box.put(rows)

    def close(self) -> None:
        self.box.close()
