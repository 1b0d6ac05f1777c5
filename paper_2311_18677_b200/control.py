"""Control channel between a prompt machine and its token machine.

Only tiny messages cross it (the KV bytes go GPU-to-GPU over NVLink):

  * reservation  token -> prompt : the KV sequence slot (and its epoch) the
    token machine reserved (final context = prompt + outputs) for each
    routed request, so the prompt machine can push each layer straight into
    those blocks (both machines are chosen at arrival, reference
    cluster.py:153-160);
  * hand-off     prompt GPU -> token host : per KV slot, a record in a
    host shared-memory table [flag, first token] that the prompt GPU writes
    itself after the last layer's push landed (``swb_kv_handoff``: the
    token, then flag = the reservation's epoch behind a full memory
    barrier) — the paper's per-request semaphore and the
    reference's TRANSFER event + token-task enqueue (engine.py:286-297).
    The prompt host never waits for its pushes; the token host polls the
    flags between (and while waiting for) decode iterations.

``HandoffWatch`` is the token host's view: reservations in FIFO order, and a
poll that returns the leading ones whose flag landed.  When the token
machine is a tensor-parallel group, every TP peer admits the same prefix at
the same scheduler iteration (a MIN all-reduce of the landed counts over the
TP group), so the peers' batches — and the collectives inside their decode
steps — stay identical.

Host-memory publication order relies on x86-64 (TSO: loads are not reordered
with older loads, stores not with older stores); ``require_tso`` refuses to
run elsewhere.
"""

from __future__ import annotations

import platform
import time
from multiprocessing import shared_memory

import numpy as np
import torch
import torch.distributed as dist

HANDOFF_FIELDS = ("request_id", "kv_slot", "prompt_tokens", "first_token", "output_tokens")


def require_tso() -> None:
    """The shared-memory records are published with plain stores and read with
    plain loads; that is ordered on x86-64 only."""
    m = platform.machine().lower()
    if m not in ("x86_64", "amd64"):
        raise RuntimeError(f"control-channel shared memory assumes x86-64 TSO, host is {m}")


def send_reservations(slots, dst: int, group, epochs=None) -> None:
    """(slot, epoch) per request; epochs default to 0."""
    epochs = list(epochs) if epochs is not None else [0] * len(slots)
    dist.send(torch.tensor(list(slots) + epochs, dtype=torch.int64), dst=dst, group=group)


def recv_reservations(n: int, src: int, group, with_epochs: bool = False):
    buf = torch.empty(2 * n, dtype=torch.int64)
    dist.recv(buf, src=src, group=group)
    v = buf.tolist()
    return (v[:n], v[n:]) if with_epochs else v[:n]


class ShmMailbox:
    """SPSC ring of int64 records in /dev/shm: header [write_seq, read_seq],
    then NSLOT slots of [n_rows, rows(MAXROWS x 5)].  The producer writes the
    slot, then publishes write_seq (an aligned 8-byte store, ordered after the
    slot writes on x86-TSO); the consumer reads it, then bumps read_seq."""

    NSLOT, MAXROWS = 64, 64
    SLOT = 1 + MAXROWS * 5

    def __init__(self, name: str | None = None, create: bool = False):
        require_tso()
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
    """Live JSQ routing at arrival for the real-time trace path: the
    reference's ``Cluster.route`` (cluster.py:153-160) makes TWO independent
    picks — the prompt machine by JSQ over the prompt pool and the token
    machine by JSQ over the token pool — each the lowest (pending, id)
    (``_argmin``, cluster.py:129-134) with pending = the machine's
    ``pending_tokens`` (cluster.py:82-84): queued prompt tokens on a prompt
    machine, one per live token task on a token machine.  Every prompt
    machine maps every token machine's KV pool, so any pairing is served.

    One /dev/shm segment per run: ``assign_p[rid]`` / ``assign_t[rid]`` (the
    picks, -1 until the request arrives; the prompt pick is published
    first), per prompt machine the prompt tokens whose prompt phase finished,
    per token machine the requests whose KV landed (token task live) and the
    requests finished — cumulative values the servers publish.  The
    router adds the prompt tokens it routed itself."""

    PROMPT_TOK = 0                # prompt machine field
    LANDED, FINISHED = 0, 1       # token machine fields

    def __init__(self, n_requests: int, prompts: int, tokens: int | None = None,
                 name: str | None = None, create: bool = False):
        tokens = prompts if tokens is None else tokens
        self.n, self.prompts, self.tokens = n_requests, prompts, tokens
        size = 8 * (2 * n_requests + prompts + 2 * tokens + 1)
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
        a = np.ndarray((2 * n_requests + prompts + 2 * tokens + 1,), dtype=np.int64,
                       buffer=self.shm.buf)
        self.assign_p = a[:n_requests]
        self.assign_t = a[n_requests:2 * n_requests]
        o = 2 * n_requests
        self.p_load = a[o:o + prompts]
        self.t_load = a[o + prompts:o + prompts + 2 * tokens].reshape(tokens, 2)
        if create:
            a[:] = 0
            self.assign_p[:] = -1
            self.assign_t[:] = -1
        self.routed_tok = [0] * prompts

    @property
    def name(self) -> str:
        return self.shm.name

    # -- servers --------------------------------------------------------
    def publish_prompt(self, machine: int, done_tokens: int) -> None:
        self.p_load[machine] = done_tokens

    def publish_token(self, machine: int, field: int, value: int) -> None:
        self.t_load[machine, field] = value

    # -- router ---------------------------------------------------------
    def pending_prompt(self, m: int) -> int:
        return self.routed_tok[m] - int(self.p_load[m])

    def pending_token(self, m: int) -> int:
        return int(self.t_load[m, self.LANDED]) - int(self.t_load[m, self.FINISHED])

    def route(self, rid: int, prompt_tokens: int) -> tuple[int, int]:
        pm = min(range(self.prompts), key=lambda m: (self.pending_prompt(m), m))
        tm = min(range(self.tokens), key=lambda m: (self.pending_token(m), m))
        self.routed_tok[pm] += prompt_tokens
        self.assign_p[rid] = pm       # publish the prompt pick first: the token
        self.assign_t[rid] = tm       # machine reads it when it reserves
        return pm, tm

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
    requests routed to this machine (``role`` "prompt" or "token") whose
    routing is already published.  With no board it is a static list."""

    def __init__(self, requests, machine: int, board: RouteBoard | None = None,
                 role: str = "prompt"):
        self.all = list(requests)
        self.machine = machine
        self.board = board
        self.assign = None if board is None else (board.assign_p if role == "prompt"
                                                  else board.assign_t)
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
            m = int(self.assign[r[0]])
            if m < 0:
                break
            if m == self.machine:
                out.append(r)
            self.cursor += 1
        self.mine += len(out)
        return out

    def complete(self) -> bool:
        """Every request has been routed (so ``mine`` is final)."""
        if self.board is None:
            return not self.all
        return self.cursor == len(self.all)


class HandoffTable:
    """Per-KV-slot hand-off records in host shared memory, int32
    [max_seqs][STRIDE/4]: word 0 = flag (epoch of the reservation whose KV
    landed), word 1 = first token, word 2 = group key of the prompt batch,
    word 3 = the group's record count in this table.  Created by the token machine's process;
    the prompt machine's process attaches by name and page-locks / maps it
    (``device_ptr``) so its GPU stores the records (swb_kv_handoff)."""

    STRIDE = 16

    def __init__(self, max_seqs: int = 0, name: str | None = None, create: bool = False):
        require_tso()
        if create:
            self.shm = shared_memory.SharedMemory(create=True, size=max(4096, max_seqs * self.STRIDE))
        else:
            self.shm = shared_memory.SharedMemory(name=name)
            try:
                from multiprocessing import resource_tracker
                resource_tracker.unregister(self.shm._name, "shared_memory")
            except Exception:
                pass
        self.owner = create
        self.max_seqs = self.shm.size // self.STRIDE
        self.a = np.ndarray((self.max_seqs, self.STRIDE // 4), dtype=np.int32, buffer=self.shm.buf)
        if create:
            self.a[:] = 0
        self._dev = None
        self._host_ptr = None

    @property
    def name(self) -> str:
        return self.shm.name

    def device_ptr(self) -> int:
        """Device address of this process's mapping (registered on first use)."""
        if self._dev is None:
            import ctypes as C
            from . import _abi
            self._host_ptr = C.addressof(C.c_char.from_buffer(self.shm.buf))
            dev = C.c_void_p()
            _abi.call("swb_host_register", self._host_ptr, self.shm.size, C.byref(dev))
            self._dev = int(dev.value)
        return self._dev

    def landed(self, seq: int, epoch: int) -> bool:
        return int(self.a[seq, 0]) == epoch

    def token(self, seq: int) -> int:
        return int(self.a[seq, 1])

    def group(self, seq: int) -> tuple[int, int]:
        return int(self.a[seq, 2]), int(self.a[seq, 3])

    def close(self) -> None:
        try:
            if self._host_ptr is not None:
                from . import _abi
                _abi.call("swb_host_unregister", self._host_ptr)
                self._host_ptr = None
            del self.a
            self.shm.close()
            if self.owner:
                self.shm.unlink()
        except Exception:
            pass


class HandoffWatch:
    """Token host: the reservations whose KV is on its way, and the first
    instant each landing was observed (the first token's emission).  A
    prompt batch's requests are admitted together (all records of its group
    landed) — the reference enqueues the token tasks of a batch at the same
    transfer time — and groups from different prompt machines in whatever
    order they land."""

    def __init__(self, table: HandoffTable, tp_group=None):
        self.table = table
        self.tp_group = tp_group
        self.pending: list = []          # [rid, seq, epoch, plen, n_out]
        self.seen: dict = {}             # rid -> host time the flag was first observed

    def expect(self, rid: int, seq: int, epoch: int, plen: int, n_out: int) -> None:
        self.pending.append([rid, seq, epoch, plen, n_out])

    def observe(self) -> list:
        """Time-stamp new landings; returns the pending indices whose whole
        group has landed."""
        now = None
        landed, count = [], {}
        for i, (rid, seq, epoch, _p, _o) in enumerate(self.pending):
            if not self.table.landed(seq, epoch):
                continue
            if rid not in self.seen:
                now = now or time.perf_counter()
                self.seen[rid] = now
            key, n = self.table.group(seq)
            landed.append((i, key, n))
            count[key] = count.get(key, 0) + 1
        return [i for i, key, n in landed if count[key] >= n]

    def poll(self) -> list:
        """Hand-off rows (rid, seq, plen, first token, n_out) of the complete
        landed groups, in reservation order — the same set on every TP peer
        (MIN all-reduce of the per-reservation ready mask)."""
        ready = self.observe()
        if self.tp_group is not None and self.pending:
            mask = torch.zeros(len(self.pending), dtype=torch.int32)
            if ready:
                mask[ready] = 1
            dist.all_reduce(mask, op=dist.ReduceOp.MIN, group=self.tp_group)
            ready = mask.nonzero().flatten().tolist()
        if not ready:
            return []
        take = set(ready)
        rows = [(rid, seq, plen, self.table.token(seq), n_out)
                for i, (rid, seq, _e, plen, n_out) in enumerate(self.pending) if i in take]
        self.pending = [r for i, r in enumerate(self.pending) if i not in take]
        return rows
