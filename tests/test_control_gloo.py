"""Multi-process (gloo, CPU) tests of the prompt -> token control channel
(paper_2311_18677_b200/control.py): reservations with epochs, hand-off
records in the shared table (written here by the peer process the way the
prompt GPU's swb_kv_handoff writes them: token, then flag), non-blocking
polling, prefix/epoch admission, and TP lockstep admission across a token
machine's TP group."""

import os
import socket
import time

import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _init(rank, world, port):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)


def _land(table, seq, epoch, token, key=0, n=1):
    """What swb_kv_handoff does from the prompt GPU: token, group key and
    size, then the flag."""
    table.a[seq, 1] = token
    table.a[seq, 2] = key
    table.a[seq, 3] = n
    table.a[seq, 0] = epoch


def _pair(rank, world, port, q):
    from paper_2311_18677_b200.control import (HandoffTable, HandoffWatch,
                                               recv_reservations, send_reservations)
    _init(rank, world, port)
    try:
        if rank == 1:                     # token machine
            table = HandoffTable(8, create=True)
            watch = HandoffWatch(table)
            dist.send_object_list([table.name], dst=0)
            send_reservations([3, 5], 0, None, epochs=[7, 2])
            watch.expect(10, 3, 7, 1024, 128)
            watch.expect(11, 5, 2, 999, 1)
            got, polls = [], 0
            while len(got) < 2:
                got += watch.poll()
                polls += 1
                time.sleep(0.005)
            seen = sorted(watch.seen)
            table.close()
            q.put(("token", got, polls, seen))
        else:                             # prompt machine
            name = [None]
            dist.recv_object_list(name, src=1)
            table = HandoffTable(name=name[0])
            slots, epochs = recv_reservations(2, 1, None, with_epochs=True)
            time.sleep(0.1)               # the token side polls meanwhile
            _land(table, slots[1], epochs[1] - 1, 99, key=1)   # stale epoch: must not admit
            _land(table, slots[0], epochs[0], 77, key=1)
            time.sleep(0.05)
            _land(table, slots[1], epochs[1], 42, key=2)
            table.close()
            q.put(("prompt", (slots, epochs), 0, None))
    finally:
        dist.destroy_process_group()


def test_reservation_and_handoff_roundtrip():
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_pair, args=(r, 2, port, q)) for r in range(2)]
    for p in procs:
        p.start()
    out = dict((k, (a, b, c)) for k, a, b, c in (q.get(timeout=120) for _ in range(2)))
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    assert out["prompt"][0] == ([3, 5], [7, 2])
    rows, polls, seen = out["token"]
    assert rows == [(10, 3, 1024, 77, 128), (11, 5, 999, 42, 1)]
    assert polls > 1          # it polled without blocking before the flags landed
    assert seen == [10, 11]


def test_handoff_groups_and_epochs():
    """A prompt batch's requests are admitted together once its whole group
    landed; groups (e.g. from different prompt machines) in landing order;
    only the current epoch of a slot counts."""
    from paper_2311_18677_b200.control import HandoffTable, HandoffWatch
    table = HandoffTable(8, create=True)
    try:
        w = HandoffWatch(table)
        w.expect(1, 0, 5, 10, 3)
        w.expect(2, 1, 1, 20, 4)          # rids 2, 3: one batch of another machine
        w.expect(3, 2, 1, 30, 5)
        _land(table, 1, 1, 8, key=7, n=2)  # half of group 7
        assert w.poll() == [] and 2 in w.seen
        _land(table, 0, 4, 9, key=6)      # previous epoch of slot 0
        assert w.poll() == []
        _land(table, 2, 1, 4, key=7, n=2)  # group 7 complete: admitted before rid 1
        assert w.poll() == [(2, 1, 20, 8, 4), (3, 2, 30, 4, 5)]
        _land(table, 0, 5, 6, key=6)
        assert w.poll() == [(1, 0, 10, 6, 3)]
        assert w.pending == [] and set(w.seen) == {1, 2, 3}
    finally:
        table.close()


def _tp_group(rank, world, port, q):
    """ranks 0,1 = prompt TP group, 2,3 = token TP group; prompt rank i lands
    on token rank i+2's table, rank 1's landing is delayed: both token ranks
    must admit at the same poll iteration."""
    from paper_2311_18677_b200.control import HandoffTable, HandoffWatch
    _init(rank, world, port)
    try:
        tok_group = dist.new_group([2, 3], backend="gloo")
        dist.new_group([0, 1], backend="gloo")
        if rank < 2:
            name = [None]
            dist.recv_object_list(name, src=rank + 2)
            table = HandoffTable(name=name[0])
            time.sleep(0.05 if rank == 0 else 0.4)
            _land(table, 1, 3, 5)
            table.close()
        else:
            table = HandoffTable(4, create=True)
            watch = HandoffWatch(table, tp_group=tok_group)
            watch.expect(7, 1, 3, 100, 9)
            dist.send_object_list([table.name], dst=rank - 2)
            it = 0
            while True:
                rows = watch.poll()
                if rows:
                    break
                it += 1
                time.sleep(0.01)
            # both peers saw it at the same iteration
            t = torch.tensor([it], dtype=torch.int64)
            lo, hi = t.clone(), t.clone()
            dist.all_reduce(lo, op=dist.ReduceOp.MIN, group=tok_group)
            dist.all_reduce(hi, op=dist.ReduceOp.MAX, group=tok_group)
            table.close()
            q.put((rank, rows, int(lo), int(hi)))
    finally:
        dist.destroy_process_group()


def test_tp_lockstep_admission():
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_tp_group, args=(r, 4, port, q)) for r in range(4)]
    for p in procs:
        p.start()
    res = [q.get(timeout=120) for _ in range(2)]
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    for rank, rows, lo, hi in res:
        assert rows == [(7, 1, 100, 5, 9)]
        assert lo == hi           # admitted in lockstep
        assert lo >= 10           # and only once the slow peer's record landed


if __name__ == "__main__":
    pytest.main([__file__, "-q"])
