"""Multi-process (gloo, CPU) tests of the prompt -> token control channel
(paper_2311_18677_b200/control.py): reservations, hand-offs, non-blocking
polling, and TP lockstep admission across a token machine's TP group."""

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


def _pair(rank, world, port, q):
    from paper_2311_18677_b200.control import (HandoffReceiver, HandoffSender,
                                               recv_reservations, send_reservations)
    _init(rank, world, port)
    try:
        if rank == 1:                     # token machine
            rx = HandoffReceiver()
            dist.send_object_list([rx.name], dst=0)
            send_reservations([3, 5], 0, None)
            got, polls = [], 0
            while len(got) < 2:
                rows = rx.poll(block=False)
                polls += 1
                if rows:
                    got += rows
                time.sleep(0.005)
            rx.close()
            q.put(("token", got, polls))
        else:                             # prompt machine
            name = [None]
            dist.recv_object_list(name, src=1)
            tx = HandoffSender(name[0])
            slots = recv_reservations(2, 1, None)
            time.sleep(0.1)               # the token side polls meanwhile
            tx.send([(10, slots[0], 1024, 77, 128)])
            time.sleep(0.05)
            tx.send([(11, slots[1], 999, 42, 1)])
            tx.close()
            q.put(("prompt", slots, 0))
    finally:
        dist.destroy_process_group()


def test_reservation_and_handoff_roundtrip():
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_pair, args=(r, 2, port, q)) for r in range(2)]
    for p in procs:
        p.start()
    out = dict((k, (a, b)) for k, a, b in (q.get(timeout=120) for _ in range(2)))
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    assert out["prompt"][0] == [3, 5]
    rows, polls = out["token"]
    assert rows == [(10, 3, 1024, 77, 128), (11, 5, 999, 42, 1)]
    assert polls > 1          # it polled without blocking before the message came


def _tp_group(rank, world, port, q):
    """ranks 0,1 = prompt TP group, 2,3 = token TP group; prompt rank i sends
    to token rank i+2, rank 1's message is delayed: both token ranks must admit
    at the same poll iteration."""
    from paper_2311_18677_b200.control import HandoffReceiver, HandoffSender
    _init(rank, world, port)
    try:
        tok_group = dist.new_group([2, 3], backend="gloo")
        dist.new_group([0, 1], backend="gloo")
        if rank < 2:
            name = [None]
            dist.recv_object_list(name, src=rank + 2)
            tx = HandoffSender(name[0])
            time.sleep(0.05 if rank == 0 else 0.4)
            tx.send([(7, 1, 100, 5, 9)])
            tx.close()
        else:
            rx = HandoffReceiver(tp_group=tok_group)
            dist.send_object_list([rx.name], dst=rank - 2)
            it = 0
            while True:
                rows = rx.poll(block=False)
                if rows is not None:
                    break
                it += 1
                time.sleep(0.01)
            # both peers saw it at the same iteration
            t = torch.tensor([it], dtype=torch.int64)
            lo, hi = t.clone(), t.clone()
            dist.all_reduce(lo, op=dist.ReduceOp.MIN, group=tok_group)
            dist.all_reduce(hi, op=dist.ReduceOp.MAX, group=tok_group)
            rx.close()
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
        assert lo >= 10           # and only once the slow peer's message arrived


if __name__ == "__main__":
    pytest.main([__file__, "-q"])
