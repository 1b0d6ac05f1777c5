"""Live JSQ routing across Splitwise pairs (control.RouteBoard / ArrivalFeed),
the real-time trace path's restatement of the reference's Cluster.route
(cluster.py:82-84 pending_tokens, :129-134 _argmin, :153-160 route)."""

import multiprocessing as mp
import random
import time

from paper_2311_18677_b200.control import ArrivalFeed, RouteBoard


def test_jsq_pick_is_argmin_pending_then_id():
    b = RouteBoard(8, 3, create=True)
    try:
        # empty pool: ties broken by the lowest pair id, then the queued
        # prompt tokens steer the next picks
        assert b.route(0, 1000) == 0
        assert b.route(1, 500) == 1
        assert b.route(2, 700) == 2
        assert b.route(3, 10) == 1            # pending 1000 / 500 / 700
        # pair 0 finishes its prompt: its request becomes one live token task
        b.publish(0, b.PROMPT_TOK, 1000)
        b.publish(0, b.PROMPT_REQ, 1)
        assert b.pending(0) == 1
        assert b.route(4, 50) == 0
        # ... and finishes decoding
        b.publish(0, b.FINISHED, 1)
        assert b.pending(0) == 50
        assert list(b.assign[:5]) == [0, 1, 2, 1, 0]
    finally:
        b.close()


def test_jsq_matches_reference_argmin_randomised():
    rng = random.Random(3)
    for _ in range(20):
        pairs = rng.randint(2, 4)
        b = RouteBoard(64, pairs, create=True)
        try:
            routed = [[] for _ in range(pairs)]     # prompt sizes per pair
            done = [0] * pairs                       # prompts finished
            fin = [0] * pairs                        # requests finished
            for rid in range(64):
                p = rng.randrange(pairs)
                if done[p] < len(routed[p]) and rng.random() < 0.5:
                    done[p] += 1
                    b.publish(p, b.PROMPT_TOK, sum(routed[p][:done[p]]))
                    b.publish(p, b.PROMPT_REQ, done[p])
                if fin[p] < done[p] and rng.random() < 0.5:
                    fin[p] += 1
                    b.publish(p, b.FINISHED, fin[p])
                pend = [sum(routed[q][done[q]:]) + (done[q] - fin[q]) for q in range(pairs)]
                want = min(range(pairs), key=lambda q: (pend[q], q))
                size = rng.randint(1, 2048)
                assert b.route(rid, size) == want
                routed[want].append(size)
        finally:
            b.close()


def test_arrival_feed_in_order_and_complete():
    b = RouteBoard(4, 2, create=True)
    try:
        reqs = [(i, 0.0, None, 1) for i in range(4)]
        f0, f1 = ArrivalFeed(reqs, 0, b), ArrivalFeed(reqs, 1, b)
        assert f0.poll() == [] and not f0.complete()
        b.assign[0] = 1
        b.assign[2] = 0          # published out of order: the feed waits for rid 1
        assert f0.poll() == [] and [r[0] for r in f1.poll()] == [0]
        b.assign[1] = 0
        assert [r[0] for r in f0.poll()] == [1, 2]
        b.assign[3] = 1
        assert [r[0] for r in f1.poll()] == [3]
        f0.poll()
        assert f0.complete() and f1.complete() and f0.mine == 2 and f1.mine == 2
        # static feed (no board): everything at once
        s = ArrivalFeed(reqs, 0)
        assert not s.complete() and len(s.poll()) == 4 and s.complete()
    finally:
        b.close()


def _server(name, pair, n, q):
    b = RouteBoard(n, 2, name=name)
    feed = ArrivalFeed([(i, 0.0, None, 1) for i in range(n)], pair, b)
    got = []
    t_end = time.time() + 20
    while not feed.complete() and time.time() < t_end:
        got += [r[0] for r in feed.poll()]
        time.sleep(1e-3)
    got += [r[0] for r in feed.poll()]
    b.publish(pair, b.FINISHED, len(got))
    q.put((pair, got))
    b.close()


def test_router_across_processes():
    n = 24
    b = RouteBoard(n, 2, create=True)
    try:
        ctx = mp.get_context("spawn")
        q = ctx.Queue()
        ps = [ctx.Process(target=_server, args=(b.name, p, n, q)) for p in range(2)]
        for p in ps:
            p.start()
        t0 = time.perf_counter()
        b.run_router([(i, 0.01 * i, 100 + i) for i in range(n)], t0)
        res = dict(q.get(timeout=60) for _ in ps)
        for p in ps:
            p.join(timeout=30)
        assert sorted(res[0] + res[1]) == list(range(n))
        assert [int(b.assign[i]) for i in res[0]] == [0] * len(res[0])
        assert res[0] == sorted(res[0]) and res[1] == sorted(res[1])
    finally:
        b.close()


def _tp_peer(rank, port, name, n, q):
    import os
    import random as _r
    import torch.distributed as dist
    from paper_2311_18677_b200.splitwise import _lockstep
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=2)
    b = RouteBoard(n, 2, name=name)
    feed = ArrivalFeed([(i, 0.0, None, 1) for i in range(n)], 1, b)
    rng = _r.Random(rank)
    pending, taken, it = [], [], 0
    while True:
        if rank == 1 and rng.random() < 0.5:
            time.sleep(2e-3)                   # this peer sees assignments late
        else:
            pending += feed.poll()
        fin = feed.complete() and len(taken) >= feed.mine
        k, _, fin = _lockstep(len(pending), dist.group.WORLD, 0.0, fin)
        if fin:
            break
        taken += [r[0] for r in pending[:k]]
        del pending[:k]
        it += 1
    q.put((rank, taken, it))
    b.close()
    dist.destroy_process_group()


def test_tp_peers_take_the_same_arrivals_and_exit_together():
    """Two TP peers of one pair (gloo, world 2) fed by the live router: the
    MIN lockstep makes them take the same requests at the same iterations
    and leave the serve loop at the same iteration although one of them
    observes the assignments late."""
    import socket
    n = 30
    b = RouteBoard(n, 2, create=True)
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        port = s.getsockname()[1]
    try:
        ctx = mp.get_context("spawn")
        q = ctx.Queue()
        ps = [ctx.Process(target=_tp_peer, args=(r, port, b.name, n, q)) for r in range(2)]
        for p in ps:
            p.start()
        time.sleep(3.0)                        # let both peers join the group
        b.run_router([(i, 0.005 * i, 100) for i in range(n)], time.perf_counter())
        res = {r: (t, it) for r, t, it in (q.get(timeout=120) for _ in ps)}
        for p in ps:
            p.join(timeout=30)
        assert res[0] == res[1]
        assert res[0][0] == [i for i in range(n) if int(b.assign[i]) == 1]
    finally:
        b.close()
