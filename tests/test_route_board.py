"""Live JSQ routing for the real-time trace path (control.RouteBoard /
ArrivalFeed): the reference's Cluster.route (cluster.py:153-160) makes two
independent picks at arrival — prompt machine by JSQ over the prompt pool,
token machine by JSQ over the token pool — each the lowest (pending, id)
(_argmin, cluster.py:129-134) with pending = pending_tokens (cluster.py:82-84):
queued prompt tokens (prompt machine), live token tasks (token machine).
The randomized test replays the reference's own Cluster with the same
machine states."""

import multiprocessing as mp
import random
import time

from paper_2311_18677_b200.control import ArrivalFeed, RouteBoard


def test_independent_jsq_picks():
    b = RouteBoard(8, 2, 3, create=True)
    try:
        assert b.route(0, 1000) == (0, 0)       # empty: lowest ids
        assert b.route(1, 500) == (1, 0)        # prompt 0 has 1000 queued; token pool idle
        assert b.route(2, 700) == (1, 0)        # 1000 vs 500
        b.publish_token(0, b.LANDED, 2)         # two token tasks live on token machine 0
        assert b.route(3, 10) == (0, 1)         # prompt 1000 vs 1200; token 2 / 0 / 0
        b.publish_prompt(0, 1000)               # prompt 0 finished its first prompt
        b.publish_token(0, b.FINISHED, 2)
        assert b.pending_prompt(0) == 10 and b.pending_token(0) == 0
        assert b.route(4, 50) == (0, 0)
        assert list(b.assign_p[:5]) == [0, 1, 1, 0, 0]
        assert list(b.assign_t[:5]) == [0, 0, 0, 1, 0]
    finally:
        b.close()


def test_picks_match_reference_cluster_route():
    """Randomised machine loads; the board's picks equal the reference's own
    Cluster.route (imported through tools/reftrace.py) for the same queued
    prompt tokens and live token tasks.  Loads stay under the reference's
    overflow threshold (queue_threshold_tokens = 4096, machine.py:35): the
    concurrent path does not run prompts on token machines (no mixed pool),
    so overflow routing is out of its scope."""
    import reftrace
    ss = reftrace.splitsim()
    if ss is None:
        import pytest
        pytest.skip("reference not importable")
    from splitsim import cluster as C
    rng = random.Random(3)
    perf = {"H100": ss.get_calibration("llama2-70b", "H100")}
    for trial in range(30):
        P, T = rng.randint(1, 4), rng.randint(1, 4)
        b = RouteBoard(64, P, T, create=True)
        cl = C.Cluster(C.ClusterConfig("Splitwise-HH", P, T), perf)
        try:
            routed = [0] * P
            for rid in range(40):
                # random progress: prompts finish, token tasks land and finish
                for m in range(P):
                    done = rng.randint(int(b.p_load[m]), routed[m])
                    b.publish_prompt(m, done)
                    cl.machines[m].pending_token_count = routed[m] - done
                for m in range(T):
                    land = int(b.t_load[m, 0]) + rng.randint(0, 2)
                    fin = rng.randint(int(b.t_load[m, 1]), land)
                    b.publish_token(m, b.LANDED, land)
                    b.publish_token(m, b.FINISHED, fin)
                    cl.machines[P + m].pending_token_count = land - fin
                size = rng.randint(1, 1500)
                dec = cl.route(rid, 0.0)
                got = b.route(rid, size)
                assert got == (dec.prompt_machine, dec.token_machine - P), (trial, rid)
                routed[got[0]] += size
                if max(routed[m] - int(b.p_load[m]) for m in range(P)) > 3000:
                    for m in range(P):          # drain: stay below the overflow threshold
                        b.publish_prompt(m, routed[m])
        finally:
            b.close()


def test_arrival_feed_in_order_and_complete():
    b = RouteBoard(4, 2, 2, create=True)
    try:
        reqs = [(i, 0.0, None, 1) for i in range(4)]
        f0, f1 = ArrivalFeed(reqs, 0, b), ArrivalFeed(reqs, 1, b)
        t1 = ArrivalFeed(reqs, 1, b, role="token")
        assert f0.poll() == [] and not f0.complete()
        b.assign_p[0], b.assign_t[0] = 1, 1
        b.assign_p[2], b.assign_t[2] = 0, 1   # published out of order: feeds wait for rid 1
        assert f0.poll() == [] and [r[0] for r in f1.poll()] == [0]
        assert [r[0] for r in t1.poll()] == [0]
        b.assign_p[1], b.assign_t[1] = 0, 0
        assert [r[0] for r in f0.poll()] == [1, 2]
        assert [r[0] for r in t1.poll()] == [2]
        b.assign_p[3], b.assign_t[3] = 1, 1
        assert [r[0] for r in f1.poll()] == [3]
        f0.poll()
        assert f0.complete() and f1.complete() and f0.mine == 2 and f1.mine == 2
        assert [r[0] for r in t1.poll()] == [3] and t1.complete() and t1.mine == 3
        s = ArrivalFeed(reqs, 0)
        assert not s.complete() and len(s.poll()) == 4 and s.complete()
    finally:
        b.close()


def _server(name, m, role, n, q):
    b = RouteBoard(n, 2, 2, name=name)
    feed = ArrivalFeed([(i, 0.0, None, 1) for i in range(n)], m, b, role=role)
    got = []
    t_end = time.time() + 20
    while not feed.complete() and time.time() < t_end:
        got += [r[0] for r in feed.poll()]
        time.sleep(1e-3)
    got += [r[0] for r in feed.poll()]
    if role == "token":
        b.publish_token(m, b.LANDED, len(got))
    q.put(((role, m), got))
    b.close()


def test_router_across_processes():
    n = 24
    b = RouteBoard(n, 2, 2, create=True)
    try:
        ctx = mp.get_context("spawn")
        q = ctx.Queue()
        ps = [ctx.Process(target=_server, args=(b.name, m, role, n, q))
              for role in ("prompt", "token") for m in range(2)]
        for p in ps:
            p.start()
        t0 = time.perf_counter()
        b.run_router([(i, 0.01 * i, 100 + i) for i in range(n)], t0)
        res = dict(q.get(timeout=60) for _ in ps)
        for p in ps:
            p.join(timeout=30)
        for role, arr in (("prompt", b.assign_p), ("token", b.assign_t)):
            got = res[(role, 0)] + res[(role, 1)]
            assert sorted(got) == list(range(n))
            for m in (0, 1):
                assert all(int(arr[i]) == m for i in res[(role, m)])
                assert res[(role, m)] == sorted(res[(role, m)])
    finally:
        b.close()


def _tp_peer(rank, port, name, n, q):
    import os
    import random as _r
    import torch.distributed as dist
    from paper_2311_18677_b200.splitwise import _lockstep
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=2)
    b = RouteBoard(n, 2, 2, name=name)
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
    """Two TP peers of one prompt machine (gloo, world 2) fed by the live
    router: the MIN lockstep makes them take the same requests at the same
    iterations and leave the serve loop at the same iteration although one
    of them observes the assignments late."""
    import socket
    n = 30
    b = RouteBoard(n, 2, 2, create=True)
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
        assert res[0][0] == [i for i in range(n) if int(b.assign_p[i]) == 1]
    finally:
        b.close()
