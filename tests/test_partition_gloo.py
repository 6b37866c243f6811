"""-m "not gpu": the multi-rank exchange logic of partitioned TPC-C (a8) with the gloo
backend, world_size 2 and 3 on CPU: requests grouped by destination reach their owner
(all-to-all #1) and responses come back aligned with each sender's buffer (#2)."""
import os
import socket

import pytest
import torch
import torch.multiprocessing as mp

REC = 48


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, q):
    import torch.distributed as dist
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    from paper_2406_10158_b200 import partition as P
    g = torch.Generator().manual_seed(rank)
    counts = [int(x) for x in torch.randint(0, 5, (world,), generator=g)]
    recs = []
    for d, c in enumerate(counts):
        for k in range(c):
            r = torch.zeros(REC, dtype=torch.uint8)
            r[0], r[1], r[2] = rank, d, k          # (source, destination, index)
            recs.append(r)
    send = torch.cat(recs) if recs else torch.empty(0, dtype=torch.uint8)
    recv, rcounts = P.exchange(send, counts)
    ok = True
    rv = recv.view(-1, REC) if recv.numel() else recv.view(0, REC)
    ok &= bool((rv[:, 1] == rank).all())                      # every record reached its owner
    srcs = rv[:, 0].tolist()
    ok &= srcs == sorted(srcs)                                 # grouped by source rank
    resp = rv.clone()
    resp[:, 3] = rv[:, 2] + 100                                # the owner's "answer"
    back = P.give_back(resp.view(-1), rcounts, counts).view(-1, REC)
    sv = send.view(-1, REC)
    ok &= bool((back[:, 0] == sv[:, 0]).all() and (back[:, 1] == sv[:, 1]).all())
    ok &= bool((back[:, 3] == sv[:, 2] + 100).all())          # aligned with the send buffer
    q.put((rank, ok, sum(counts), sum(rcounts)))
    dist.destroy_process_group()


@pytest.mark.parametrize("world", [2, 3])
def test_exchange_routing(world):
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    ps = [ctx.Process(target=_worker, args=(r, world, port, q)) for r in range(world)]
    for p in ps:
        p.start()
    out = [q.get(timeout=120) for _ in range(world)]
    for p in ps:
        p.join(timeout=60)
    assert all(o[1] for o in out), out
    assert sum(o[2] for o in out) == sum(o[3] for o in out)


class _FakeDB:
    """Stands in for a rank's DB in dist_round_2pc (host logic only): each round it sends
    one request to every rank, grants everything, and finishes after `done_after` rounds;
    it records what it saw so the test can check routing and alignment."""

    def __init__(self, rank, world, done_after):
        self.rank, self.world, self.done_after = rank, world, done_after
        self.round, self.commits, self.finished = 0, [], False
        self.stream = type("S", (), {"synchronize": staticmethod(lambda: None)})()

    def submit(self, batch, scheme, flags=0, result=None, **kw):
        from paper_2406_10158_b200 import gcctb as G
        assert flags & G.CC_FLAG_PART_2PC and flags & G.CC_FLAG_PARTITIONED
        return "res"

    def part_send(self):
        pending = self.round < self.done_after
        counts = [1 if pending else 0] * self.world
        recs = []
        for d in range(self.world):
            for _ in range(counts[d]):
                r = torch.zeros(REC, dtype=torch.uint8)
                r[0], r[1], r[2] = self.rank, d, self.round
                recs.append(r)
        return (torch.cat(recs) if recs else torch.empty(0, dtype=torch.uint8)), counts

    def part_apply(self, recv):
        rv = recv.view(-1, REC)
        assert bool((rv[:, 1] == self.rank).all())
        self._recv_src = rv[:, 0].tolist()
        out = rv.clone()
        out[:, 5 * 8] = 1                                   # vote: granted (word 5)
        return out.view(-1)

    def part_decide(self, back):
        bv = back.view(-1, REC)
        assert bool((bv[:, 0] == self.rank).all()) and bool((bv[:, 5 * 8] == 1).all())
        dec = torch.zeros(bv.shape[0], 8, dtype=torch.uint8)
        dec[:, 0] = 1
        dec[:, 1] = self.rank                              # who decided
        return dec.view(-1)

    def part_commit(self, recv, rdec):
        dv = rdec.view(-1, 8)
        assert dv[:, 1].tolist() == self._recv_src          # decisions aligned with requests
        self.commits.append(int(dv.shape[0]))

    def part_next(self):
        self.round += 1
        return max(0, self.done_after - self.round)

    def part_finish(self, resp):
        self.finished = True


def _worker_2pc(rank, world, port, q):
    import torch.distributed as dist
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    from paper_2406_10158_b200 import partition as P
    db = _FakeDB(rank, world, done_after=rank + 1)         # ranks finish at different rounds
    res, rounds = P.dist_round_2pc(db, None, "tpl_nw")
    q.put((rank, rounds, db.finished, db.commits))
    dist.destroy_process_group()


@pytest.mark.parametrize("world", [2, 3])
def test_2pc_rounds_until_every_rank_is_done(world):
    """f-2 host loop: all ranks keep exchanging (possibly empty) rounds until the slowest
    is done; decisions come back aligned with each owner's received requests."""
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    ps = [ctx.Process(target=_worker_2pc, args=(r, world, port, q)) for r in range(world)]
    for p in ps:
        p.start()
    out = [q.get(timeout=120) for _ in range(world)]
    for p in ps:
        p.join(timeout=60)
    for rank, rounds, finished, commits in out:
        assert rounds == world and finished
        # round k: every rank still pending (rank >= k) sends one request here
        assert commits == [sum(1 for s in range(world) if s >= k) for k in range(world)]


class _WinDB:
    """Stands in for a rank's DB in p2p_setup: its window handle names its rank."""

    def __init__(self, rank, world):
        self.rank, self.world, self.got = rank, world, None

    def part_window(self):
        return bytes([self.rank]) * 80   # sizeof(cc_ipc_handle)

    def part_connect(self, handles):
        self.got = handles


def _worker_p2p_setup(rank, world, port, q):
    import torch.distributed as dist
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    from paper_2406_10158_b200 import partition as P
    db = _WinDB(rank, world)
    P.p2p_setup(db)
    q.put((rank, [h[0] for h in db.got], [len(h) for h in db.got]))
    dist.destroy_process_group()


@pytest.mark.parametrize("world", [2, 3])
def test_p2p_setup_gathers_handles_in_rank_order(world):
    """CC_FLAG_PART_P2P set-up: every rank receives all window handles, indexed by rank
    (cc_part_connect checks handle r is rank r's)."""
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    ps = [ctx.Process(target=_worker_p2p_setup, args=(r, world, port, q)) for r in range(world)]
    for p in ps:
        p.start()
    out = [q.get(timeout=120) for _ in range(world)]
    for p in ps:
        p.join(timeout=60)
    for rank, firsts, lens in out:
        assert firsts == list(range(world)) and lens == [80] * world
