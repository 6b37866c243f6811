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
