"""Warehouse-partitioned TPC-C orchestration.

Per round each rank: cc_submit(PARTITIONED) -> phase A under the chosen scheme + packed
phase-B requests; all-to-all #1 (requests to item owners); cc_part_apply (owners apply
each item's chain in global gid order); all-to-all #2 (responses back, reverse splits);
cc_part_finish (home assembles outputs / reserved slots, a7).  The collectives are NCCL
all_to_all_single through torch.distributed (plumbing); `loopback_round` runs G
partitions held by G dbs on one GPU with the same kernels, the exchange being a
device-side permutation (concatenation of the per-destination slices).
`dist_round_2pc` / `loopback_round_2pc`: the scheme-native variant (f-2) for the six
non-deterministic schemes, phase B in two-phase-commit rounds with a third all-to-all
(decisions); owners grant under 2PL locks or, for TO / MVCC / Silo / TicToc, in the
round's timestamp order.
`p2p_setup` / `p2p_round` / `loopback_p2p`: the deterministic phase B with the exchange
inside the library (CC_FLAG_PART_P2P): requests and responses are stored straight into
the peers' exchange windows over peer memory, so a round involves neither the host nor a
collective call -- the only torch.distributed use is gathering the window handles once.
"""
from __future__ import annotations

import torch

from . import gcctb as G

REC = G.PART_REC_BYTES


def exchange(send: torch.Tensor, send_counts, group=None, via_cpu: bool = False, rec: int = REC):
    """All-to-all of `rec`-byte records grouped by destination.  Returns (recv, recv_counts)."""
    import torch.distributed as dist
    dev = send.device if not via_cpu else torch.device("cpu")
    sc = torch.tensor(send_counts, dtype=torch.int64, device=dev)
    rc = torch.empty_like(sc)
    dist.all_to_all_single(rc, sc, group=group)
    recv_counts = [int(x) for x in rc.tolist()]
    src = send if not via_cpu else send.cpu()
    recv = torch.empty(sum(recv_counts) * rec, dtype=torch.uint8, device=dev)
    dist.all_to_all_single(recv, src, [c * rec for c in recv_counts], [c * rec for c in send_counts], group=group)
    return (recv if not via_cpu else recv.to(send.device)), recv_counts


def give_back(resp: torch.Tensor, recv_counts, send_counts, group=None, via_cpu: bool = False):
    """Reverse all-to-all: responses (aligned with the received requests) return to the
    senders, aligned with their send buffers."""
    import torch.distributed as dist
    dev = resp.device if not via_cpu else torch.device("cpu")
    out = torch.empty(sum(send_counts) * REC, dtype=torch.uint8, device=dev)
    src = resp if not via_cpu else resp.cpu()
    dist.all_to_all_single(out, src, [c * REC for c in send_counts], [c * REC for c in recv_counts], group=group)
    return out if not via_cpu else out.to(resp.device)


def dist_round(db, batch, scheme, result=None, group=None, via_cpu=False, **kw):
    """One partitioned submit on this rank (all ranks call it collectively)."""
    flags = kw.pop("flags", 0) | G.CC_FLAG_PARTITIONED
    res = db.submit(batch, scheme, flags=flags, result=result, **kw)
    send, counts = db.part_send()
    recv, recv_counts = exchange(send, counts, group, via_cpu)
    resp = db.part_apply(recv)
    db.stream.synchronize()
    back = give_back(resp, recv_counts, counts, group, via_cpu)
    db.part_finish(back)
    return res


def dist_round_2pc(db, batch, scheme, result=None, group=None, via_cpu=False, **kw):
    """One partitioned submit whose distributed transactions run in 2PC rounds under the
    scheme's round rule (f-2; all ranks call it collectively): per round requests (#1), grants + votes back
    (#2), decisions (#3, 8 bytes per request), until no rank has pending transactions."""
    import torch.distributed as dist
    flags = kw.pop("flags", 0) | G.CC_FLAG_PARTITIONED | G.CC_FLAG_PART_2PC
    res = db.submit(batch, scheme, flags=flags, result=result, **kw)
    rounds = 0
    while True:
        send, counts = db.part_send()
        recv, recv_counts = exchange(send, counts, group, via_cpu)
        resp = db.part_apply(recv)
        db.stream.synchronize()
        back = give_back(resp, recv_counts, counts, group, via_cpu)
        dec = db.part_decide(back)
        db.stream.synchronize()
        rdec, _ = exchange(dec, counts, group, via_cpu, rec=8)
        db.part_commit(recv, rdec)
        pending = torch.tensor([db.part_next()], dtype=torch.int64,
                               device=send.device if not via_cpu else torch.device("cpu"))
        dist.all_reduce(pending, op=dist.ReduceOp.MAX, group=group)
        rounds += 1
        if int(pending.item()) == 0:
            break
    db.part_finish(torch.empty(0, dtype=torch.uint8, device=send.device))
    return res, rounds


def p2p_setup(db, group=None):
    """Collective: create this rank's exchange window, all_gather the handles, map the peers'
    windows (CC_FLAG_PART_P2P).  Afterwards `p2p_round` needs no host participation."""
    import torch.distributed as dist
    mine = db.part_window()
    handles = [None] * db.world
    dist.all_gather_object(handles, mine, group=group)
    db.part_connect(handles)


def p2p_round(db, batch, scheme, result=None, **kw):
    """One partitioned submit with the exchange inside the library: phase A, the request /
    response transfers over peer memory, phase B and a7 are all enqueued on the db stream
    (every rank issues the same sequence of these submits)."""
    flags = kw.pop("flags", 0) | G.CC_FLAG_PARTITIONED | G.CC_FLAG_PART_P2P
    return db.submit(batch, scheme, flags=flags, result=result, **kw)


def loopback_p2p(dbs, batches, scheme, results=None, **kw):
    """G partitions held by G dbs of this process (connected with DB.part_connect_local):
    the partitioned submits are enqueued back to back and the exchange runs between their
    streams over device memory -- no host synchronisation anywhere in the round."""
    return [p2p_round(db, b, scheme, result=None if results is None else results[i], **kw)
            for i, (db, b) in enumerate(zip(dbs, batches))]


def _slices(buf, counts, rec):
    o = [0]
    for c in counts:
        o.append(o[-1] + c * rec)
    return [buf[o[d]:o[d + 1]] for d in range(len(counts))]


def loopback_round_2pc(dbs, batches, scheme, results=None, **kw):
    """dist_round_2pc for G partitions on one GPU (exchanges are slicing + concatenation)."""
    flags = kw.pop("flags", 0) | G.CC_FLAG_PARTITIONED | G.CC_FLAG_PART_2PC
    res = [db.submit(b, scheme, flags=flags, result=None if results is None else results[i], **kw)
           for i, (db, b) in enumerate(zip(dbs, batches))]
    world, rounds = len(dbs), 0
    while True:
        sends = [db.part_send() for db in dbs]
        parts = [_slices(buf, counts, REC) for buf, counts in sends]            # [src][dst]
        recvs = [torch.cat([parts[s][d] for s in range(world)]) for d in range(world)]
        resps = []
        for d, db in enumerate(dbs):
            resps.append(db.part_apply(recvs[d]))
            db.stream.synchronize()
        decs = []
        for s, db in enumerate(dbs):   # responses return to the senders in their send order
            pieces = []
            for d in range(world):
                start = sum(sends[q][1][d] for q in range(s)) * REC
                pieces.append(resps[d][start:start + sends[s][1][d] * REC])
            decs.append(db.part_decide(torch.cat(pieces)))
            db.stream.synchronize()
        dparts = [_slices(dec, counts, 8) for dec, (_, counts) in zip(decs, sends)]
        pending = 0
        for d, db in enumerate(dbs):
            db.part_commit(recvs[d], torch.cat([dparts[s][d] for s in range(world)]))
        for db in dbs:
            pending = max(pending, db.part_next())
        rounds += 1
        if pending == 0:
            break
    for db in dbs:
        db.part_finish(torch.empty(0, dtype=torch.uint8, device=torch.device("cuda", db.device)))
    return res, rounds


def loopback_round(dbs, batches, scheme, results=None, **kw):
    """G partitions on one GPU: the same protocol, the all-to-all being slicing and
    concatenation of device buffers."""
    flags = kw.pop("flags", 0) | G.CC_FLAG_PARTITIONED
    res = [db.submit(b, scheme, flags=flags, result=None if results is None else results[i], **kw)
           for i, (db, b) in enumerate(zip(dbs, batches))]
    sends = [db.part_send() for db in dbs]
    world = len(dbs)
    offs = []
    for buf, counts in sends:
        o = [0]
        for c in counts:
            o.append(o[-1] + c * REC)
        offs.append(o)
    recvs, recv_parts = [], []
    for d in range(world):
        parts = [sends[s][0][offs[s][d]:offs[s][d + 1]] for s in range(world)]
        recv_parts.append([p.numel() for p in parts])
        recvs.append(torch.cat(parts) if parts else torch.empty(0, dtype=torch.uint8))
    resps = []
    for d, db in enumerate(dbs):
        resps.append(db.part_apply(recvs[d]))
        db.stream.synchronize()
    for s, db in enumerate(dbs):
        pieces = []
        for d in range(world):
            start = sum(recv_parts[d][:s])
            pieces.append(resps[d][start:start + recv_parts[d][s]])
        back = torch.cat(pieces)
        db.part_finish(back)
    return res
