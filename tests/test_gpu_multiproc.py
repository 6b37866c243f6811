"""-m gpu: partitioned TPC-C (a8) across real processes.

G processes (G = 2, 4) share the one B200 of this run; each is rank r of a gloo process
group, holds warehouse partition r in its own db (its own CUDA context, its own stream)
and runs the product path exactly as a multi-GPU job would -- cc_submit(PARTITIONED),
cc_part_send / apply / finish (deterministic phase B) or the 2PC rounds (f-2) -- with the
all-to-alls going through torch.distributed (`exchange(..., via_cpu=True)`: gloo moves
host copies; on a multi-GPU box the same calls run on NCCL) -- and with the exchange
inside the library (CC_FLAG_PART_P2P): the processes' exchange windows are mapped into
each other through CUDA IPC and the round runs between their kernels, no host step.
Every scheme runs on the same initial state (cc_snapshot).  The parent merges the ranks' results and final tables
and checks them against the oracle's serial replay of [phase A of every rank in its
reported order] + [phase B in (round, gid) order] (reading R9)."""
import os
import socket
import tempfile

import numpy as np
import pytest

from inputs import tpcc as IT

pytestmark = pytest.mark.gpu
SCHEMES = ["tpl_nw", "tpl_wd", "to", "mvcc", "silo", "tictoc", "gputx", "gacco"]
TWO_PC = ["tpl_nw", "tpl_wd", "to", "mvcc", "silo", "tictoc"]
POP = ["warehouse", "district", "customer", "stock"]
W, N, SEED = 8, 2048, 23


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _rank_main(rank, world, port, outdir):
    import torch
    import torch.distributed as dist
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    torch.cuda.set_device(0)
    from paper_2406_10158_b200.api import DB
    from paper_2406_10158_b200.partition import dist_round, dist_round_2pc, p2p_round, p2p_setup
    wpr = W // world
    db = DB(0, rank=rank, world=world)
    db.load_tpcc(W, SEED, N, w_first=rank * wpr, w_count=wpr)
    db.snapshot(True)
    p2p_setup(db)   # exchange windows mapped across the processes through CUDA IPC
    b = db.gen_tpcc(N, 500 + rank, 5114, w_lo=rank * wpr, w_hi=(rank + 1) * wpr)
    tx = b.export_tpcc()
    runs = [(s, 0) for s in SCHEMES] + [(s, 1) for s in TWO_PC] + [(s, 2) for s in SCHEMES]
    for scheme, mode in runs:
        db.snapshot(False)
        dist.barrier()
        if mode == 1:
            res, rounds = dist_round_2pc(db, b, scheme, via_cpu=True, bs=8, lanes=32, watchdog_s=60)
        elif mode == 2:   # no host step: the exchange runs between the processes' kernels
            res, rounds = p2p_round(db, b, scheme, bs=8, lanes=32, watchdog_s=120), 0
        else:
            res, rounds = dist_round(db, b, scheme, via_cpu=True, bs=8, lanes=32, watchdog_s=60), 0
        st = db.sync()
        h = res.host(db.stream)
        tabs = {k: db.read_table(db.tpcc_ids[k]) for k in POP}
        for k in ("order", "new_order", "history"):
            tabs[k] = db.read_table(db.tpcc_ids[k])[:N]
        tabs["order_line"] = db.read_table(db.tpcc_ids["order_line"])[:N * 15]
        np.savez(os.path.join(outdir, f"{scheme}_{mode}_{rank}.npz"), tx=tx, commits=st.commits,
                 rounds=rounds, **{"r_" + k: v for k, v in h.items()}, **{"t_" + k: v for k, v in tabs.items()})
    b.free()
    db.close()
    dist.barrier()
    dist.destroy_process_group()


def _merged_check(scheme, world, outdir, mode, S0):
    from oracle import order_from_result
    from oracle import tpcc as OT
    two_pc = mode == 1
    parts = [np.load(os.path.join(outdir, f"{scheme}_{mode}_{r}.npz")) for r in range(world)]
    for p in parts:
        assert int(p["commits"]) == N
        order_from_result(p["r_committed"], p["r_commit_pos"], p["r_order_hi"], p["r_order_lo"])
    m = {k: np.concatenate([p["r_" + k] for p in parts]) for k in
         ("committed", "order_hi", "order_lo", "restarts", "read_out")}
    pos = np.empty(len(m["committed"]), np.uint32)
    pos[np.lexsort((m["order_lo"], m["order_hi"]))] = np.arange(len(pos))
    m["commit_pos"] = pos
    state = {k: np.concatenate([p["t_" + k] for p in parts]) for k in
             POP + ["order", "new_order", "history", "order_line"]}
    OT.check(("part-", "2pc-", "p2p-")[mode] + scheme, S0, np.concatenate([p["tx"] for p in parts]), W, m, state)
    b = m["order_hi"] >= np.uint64(1 << 63)
    assert b.any()   # some transactions crossed partitions and went through phase B
    if two_pc:
        rounds = int(parts[0]["rounds"])
        assert rounds >= 1 and all(int(p["rounds"]) == rounds for p in parts)
        assert ((m["order_hi"][b] & np.uint64(0xFFFFFFFF)) < np.uint64(rounds)).all()


@pytest.mark.parametrize("world", [2, 4])
def test_multiprocess_partitions(orc, world):
    torch = pytest.importorskip("torch")
    if not torch.cuda.is_available():
        pytest.skip("no GPU")
    import torch.multiprocessing as mp
    ctx = mp.get_context("spawn")
    port = _free_port()
    with tempfile.TemporaryDirectory() as outdir:
        ps = [ctx.Process(target=_rank_main, args=(r, world, port, outdir)) for r in range(world)]
        for p in ps:
            p.start()
        for p in ps:
            p.join(timeout=600)
        assert all(p.exitcode == 0 for p in ps), [p.exitcode for p in ps]
        S0 = IT.population(SEED, W)
        for scheme in SCHEMES:
            _merged_check(scheme, world, outdir, 0, S0)
            _merged_check(scheme, world, outdir, 2, S0)
        for scheme in TWO_PC:
            _merged_check(scheme, world, outdir, 1, S0)
