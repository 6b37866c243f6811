"""-m gpu: parity at BASELINE.json configs[4] size -- TPC-C with 512 warehouses (27 GB of
rows), 65,536 transactions per batch (per partition in the loopback case), 45:43 mix
 -- in exactly the launches bench.py times:
  * one GPU holding all 512 warehouses, every scheme in bench.TPCC_CONFIGS' configs[4]
    launch (the `tpcc` block of the bench line);
  * four 128-warehouse partitions on this GPU (bench --workload tpcc --loopback 4),
    deterministic phase B and 2PC (f-2).
The oracle replays the full 512-warehouse S0 (generated in parallel, tests/bigpop.py) in
the GPU-reported order and every table byte is compared."""
import numpy as np
import pytest

pytestmark = pytest.mark.gpu
SCHEMES = ["tpl_nw", "tpl_wd", "to", "mvcc", "silo", "tictoc", "gputx", "gacco"]
W, N, SEED = 512, 65536, 29


@pytest.fixture(scope="module")
def torch_cuda():
    torch = pytest.importorskip("torch")
    if not torch.cuda.is_available():
        pytest.skip("no GPU")
    return torch


@pytest.fixture(scope="module")
def S0():
    import bigpop
    P = bigpop.population(SEED, W)
    yield P
    P.close()


@pytest.fixture(scope="module")
def db512(torch_cuda):
    from paper_2406_10158_b200.api import DB
    db = DB(0)
    db.load_tpcc(W, SEED, N)
    db.snapshot(True)
    yield db
    db.close()


def _bench_launch(scheme, n_sms):
    import bench
    cfg = [c for c in bench.TPCC_CONFIGS if c["W"] == W][0]
    bs, per_sm = cfg["launch"].get(scheme, cfg["launch"]["*"])
    return {"bs": bs, "grid": n_sms if per_sm else 0}, cfg["mix"]


@pytest.mark.parametrize("scheme", SCHEMES)
def test_c4_single_gpu_bench_launch(orc, db512, S0, scheme):
    from oracle import tpcc as OT
    db = db512
    la, mix = _bench_launch(scheme, db.num_sms)
    db.snapshot(False)
    b = db.gen_tpcc(N, 41, mix)
    tx = b.export_tpcc()
    res = db.submit(b, scheme, lanes=32, watchdog_s=120, **la)
    assert db.sync().commits == N
    OT.check(scheme, S0, tx, W, res.host(db.stream), db.read_tpcc(list(OT.TABLES + OT.SLOTS)))
    b.free()


@pytest.mark.parametrize("scheme,two_pc", [("silo", False), ("gacco", False), ("tpl_wd", True), ("to", True)])
def test_c4_loopback_4x128(orc, torch_cuda, S0, scheme, two_pc):
    import bench
    from oracle import order_from_result
    from oracle import tpcc as OT
    from paper_2406_10158_b200.api import DB, Result
    from paper_2406_10158_b200.partition import loopback_round, loopback_round_2pc
    G = 4
    wpr = W // G
    dev = torch_cuda.device("cuda", 0)
    dbs, batches = [], []
    for r in range(G):
        db = DB(0, rank=r, world=G)
        db.load_tpcc(W, SEED, N, w_first=r * wpr, w_count=wpr)
        dbs.append(db)
        batches.append(db.gen_tpcc(N, 900 + r, 5114, w_lo=r * wpr, w_hi=(r + 1) * wpr))
    la = {"bs": bench.LOOPBACK_TPCC_BS[scheme], "grid": dbs[0].num_sms}
    results = [Result.alloc(N, 18, dev, stream=db.stream, out_words=48) for db in dbs]
    if two_pc:
        loopback_round_2pc(dbs, batches, scheme, results=results, lanes=32, watchdog_s=120, **la)
    else:
        loopback_round(dbs, batches, scheme, results=results, lanes=32, watchdog_s=120, **la)
    for db in dbs:
        assert db.sync().commits == N
    hs = [r.host(db.stream) for r, db in zip(results, dbs)]
    for h in hs:
        order_from_result(h["committed"], h["commit_pos"], h["order_hi"], h["order_lo"])
    m = {k: np.concatenate([h[k] for h in hs]) for k in ("committed", "order_hi", "order_lo", "restarts", "read_out")}
    pos = np.empty(len(m["committed"]), np.uint32)
    pos[np.lexsort((m["order_lo"], m["order_hi"]))] = np.arange(len(pos))
    m["commit_pos"] = pos
    state = {k: np.concatenate([db.read_table(db.tpcc_ids[k]) for db in dbs])
             for k in ("warehouse", "district", "customer", "stock")}
    for k in ("order", "new_order", "history"):
        state[k] = np.concatenate([db.read_table(db.tpcc_ids[k])[:N] for db in dbs])
    state["order_line"] = np.concatenate([db.read_table(db.tpcc_ids["order_line"])[:N * 15] for db in dbs])
    txs = np.concatenate([b.export_tpcc() for b in batches])
    OT.check(("2pc-" if two_pc else "part-") + scheme, S0, txs, W, m, state)
    assert (m["order_hi"] >= np.uint64(1 << 63)).any()   # phase B ran
    for b in batches:
        b.free()
    for db in dbs:
        db.close()
