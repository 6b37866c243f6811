"""-m gpu: partitioned TPC-C (a8).  Phase B alone on one partition (CC_FLAG_PART_ALL)
must equal serial replay in global gid order; G = 2 and 4 warehouse partitions held by
G dbs on one GPU (loopback exchange through the same pack/apply/finish kernels) must
equal serial replay of [phase A of every rank in its reported order] + [phase B in gid
order] over the merged state."""
import numpy as np
import pytest

from inputs import tpcc as IT

pytestmark = pytest.mark.gpu
SCHEMES = ["tpl_nw", "tpl_wd", "to", "mvcc", "silo", "tictoc", "gputx", "gacco"]
POP = ["warehouse", "district", "customer", "stock"]


@pytest.fixture(scope="module")
def torch_cuda():
    torch = pytest.importorskip("torch")
    if not torch.cuda.is_available():
        pytest.skip("no GPU")
    return torch


def _merged_check(scheme, W, dbs, batches, results, S0, n_local):
    from oracle import tpcc as OT
    txs = [b.export_tpcc() for b in batches]
    hs = [r.host(db.stream) for r, db in zip(results, dbs)]
    for h in hs:   # each rank's dense commit positions follow its keys
        from oracle import order_from_result
        order_from_result(h["committed"], h["commit_pos"], h["order_hi"], h["order_lo"])
    m = {k: np.concatenate([h[k] for h in hs]) for k in ("committed", "order_hi", "order_lo", "restarts")}
    m["read_out"] = np.concatenate([h["read_out"] for h in hs])
    pos = np.empty(len(m["committed"]), np.uint32)
    pos[np.lexsort((m["order_lo"], m["order_hi"]))] = np.arange(len(pos))
    m["commit_pos"] = pos
    state = {}
    for k in POP:
        state[k] = np.concatenate([db.read_table(db.tpcc_ids[k]) for db in dbs])
    for k in ("order", "new_order", "history"):
        state[k] = np.concatenate([db.read_table(db.tpcc_ids[k])[:n_local] for db in dbs])
    state["order_line"] = np.concatenate([db.read_table(db.tpcc_ids["order_line"])[:n_local * 15] for db in dbs])
    OT.check("part-" + scheme, S0, np.concatenate(txs), W, m, state)
    # phase B transactions are ordered after every phase A transaction, by global gid
    hi = m["order_hi"]
    phase_b = hi >= np.uint64(1 << 63)
    assert phase_b.any() or W == len(dbs)


@pytest.mark.parametrize("scheme", SCHEMES)
def test_phase_b_only(torch_cuda, orc, scheme):
    from paper_2406_10158_b200.api import DB
    from paper_2406_10158_b200 import gcctb as G
    from paper_2406_10158_b200.partition import loopback_round
    W, n = 2, 2048
    db = DB(0, rank=0, world=1)
    db.load_tpcc(W, 13, n)
    S0 = IT.population(13, W)
    b = db.gen_tpcc(n, 5, 5114)
    res = loopback_round([db], [b], scheme, flags=G.CC_FLAG_PART_ALL, bs=8, lanes=32)
    st = db.sync()
    assert st.commits == n and st.aborts == 0
    h = res[0].host(db.stream)
    assert (h["order_hi"] == np.uint64(1 << 63)).all()
    _merged_check(scheme, W, [db], [b], res, S0, n)
    db.close()


@pytest.mark.parametrize("G_", [2, 4])
@pytest.mark.parametrize("scheme", SCHEMES)
def test_loopback_partitions(torch_cuda, orc, scheme, G_):
    from paper_2406_10158_b200.api import DB
    from paper_2406_10158_b200.partition import loopback_round
    W, n = 8, 2048
    wpr = W // G_
    dbs, batches = [], []
    for r in range(G_):
        db = DB(0, rank=r, world=G_)
        db.load_tpcc(W, 17, n, w_first=r * wpr, w_count=wpr)
        dbs.append(db)
        batches.append(db.gen_tpcc(n, 100 + r, 5114, w_lo=r * wpr, w_hi=(r + 1) * wpr))
    S0 = IT.population(17, W)
    res = loopback_round(dbs, batches, scheme, bs=8, lanes=32)
    for db in dbs:
        assert db.sync().commits == n
    _merged_check(scheme, W, dbs, batches, res, S0, n)
    for db in dbs:
        db.close()


# ------------------------------------------------- in-library exchange over peer memory
def _partitions(G_, seed, n=2048, W=8):
    from paper_2406_10158_b200.api import DB
    wpr = W // G_
    dbs, batches = [], []
    for r in range(G_):
        db = DB(0, rank=r, world=G_)
        db.load_tpcc(W, 17, n, w_first=r * wpr, w_count=wpr)
        dbs.append(db)
        batches.append(db.gen_tpcc(n, seed + r, 5114, w_lo=r * wpr, w_hi=(r + 1) * wpr))
    return dbs, batches


@pytest.mark.parametrize("G_", [2, 4])
@pytest.mark.parametrize("scheme", SCHEMES)
def test_loopback_p2p(torch_cuda, orc, scheme, G_):
    """CC_FLAG_PART_P2P: phase A, the exchange over the dbs' windows, phase B and a7 all
    enqueued by one cc_submit per partition (no host step in between); twice in a row, so
    the windows and epochs are reused."""
    from paper_2406_10158_b200.api import DB
    from paper_2406_10158_b200.partition import loopback_p2p
    W, n = 8, 2048
    dbs, batches = _partitions(G_, 100)
    DB.part_connect_local(dbs)
    for db in dbs:
        db.snapshot(True)
    S0 = IT.population(17, W)
    for rep in range(2):
        for db in dbs:
            db.snapshot(False)
        res = loopback_p2p(dbs, batches, scheme, bs=8, lanes=32, watchdog_s=60)
        for db in dbs:
            assert db.sync().commits == n
        _merged_check(scheme, W, dbs, batches, res, S0, n)
    for db in dbs:
        db.close()


@pytest.mark.parametrize("scheme", ["gputx", "gacco"])
def test_p2p_equals_host_exchange(torch_cuda, orc, scheme):
    """The deterministic schemes' partitioned results are a function of the input alone:
    the in-library exchange and the host-driven one give identical outputs and tables."""
    from paper_2406_10158_b200.api import DB
    from paper_2406_10158_b200.partition import loopback_p2p, loopback_round
    G_ = 4
    dbs, batches = _partitions(G_, 700)
    DB.part_connect_local(dbs)
    for db in dbs:
        db.snapshot(True)
    out = []
    for run in (loopback_round, loopback_p2p):
        for db in dbs:
            db.snapshot(False)
        res = run(dbs, batches, scheme, bs=8, lanes=32, watchdog_s=60)
        hs = [r.host(db.stream) for r, db in zip(res, dbs)]
        tabs = [db.read_tpcc(["warehouse", "district", "customer", "stock", "order", "new_order", "order_line",
                              "history"]) for db in dbs]
        out.append((hs, tabs))
    (h1, t1), (h2, t2) = out
    for a, b in zip(h1, h2):
        for k in a:
            assert np.array_equal(a[k], b[k]), k
    for a, b in zip(t1, t2):
        for k in a:
            assert np.array_equal(a[k], b[k]), k
    for db in dbs:
        db.close()


def test_p2p_phase_b_only(torch_cuda, orc):
    """CC_FLAG_PART_ALL with the in-library exchange on one partition: every transaction
    through phase B over the window, equal to serial replay in gid order."""
    from paper_2406_10158_b200.api import DB
    from paper_2406_10158_b200 import gcctb as G
    from paper_2406_10158_b200.partition import loopback_p2p
    W, n = 2, 2048
    db = DB(0, rank=0, world=1)
    db.load_tpcc(W, 13, n)
    DB.part_connect_local([db])
    S0 = IT.population(13, W)
    b = db.gen_tpcc(n, 5, 5114)
    res = loopback_p2p([db], [b], "tpl_nw", flags=G.CC_FLAG_PART_ALL, bs=8, lanes=32)
    st = db.sync()
    assert st.commits == n and st.aborts == 0
    assert (res[0].host(db.stream)["order_hi"] == np.uint64(1 << 63)).all()
    _merged_check("tpl_nw", W, [db], [b], res, S0, n)
    db.close()


# ---------------------------------------------------------------- f-2: 2PC phase B
TWO_PC = ["tpl_nw", "tpl_wd", "to", "mvcc", "silo", "tictoc"]


@pytest.mark.parametrize("G_", [2, 4])
@pytest.mark.parametrize("scheme", TWO_PC)
def test_loopback_2pc(torch_cuda, orc, scheme, G_):
    """Distributed transactions in 2PC rounds under the scheme's round rule (2PL locks,
    or timestamp order for TO / MVCC / Silo / TicToc): the merged result equals serial
    replay of phase A then the 2PC rounds in (round, gid) order."""
    from paper_2406_10158_b200.api import DB
    from paper_2406_10158_b200.partition import loopback_round_2pc
    W, n = 8, 2048
    wpr = W // G_
    dbs, batches = [], []
    for r in range(G_):
        db = DB(0, rank=r, world=G_)
        db.load_tpcc(W, 17, n, w_first=r * wpr, w_count=wpr)
        dbs.append(db)
        batches.append(db.gen_tpcc(n, 300 + r, 5114, w_lo=r * wpr, w_hi=(r + 1) * wpr))
    S0 = IT.population(17, W)
    res, rounds = loopback_round_2pc(dbs, batches, scheme, bs=8, lanes=32)
    assert rounds >= 1
    for db in dbs:
        assert db.sync().commits == n
    _merged_check(scheme, W, dbs, batches, res, S0, n)
    hs = [r.host(db.stream) for r, db in zip(res, dbs)]
    hi = np.concatenate([h["order_hi"] for h in hs])
    b = hi >= np.uint64(1 << 63)
    assert b.any()
    assert ((hi[b] & np.uint64(0xFFFFFFFF)) < np.uint64(rounds)).all()   # round number in the key
    for db in dbs:
        db.close()


@pytest.mark.parametrize("scheme", TWO_PC)
def test_2pc_all_distributed_contention(torch_cuda, orc, scheme):
    """Every transaction through 2PC on one partition of 2 warehouses: heavy conflicts,
    many rounds, each committing a conflict-free set; aborts are counted as restarts."""
    from paper_2406_10158_b200.api import DB
    from paper_2406_10158_b200 import gcctb as G
    from paper_2406_10158_b200.partition import loopback_round_2pc
    W, n = 2, 2048
    db = DB(0, rank=0, world=1)
    db.load_tpcc(W, 13, n)
    S0 = IT.population(13, W)
    b = db.gen_tpcc(n, 6, 5114)
    res, rounds = loopback_round_2pc([db], [b], scheme, flags=G.CC_FLAG_PART_ALL, bs=8, lanes=32)
    st = db.sync()
    assert st.commits == n and st.aborts > 0 and rounds > 10
    h = res[0].host(db.stream)
    assert (h["order_hi"] >= np.uint64(1 << 63)).all()
    _merged_check(scheme, W, [db], [b], res, S0, n)
    db.close()


def test_2pc_rejects_other_schemes(torch_cuda):
    from paper_2406_10158_b200.api import DB
    from paper_2406_10158_b200 import gcctb as G
    db = DB(0, rank=0, world=1)
    db.load_tpcc(1, 3, 256)
    b = db.gen_tpcc(256, 1, 5000)
    with pytest.raises(G.CCError, match="UNSUPPORTED"):
        db.submit(b, "gacco", flags=G.CC_FLAG_PARTITIONED | G.CC_FLAG_PART_2PC, lanes=32, bs=8)
    db.close()
