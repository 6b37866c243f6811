"""-m gpu: TPC-C NewOrder/Payment parity of the CUDA path against the oracle
(BASELINE.json configs[2..3]): device population == input generator, a1 generator
bit-exact, and for every scheme the outputs, CC tables and reserved slots equal the
oracle's serial replay in the reported order (GPUTx/GaccO: batch order)."""
import numpy as np
import pytest

import inputs
from inputs import tpcc as IT

pytestmark = pytest.mark.gpu
SCHEMES = ["tpl_nw", "tpl_wd", "to", "mvcc", "silo", "tictoc", "gputx", "gacco"]
POP = ["warehouse", "district", "customer", "stock", "item"]


@pytest.fixture(scope="module")
def torch_cuda():
    torch = pytest.importorskip("torch")
    if not torch.cuda.is_available():
        pytest.skip("no GPU")
    return torch


def _db(W, seed, max_txn):
    from paper_2406_10158_b200.api import DB
    db = DB(0)
    db.load_tpcc(W, seed, max_txn)
    return db


@pytest.fixture(scope="module")
def w4(torch_cuda, orc):
    db = _db(4, 21, 8192)
    S0 = IT.population(21, 4)
    got = db.read_tpcc(POP)
    for k in POP:
        assert np.array_equal(got[k], S0[k]), f"device population differs in {k}"
    db.snapshot(True)
    yield db, S0
    db.close()


def _run(db, S0, W, tx_batch, scheme, lanes, orc, flags=0, launch=None):
    from oracle import tpcc as OT
    tx = tx_batch.export_tpcc()
    db.snapshot(False)
    la = launch or {"bs": 32 if lanes == 1 else 8}
    res = db.submit(tx_batch, scheme, wd=0, lanes=lanes, watchdog_s=60, flags=flags, **la)
    st = db.sync()
    assert st.commits == tx_batch.n_txn
    h = res.host(db.stream)
    S_gpu = db.read_tpcc(list(OT.TABLES + OT.SLOTS))
    n = tx_batch.n_txn
    S_gpu = {k: (v[:n * 15] if k == "order_line" else v[:n]) if k in OT.SLOTS else v for k, v in S_gpu.items()}
    OT.check(scheme, S0, tx, W, h, S_gpu)
    return st


def test_generator_bitexact(w4, orc):
    from oracle import tpcc as OT
    db, _ = w4
    for seed, pm in [(1, 5000), (2, 5114), (3, 10000), (4, 0)]:
        b = db.gen_tpcc(4096, seed, pm)
        exp = OT.gen(seed, 4, 4096, pm, IT.nurand_consts(21))
        assert np.array_equal(b.export_tpcc(), exp)
        b.free()


@pytest.mark.parametrize("lanes", [1, 32])
@pytest.mark.parametrize("scheme", SCHEMES)
def test_w4_parity(w4, orc, scheme, lanes):
    db, S0 = w4
    for seed in (7, 8):
        b = db.gen_tpcc(4096, seed, 5114)
        _run(db, S0, 4, b, scheme, lanes, orc)
        b.free()


@pytest.mark.parametrize("scheme", SCHEMES)
def test_payment_only_by_name_heavy(w4, orc, scheme):
    """All Payments (60% by last name, 15% remote): W/D hot rows and BC c_data shifts."""
    db, S0 = w4
    b = db.gen_tpcc(4096, 99, 0)
    _run(db, S0, 4, b, scheme, 32, orc)
    b.free()


@pytest.fixture(scope="module")
def c3(torch_cuda, orc):
    """BASELINE.json configs[2]: 1 warehouse, NewOrder/Payment 50/50, batch 16K."""
    db = _db(1, 5, 16384)
    S0 = IT.population(5, 1)
    got = db.read_tpcc(POP)
    for k in POP:
        assert np.array_equal(got[k], S0[k])
    db.snapshot(True)
    yield db, S0
    db.close()


@pytest.mark.parametrize("lanes", [1, 32])
@pytest.mark.parametrize("scheme", SCHEMES)
def test_c3_full_size_parity(c3, orc, scheme, lanes):
    db, S0 = c3
    b = db.gen_tpcc(16384, 31, 5000)
    _run(db, S0, 1, b, scheme, lanes, orc)
    b.free()


@pytest.fixture(scope="module")
def c4(torch_cuda, orc):
    """BASELINE.json configs[3]: 64 warehouses, 45:43 NewOrder/Payment, batch 64K."""
    db = _db(64, 9, 65536)
    S0 = IT.population(9, 64)
    got = db.read_tpcc(["warehouse", "district"])
    assert np.array_equal(got["warehouse"], S0["warehouse"]) and np.array_equal(got["district"], S0["district"])
    for k in ("customer", "stock"):   # sampled rows of the big tables (the full compare is below)
        t = db.read_table(db.tpcc_ids[k])
        idx = np.random.default_rng(1).integers(0, t.shape[0], 4096)
        assert np.array_equal(t[idx], S0[k][idx])
    db.snapshot(True)
    yield db, S0
    db.close()


@pytest.mark.parametrize("lanes", [1, 32])
@pytest.mark.parametrize("scheme", SCHEMES)
def test_c4_full_size_parity(c4, orc, scheme, lanes):
    db, S0 = c4
    b = db.gen_tpcc(65536, 41, 5114)
    _run(db, S0, 64, b, scheme, lanes, orc)
    b.free()


@pytest.mark.parametrize("loopback", [False, True])
@pytest.mark.parametrize("scheme", SCHEMES)
def test_c4_full_size_parity_bench_launch(c4, orc, scheme, loopback):
    """configs[3] in the launches bench.py times for TPC-C (bench.tpcc_launch: per-scheme
    warps per SM, one block per SM where tuned; the loopback partitions' launch)."""
    import types
    import bench
    db, S0 = c4
    if loopback:
        la = bench.tpcc_launch(types.SimpleNamespace(launch="tuned"), scheme, db.num_sms, loopback)
    else:   # the `tpcc` block of the bench line (bench.TPCC_CONFIGS, configs[3])
        cfg = [c for c in bench.TPCC_CONFIGS if c["W"] == 64][0]
        bs, per_sm = cfg["launch"].get(scheme, cfg["launch"]["*"])
        la = {"bs": bs, "grid": db.num_sms if per_sm else 0}
    b = db.gen_tpcc(65536, 43, 5114)
    _run(db, S0, 64, b, scheme, 32, orc, launch=la)
    b.free()


@pytest.mark.parametrize("lanes", [1, 32])
def test_mvcc_split_layout(w4, orc, lanes):
    """f-3 metadata ablation (CC_FLAG_MVCC_SPLIT) on TPC-C: same results as interleaved."""
    from paper_2406_10158_b200.gcctb import CC_FLAG_MVCC_SPLIT
    db, S0 = w4
    b = db.gen_tpcc(8192, 41, 5000)
    _run(db, S0, 4, b, "mvcc", lanes, orc, flags=CC_FLAG_MVCC_SPLIT)
    b.free()


@pytest.mark.parametrize("scheme", SCHEMES)
@pytest.mark.parametrize("n,mix", [(1, 10000), (1, 0), (37, 10000), (1029, 5114)])
def test_ragged_batches_and_pure_mixes(w4, orc, scheme, n, mix):
    """A single transaction, batches that leave a partial last warp / block, and a
    NewOrder-only mix (every line a stock RMW; Payment-only is covered above)."""
    db, S0 = w4
    b = db.gen_tpcc(n, 500 + n + mix, mix)
    for lanes in (1, 32):
        _run(db, S0, 4, b, scheme, lanes, orc, launch={"bs": 32 if n > 64 else 1})
    b.free()


@pytest.mark.parametrize("mode", ["latched", "immediate", "stages", "binary_index", "meta_pad"])
@pytest.mark.parametrize("scheme", SCHEMES)
def test_w4_parity_flags(w4, orc, scheme, mode):
    """The execution flags change timing / instrumentation only: Exp-7 latched words
    (PAPER.md:836-852), the paper's immediate restart, Exp-6 stage clocks
    (PAPER.md:473), the paper's binary-search index and the padded control-word layout
    (f-3) keep TPC-C serial-replay parity."""
    from paper_2406_10158_b200 import gcctb as G
    flags = {"latched": G.CC_FLAG_LATCHED, "immediate": G.CC_FLAG_IMMEDIATE_RETRY,
             "stages": G.CC_FLAG_STAGES, "binary_index": G.CC_FLAG_INDEX_BINARY,
             "meta_pad": G.CC_FLAG_META_PAD}[mode]
    db, S0 = w4
    b = db.gen_tpcc(2048, 61, 5114)
    for lanes in (1, 32):
        _run(db, S0, 4, b, scheme, lanes, orc, flags=flags)
    b.free()


@pytest.mark.parametrize("lanes", [1, 32])
@pytest.mark.parametrize("scheme", ["tpl_nw", "tpl_wd", "to", "silo", "tictoc", "gputx", "gacco"])
def test_w4_event_log_conflict_graph(w4, orc, scheme, lanes):
    """f-4 debug mode on TPC-C: the device event log of the CC-managed accesses (W, D, C,
    stock rows) yields an acyclic conflict graph with one commit event per
    transaction.  (MVCC reads of older versions are not physical-order conflicts: MVCC is
    covered by the replay.)"""
    from paper_2406_10158_b200.gcctb import CC_FLAG_EVENTS
    from paper_2406_10158_b200.verify import check_serializable
    db, S0 = w4
    b = db.gen_tpcc(2048, 71, 5000)
    db.events_capacity(1 << 22)
    st = _run(db, S0, 4, b, scheme, lanes, orc, flags=CC_FLAG_EVENTS)
    ev = db.events()
    assert int((ev["kind"] == 2).sum()) == 2048
    assert int((ev["kind"] == 3).sum()) == st.aborts
    assert int((ev["kind"] == 0).sum()) > 0 and int((ev["kind"] == 1).sum()) > 0   # reads and installs logged
    ok, info = check_serializable(ev)
    assert ok, f"cycle {info}"
    db.events_capacity(0)
    b.free()
