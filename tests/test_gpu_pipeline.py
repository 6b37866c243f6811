"""f-4: GPUTx / GaccO preprocessing prepared ahead on the
second stream (cc_prepare) gives exactly the results of the inline a3, while the main stream
executes another batch."""
import numpy as np
import pytest

import inputs

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def torch_cuda():
    torch = pytest.importorskip("torch")
    if not torch.cuda.is_available():
        pytest.skip("no GPU")
    return torch


@pytest.fixture(scope="module")
def c1(torch_cuda, orc):
    from paper_2406_10158_b200.api import DB
    db = DB(0)
    db.load_ycsb(1024, 11)
    S0 = db.read_table(0)
    db.snapshot(True)
    yield db, S0
    db.close()


def _gen(db, orc, seed):
    T = inputs.zipf_thresholds(1024, 0.8)
    A = inputs.scramble_mult(1024)
    b = db.gen_ycsb(1024, 4, 0.5, seed, T, A)
    keys, ops = orc.ycsb_gen(seed, 1024, 1024, 4, 0.5, T, A)
    return b, keys, ops


@pytest.mark.parametrize("lanes", [1, 4])
@pytest.mark.parametrize("scheme", ["gputx", "gacco"])
def test_prepared_matches_inline(c1, orc, scheme, lanes):
    db, S0 = c1
    b, keys, ops = _gen(db, orc, 91)
    outs = []
    for prepared in (False, True):
        db.snapshot(False)
        if prepared:
            db.prepare(b, scheme)
        res = db.submit(b, scheme, wd=0, bs=32, lanes=lanes)
        db.sync()
        h = res.host(db.stream)
        orc.check_ycsb(scheme, S0, keys, ops, 4, h, db.read_table(0))
        outs.append(h)
    for k in ("committed", "order_lo", "commit_pos", "read_out"):
        assert np.array_equal(outs[0][k], outs[1][k]), k
    b.free()


def test_prepare_overlaps_previous_batch(c1, orc):
    """Pipeline: batch i+1 is prepared while batch i executes; each batch is checked against
    the oracle from its own starting state; a prepared result is consumed once (a second
    submit of the same batch prepares inline)."""
    db, S0 = c1
    for scheme in ("gacco", "gputx"):
        b1, k1, o1 = _gen(db, orc, 92)
        b2, k2, o2 = _gen(db, orc, 93)
        db.snapshot(False)
        db.prepare(b1, scheme)
        r1 = db.submit(b1, scheme, wd=0, bs=32, lanes=4)
        db.prepare(b2, scheme)                      # runs beside b1's execution
        db.sync()
        h1 = r1.host(db.stream)
        S1 = db.read_table(0)
        orc.check_ycsb(scheme, S0, k1, o1, 4, h1, S1)
        r2 = db.submit(b2, scheme, wd=0, bs=32, lanes=4)
        db.sync()
        orc.check_ycsb(scheme, S1, k2, o2, 4, r2.host(db.stream), db.read_table(0))
        S2 = db.read_table(0)
        r3 = db.submit(b2, scheme, wd=0, bs=32, lanes=4)   # not prepared again: inline a3
        db.sync()
        orc.check_ycsb(scheme, S2, k2, o2, 4, r3.host(db.stream), db.read_table(0))
        b1.free()
        b2.free()


def test_prepare_other_schemes_is_noop(c1, orc):
    db, S0 = c1
    b, keys, ops = _gen(db, orc, 94)
    db.snapshot(False)
    db.prepare(b, "silo")
    res = db.submit(b, "silo", wd=0, bs=32, lanes=4)
    db.sync()
    orc.check_ycsb("silo", S0, keys, ops, 4, res.host(db.stream), db.read_table(0))
    b.free()


def test_prepare_key_not_found_surfaces_at_submit(c1):
    from paper_2406_10158_b200.gcctb import CCError
    db, _ = c1
    keys = np.full(64 * 4, 5000, np.uint32)   # beyond the 1,024-row table
    ops = np.zeros(keys.size, np.uint8)
    b = db.import_ycsb(keys, ops, 4)
    db.prepare(b, "gacco")
    db.submit(b, "gacco", wd=0, bs=32, lanes=4)
    with pytest.raises(CCError, match="KEY_NOT_FOUND"):
        db.sync()
    b.free()


@pytest.mark.parametrize("scheme", ["gputx", "gacco"])
def test_prepared_tpcc(torch_cuda, orc, scheme):
    import inputs.tpcc as IT
    from oracle import tpcc as OT
    from paper_2406_10158_b200.api import DB
    db = DB(0)
    db.load_tpcc(2, 23, 4096)
    S0 = IT.population(23, 2)
    db.snapshot(True)
    b = db.gen_tpcc(4096, 5, 5000)
    tx = b.export_tpcc()
    db.prepare(b, scheme)
    res = db.submit(b, scheme, wd=0, bs=8, lanes=32, watchdog_s=60)
    st = db.sync()
    assert st.commits == 4096
    h = res.host(db.stream)
    S = db.read_tpcc(list(OT.TABLES + OT.SLOTS))
    S = {k: (v[:4096 * 15] if k == "order_line" else v[:4096]) if k in OT.SLOTS else v for k, v in S.items()}
    OT.check(scheme, S0, tx, 2, h, S)
    b.free()
    db.close()
