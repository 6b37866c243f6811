"""Pins for the TPC-C oracle (-m "not gpu"): TPC-C §3.3.2 consistency conditions
(delta forms), conservation per customer and stock row, a hand-worked
NewOrder (tests/golden/tpcc_neworder.json), the by-name rule, generator rates."""
import json
import os

import numpy as np
import pytest

import inputs
from inputs import tpcc as IT

GOLD = json.load(open(os.path.join(os.path.dirname(__file__), "golden", "tpcc_neworder.json")))
TXW = 40


@pytest.fixture(scope="module")
def pop2():
    return IT.population(3, 2)


def _gen(orc, seed, W, B, no_pm=5000):
    from oracle import tpcc as OT
    return OT.gen(seed, W, B, no_pm, IT.nurand_consts(3))


def test_neworder_hand_example(orc):
    from oracle import tpcc as OT
    g = GOLD
    P = IT.population(3, 1)
    P["warehouse"][0, 1] = g["w_tax"]
    P["district"][0, 1] = g["d_tax"] | (g["d_next_o_id"] << 32)
    P["customer"][5, 3] = (P["customer"][5, 3] & np.uint64(0xFFFFFFFF00000000)) | np.uint64(g["c_discount"])
    tx = np.zeros(TXW, np.uint32)
    tx[0], tx[1], tx[2], tx[3], tx[4], tx[5], tx[6], tx[8], tx[9] = 0, 0, 0, 0, 0, 5, 0xFFFFFFFF, 2, 1
    for j, ln in enumerate(g["lines"]):
        P["item"][ln["item"], 0] = (P["item"][ln["item"], 0] & np.uint64(0xFFFFFFFF00000000)) | np.uint64(ln["price"])
        P["stock"][ln["item"], 0] = np.uint64(ln["s_quantity"])
        tx[10 + j] = ln["item"]
        tx[25 + j] = (0 << 8) | ln["qty"]
    S, out = OT.replay(P, tx, [0], 1)
    e = g["expect"]
    assert out[0] == e["o_id"] and out[1] == e["total"]
    assert [int(out[4 + 3 * j]) for j in range(2)] == e["ol_amount"]
    assert [int(out[2 + 3 * j]) for j in range(2)] == [ln["s_quantity"] for ln in g["lines"]]
    for j, ln in enumerate(g["lines"]):
        s = S["stock"][ln["item"]]
        assert int(s[0]) & 0xFFFFFFFF == e["s_quantity_after"][j]
        assert int(s[0]) >> 32 == e["s_order_cnt"][j] and int(s[1]) == e["s_ytd"][j]
    assert int(S["district"][0, 1]) >> 32 == e["d_next_o_id_after"]
    assert int(S["order"][0, 5]) == 2 and int(S["order_line"][0, 4]) == 3000


def test_consistency_conditions(orc, pop2):
    from oracle import tpcc as OT
    W, B = 2, 3000
    tx = _gen(orc, 11, W, B)
    T = tx.reshape(B, TXW)
    order = np.random.default_rng(5).permutation(B)
    S, out = OT.replay(pop2, tx, order, W)
    P = pop2
    no = T[:, 0] == 0
    pay = ~no
    wy = S["warehouse"][:, 0].astype(np.int64)
    dy = S["district"][:, 0].astype(np.int64).reshape(W, 10)
    # condition 1: W_YTD = sum(D_YTD)
    assert np.array_equal(wy, dy.sum(axis=1))
    # conditions 8/9 (delta): W_YTD - 300,000.00 = sum h_amount; D_YTD - 30,000.00 likewise
    for w in range(W):
        assert wy[w] - 30000000 == int(T[pay & (T[:, 1] == w), 7].astype(np.int64).sum())
        for d in range(10):
            sel = pay & (T[:, 1] == w) & (T[:, 2] == d)
            assert dy[w, d] - 3000000 == int(T[sel, 7].astype(np.int64).sum())
    # condition 2 (delta): D_NEXT_O_ID - 3001 = #NewOrders of the district, ids contiguous
    nxt = (S["district"][:, 1] >> np.uint64(32)).astype(np.int64).reshape(W, 10)
    for w in range(W):
        for d in range(10):
            sel = no & (T[:, 1] == w) & (T[:, 2] == d)
            assert nxt[w, d] - 3001 == int(sel.sum())
            ids = np.sort(S["order"][np.nonzero(sel)[0], 0].astype(np.int64))
            assert np.array_equal(ids, np.arange(3001, 3001 + sel.sum()))
    # conditions 3/4: NO row and OL rows agree with the O row
    for g in np.nonzero(no)[0][:300]:
        o = S["order"][g]
        assert np.array_equal(S["new_order"][g][:3], o[:3])
        n = int(o[5])
        assert n == T[g, 8]
        ol = S["order_line"][g * 15:(g + 1) * 15]
        assert all(int(ol[j, 0]) & 0xFFFFFFFF == int(o[0]) for j in range(n))
        assert not ol[n:].any()
    # per-customer conservation via the history slots
    hist = S["history"][pay]
    cid = (hist[:, 0] & np.uint64(0xFFFFFFFF)).astype(np.int64) - 1
    cd = (hist[:, 0] >> np.uint64(32)).astype(np.int64) - 1
    cw = (hist[:, 1] & np.uint64(0xFFFFFFFF)).astype(np.int64) - 1
    row = (cw * 10 + cd) * 3000 + cid
    amt = hist[:, 4].astype(np.int64)
    exp_ytd = np.zeros(W * 30000, np.int64)
    np.add.at(exp_ytd, row, amt)
    cnt = np.zeros(W * 30000, np.int64)
    np.add.at(cnt, row, 1)
    c0, c1 = P["customer"], S["customer"]
    assert np.array_equal(c1[:, 1].astype(np.int64) - c0[:, 1].astype(np.int64), exp_ytd)
    assert np.array_equal(c0[:, 0].astype(np.int64) - c1[:, 0].astype(np.int64), exp_ytd)
    assert np.array_equal((c1[:, 2] & np.uint64(0xFFFFFFFF)).astype(np.int64) - 1, cnt)
    # per-stock conservation: s_ytd, s_order_cnt, s_remote_cnt over committed lines
    ytd = np.zeros(W * 100000, np.int64); oc = np.zeros_like(ytd); rc = np.zeros_like(ytd)
    for g in np.nonzero(no)[0]:
        for j in range(T[g, 8]):
            sw = int(T[g, 25 + j]) >> 8
            r = sw * 100000 + int(T[g, 10 + j])
            ytd[r] += int(T[g, 25 + j]) & 0xFF
            oc[r] += 1
            rc[r] += sw != int(T[g, 1])
    s1 = S["stock"]
    assert np.array_equal(s1[:, 1].astype(np.int64), ytd)
    assert np.array_equal((s1[:, 0] >> np.uint64(32)).astype(np.int64), oc)
    assert np.array_equal((s1[:, 2] & np.uint64(0xFFFFFFFF)).astype(np.int64), rc)


def test_serial_order_matters(orc, pop2):
    """Two NewOrders of one district swap their o_ids when their order swaps."""
    from oracle import tpcc as OT
    tx = _gen(orc, 4, 2, 400, no_pm=10000)
    T = tx.reshape(400, TXW)
    a, b = [int(x) for x in np.nonzero((T[:, 1] == T[0, 1]) & (T[:, 2] == T[0, 2]))[0][:2]]
    _, o1 = OT.replay(pop2, tx, [a, b], 2)
    _, o2 = OT.replay(pop2, tx, [b, a], 2)
    assert o1[a * 48] == o2[b * 48] == 3001 and o1[b * 48] == o2[a * 48] == 3002


def test_by_name_rule(orc, pop2):
    from oracle import tpcc as OT
    C = pop2["customer"]
    for (w, d, last) in [(0, 0, 0), (1, 3, 371), (0, 9, 999), (1, 0, 123)]:
        base = (w * 10 + d) * 3000
        name = IT.last_name(last).ljust(16, b"\0")
        ids = [c for c in range(3000) if C[base + c, 4:6].tobytes() == name]
        ids.sort(key=lambda c: (C[base + c, 6:8].tobytes(), c))
        assert OT.by_name(C, w, d, last) == ids[(len(ids) + 1) // 2 - 1]


def test_generator_rates(orc):
    W, B = 64, 40000
    tx = _gen(orc, 9, W, B, no_pm=5114).reshape(B, TXW)    # 45:43 mix
    no = tx[:, 0] == 0
    assert abs(no.mean() - 0.5114) < 5 * np.sqrt(0.25 / B)
    olc = tx[no, 8]
    assert olc.min() == 5 and olc.max() == 15 and abs(olc.mean() - 10) < 0.1
    lines = [(tx[g, 10:10 + tx[g, 8]], tx[g, 25:25 + tx[g, 8]]) for g in np.nonzero(no)[0]]
    remote_lines = sum(int(((sq >> 8) != tx[g, 1]).sum()) for g, (_, sq) in zip(np.nonzero(no)[0], lines))
    n_lines = int(olc.sum())
    assert abs(remote_lines / n_lines - 0.01) < 0.002
    any_remote = np.mean([((sq >> 8) != tx[g, 1]).any() for g, (_, sq) in zip(np.nonzero(no)[0], lines)])
    assert abs(any_remote - 0.0952) < 0.01       # 9.52% of NewOrders
    for (it, sq) in lines[:2000]:
        key = (sq >> 8).astype(np.int64) * 100000 + it
        assert (np.diff(key) > 0).all()           # stock-key order, distinct
    pay = tx[~no]
    assert abs((pay[:, 3] != pay[:, 1]).mean() - 0.15) < 0.01
    assert abs((pay[:, 5] == 0xFFFFFFFF).mean() - 0.60) < 0.01
    assert pay[:, 7].min() >= 100 and pay[:, 7].max() <= 500000
    assert (tx[:, 1] < W).all() and (tx[:, 2] < 10).all()


def test_nurand_nonuniform(orc):
    W, B = 1, 40000
    tx = _gen(orc, 2, W, B, no_pm=10000).reshape(B, TXW)
    c = tx[:, 5]
    assert c.min() >= 0 and c.max() < 3000
    counts = np.bincount(c, minlength=3000)
    # NURand is skewed: the most popular customers are far above uniform (B/3000)
    assert counts.max() > 3 * B / 3000
