"""Pins for the oracle parts the other CPU tests reach only through invariants
(-m "not gpu"; VERDICT r01 "parity unpinned" items):

* the YCSB row fingerprint fp and the affine write of reading Z11 (SURVEY.md §8(c),
  DESIGN.md §4) -- closed forms on rows of special structure, derived by hand from the
  reading's definition, so a rotation by j+1, a shift instead of a rotation, a dropped
  word, a dropped "+1", a wrong field or a missing write-counter increment each fail;
* Payment's BC c_data rewrite and h_data (TPC-C §2.5.2.2; reading R7) -- a hand-worked
  example in tests/golden/tpcc_payment_bc.json;
* orc_tpcc_accesses (the CC-managed records of a transaction, PAPER.md:343 record ids
  "arranged consecutively" W | D | C | S) -- against the rows a serial replay actually
  writes, and against the rows whose perturbation changes the transaction's output.
"""
import json
import os

import numpy as np
import pytest

M64 = (1 << 64) - 1
G = 0x9E3779B97F4A7C15   # the reading's multiplier (Z11)


def test_fp_closed_forms(orc):
    # a single word 1 in position k: fp = rotl(1, k) = 2^k (the rotation amount is j)
    for k in range(16):
        r = np.zeros(16, np.uint64)
        r[k] = 1
        assert orc.ycsb_fp(r) == 1 << k, k
    # the top bit in position k >= 1 wraps around to bit k-1: a rotation, not a shift
    for k in range(1, 16):
        r = np.zeros(16, np.uint64)
        r[k] = 1 << 63
        assert orc.ycsb_fp(r) == 1 << (k - 1), k
    # every word all-ones: each rotation is all-ones, the sum of 16 is -16 mod 2^64
    assert orc.ycsb_fp(np.full(16, M64, np.uint64)) == (16 * M64) & M64
    # every word 1: sum_j 2^j = 2^16 - 1 (all sixteen words, word 15 included)
    assert orc.ycsb_fp(np.ones(16, np.uint64)) == (1 << 16) - 1


def _exec_one(orc, rows, gid, keys, ops):
    """orc_ycsb_exec of transaction `gid` on `rows` (in place); returns out[K]."""
    K = len(keys)
    k = np.ascontiguousarray(keys, np.uint32)
    o = np.ascontiguousarray(ops, np.uint8)
    out = np.zeros(K, np.uint64)
    st = orc.lib().orc_ycsb_exec(orc._ptr(rows), rows.shape[0], gid, K, orc._ptr(k), orc._ptr(o), orc._ptr(out))
    assert st == 0
    return out


def test_affine_write_closed_forms(orc):
    rows = np.zeros((2, 16), np.uint64)
    rows[1, 7] = 1
    # txn gid 3: op 0 writes field 4 of row 0 (was 0), op 1 writes field 7 of row 1 (was 1)
    out = _exec_one(orc, rows, 3, [0, 1], [0x80 | 4, 0x80 | 7])
    # fp before the writes: row 0 all zero -> 0; row 1 has word 7 = 1 -> 2^7
    assert int(out[0]) == 0 and int(out[1]) == 1 << 7
    # r[f] = r[f] * G + ((gid << 4) | i) + 1: (3 << 4 | 0) + 1 = 49 and G + (3 << 4 | 1) + 1 = G + 50
    assert int(rows[0, 4]) == 49
    assert int(rows[1, 7]) == (G + 50) & M64
    # the write counter r[15] += 1 on every write, nothing else changes
    assert int(rows[0, 15]) == 1 and int(rows[1, 15]) == 1
    assert np.count_nonzero(rows[0]) == 2 and np.count_nonzero(rows[1]) == 2
    # a read changes nothing and outputs fp of the row as written: row 0 = 49 at word 4
    # (rotl 4 -> 49 * 16) plus 1 at word 15 (rotl 15 -> 2^15)
    before = rows.copy()
    out = _exec_one(orc, rows, 9, [0], [0x04])
    assert np.array_equal(rows, before)
    assert int(out[0]) == 49 * 16 + (1 << 15)
    # the same write twice from two transactions composes: 49 * G + (5 << 4 | 0) + 1
    _exec_one(orc, rows, 5, [0], [0x80 | 4])
    assert int(rows[0, 4]) == (49 * G + 81) & M64 and int(rows[0, 15]) == 2


# ------------------------------------------------------------------------------ TPC-C
GOLD_BC = json.load(open(os.path.join(os.path.dirname(__file__), "golden", "tpcc_payment_bc.json")))


def _u64(x):
    return np.uint64(x & M64)


def _bytes_words(b, n):
    return np.frombuffer(b.ljust(8 * n, b"\0"), dtype="<u8").copy()


def test_payment_bc_cdata_hdata(orc):
    from inputs import tpcc as IT
    from oracle import tpcc as OT
    e, x = GOLD_BC["example"], GOLD_BC["expect"]
    P = IT.population(3, 1)
    w, d, cw, cd, c, h = e["w"], e["d"], e["c_w"], e["c_d"], e["c"], e["h_amount"]
    crow = (cw * 10 + cd) * 3000 + c
    other = crow + 1                                   # a GC customer, untouched
    for row, credit in ((crow, b"BC"), (other, b"GC")):
        cr = P["customer"][row]
        cr[0] = _u64(e["c_balance_before"])
        cr[1] = _u64(e["c_ytd_before"])
        cr[2] = _u64(e["c_cnt_before"])
        cr[3] = np.uint64(int(cr[3]) & 0xFFFFFFFF | (int.from_bytes(credit, "little") << 32))
        cr[25:88] = np.arange(1000, 1063, dtype=np.uint64)
    P["warehouse"][w, 0] = _u64(e["w_ytd_before"])
    P["warehouse"][w, 2:4] = _bytes_words(e["w_name"].encode(), 2)
    P["district"][w * 10 + d, 0] = _u64(e["d_ytd_before"])
    P["district"][w * 10 + d, 2:4] = _bytes_words(e["d_name"].encode(), 2)
    other_before = P["customer"][other].copy()
    tx = np.zeros(40, np.uint32)
    tx[0:8] = [1, w, d, cw, cd, c, 0xFFFFFFFF, h]
    S, out = OT.replay(P, tx, [0], 1)
    cr = S["customer"][crow]
    assert [int(v) for v in cr[25:29]] == x["c_data_words_0_3"]
    assert np.array_equal(cr[29:88], np.arange(1000, 1059, dtype=np.uint64))
    assert int(cr[0]) == x["c_balance_after"] & M64 and int(cr[1]) == x["c_ytd_after"]
    assert int(cr[2]) & 0xFFFFFFFF == x["c_cnt_after"]
    assert int(S["warehouse"][w, 0]) == x["w_ytd_after"]
    assert int(S["district"][w * 10 + d, 0]) == x["d_ytd_after"]
    hist = S["history"][0]
    assert [int(v) for v in hist[0:5]] == x["history_words_0_4"]
    assert hist[5:8].tobytes() == x["h_data"].encode()
    o = out[:3]
    assert [int(o[0]), int(o[1]), int(o[2])] == [x["out"][0], x["out"][1] & M64, x["out"][2]]
    # the same Payment on the GC customer leaves c_data alone
    tx[5] = c + 1
    S2, out2 = OT.replay(P, tx, [0], 1)
    assert np.array_equal(S2["customer"][other][25:88], other_before[25:88])
    assert int(out2[2]) == int.from_bytes(b"GC", "little")


def _record_of(W, table, row):
    """CC-managed records numbered consecutively W | D | C | S."""
    base = {"warehouse": 0, "district": W, "customer": W + W * 10, "stock": W + W * 10 + W * 30000}
    return base[table] + row


@pytest.mark.parametrize("seed", [1, 2])
def test_tpcc_accesses_match_replay(orc, seed):
    from inputs import tpcc as IT
    from oracle import tpcc as OT
    W, B = 2, 40
    P = IT.population(3, W)
    tx = OT.gen(seed, W, B, 5000, IT.nurand_consts(3)).reshape(B, 40)
    for t in tx:
        rec, mode = OT.accesses(W, P["customer"], t)
        assert np.all(np.diff(rec.astype(np.int64)) != 0)
        S, out = OT.replay(P, t, [0], W)
        written = set()
        for k in ("warehouse", "district", "customer", "stock"):
            rows = np.nonzero((S[k] != P[k]).any(axis=1))[0]
            written |= {_record_of(W, k, int(r)) for r in rows}
        # every record the replay wrote is a write access, and every write access is written
        assert written == {int(r) for r, m in zip(rec, mode) if m & 1}
        # read accesses: perturbing the record changes the output (NewOrder reads W's
        # w_tax and C's c_discount; a perturbation of the next record does not)
        for r, m in zip(rec, mode):
            if m & 1:
                continue
            for k, base in (("warehouse", 0), ("customer", W + W * 10)):
                row = int(r) - base
                if 0 <= row < len(P[k]) and (k == "warehouse") == (int(r) < W):
                    Q = {kk: v.copy() for kk, v in P.items()}
                    Q[k][row, 1 if k == "warehouse" else 3] ^= np.uint64(0x7)   # w_tax / c_discount
                    _, out2 = OT.replay(Q, t, [0], W)
                    assert int(out2[1]) != int(out[1]), (k, row)
                    if row + 1 < len(P[k]):
                        Q = {kk: v.copy() for kk, v in P.items()}
                        Q[k][row + 1, 1 if k == "warehouse" else 3] ^= np.uint64(0x7)
                        _, out3 = OT.replay(Q, t, [0], W)
                        assert np.array_equal(out3, out)
