"""cc_roofline_probe (SURVEY.md §8(d) ceilings) returns physical numbers on a B200, and the
bench's bound bookkeeping is consistent (host logic: -m "not gpu")."""
import numpy as np
import pytest

import bench


def test_hot_record_counts_and_atomics():
    keys = np.array([[5, 7, 9, 11], [5, 6, 9, 12], [1, 5, 9, 13]], dtype=np.uint32)
    ops = np.zeros_like(keys, dtype=np.uint8)
    ops[0, 0] = ops[1, 0] = 0x80   # two writes of record 5; record 9 read three times
    acc, w = bench.hot_record_counts(keys, ops, 16)
    assert (acc, w) == (3, 2)
    # 2PL: acquire + release per op, a ticket and a claim per transaction
    assert bench.atomics_per_batch(3, 4, 2, "tpl_nw") == 2 * 12 + 3 + 3
    assert bench.atomics_per_batch(3, 4, 2, "gacco") == 0


def test_scheme_bounds_binding():
    ceil = {"gather_gbs": 1000.0, "cas_l2_per_s": 1e10, "cas_hbm_per_s": 1e9,
            "handoff_row_ns": 1000.0, "handoff_ns": 500.0}
    # 1 ms exec, 100 MB -> 100 GB/s = 10 % of gather; 1e6 atomics -> 1e9/s = 10 %;
    # GaccO chain of 500 accesses x 1 us = 0.5 ms -> 50 %: serialization binds
    b = bench.scheme_bounds("gacco", 1.0, 100e6, 0, 500, 50, 0, ceil)
    assert b["binding"] == "serial" and abs(b["serial_frac"] - 0.5) < 1e-9
    assert b["atomic_frac"] is None and abs(b["gather_frac"] - 0.1) < 1e-9
    b = bench.scheme_bounds("gputx", 1.0, 100e6, 10**6, 500, 50, 299, ceil)
    assert b["serial_chain"] == 300 and b["binding"] == "serial"
    b = bench.scheme_bounds("silo", 1.0, 600e6, 10**6, 500, 50, 0, ceil)
    assert b["serial_chain"] == 50 and b["binding"] == "gather"


@pytest.mark.gpu
def test_roofline_probe_values():
    from paper_2406_10158_b200.api import DB
    db = DB(0)
    r = db.roofline_probe()
    db.close()
    assert 100.0 < r["gather_gbs"] < 8000.0, r
    assert 1e8 < r["cas_hbm_per_s"] <= r["cas_l2_per_s"] * 1.5 < 1e12, r
    assert 50.0 < r["handoff_ns"] < 20000.0, r
    assert r["handoff_row_ns"] > r["handoff_ns"] * 0.8, r
