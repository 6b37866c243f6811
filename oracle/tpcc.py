"""ctypes marshalling + checks for the TPC-C oracle (oracle_tpcc.c).  TEST
INFRASTRUCTURE ONLY (see oracle/__init__.py)."""
from __future__ import annotations

import ctypes

import numpy as np

TX_WORDS = 40
OUT_WORDS = 48
TABLES = ("warehouse", "district", "customer", "stock")
SLOTS = ("order", "new_order", "order_line", "history")
_L = None


def _bind(L):
    global _L
    u32, u64, i32, p = ctypes.c_uint32, ctypes.c_uint64, ctypes.c_int, ctypes.c_void_p
    L.orc_tpcc_gen.restype = i32
    L.orc_tpcc_gen.argtypes = [u64, u32, u32, u32, u32, u32, u32, u32, u32, p]
    L.orc_tpcc_replay.restype = i32
    L.orc_tpcc_replay.argtypes = [u32, p, p, p, p, p, p, p, p, p, u64, u32, p, p, u32, p]
    L.orc_tpcc_by_name.restype = ctypes.c_int64
    L.orc_tpcc_by_name.argtypes = [p, u32, u32, u32]
    L.orc_tpcc_accesses.restype = i32
    L.orc_tpcc_accesses.argtypes = [u32, p, p, p, p]
    _L = L


def _lib():
    from . import lib
    lib()
    return _L


def _ptr(a):
    assert a.flags["C_CONTIGUOUS"]
    return a.ctypes.data_as(ctypes.c_void_p)


def gen(seed, W, n_txn, no_permyriad, consts, w_lo=0, w_hi=None):
    """The a1 TPC-C generator (oracle copy).  consts = (c_last_load, c_last_run, c_id, c_ol_i_id)."""
    tx = np.zeros(n_txn * TX_WORDS, np.uint32)
    st = _lib().orc_tpcc_gen(seed, W, w_lo, W if w_hi is None else w_hi, n_txn, no_permyriad,
                             consts[1], consts[2], consts[3], _ptr(tx))
    if st:
        from . import OracleError
        raise OracleError(f"orc_tpcc_gen status {st}")
    return tx


def empty_slots(n_txn):
    return {"order": np.zeros((n_txn, 8), np.uint64), "new_order": np.zeros((n_txn, 4), np.uint64),
            "order_line": np.zeros((n_txn * 15, 8), np.uint64), "history": np.zeros((n_txn, 8), np.uint64)}


def replay(S0: dict, tx, order, W, entry_date=20240601):
    """Serial replay in `order`.  S0: dict with warehouse/district/customer/stock/item
    arrays (and optionally slot arrays).  Returns (state dict, out u64[n_txn*48])."""
    n_txn = tx.size // TX_WORDS
    S = {k: np.array(S0[k], dtype=np.uint64, copy=True, order="C") for k in TABLES}
    S["item"] = np.ascontiguousarray(S0["item"], dtype=np.uint64)
    sl = empty_slots(n_txn)
    for k in SLOTS:
        S[k] = np.array(S0[k], np.uint64, copy=True, order="C") if k in S0 else sl[k]
    out = np.zeros(n_txn * OUT_WORDS, np.uint64)
    order = np.ascontiguousarray(order, dtype=np.uint32)
    st = _lib().orc_tpcc_replay(W, _ptr(S["warehouse"]), _ptr(S["district"]), _ptr(S["customer"]),
                                _ptr(S["stock"]), _ptr(S["item"]), _ptr(S["order"]), _ptr(S["new_order"]),
                                _ptr(S["order_line"]), _ptr(S["history"]), entry_date, n_txn,
                                _ptr(np.ascontiguousarray(tx, np.uint32)), _ptr(order), order.size, _ptr(out))
    if st:
        from . import OracleError
        raise OracleError(f"orc_tpcc_replay status {st}")
    return S, out


def by_name(customer, w, d, last):
    c = np.ascontiguousarray(customer, np.uint64)
    return int(_lib().orc_tpcc_by_name(_ptr(c), w, d, last))


def accesses(W, customer, tx_row):
    c = np.ascontiguousarray(customer, np.uint64)
    rec = np.zeros(18, np.uint64)
    mode = np.zeros(18, np.uint8)
    n = _lib().orc_tpcc_accesses(W, _ptr(c), _ptr(np.ascontiguousarray(tx_row, np.uint32)), _ptr(rec), _ptr(mode))
    return rec[:n], mode[:n]


def check(scheme, S0, tx, W, res, S_gpu, entry_date=20240601, require_all=True):
    """SURVEY.md §8(c) steps 1-5 for a TPC-C submit: order permutation (+ gid order for
    GPUTx/GaccO), serial replay equality of outputs and every table byte (CC tables and
    reserved slots of committed transactions)."""
    from . import DETERMINISTIC, order_from_result
    n_txn = tx.size // TX_WORDS
    committed = np.asarray(res["committed"]).astype(bool)
    if require_all and not committed.all():
        raise AssertionError(f"{(~committed).sum()} transactions did not commit")
    pi = order_from_result(committed, res["commit_pos"], res.get("order_hi"), res.get("order_lo"))
    if scheme in DETERMINISTIC:
        if not np.array_equal(pi, np.sort(pi)):
            raise AssertionError(f"{scheme}: reported order is not ascending gid")
        if np.asarray(res["restarts"]).any():
            raise AssertionError(f"{scheme}: deterministic scheme aborted")
    S, out = replay(S0, tx, pi, W, entry_date)
    og = np.asarray(res["read_out"], np.uint64).reshape(n_txn, OUT_WORDS)
    oe = out.reshape(n_txn, OUT_WORDS)
    bad = np.nonzero((og != oe).any(axis=1) & committed)[0]
    if bad.size:
        t = int(bad[0])
        raise AssertionError(f"{scheme}: outputs differ for {bad.size} txns; first {t} "
                             f"(type {tx[t*TX_WORDS]}): gpu {og[t][:6]} exp {oe[t][:6]}")
    for k in TABLES + SLOTS:
        a = np.asarray(S_gpu[k], np.uint64).reshape(S[k].shape)
        if not np.array_equal(a, S[k]):
            rows = np.nonzero((a != S[k]).any(axis=1))[0]
            raise AssertionError(f"{scheme}: table {k} differs from serial replay in {rows.size} rows "
                                 f"(first {int(rows[0])})")
    return {"committed": int(committed.sum())}
