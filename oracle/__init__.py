"""CPU oracle -- TEST INFRASTRUCTURE ONLY.

Only ``tests/``, ``__graft_entry__.smoke()`` and ``bench.py``'s ``cpu_baseline`` /
``--impl reference`` legs may import this package.  The product path
(``paper_2406_10158_b200``) never imports it, and it never imports the product path:
the two share no code.  The arithmetic lives in plain single-threaded C
(``oracle_ycsb.c``, ``oracle_tpcc.c``) built by ``__graft_entry__.build()`` into
``oracle/liboracle.so``; this module is ctypes marshalling plus the order / replay /
invariant checks of SURVEY.md §8(c) "The definition" (steps 1-6).
"""
from __future__ import annotations

import ctypes
import itertools
import os
import subprocess

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
_LIB_PATH = os.path.join(_HERE, "liboracle.so")
_SOURCES = ["oracle_ycsb.c", "oracle_tpcc.c"]
_lib = None


def build(force: bool = False) -> str:
    """Compile the C oracle with gcc (building the checker is not using it)."""
    srcs = [os.path.join(_HERE, s) for s in _SOURCES if os.path.exists(os.path.join(_HERE, s))]
    if not force and os.path.exists(_LIB_PATH):
        mt = os.path.getmtime(_LIB_PATH)
        if all(os.path.getmtime(s) <= mt for s in srcs):
            return _LIB_PATH
    cmd = ["gcc", "-O2", "-std=c11", "-Wall", "-Wextra", "-shared", "-fPIC", "-o", _LIB_PATH] + srcs
    subprocess.check_call(cmd)
    return _LIB_PATH


def lib():
    global _lib
    if _lib is None:
        build()
        L = ctypes.CDLL(_LIB_PATH)
        u64, u32, i32, dbl = ctypes.c_uint64, ctypes.c_uint32, ctypes.c_int, ctypes.c_double
        p = ctypes.c_void_p
        L.orc_rng.restype = u64
        L.orc_rng.argtypes = [u64, u64, u64]
        L.orc_ycsb_fp.restype = u64
        L.orc_ycsb_fp.argtypes = [p]
        L.orc_ycsb_exec.restype = i32
        L.orc_ycsb_exec.argtypes = [p, u64, u32, u32, p, p, p]
        L.orc_ycsb_replay.restype = i32
        L.orc_ycsb_replay.argtypes = [p, u64, u32, u32, p, p, p, u32, p]
        L.orc_ycsb_gen.restype = i32
        L.orc_ycsb_gen.argtypes = [u64, u64, u32, u32, dbl, p, u64, p, p]
        L.orc_gputx_ranks.restype = i32
        L.orc_gputx_ranks.argtypes = [u32, u32, p, p, u64, p]
        L.orc_gacco_positions.restype = i32
        L.orc_gacco_positions.argtypes = [u32, u32, p, u64, p]
        if hasattr(L, "orc_tpcc_replay"):
            from . import tpcc as _t
            _t._bind(L)
        _lib = L
    return _lib


def _ptr(a: np.ndarray):
    assert a.flags["C_CONTIGUOUS"]
    return a.ctypes.data_as(ctypes.c_void_p)


class OracleError(RuntimeError):
    pass


# ----------------------------------------------------------------------------- YCSB

def ycsb_fp(row) -> int:
    r = np.ascontiguousarray(row, dtype=np.uint64)
    return int(lib().orc_ycsb_fp(_ptr(r)))


def ycsb_gen(seed: int, n_rows: int, n_txn: int, K: int, W: float,
             thresholds: np.ndarray, mult: int):
    """The a1 YCSB generator (oracle copy).  Returns (keys u32[n*K], ops u8[n*K])."""
    T = np.ascontiguousarray(thresholds, dtype=np.uint64)
    keys = np.zeros(n_txn * K, dtype=np.uint32)
    ops = np.zeros(n_txn * K, dtype=np.uint8)
    st = lib().orc_ycsb_gen(seed, n_rows, n_txn, K, float(W), _ptr(T), mult, _ptr(keys), _ptr(ops))
    if st:
        raise OracleError(f"orc_ycsb_gen status {st}")
    return keys, ops


def ycsb_replay(rows0: np.ndarray, keys: np.ndarray, ops: np.ndarray, K: int, order):
    """Serial replay in `order`.  Returns (final rows, out u64[n_txn*K])."""
    rows = np.array(rows0, dtype=np.uint64, copy=True, order="C")
    keys = np.ascontiguousarray(keys, dtype=np.uint32)
    ops = np.ascontiguousarray(ops, dtype=np.uint8)
    order = np.ascontiguousarray(order, dtype=np.uint32)
    n_txn = keys.size // K
    out = np.zeros(n_txn * K, dtype=np.uint64)
    st = lib().orc_ycsb_replay(_ptr(rows), rows.shape[0], n_txn, K, _ptr(keys), _ptr(ops),
                               _ptr(order), order.size, _ptr(out))
    if st:
        raise OracleError(f"orc_ycsb_replay status {st}")
    return rows, out


def gputx_ranks(keys, ops, K: int, n_items: int) -> np.ndarray:
    keys = np.ascontiguousarray(keys, dtype=np.uint32)
    ops = np.ascontiguousarray(ops, dtype=np.uint8)
    n_txn = keys.size // K
    r = np.zeros(n_txn, dtype=np.uint32)
    st = lib().orc_gputx_ranks(n_txn, K, _ptr(keys), _ptr(ops), n_items, _ptr(r))
    if st:
        raise OracleError(f"orc_gputx_ranks status {st}")
    return r


def gacco_positions(keys, K: int, n_items: int) -> np.ndarray:
    keys = np.ascontiguousarray(keys, dtype=np.uint32)
    pos = np.zeros(keys.size, dtype=np.uint32)
    st = lib().orc_gacco_positions(keys.size // K, K, _ptr(keys), n_items, _ptr(pos))
    if st:
        raise OracleError(f"orc_gacco_positions status {st}")
    return pos


# ---------------------------------------------------------------- order + replay check

DETERMINISTIC = {"gputx", "gacco"}


def order_from_result(committed, commit_pos, order_hi=None, order_lo=None):
    """commit_pos must be a permutation of
    [0, n_committed) over the committed transactions, and, when order keys are
    given, the keys must be strictly increasing along that permutation.
    Returns pi (txn ids in serialization order)."""
    committed = np.asarray(committed).astype(bool)
    ids = np.nonzero(committed)[0]
    pos = np.asarray(commit_pos, dtype=np.int64)[ids]
    if ids.size and not np.array_equal(np.sort(pos), np.arange(ids.size)):
        raise AssertionError("commit_pos is not a permutation of the committed set")
    pi = np.empty(ids.size, dtype=np.uint32)
    pi[pos] = ids
    if order_hi is not None and order_lo is not None and pi.size > 1:
        hi = np.asarray(order_hi, dtype=np.uint64)[pi]
        lo = np.asarray(order_lo, dtype=np.uint64)[pi]
        inc = (hi[1:] > hi[:-1]) | ((hi[1:] == hi[:-1]) & (lo[1:] > lo[:-1]))
        if not inc.all():
            bad = int(np.nonzero(~inc)[0][0])
            raise AssertionError(f"order keys not strictly increasing along commit_pos at {bad}")
    return pi


def check_ycsb(scheme: str, rows0, keys, ops, K: int, res: dict, rows_gpu, *,
               require_all=True) -> dict:
    """Full SURVEY.md §8(c) check of one GPU submit on YCSB.

    res: committed u8[n], commit_pos u32[n], order_hi/order_lo u64[n], read_out u64[n*K],
         restarts u32[n].  rows_gpu: final table (n_rows, 16) u64.
    Raises AssertionError on the first violation; returns a small report."""
    n_txn = keys.size // K
    committed = np.asarray(res["committed"]).astype(bool)
    if require_all and not committed.all():
        raise AssertionError(f"{(~committed).sum()} transactions did not commit")
    pi = order_from_result(committed, res["commit_pos"], res.get("order_hi"), res.get("order_lo"))
    if scheme in DETERMINISTIC:
        # step 2: deterministic schemes serialize in batch (gid) order
        if not np.array_equal(pi, np.sort(pi)):
            raise AssertionError(f"{scheme}: reported order is not ascending gid")
        if np.asarray(res["restarts"]).any():
            raise AssertionError(f"{scheme}: deterministic scheme aborted")
    rows_exp, out_exp = ycsb_replay(rows0, keys, ops, K, pi)
    out_gpu = np.asarray(res["read_out"], dtype=np.uint64).reshape(n_txn, K)
    out_exp = out_exp.reshape(n_txn, K)
    bad = np.nonzero((out_gpu != out_exp).any(axis=1) & committed)[0]
    if bad.size:
        t = int(bad[0])
        raise AssertionError(f"{scheme}: read outputs differ from serial replay for {bad.size} "
                             f"txns, first gid {t}: gpu {out_gpu[t][:4]} exp {out_exp[t][:4]}")
    rows_gpu = np.asarray(rows_gpu, dtype=np.uint64).reshape(rows_exp.shape)
    if not np.array_equal(rows_gpu, rows_exp):
        diff = np.nonzero((rows_gpu != rows_exp).any(axis=1))[0]
        raise AssertionError(f"{scheme}: final state differs from serial replay in {diff.size} rows "
                             f"(first row {int(diff[0])})")
    # step 5, order-free invariant: write counter conservation
    n_writes = int(((np.asarray(ops).reshape(n_txn, K) & 0x80) != 0)[committed].sum())
    d15 = int((rows_gpu[:, 15].astype(np.int64) - np.asarray(rows0)[:, 15].astype(np.int64)).sum())
    if d15 != n_writes:
        raise AssertionError(f"{scheme}: sum of write counters moved by {d15}, expected {n_writes}")
    return {"committed": int(committed.sum()), "aborts": int(np.asarray(res["restarts"]).sum())}


def ycsb_serial_outcomes(rows0, keys, ops, K: int, ids):
    """Brute force: the set of (final rows bytes, outputs bytes)
    over every serial order of the transactions `ids` (n <= 7)."""
    ids = list(ids)
    if len(ids) > 7:
        raise ValueError("brute force limited to 7 transactions")
    outs = set()
    for perm in itertools.permutations(ids):
        r, o = ycsb_replay(rows0, keys, ops, K, np.array(perm, dtype=np.uint32))
        outs.add((r.tobytes(), o.reshape(-1, K)[ids].tobytes()))
    return outs
