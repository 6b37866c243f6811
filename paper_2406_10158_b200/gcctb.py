"""Thin ctypes binding of libgcctb.so (include/gcctb.h).  Argument marshalling only:
every step of the hot path runs in the library's CUDA kernels.  Device buffers are
passed as raw pointers (torch tensors' data_ptr()); torch is plumbing only.

The library is loaded from this package directory; if it is missing the import of
``lib()`` raises -- there is no CPU fallback."""
from __future__ import annotations

import ctypes
import os

HERE = os.path.dirname(os.path.abspath(__file__))
# GCCTB_LIB: an experiment variant built by build.py --out (never set by the tests or bench)
LIB_PATH = os.environ.get("GCCTB_LIB") or os.path.join(HERE, "libgcctb.so")

CC_OK = 0
STATUS_NAMES = {0: "OK", 1: "INVALID_ARG", 2: "CONFIG", 3: "OOM", 4: "CUDA", 5: "NCCL",
                6: "KEY_NOT_FOUND", 7: "TS_OVERFLOW", 8: "VERSION_EXHAUSTED", 9: "WATCHDOG",
                10: "STATE", 11: "UNSUPPORTED"}

SCHEMES = ["tpl_nw", "tpl_wd", "to", "mvcc", "silo", "tictoc", "gputx", "gacco"]
SCHEME_ID = {s: i for i, s in enumerate(SCHEMES)}

CC_FLAG_IMMEDIATE_RETRY = 0x1
CC_FLAG_TIMING = 0x2
CC_FLAG_PARTITIONED = 0x4
CC_FLAG_PART_ALL = 0x8
CC_FLAG_INDEX_BINARY = 0x10
CC_FLAG_LATCHED = 0x20
CC_FLAG_STAGES = 0x40
CC_FLAG_EVENTS = 0x80
CC_FLAG_INDEX_TREE = 0x100
CC_FLAG_FLAT_JITTER = 0x200
CC_FLAG_MVCC_SPLIT = 0x400
CC_FLAG_PART_2PC = 0x800
CC_FLAG_INDEX_EYTZ = 0x1000
CC_FLAG_WARM = 0x2000
CC_FLAG_PART_P2P = 0x4000
CC_FLAG_L2_PERSIST = 0x8000
CC_FLAG_META_PAD = 0x10000
CC_SRC_HOST_ASYNC = 2
STAGES = ["index", "ts_alloc", "wait", "cc_manager", "abort", "useful", "attempts"]
PART_REC_BYTES = 48
CC_STATS_WORDS = 16


class cc_db_desc(ctypes.Structure):
    _fields_ = [("device", ctypes.c_int), ("stream", ctypes.c_void_p), ("rank", ctypes.c_int),
                ("world", ctypes.c_int)]


class cc_ycsb_db_desc(ctypes.Structure):
    _fields_ = [("n_rows", ctypes.c_uint64), ("seed", ctypes.c_uint64)]


class cc_ycsb_gen_desc(ctypes.Structure):
    _fields_ = [("n_txn", ctypes.c_uint32), ("ops_per_txn", ctypes.c_uint32),
                ("write_frac", ctypes.c_double), ("seed", ctypes.c_uint64),
                ("thresholds", ctypes.c_void_p), ("thresholds_on_device", ctypes.c_int),
                ("scramble_mult", ctypes.c_uint64)]


class cc_tpcc_db_desc(ctypes.Structure):
    _fields_ = [("warehouses", ctypes.c_uint32), ("w_first", ctypes.c_uint32), ("w_count", ctypes.c_uint32),
                ("max_txn", ctypes.c_uint32), ("seed", ctypes.c_uint64)]


class cc_tpcc_gen_desc(ctypes.Structure):
    _fields_ = [("n_txn", ctypes.c_uint32), ("neworder_permyriad", ctypes.c_uint32), ("seed", ctypes.c_uint64),
                ("w_lo", ctypes.c_uint32), ("w_hi", ctypes.c_uint32)]


class cc_exec_desc(ctypes.Structure):
    _fields_ = [("scheme", ctypes.c_int), ("wd", ctypes.c_uint32), ("bs", ctypes.c_uint32),
                ("flags", ctypes.c_uint32), ("grid", ctypes.c_uint32),
                ("lanes_per_txn", ctypes.c_uint32), ("watchdog_s", ctypes.c_double),
                ("claim_chunk", ctypes.c_uint32)]


class cc_result(ctypes.Structure):
    _fields_ = [("committed", ctypes.c_void_p), ("restarts", ctypes.c_void_p),
                ("order_hi", ctypes.c_void_p), ("order_lo", ctypes.c_void_p),
                ("commit_pos", ctypes.c_void_p), ("read_out", ctypes.c_void_p),
                ("stats", ctypes.c_void_p)]


class cc_stats(ctypes.Structure):
    _fields_ = [("commits", ctypes.c_uint64), ("aborts", ctypes.c_uint64),
                ("attempts", ctypes.c_uint64), ("error", ctypes.c_uint64),
                ("max_rank", ctypes.c_uint64), ("ts_last", ctypes.c_uint64),
                ("reserved", ctypes.c_uint64 * 2), ("stage_cycles", ctypes.c_uint64 * 7),
                ("sm_clock_khz", ctypes.c_uint64)]


class cc_roofline(ctypes.Structure):
    _fields_ = [("gather_gbs", ctypes.c_double), ("cas_l2_per_s", ctypes.c_double),
                ("cas_hbm_per_s", ctypes.c_double), ("handoff_row_ns", ctypes.c_double),
                ("handoff_ns", ctypes.c_double), ("handoff_acq_row_ns", ctypes.c_double)]


class cc_ipc_handle(ctypes.Structure):
    _fields_ = [("ipc", ctypes.c_ubyte * 64), ("rank", ctypes.c_uint32), ("world", ctypes.c_uint32),
                ("cap", ctypes.c_uint32), ("max_txn", ctypes.c_uint32)]


_lib = None

# name -> (restype, argtypes)
_P = ctypes.c_void_p
_SIGS = {
    "cc_version": (ctypes.c_char_p, []),
    "cc_last_error": (ctypes.c_char_p, [_P]),
    "cc_db_create": (ctypes.c_int, [ctypes.POINTER(cc_db_desc), ctypes.POINTER(_P)]),
    "cc_db_destroy": (ctypes.c_int, [_P]),
    "cc_table_create": (ctypes.c_int, [_P, ctypes.c_char_p, ctypes.c_uint32, ctypes.c_uint64,
                                       ctypes.POINTER(ctypes.c_uint32)]),
    "cc_table_load": (ctypes.c_int, [_P, ctypes.c_uint32, ctypes.c_uint64, ctypes.c_uint64, _P,
                                     ctypes.c_int]),
    "cc_table_read": (ctypes.c_int, [_P, ctypes.c_uint32, ctypes.c_uint64, ctypes.c_uint64, _P,
                                     ctypes.c_int]),
    "cc_table_info": (ctypes.c_int, [_P, ctypes.c_uint32, ctypes.POINTER(ctypes.c_uint64),
                                     ctypes.POINTER(ctypes.c_uint32)]),
    "cc_index_create": (ctypes.c_int, [_P, ctypes.c_uint32, _P, _P, ctypes.c_uint64, ctypes.c_int,
                                       ctypes.POINTER(ctypes.c_uint32)]),
    "cc_load_ycsb": (ctypes.c_int, [_P, ctypes.POINTER(cc_ycsb_db_desc)]),
    "cc_index_lookup": (ctypes.c_int, [_P, ctypes.c_uint32, _P, ctypes.c_uint64, _P, ctypes.c_uint32]),
    "cc_batch_gen_ycsb": (ctypes.c_int, [_P, ctypes.POINTER(cc_ycsb_gen_desc), ctypes.POINTER(_P)]),
    "cc_batch_import_ycsb": (ctypes.c_int, [_P, _P, _P, ctypes.c_uint32, ctypes.c_uint32,
                                            ctypes.c_int, ctypes.POINTER(_P)]),
    "cc_batch_export_ycsb": (ctypes.c_int, [_P, _P, _P, _P]),
    "cc_batch_info": (ctypes.c_int, [_P, _P, ctypes.POINTER(ctypes.c_uint32),
                                     ctypes.POINTER(ctypes.c_uint32), ctypes.POINTER(ctypes.c_uint32)]),
    "cc_batch_free": (ctypes.c_int, [_P, _P]),
    "cc_pool_trim": (ctypes.c_int, [_P]),
    "cc_mem_stats": (ctypes.c_int, [_P, ctypes.POINTER(ctypes.c_uint64), ctypes.POINTER(ctypes.c_uint64),
                                    ctypes.POINTER(ctypes.c_uint64)]),
    "cc_submit": (ctypes.c_int, [_P, _P, ctypes.POINTER(cc_exec_desc), ctypes.POINTER(cc_result)]),
    "cc_prepare": (ctypes.c_int, [_P, _P, ctypes.c_int, ctypes.c_uint32]),
    "cc_sync": (ctypes.c_int, [_P, ctypes.POINTER(cc_stats)]),
    "cc_join": (ctypes.c_int, [_P]),
    "cc_timing_read": (ctypes.c_int, [_P, ctypes.POINTER(ctypes.c_double * 5),
                                      ctypes.POINTER(ctypes.c_uint64), ctypes.c_int]),
    "cc_snapshot": (ctypes.c_int, [_P, ctypes.c_int]),
    "cc_load_tpcc": (ctypes.c_int, [_P, ctypes.POINTER(cc_tpcc_db_desc)]),
    "cc_tpcc_tables": (ctypes.c_int, [_P, ctypes.POINTER(ctypes.c_uint32 * 9)]),
    "cc_batch_gen_tpcc": (ctypes.c_int, [_P, ctypes.POINTER(cc_tpcc_gen_desc), ctypes.POINTER(_P)]),
    "cc_batch_import_tpcc": (ctypes.c_int, [_P, _P, ctypes.c_uint32, ctypes.c_int, ctypes.POINTER(_P)]),
    "cc_batch_export_tpcc": (ctypes.c_int, [_P, _P, _P]),
    "cc_part_send": (ctypes.c_int, [_P, ctypes.POINTER(_P), _P]),
    "cc_events_capacity": (ctypes.c_int, [_P, ctypes.c_uint64]),
    "cc_events_read": (ctypes.c_int, [_P, _P, ctypes.c_uint64, ctypes.POINTER(ctypes.c_uint64)]),
    "cc_part_apply": (ctypes.c_int, [_P, _P, ctypes.c_uint64, _P]),
    "cc_part_finish": (ctypes.c_int, [_P, _P, ctypes.c_uint64]),
    "cc_part_decide": (ctypes.c_int, [_P, _P, ctypes.c_uint64, ctypes.POINTER(_P)]),
    "cc_part_commit": (ctypes.c_int, [_P, _P, _P, ctypes.c_uint64]),
    "cc_part_next": (ctypes.c_int, [_P, ctypes.POINTER(ctypes.c_uint64)]),
    "cc_roofline_probe": (ctypes.c_int, [_P, ctypes.POINTER(cc_roofline)]),
    "cc_gather_sweep": (ctypes.c_int, [_P, ctypes.POINTER(ctypes.c_double * 4)]),
    "cc_part_window": (ctypes.c_int, [_P, ctypes.POINTER(cc_ipc_handle)]),
    "cc_part_connect": (ctypes.c_int, [_P, ctypes.POINTER(cc_ipc_handle)]),
    "cc_part_connect_local": (ctypes.c_int, [ctypes.POINTER(_P), ctypes.c_int]),
}

TPCC_TX_WORDS = 40
TPCC_OUT_WORDS = 48
TPCC_TABLES = ["warehouse", "district", "customer", "stock", "item", "order", "new_order", "order_line", "history"]

EXPORTED = sorted(_SIGS)


def lib(path: str | None = None):
    """Load libgcctb.so (raises if it was not built: there is no fallback)."""
    global _lib
    if _lib is None:
        p = path or LIB_PATH
        if not os.path.exists(p):
            raise RuntimeError(f"{p} missing: run __graft_entry__.build() (no CPU fallback exists)")
        L = ctypes.CDLL(p)
        for name, (res, args) in _SIGS.items():
            f = getattr(L, name)
            f.restype = res
            f.argtypes = args
        _lib = L
    return _lib


class CCError(RuntimeError):
    def __init__(self, status, msg):
        super().__init__(f"{STATUS_NAMES.get(status, status)}: {msg}")
        self.status = status


def check(db, st):
    if st != CC_OK:
        msg = lib().cc_last_error(db).decode() if db else ""
        raise CCError(st, msg)
