"""Python convenience layer over the C ABI: torch tensors as caller-owned device result
buffers, the db stream = the current torch stream.  Marshalling only."""
from __future__ import annotations

import ctypes
from dataclasses import dataclass

import numpy as np
import torch

from . import gcctb as G


@dataclass
class Result:
    committed: torch.Tensor
    restarts: torch.Tensor
    order_hi: torch.Tensor
    order_lo: torch.Tensor
    commit_pos: torch.Tensor
    read_out: torch.Tensor | None
    stats: torch.Tensor

    @staticmethod
    def alloc(n_txn: int, K: int, device, read_out=True, stream=None, out_words=None) -> "Result":
        """Allocate on `stream` (the db's stream) so the zero-fill is ordered before
        the library's kernels on that stream."""
        if stream is not None:
            with torch.cuda.stream(stream):
                return Result.alloc(n_txn, K, device, read_out, out_words=out_words)
        z = dict(device=device)
        return Result(
            committed=torch.zeros(n_txn, dtype=torch.uint8, **z),
            restarts=torch.zeros(n_txn, dtype=torch.int32, **z),
            order_hi=torch.zeros(n_txn, dtype=torch.int64, **z),
            order_lo=torch.zeros(n_txn, dtype=torch.int64, **z),
            commit_pos=torch.zeros(n_txn, dtype=torch.int32, **z),
            read_out=torch.zeros(n_txn * (out_words or K), dtype=torch.int64, **z) if read_out else None,
            stats=torch.zeros(G.CC_STATS_WORDS, dtype=torch.int64, **z),
        )

    @staticmethod
    def alloc_host(n_txn: int, K: int, read_out=True, out_words=None) -> "Result":
        """Pinned host buffers: the submit stages the results on the device and copies them
        out asynchronously (complete at the next sync)."""
        z = dict(device="cpu", pin_memory=True)
        return Result(
            committed=torch.zeros(n_txn, dtype=torch.uint8, **z),
            restarts=torch.zeros(n_txn, dtype=torch.int32, **z),
            order_hi=torch.zeros(n_txn, dtype=torch.int64, **z),
            order_lo=torch.zeros(n_txn, dtype=torch.int64, **z),
            commit_pos=torch.zeros(n_txn, dtype=torch.int32, **z),
            read_out=torch.zeros(n_txn * (out_words or K), dtype=torch.int64, **z) if read_out else None,
            stats=torch.zeros(G.CC_STATS_WORDS, dtype=torch.int64, **z),
        )

    def c(self) -> G.cc_result:
        p = lambda t: ctypes.c_void_p(t.data_ptr()) if t is not None else None  # noqa: E731
        return G.cc_result(p(self.committed), p(self.restarts), p(self.order_hi), p(self.order_lo),
                           p(self.commit_pos), p(self.read_out), p(self.stats))

    def host(self, stream=None) -> dict:
        if stream is not None:
            stream.synchronize()
        u = lambda t: t.cpu().numpy()  # noqa: E731
        d = {
            "committed": u(self.committed),
            "restarts": u(self.restarts).view(np.uint32),
            "order_hi": u(self.order_hi).view(np.uint64),
            "order_lo": u(self.order_lo).view(np.uint64),
            "commit_pos": u(self.commit_pos).view(np.uint32),
        }
        if self.read_out is not None:
            d["read_out"] = u(self.read_out).view(np.uint64)
        return d


class _CudaBytes:
    """__cuda_array_interface__ view of library-owned device memory (no copy)."""

    def __init__(self, ptr: int, nbytes: int):
        self.__cuda_array_interface__ = {"shape": (nbytes,), "typestr": "|u1", "data": (ptr, False),
                                         "version": 3}


def _device_bytes(ptr: int, nbytes: int, device: int) -> torch.Tensor:
    return torch.as_tensor(_CudaBytes(ptr, nbytes), device=torch.device("cuda", device))


class Batch:
    def __init__(self, db: "DB", handle):
        self.db = db
        self.h = handle
        n, k, kind = ctypes.c_uint32(), ctypes.c_uint32(), ctypes.c_uint32()
        G.check(db.h, G.lib().cc_batch_info(db.h, handle, ctypes.byref(n), ctypes.byref(k),
                                            ctypes.byref(kind)))
        self.n_txn, self.K, self.kind = n.value, k.value, kind.value

    def export_ycsb(self):
        keys = np.zeros(self.n_txn * self.K, dtype=np.uint32)
        ops = np.zeros(self.n_txn * self.K, dtype=np.uint8)
        G.check(self.db.h, G.lib().cc_batch_export_ycsb(self.db.h, self.h, keys.ctypes.data,
                                                        ops.ctypes.data))
        return keys, ops

    def export_tpcc(self):
        tx = np.zeros(self.n_txn * G.TPCC_TX_WORDS, dtype=np.uint32)
        G.check(self.db.h, G.lib().cc_batch_export_tpcc(self.db.h, self.h, tx.ctypes.data))
        return tx

    @property
    def out_words(self):
        return G.TPCC_OUT_WORDS if self.kind == 2 else self.K

    def free(self):
        if self.h:
            G.lib().cc_batch_free(self.db.h, self.h)
            self.h = None


class DB:
    """One db on one device.  All library work runs on ``self.stream`` (an explicit
    torch stream, never the legacy default stream, which would make the library create
    an unordered stream of its own).  Result buffers are allocated on it; callers that
    touch results with torch ops must use ``with torch.cuda.stream(db.stream)`` or
    synchronise first (``sync()``)."""

    def __init__(self, device: int = 0, stream=None, rank: int = 0, world: int = 1):
        L = G.lib()
        if stream is None or stream.cuda_stream == 0:
            # highest priority: pending blocks of the executor are scheduled before those of
            # the library's low-priority preprocessing stream (cc_prepare)
            stream = torch.cuda.Stream(device, priority=-8)
        self.stream = stream
        self.device = device
        d = G.cc_db_desc(device, ctypes.c_void_p(stream.cuda_stream), rank, world)
        self.rank, self.world = rank, world
        h = ctypes.c_void_p()
        G.check(None, L.cc_db_create(ctypes.byref(d), ctypes.byref(h)))
        self.h = h
        self.ycsb_rows = 0
        self.num_sms = torch.cuda.get_device_properties(device).multi_processor_count

    def close(self):
        if self.h:
            G.lib().cc_db_destroy(self.h)
            self.h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    def _chk(self, st):
        G.check(self.h, st)

    # ----------------------------------------------------------- YCSB
    def load_ycsb(self, n_rows: int, seed: int):
        d = G.cc_ycsb_db_desc(n_rows, seed)
        self._chk(G.lib().cc_load_ycsb(self.h, ctypes.byref(d)))
        self.ycsb_rows = n_rows
        self.ycsb_table = 0

    def gen_ycsb(self, n_txn: int, K: int, W: float, seed: int, thresholds, mult: int) -> Batch:
        """thresholds: torch uint64/int64 cuda tensor or numpy uint64 array."""
        if isinstance(thresholds, torch.Tensor):
            self._use(thresholds)
            ptr, on_dev = thresholds.data_ptr(), 1
            keep = thresholds
        else:
            keep = np.ascontiguousarray(thresholds, dtype=np.uint64)
            ptr, on_dev = keep.ctypes.data, 0
        g = G.cc_ycsb_gen_desc(n_txn, K, float(W), seed, ctypes.c_void_p(ptr), on_dev, mult)
        h = ctypes.c_void_p()
        self._chk(G.lib().cc_batch_gen_ycsb(self.h, ctypes.byref(g), ctypes.byref(h)))
        del keep
        return Batch(self, h)

    def import_ycsb(self, keys, ops, K: int, async_host: bool = False) -> Batch:
        """keys/ops: device tensors, or host arrays / CPU tensors.  async_host: copy host
        buffers on the copy stream without waiting (CC_SRC_HOST_ASYNC; pass pinned CPU
        tensors and keep them unchanged until the batch's first submit has completed)."""
        h = ctypes.c_void_p()
        keep = None
        if isinstance(keys, torch.Tensor) and keys.is_cuda:
            self._use(keys, ops)
            st = G.lib().cc_batch_import_ycsb(self.h, keys.data_ptr(), ops.data_ptr(),
                                              keys.numel() // K, K, 1, ctypes.byref(h))
        else:
            if isinstance(keys, torch.Tensor):
                k, o = keys.contiguous(), ops.contiguous()
                kp, op, n = k.data_ptr(), o.data_ptr(), k.numel()
            else:
                k = np.ascontiguousarray(keys, dtype=np.uint32)
                o = np.ascontiguousarray(ops, dtype=np.uint8)
                kp, op, n = k.ctypes.data, o.ctypes.data, k.size
            keep = (k, o)
            st = G.lib().cc_batch_import_ycsb(self.h, kp, op, n // K, K, G.CC_SRC_HOST_ASYNC if async_host else 0,
                                              ctypes.byref(h))
        self._chk(st)
        b = Batch(self, h)
        b._keep = keep if async_host else None   # host buffers stay alive with the batch
        return b

    # ----------------------------------------------------------- TPC-C
    def load_tpcc(self, warehouses: int, seed: int, max_txn: int, w_first: int = 0, w_count: int | None = None):
        d = G.cc_tpcc_db_desc(warehouses, w_first, warehouses if w_count is None else w_count, max_txn, seed)
        self._chk(G.lib().cc_load_tpcc(self.h, ctypes.byref(d)))
        ids = (ctypes.c_uint32 * 9)()
        self._chk(G.lib().cc_tpcc_tables(self.h, ctypes.byref(ids)))
        self.tpcc_ids = dict(zip(G.TPCC_TABLES, list(ids)))

    def gen_tpcc(self, n_txn: int, seed: int, neworder_permyriad: int = 5000, w_lo: int = 0, w_hi=None) -> Batch:
        if w_hi is None:
            rows = ctypes.c_uint64()
            self._chk(G.lib().cc_table_info(self.h, self.tpcc_ids["warehouse"], ctypes.byref(rows), None))
            w_hi = w_lo + rows.value
        g = G.cc_tpcc_gen_desc(n_txn, neworder_permyriad, seed, w_lo, w_hi)
        h = ctypes.c_void_p()
        self._chk(G.lib().cc_batch_gen_tpcc(self.h, ctypes.byref(g), ctypes.byref(h)))
        return Batch(self, h)

    def import_tpcc(self, tx) -> Batch:
        t = np.ascontiguousarray(tx, dtype=np.uint32)
        h = ctypes.c_void_p()
        self._chk(G.lib().cc_batch_import_tpcc(self.h, t.ctypes.data, t.size // G.TPCC_TX_WORDS, 0, ctypes.byref(h)))
        return Batch(self, h)

    def read_tpcc(self, names=None) -> dict:
        return {k: self.read_table(self.tpcc_ids[k]) for k in (names or G.TPCC_TABLES)}

    def create_table(self, name: str, row_bytes: int, rows: int) -> int:
        tid = ctypes.c_uint32()
        self._chk(G.lib().cc_table_create(self.h, name.encode(), row_bytes, rows, ctypes.byref(tid)))
        return tid.value

    def create_index(self, table_id: int, sorted_keys, row_ids) -> int:
        k = np.ascontiguousarray(sorted_keys, dtype=np.uint64)
        r = np.ascontiguousarray(row_ids, dtype=np.uint64)
        iid = ctypes.c_uint32()
        self._chk(G.lib().cc_index_create(self.h, table_id, k.ctypes.data, r.ctypes.data, k.size, 0,
                                          ctypes.byref(iid)))
        return iid.value

    def index_lookup(self, index_id: int, keys, method: str = "auto") -> np.ndarray:
        """method: "auto" (direct addressing on a dense key range, else the tree), "tree",
        "eytz" (Eytzinger layout) or "binary"; all return the same rows."""
        flags = {"auto": 0, "tree": G.CC_FLAG_INDEX_TREE, "binary": G.CC_FLAG_INDEX_BINARY,
                 "eytz": G.CC_FLAG_INDEX_EYTZ}[method]
        dev = torch.device("cuda", self.device)
        with torch.cuda.stream(self.stream):
            k = torch.from_numpy(np.ascontiguousarray(keys, dtype=np.uint64).view(np.int64)).to(dev)
            out = torch.empty_like(k)
        self._chk(G.lib().cc_index_lookup(self.h, index_id, k.data_ptr(), k.numel(), out.data_ptr(),
                                          flags))
        self.stream.synchronize()
        return out.cpu().numpy().view(np.uint64)

    def read_table(self, table_id: int = 0) -> np.ndarray:
        rows, rb = ctypes.c_uint64(), ctypes.c_uint32()
        self._chk(G.lib().cc_table_info(self.h, table_id, ctypes.byref(rows), ctypes.byref(rb)))
        out = np.zeros(rows.value * rb.value // 8, dtype=np.uint64)
        self._chk(G.lib().cc_table_read(self.h, table_id, 0, rows.value, out.ctypes.data, 0))
        return out.reshape(rows.value, rb.value // 8)

    def load_table(self, table_id: int, rows: np.ndarray, first: int = 0):
        r = np.ascontiguousarray(rows)
        rb = r.shape[1] * r.itemsize if r.ndim == 2 else None
        n = r.shape[0]
        self._chk(G.lib().cc_table_load(self.h, table_id, first, n, r.ctypes.data, 0))

    # ----------------------------------------------------------- execution
    def submit(self, batch: Batch, scheme, wd: int = 0, bs: int = 32, flags: int = 0,
               grid: int = 0, watchdog_s: float = 30.0, result: Result | None = None,
               read_out=True, lanes: int = 1, claim_chunk: int = 1) -> Result:
        sid = G.SCHEME_ID[scheme] if isinstance(scheme, str) else int(scheme)
        if result is None:
            result = Result.alloc(batch.n_txn, batch.K, torch.device("cuda", self.device), read_out,
                                  stream=self.stream, out_words=batch.out_words)
        d = G.cc_exec_desc(sid, wd, bs, flags, grid, lanes, watchdog_s, claim_chunk)
        r = result.c()
        self._chk(G.lib().cc_submit(self.h, batch.h, ctypes.byref(d), ctypes.byref(r)))
        return result

    def prepare(self, batch: Batch, scheme, flags: int = 0):
        """f-4: run a3 of GPUTx / GaccO for `batch` on the preprocessing stream (overlaps the
        main stream); the next submit of `batch` with `scheme` consumes it."""
        sid = G.SCHEME_ID[scheme] if isinstance(scheme, str) else int(scheme)
        self._chk(G.lib().cc_prepare(self.h, batch.h, sid, flags))

    # ----------------------------------------------------------- partitioned TPC-C (a8)
    def _use(self, *tensors):
        """The db stream waits for the current stream, and each caller tensor is marked as
        in use by the db stream: the caching allocator must not hand its memory to a later
        allocation (e.g. the next torch.cat of a loopback round) before the library's
        kernels on the db stream have read it -- otherwise a temporary freed right after
        the call (a concatenated decision buffer) could be overwritten under them."""
        self.stream.wait_stream(torch.cuda.current_stream(self.device))
        for t in tensors:
            if t is not None and t.is_cuda and t.numel():
                t.record_stream(self.stream)

    def part_send(self):
        """(device uint8 tensor of the phase-B requests grouped by destination, counts list)."""
        ptr = ctypes.c_void_p()
        counts = np.zeros(self.world, dtype=np.uint64)
        self._chk(G.lib().cc_part_send(self.h, ctypes.byref(ptr), counts.ctypes.data))
        n = int(counts.sum())
        buf = _device_bytes(ptr.value, n * G.PART_REC_BYTES, self.device) if n else \
            torch.empty(0, dtype=torch.uint8, device=torch.device("cuda", self.device))
        return buf, [int(c) for c in counts]

    def part_apply(self, recv: torch.Tensor) -> torch.Tensor:
        n = recv.numel() // G.PART_REC_BYTES
        with torch.cuda.stream(self.stream):
            resp = torch.empty(n * G.PART_REC_BYTES, dtype=torch.uint8, device=recv.device)
        self._use(recv)
        self._chk(G.lib().cc_part_apply(self.h, recv.data_ptr() if n else None, n, resp.data_ptr() if n else None))
        return resp

    def part_finish(self, resp: torch.Tensor):
        n = resp.numel() // G.PART_REC_BYTES
        self._use(resp)
        self._chk(G.lib().cc_part_finish(self.h, resp.data_ptr() if n else None, n))

    # in-library exchange over peer memory (CC_FLAG_PART_P2P)
    def part_window(self) -> bytes:
        """This db's exchange window handle (bytes of cc_ipc_handle), to be gathered by all ranks."""
        h = G.cc_ipc_handle()
        self._chk(G.lib().cc_part_window(self.h, ctypes.byref(h)))
        return bytes(h)

    def part_connect(self, handles: list[bytes]):
        arr = (G.cc_ipc_handle * len(handles))()
        for i, hb in enumerate(handles):
            ctypes.memmove(ctypes.byref(arr[i]), hb, ctypes.sizeof(G.cc_ipc_handle))
        self._chk(G.lib().cc_part_connect(self.h, arr))

    @staticmethod
    def part_connect_local(dbs: list["DB"]):
        arr = (ctypes.c_void_p * len(dbs))(*[db.h.value for db in dbs])
        G.check(dbs[0].h, G.lib().cc_part_connect_local(arr, len(dbs)))

    # 2PC phase B (f-2)
    def part_decide(self, back: torch.Tensor) -> torch.Tensor:
        """Home: decide this round from the returned responses; device u64 decisions
        aligned with this round's send buffer (as a uint8 tensor of 8 bytes each)."""
        n = back.numel() // G.PART_REC_BYTES
        self._use(back)
        ptr = ctypes.c_void_p()
        self._chk(G.lib().cc_part_decide(self.h, back.data_ptr() if n else None, n, ctypes.byref(ptr)))
        if n == 0:
            return torch.empty(0, dtype=torch.uint8, device=torch.device("cuda", self.device))
        return _device_bytes(ptr.value, n * 8, self.device)

    def part_commit(self, recv: torch.Tensor, dec: torch.Tensor):
        n = dec.numel() // 8
        self._use(recv, dec)
        self._chk(G.lib().cc_part_commit(self.h, recv.data_ptr() if n else None, dec.data_ptr() if n else None, n))

    def part_next(self) -> int:
        p = ctypes.c_uint64()
        self._chk(G.lib().cc_part_next(self.h, ctypes.byref(p)))
        return int(p.value)

    # ----------------------------------------------------------- debug event log (f-4)
    EVENT_DTYPE = np.dtype([("seq", "<u8"), ("gid", "<u4"), ("rec", "<u4"), ("attempt", "<u4"), ("kind", "<u4")])

    def events_capacity(self, cap: int):
        self._chk(G.lib().cc_events_capacity(self.h, cap))
        self._events_cap = cap

    def events(self) -> np.ndarray:
        cap = getattr(self, "_events_cap", 0)
        buf = np.zeros(cap, dtype=self.EVENT_DTYPE)
        n = ctypes.c_uint64()
        self._chk(G.lib().cc_events_read(self.h, buf.ctypes.data, cap, ctypes.byref(n)))
        if n.value > cap:
            raise RuntimeError(f"event log overflow: {n.value} events > capacity {cap}")
        return buf[:n.value]

    def join(self) -> None:
        """The db stream waits (on the device) for the library's background zeroing of CC
        words, so an event recorded after it covers every submit so far (cc_join)."""
        self._chk(G.lib().cc_join(self.h))

    def sync(self) -> G.cc_stats:
        s = G.cc_stats()
        self._chk(G.lib().cc_sync(self.h, ctypes.byref(s)))
        return s

    def timing(self, reset: bool = False):
        ms = (ctypes.c_double * 5)()
        n = ctypes.c_uint64()
        self._chk(G.lib().cc_timing_read(self.h, ctypes.byref(ms), ctypes.byref(n), int(reset)))
        return list(ms), n.value

    def roofline_probe(self) -> dict:
        """Memory-system ceilings (cc_roofline_probe): random-line gather GB/s, distinct-
        address CAS/s (L2-resident and > L2), per-record hand-off ns (with / without row)."""
        r = G.cc_roofline()
        self._chk(G.lib().cc_roofline_probe(self.h, ctypes.byref(r)))
        return {k: getattr(r, k) for k, _ in r._fields_}

    def mem_stats(self) -> tuple[int, int, int]:
        """(cudaMalloc calls, cudaFree calls, bytes allocated) of the driver so far."""
        a, f, b = ctypes.c_uint64(), ctypes.c_uint64(), ctypes.c_uint64()
        self._chk(G.lib().cc_mem_stats(self.h, ctypes.byref(a), ctypes.byref(f), ctypes.byref(b)))
        return a.value, f.value, b.value

    def pool_trim(self):
        self._chk(G.lib().cc_pool_trim(self.h))

    def gather_sweep(self) -> dict:
        """GB/s of random 32 / 64 / 128 / 256 B reads over 1 GiB (cc_gather_sweep)."""
        out = (ctypes.c_double * 4)()
        self._chk(G.lib().cc_gather_sweep(self.h, ctypes.byref(out)))
        return {32: out[0], 64: out[1], 128: out[2], 256: out[3]}

    def snapshot(self, save: bool):
        self._chk(G.lib().cc_snapshot(self.h, 1 if save else 0))
