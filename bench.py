"""bench.py -- committed txn/s + abort rate per CC scheme on YCSB (BASELINE.json
metric; workload = configs[1]: 10,485,760-row table, batch 64K x 16 ops).

One step = one pass of the whole hot path over one synthetic batch: a1 on-device batch
generation, then for each of the 8 schemes a2 reset, a3 preprocessing (GPUTx/GaccO),
a4-a6 execution with abort compaction, a7 result emission.  value = committed
transactions of all schemes / step time (whole job, summed over ranks).

YCSB does not shard: with N GPUs every rank runs an independent
replica on its own batch ("replicas only", weak scaling); no data-path collective.

  python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference]
"""
from __future__ import annotations

import argparse
import json
import os
import subprocess
import sys
import threading
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

SCHEMES = ["tpl_nw", "tpl_wd", "to", "mvcc", "silo", "tictoc", "gputx", "gacco"]
METRIC = "committed txn/s + abort rate per CC scheme, YCSB & TPC-C, at 1/2/4/8 B200"


def parse():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=5)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--rows", type=int, default=10 * (1 << 20))
    ap.add_argument("--batch", type=int, default=1 << 16)
    ap.add_argument("--ops", type=int, default=16)
    ap.add_argument("--theta", type=float, default=0.6)   # MC preset
    ap.add_argument("--write-frac", type=float, default=0.1)
    ap.add_argument("--wd", type=int, default=0)          # paper launch wd=0, bs=32
    ap.add_argument("--bs", type=int, default=32)
    ap.add_argument("--launch", choices=["tuned", "fixed"], default="tuned",
                    help="tuned: per-scheme warps per SM measured best at configs[1] theta=0.6 "
                         "(profiles/r01_tune_bs.jsonl; one block per SM); fixed: --wd/--bs for "
                         "every scheme with a full-occupancy grid")
    ap.add_argument("--phase-events", action=argparse.BooleanOptionalAction, default=False,
                    help="CC_FLAG_TIMING (library phase events) on the timed submits: five CUDA "
                         "events per submit, ~2 %% of the step (off: the exec share comes from the "
                         "per-scheme pass)")
    ap.add_argument("--scheme-events", action=argparse.BooleanOptionalAction, default=True,
                    help="a CUDA event between the schemes of each timed step (step_scheme_ms)")
    ap.add_argument("--lanes", type=int, default=32)      # tile mode: lane i owns op i (32: one txn per warp); 1 = thread per txn (paper)
    ap.add_argument("--schemes", default=",".join(SCHEMES))
    ap.add_argument("--index", default="dense", choices=["dense", "tree", "binary", "eytz"],
                    help="dense = direct addressing on the dense YCSB key range (default); tree = cache-line "
                         "search tree over the sorted keys; binary = PAPER.md:344 (identical results)")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-ceilings", action="store_true",
                    help="skip cc_roofline_probe (for ncu launch lists: its ring kernel is long)")
    ap.add_argument("--pipeline", action=argparse.BooleanOptionalAction, default=True,
                    help="f-4 (default on): prepare GPUTx / GaccO for each step's batch on the low-priority "
                         "prep stream (cc_prepare) while the other schemes execute.  With the tuned launch "
                         "(one block of 8-24 warps per SM) the rank pass runs beside the executors: 78 -> 85 M "
                         "txn/s (profiles/r01_bench_v24_pipeline.jsonl); with full-occupancy grids it was "
                         "slower (profiles/r01_bench_v5_*).  --no-pipeline: inline a3")
    ap.add_argument("--workload", default="ycsb", choices=["ycsb", "tpcc"],
                    help="ycsb = configs[1] (default); tpcc = configs[4]: W warehouses partitioned over the ranks")
    ap.add_argument("--warehouses", type=int, default=512)
    ap.add_argument("--tpcc-batch", type=int, default=65536, help="transactions per rank per step")
    ap.add_argument("--tpcc-mix", type=int, default=5114, help="NewOrder share in 1/10,000 (45:43, PAPER.md:468)")
    ap.add_argument("--two-pc", action="store_true",
                    help="TPC-C: distributed transactions of tpl_nw / tpl_wd in 2PC rounds (f-2); the other "
                         "schemes keep the deterministic phase B")
    ap.add_argument("--exchange", choices=["p2p", "host"], default="p2p",
                    help="tpcc partitions: p2p = the exchange inside the library over peer memory "
                         "(CC_FLAG_PART_P2P, no host step per round); host = cc_part_send/apply/finish "
                         "with torch.distributed all-to-alls (or device copies in --loopback)")
    ap.add_argument("--loopback", type=int, default=0,
                    help="tpcc: run G warehouse partitions as G dbs on this one GPU (a8 with a device-side exchange)")
    ap.add_argument("--cpu-seconds", type=float, default=10.0)
    ap.add_argument("--no-tpcc", action="store_true", help="skip the TPC-C block of the YCSB line")
    ap.add_argument("--no-index-binary", action="store_true", help="skip the binary-index pass")
    return ap.parse_args()


def dist_env():
    rank = int(os.environ.get("RANK", "0"))
    world = int(os.environ.get("WORLD_SIZE", "1"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    return rank, world, local


class Clocks:
    """nvidia-smi sampling during the timed region (B200_PROFILING.md clocks line)."""
    Q = ("index,clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,"
         "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
         "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")

    def __init__(self, index: int):
        self.index = index
        self.samples = []
        self.proc = None

    def start(self):
        try:
            self.proc = subprocess.Popen(["nvidia-smi", "-i", str(self.index), f"--query-gpu={self.Q}",
                                          "--format=csv,noheader,nounits", "-lms", "200"],
                                         stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            self.t = threading.Thread(target=self._read, daemon=True)
            self.t.start()
        except Exception:
            self.proc = None

    def _read(self):
        for line in self.proc.stdout:
            self.samples.append([x.strip() for x in line.split(",")])

    def stop(self):
        if not self.proc:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["nvidia-smi unavailable"]}
        time.sleep(0.25)
        self.proc.terminate()
        try:
            self.proc.wait(timeout=2)
        except Exception:
            self.proc.kill()
        sm = [float(s[1]) for s in self.samples if len(s) >= 9 and s[1].replace(".", "").isdigit()]
        mx = [float(s[2]) for s in self.samples if len(s) >= 9 and s[2].replace(".", "").isdigit()]
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        reasons = set()
        for s in self.samples:
            if len(s) >= 9:
                for n, v in zip(names, s[5:9]):
                    if v.lower() == "active":
                        reasons.add(n)
        sm.sort()
        return {"sm_mhz": sm[len(sm) // 2] if sm else None, "sm_max_mhz": max(mx) if mx else None,
                "reasons": sorted(reasons), "samples": len(self.samples)}


def algorithmic_bytes(n_txn, K, n_writes, scheme):
    """SURVEY.md §8(d) per-op bytes: read = 8 (CC word) + 128 (row) + 8 (out); a write
    adds 16 (two updated row words) + 8 (word release); MVCC adds 144 per write
    (history node); + 5 B per op of batch input (u32 key + u8 op)."""
    reads = n_txn * K - n_writes
    b = reads * 144 + n_writes * 168 + n_txn * K * 5
    if scheme == "mvcc":
        b += n_writes * 144
    return b


def atomics_per_batch(n_txn, K, n_writes, scheme):
    """SURVEY.md §8(d) 'Atomics per transaction' (committed attempts, one claim each):
    2PL acquire + release per op and a lock-point ticket; TO one CAS per op + one per
    write (pending bit) + ts; MVCC one per op + two per write + ts; Silo write lock +
    release + serialization ticket; TicToc the same (rts extensions only when needed:
    not counted); GPUTx the K-set completion counter; GaccO none (release stores and
    polls only: no L2-atomic ceiling)."""
    n, w = n_txn * K, n_writes
    a = {"tpl_nw": 2 * n + n_txn, "tpl_wd": 2 * n + n_txn, "to": n + w + n_txn,
         "mvcc": n + 2 * w + n_txn, "silo": 2 * w + n_txn, "tictoc": 2 * w + n_txn,
         "gputx": n_txn, "gacco": 0}[scheme]
    return a + (n_txn if a else 0)


def hot_record_counts(keys, ops, n_rows):
    """Accesses and writes to the most-accessed / most-written record of a batch (keys map
    to records one-to-one)."""
    import numpy as np
    k = keys.astype(np.int64).ravel()
    w = (ops.ravel() & 0x80) != 0
    acc = np.bincount(k, minlength=1)
    wr = np.bincount(k[w], minlength=1) if w.any() else np.zeros(1, np.int64)
    return int(acc.max()), int(wr.max())


def scheme_bounds(scheme, exec_ms, alg_bytes, atomics, acc_max, w_max, max_rank, ceil):
    """The three memory-system fractions of SURVEY.md §8(d) for one exec launch, and the
    one that binds (closest to its ceiling):
      gather        algorithmic bytes / time vs the measured random-128 B-line gather rate;
      l2_atomic     atomics / time vs measured distinct-address CAS/s (L2-resident);
      serialization (conflicting accesses on the hottest record) x measured hand-off /
                    time: GaccO serialises every access of an item,
                    GPUTx every K-set (max_rank + 1 of them), the other
                    schemes at least every write of the hot record."""
    t = exec_ms / 1e3
    out = {"gather_frac": alg_bytes / t / 1e9 / ceil["gather_gbs"] if ceil["gather_gbs"] > 0 else None,
           "atomic_frac": atomics / t / ceil["cas_l2_per_s"] if atomics and ceil["cas_l2_per_s"] > 0 else None}
    chain = acc_max if scheme == "gacco" else (max_rank + 1 if scheme == "gputx" else w_max)
    # the executor's waits poll with ld.acquire: the faster of the two measured idioms
    h = min(x for x in (ceil["handoff_row_ns"], ceil.get("handoff_acq_row_ns", -1), float("inf")) if x > 0)
    h = h if h != float("inf") else -1
    out["serial_chain"] = chain
    out["serial_bound_ms"] = chain * h / 1e6 if h > 0 else None
    out["serial_frac"] = chain * h / 1e9 / t if h > 0 else None
    fr = {k[:-5]: v for k, v in out.items() if k.endswith("_frac") and v is not None}
    out["binding"] = max(fr, key=fr.get) if fr else None
    return out


def load_peaks():
    try:
        return json.load(open(os.path.join(ROOT, "MEASURED_PEAKS.json")))
    except Exception:
        return None


def load_traffic():
    try:
        return json.load(open(os.path.join(ROOT, "profiles", "ncu_traffic.json")))
    except Exception:
        return None


# ------------------------------------------------------------------ CPU oracle legs
def oracle_replay_timed(args, seconds, max_batches=None):
    """The oracle as it stands (oracle/: plain C serial executor), one host core.
    Generates S0 (inputs) and batches with the oracle's own generator, then times only
    the serial replay loop.  Returns (txn/s, txns replayed, seconds, sample string)."""
    import numpy as np
    import inputs
    import oracle
    try:
        os.sched_setaffinity(0, {sorted(os.sched_getaffinity(0))[0]})
    except Exception:
        pass
    S = inputs.ycsb_rows(1, args.rows)
    T = inputs.zipf_thresholds(args.rows, args.theta)
    A = inputs.scramble_mult(args.rows)
    keys, ops = oracle.ycsb_gen(123, args.rows, args.batch, args.ops, args.write_frac, T, A)
    order = np.arange(args.batch, dtype=np.uint32)
    out = np.zeros(args.batch * args.ops, dtype=np.uint64)
    L = oracle.lib()
    done = 0
    t0 = time.perf_counter()
    n = 0
    while True:
        st = L.orc_ycsb_replay(oracle._ptr(S), args.rows, args.batch, args.ops, oracle._ptr(keys),
                               oracle._ptr(ops), oracle._ptr(order), args.batch, oracle._ptr(out))
        assert st == 0
        done += args.batch
        n += 1
        el = time.perf_counter() - t0
        if el >= seconds or (max_batches and n >= max_batches):
            break
    sample = (f"serial replay of {n} x {args.batch}-txn YCSB batches (K={args.ops}, theta={args.theta}, "
              f"W={args.write_frac}) over the {args.rows}-row table, 1 core")
    return done / el, done, el, sample


def run_reference(args, rank, world):
    if rank != 0:
        return
    # each step: serial replay of one step's worth of transactions (8 schemes x batch),
    # bounded so --steps K --warmup W finishes in minutes
    import numpy as np  # noqa: F401
    per_step = len(args.schemes.split(",")) * args.batch
    tps, done, el, sample = oracle_replay_timed(args, seconds=min(args.cpu_seconds, 30.0))
    ms_per_step = per_step / tps * 1e3
    line = {
        "metric": METRIC, "value": tps, "unit": "txn/s", "n_gpus": args.gpus, "steps": args.steps,
        "warmup": args.warmup, "ms_per_step": ms_per_step, "higher_is_better": True, "scaling": "weak",
        "vs_baseline": None, "dtype": "u64", "data": "synthetic", "impl": "reference",
        "config": config_of(args, world),
        "cpu_baseline": {"value": tps, "unit": "txn/s", "cores": 1, "kind": "oracle", "sample": sample},
        "e2e": {"value": tps, "unit": "txn/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line), flush=True)


# YCSB tile mode: warps per SM (one block per SM) with the lowest exec time at the bench
# workload (configs[1], theta 0.6, 2 seeds).  Round 2: one transaction per warp (32-lane
# tiles, lanes 16-31 idle for K = 16) beats two 16-lane tiles per warp for every scheme
# (sum of the best exec times 3.99 -> 3.60 ms, GPUTx 0.74 -> 0.66, GaccO 0.78 -> 0.70):
# a tile that waits or paces no longer shares its warp's issue slots and sleeps with
# another transaction (profiles/r02_tune_lanes32.jsonl vs r02_tune_lanes16.jsonl).
# Round 1 (16 lanes): profiles/r01_tune_bs.jsonl.
# GPUTx re-tuned after its reads moved before the gate (more transactions in flight now
# pay: 0.57 ms at 8 warps -> 0.49 at 20, profiles/r02_tune_gputx_early.log).
TUNED_BS = {"tpl_nw": 32, "tpl_wd": 32, "to": 16, "mvcc": 24, "silo": 24, "tictoc": 24, "gputx": 20, "gacco": 8}
TUNED_BS_16 = {"tpl_nw": 20, "tpl_wd": 20, "to": 8, "mvcc": 20, "silo": 12, "tictoc": 16, "gputx": 8, "gacco": 24}


# TPC-C tile mode (32 lanes), configs[4] shape on one GPU (512 warehouses, 64K batch;
# profiles/r01_tpcc_launch.txt): the full-occupancy grid is best for every scheme but
# GaccO, whose hand-off chains prefer 16 warps on one block per SM (49 -> 55 M txn/s).
# (At 64 warehouses one block of 4-8 warps per SM wins instead: contention decides.)
TUNED_TPCC = {"gacco": (16, True)}


# Loopback partitions share one GPU: each partition's executor takes one block per SM so
# the G partitions run side by side (warps per SM as at 64 warehouses; 4 partitions x
# 128 warehouses: 9.0 -> 45 M txn/s against full-occupancy grids that serialise them).
LOOPBACK_TPCC_BS = {"tpl_nw": 8, "tpl_wd": 8, "to": 8, "mvcc": 8, "silo": 4, "tictoc": 8, "gputx": 8, "gacco": 4}


def tpcc_launch(args, scheme, n_sms, loopback=False):
    if loopback and args.launch == "tuned":
        return {"bs": LOOPBACK_TPCC_BS[scheme], "grid": n_sms}
    bs, one_block = TUNED_TPCC.get(scheme, (8, False)) if args.launch == "tuned" else (8, False)
    return {"bs": bs, "grid": n_sms if one_block else 0}


def launch_of(args, scheme, n_sms):
    if args.launch == "tuned" and args.lanes > 1 and args.wd == 0:
        return {"wd": 0, "bs": (TUNED_BS if args.lanes == 32 else TUNED_BS_16)[scheme], "grid": n_sms}
    return {"wd": args.wd, "bs": args.bs, "grid": 0}


def config_of(args, world):
    return {"workload": "ycsb_configs1_10Mrows_64Kx16", "rows": args.rows, "batch": args.batch,
            "ops_per_txn": args.ops, "theta": args.theta, "write_frac": args.write_frac,
            "schemes": args.schemes.split(","), "wd": args.wd, "bs": args.bs, "lanes_per_txn": args.lanes, "index": args.index,
            "launch": ({s: launch_of(args, s, 148)["bs"] for s in args.schemes.split(",")} | {"grid": "1 block/SM"})
            if args.launch == "tuned" and args.lanes > 1 and args.wd == 0 else "fixed (wd, bs), full-occupancy grid",
            "prep": "pipelined (cc_prepare on a second stream)" if args.pipeline else "inline",
            "parallelism": f"replicas{world}", "l2": "inputs larger than L2 (1.34 GB table, 168 MB CC words)"}


# ------------------------------------------------------------------ GPU arm
def run_ours(args, rank, world, local):
    import numpy as np
    import torch
    import torch.distributed as dist

    import inputs
    from paper_2406_10158_b200.api import DB, Result
    from paper_2406_10158_b200.gcctb import CC_FLAG_TIMING

    torch.cuda.set_device(local)
    if world > 1:
        dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    dev = torch.device("cuda", local)
    schemes = args.schemes.split(",")
    db = DB(local)
    db.load_ycsb(args.rows, 1 + rank)
    T = torch.from_numpy(inputs.zipf_thresholds(args.rows, args.theta).view(np.int64)).to(dev)
    A = inputs.scramble_mult(args.rows)
    res = {s: Result.alloc(args.batch, args.ops, dev, stream=db.stream) for s in schemes}
    stream = db.stream   # every library launch goes to this stream; events are recorded on it
    LA = {s: launch_of(args, s, db.num_sms) for s in schemes}

    from paper_2406_10158_b200.gcctb import CC_FLAG_INDEX_BINARY, CC_FLAG_INDEX_TREE
    xflags = {"dense": 0, "tree": CC_FLAG_INDEX_TREE, "binary": CC_FLAG_INDEX_BINARY,
              "eytz": 0x1000}[args.index]   # CC_FLAG_INDEX_EYTZ

    def prepare(b):
        """f-4: GPUTx / GaccO a3 on the prep stream, overlapping the other schemes' execution."""
        if args.pipeline:
            for s in schemes:
                db.prepare(b, s, xflags)

    scheme_ev = []   # timed steps: an event after each scheme's submit (per-step attribution)
    ev_pool = [[torch.cuda.Event(enable_timing=True) for _ in range(len(schemes) + 1)] for _ in range(args.steps)]

    def step(i, timing=False, keep=False):
        """One step: a1 generation, f-4 preparation, then a2-a7 under every scheme.  The
        batch is released after its last submit (its buffers return to the pool and the next
        step's generation reuses them in stream order; cc_batch_free never blocks)."""
        b = db.gen_ycsb(args.batch, args.ops, args.write_frac, 1000 * (rank + 1) + i, T, A)
        prepare(b)
        sev = timing and args.scheme_events
        evs = ev_pool[len(scheme_ev)] if sev else None   # created before the timed region
        for k, s in enumerate(schemes):
            if sev:
                evs[k].record(stream)
            db.submit(b, s, **LA[s], flags=xflags | (CC_FLAG_TIMING if timing and args.phase_events else 0),
                      result=res[s], watchdog_s=60, lanes=args.lanes)
        db.join()   # the last submit's a2 zeroing (reset stream) belongs to this step
        if sev:
            evs[-1].record(stream)
            scheme_ev.append(evs)
        if keep:
            return b
        b.free()
        return None

    def barrier():
        torch.cuda.synchronize(dev)
        if world > 1:
            dist.barrier()
        torch.cuda.synchronize(dev)

    # nvidia-smi starts (and initialises NVML, which can hold driver locks for tens of ms)
    # before the warm-up, not inside the timed region; it samples through both
    clocks = Clocks(local)
    clocks.start()
    time.sleep(0.5)
    for i in range(args.warmup):
        step(i)
        db.sync()
    # the pool holds two prepared buffer sets (the steady loop recycles one; the last
    # step keeps its batch): no cudaMalloc / cudaFree while timing -- asserted below
    pre = [db.gen_ycsb(args.batch, args.ops, args.write_frac, 0, T, A) for _ in range(2)]
    for b in pre:
        prepare(b)
    db.sync()
    torch.cuda.synchronize(dev)
    for b in pre:
        b.free()
    barrier()
    # ---- timed region
    db.timing(reset=True)
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    ev = [torch.cuda.Event(enable_timing=True) for _ in range(args.steps)]
    batches = []
    barrier()
    mem0 = db.mem_stats()
    e0.record(stream)
    for i in range(args.steps):
        b = step(args.warmup + i, timing=True, keep=i == args.steps - 1)
        if b is not None:
            batches.append(b)
        ev[i].record(stream)
    e1.record(stream)
    mem1 = db.mem_stats()
    barrier()
    clk = clocks.stop()
    st = db.sync()
    allocs_timed = (mem1[0] - mem0[0], mem1[1] - mem0[1])
    assert allocs_timed == (0, 0), f"device allocations inside the timed region: {allocs_timed}"
    ms = e0.elapsed_time(e1)
    step_ms = [e0.elapsed_time(ev[0])] + [ev[i - 1].elapsed_time(ev[i]) for i in range(1, args.steps)]
    step_scheme_ms = {s: [round(evs[k].elapsed_time(evs[k + 1]), 4) for evs in scheme_ev]
                      for k, s in enumerate(schemes)}
    phase_ms, n_sub = db.timing(reset=True)
    # per-scheme stats from the last step (committed + aborts), checked complete
    per = {}
    last = batches[-1]
    for s in schemes:
        h = res[s].stats.cpu().numpy().view(np.uint64)   # after db.sync()
        per[s] = {"commits": int(h[0]), "aborts": int(h[1]), "abort_rate": float(h[1]) / max(1, int(h[0]))}
        assert int(h[0]) == args.batch, (s, int(h[0]))
    keys, ops = last.export_ycsb()
    n_writes = int(((ops & 0x80) != 0).sum())
    for b in batches:
        b.free()
    # per-scheme exec timing (one extra timed pass per scheme on a fresh batch, untimed overall)
    b = db.gen_ycsb(args.batch, args.ops, args.write_frac, 999_999 + rank, T, A)
    bk, bo = b.export_ycsb()
    nw2 = int(((bo & 0x80) != 0).sum())
    acc_max, w_max = hot_record_counts(bk, bo, args.rows)
    ceil = db.roofline_probe() if rank == 0 and not args.no_ceilings else None   # untimed ceilings
    exec_ms_total, alg_bytes_total = 0.0, 0
    for s in schemes:
        db.timing(reset=True)
        db.submit(b, s, **LA[s], flags=xflags | CC_FLAG_TIMING, result=res[s], watchdog_s=60,
                  lanes=args.lanes)
        db.sync()
        pm, _ = db.timing(reset=True)
        per[s]["exec_ms"] = pm[2]
        per[s]["submit_ms"] = pm[4]
        per[s]["txn_s"] = args.batch / (pm[4] / 1e3)
        ab = algorithmic_bytes(args.batch, args.ops, nw2, s)
        per[s]["exec_GBps"] = ab / (pm[2] / 1e3) / 1e9
        if ceil is not None:
            max_rank = int(res[s].stats.cpu().numpy().view(np.uint64)[4])
            per[s]["bounds"] = scheme_bounds(s, pm[2], ab, atomics_per_batch(args.batch, args.ops, nw2, s),
                                             acc_max, w_max, max_rank, ceil)
        exec_ms_total += pm[2]
        alg_bytes_total += ab
    # ---- e2e through the public API with host buffers
    # the paper's index (binary search over the sorted keys) beside the
    # direct-addressed headline: same batch, same launches, identical results
    idx_bin = None
    if args.index == "dense" and not args.no_index_binary:
        idx_bin = index_pass(args, db, b, schemes, LA, res, CC_FLAG_INDEX_BINARY)
    e2e = run_e2e(args, db, bk, bo, schemes, res, dev, stream, barrier, world, xflags)
    b.free()

    ms_t = torch.tensor([ms], device=dev, dtype=torch.float64)
    if world > 1:
        dist.all_reduce(ms_t, op=dist.ReduceOp.MAX)
    ms_max = float(ms_t.item())
    total_commits = args.steps * args.batch * len(schemes) * world
    value = total_commits / (ms_max / 1e3)
    if rank == 0:
        peaks = load_peaks()
        peak = peaks["hbm_gbs"] if peaks else 6650.0
        achieved = alg_bytes_total / (exec_ms_total / 1e3) / 1e9
        traffic = None
        for tr in load_traffic() or []:   # ncu --set full DRAM bytes per launch, this exact config
            if tr.get("config") == config_key(args):
                traffic = tr.get("dram_bytes_per_launch")
        # exec share of the step: the timed submits' own phase events when on, else the
        # per-scheme pass's exec times against the step time
        exec_share = (phase_ms[2] / phase_ms[4]) if phase_ms[4] else exec_ms_total / (ms_max / args.steps)
        line = {
            "metric": METRIC, "value": value, "unit": "txn/s", "n_gpus": world, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": ms_max / args.steps, "higher_is_better": True,
            "scaling": "weak", "vs_baseline": None, "dtype": "u64", "data": "synthetic",
            "config": config_of(args, world),
            "abort_rate": sum(p["aborts"] for p in per.values()) / max(1, sum(p["commits"] for p in per.values())),
            "per_scheme": per,
            "step_ms": step_ms,
            "step_scheme_ms": step_scheme_ms,
            "clocks": clk,
            "e2e": e2e,
            "gpu_launches": launches_per_step(schemes, args.pipeline) * args.steps,
            "device_allocs_in_timed_region": {"cudaMalloc": allocs_timed[0], "cudaFree": allocs_timed[1]},
            "step_ms_max_over_median": max(step_ms) / sorted(step_ms)[len(step_ms) // 2],
            "roofline": {"bound": "hbm", "achieved": achieved, "peak": peak, "unit": "GB/s",
                         "frac": achieved / peak, "traffic": traffic,
                         "kernel": "exec_kernel (a4-a6), all schemes",
                         "peak_source": "MEASURED_PEAKS.json hbm_gbs (measured)" if peaks else "fallback 6.65 TB/s",
                         "exec_share_of_step": exec_share,
                         # the ceilings a random-access, atomic, hand-off
                         # bound path actually meets (cc_roofline_probe), per scheme in
                         # per_scheme[s]["bounds"]
                         "ceilings": ceil,
                         "frac_gather": achieved / ceil["gather_gbs"] if ceil and ceil["gather_gbs"] > 0 else None,
                         "hot_record": {"accesses": acc_max, "writes": w_max},
                         "binding": {s: per[s].get("bounds", {}).get("binding") for s in schemes}},
        }
        if not args.no_cpu_baseline and world >= 1:
            tps, done, el, sample = oracle_replay_timed(args, args.cpu_seconds)
            line["cpu_baseline"] = {"value": tps, "unit": "txn/s", "cores": 1, "kind": "oracle",
                                    "sample": sample}
        if idx_bin is not None:
            line["index_binary"] = idx_bin
    db.close()
    if rank == 0 and not args.no_tpcc:
        line["tpcc"] = tpcc_block(args, local, schemes)
    if world > 1 and not args.no_tpcc:
        # the path that shards: configs[4], 512 warehouses partitioned over the ranks, the
        # exchange inside the library over NVLink peer memory (every rank takes part)
        part = tpcc_partitioned_block(args, rank, world, local, schemes)
        if rank == 0:
            line["tpcc_partitioned"] = part
    if rank == 0:
        print(json.dumps(line), flush=True)
    if world > 1:
        dist.destroy_process_group()


def tpcc_partitioned_block(args, rank, world, local, schemes, steps=3):
    """configs[4] on `world` GPUs: W = 512 warehouses in contiguous ranges, 65,536 home
    transactions per rank per step, every scheme per step with the deterministic phase B
    exchanged over peer memory (CC_FLAG_PART_P2P: no host step, no collective per round).
    Device-timed on each rank's db stream, max over ranks; value = all ranks' commits / time."""
    import torch
    import torch.distributed as dist

    from paper_2406_10158_b200.api import DB, Result
    from paper_2406_10158_b200.partition import p2p_round, p2p_setup
    dev = torch.device("cuda", local)
    W, n = args.warehouses, args.tpcc_batch
    wpr = W // world
    out = {"workload": "tpcc_configs4_partitioned", "warehouses": W, "batch_per_rank": n, "ranks": world,
           "exchange": "in-library over NVLink peer memory (CC_FLAG_PART_P2P)"}
    db, err = None, None
    try:
        db = DB(local, rank=rank, world=world)
        db.load_tpcc(W, 1, n, w_first=rank * wpr, w_count=wpr)
        p2p_setup(db)
    except Exception as e:
        err = f"{type(e).__name__}: {e}"
    ok = torch.tensor([0 if err else 1], device=dev, dtype=torch.int32)
    dist.all_reduce(ok, op=dist.ReduceOp.MIN)   # every rank connected, or nobody runs
    if int(ok.item()) == 0:
        out["error"] = err or "another rank failed to connect its exchange window"
        if db is not None:
            db.close()
        return out
    ms_local = -1.0
    try:
        res = {s: Result.alloc(n, 18, dev, stream=db.stream, out_words=48) for s in schemes}

        def step(i):
            b = db.gen_tpcc(n, 7919 * (rank + 1) + i, args.tpcc_mix, w_lo=rank * wpr, w_hi=(rank + 1) * wpr)
            for s in schemes:
                p2p_round(db, b, s, result=res[s], **tpcc_launch(args, s, db.num_sms), lanes=32, watchdog_s=60)
            b.free()

        step(0)
        db.sync()
        torch.cuda.synchronize(dev)
        dist.barrier()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(db.stream)
        for i in range(steps):
            step(1 + i)
        e1.record(db.stream)
        db.sync()
        ms_local = e0.elapsed_time(e1)
    except Exception as e:   # reported, never fatal for the headline line
        out["error"] = f"{type(e).__name__}: {e}"
    # every rank reaches these collectives, also after an error (no rank waits forever)
    ok = torch.tensor([0 if "error" in out else 1], device=dev, dtype=torch.int32)
    dist.all_reduce(ok, op=dist.ReduceOp.MIN)
    ms = torch.tensor([ms_local], device=dev, dtype=torch.float64)
    dist.all_reduce(ms, op=dist.ReduceOp.MAX)
    if int(ok.item()) == 1:
        ms = float(ms.item())
        out.update({"value": steps * n * len(schemes) * world / (ms / 1e3), "unit": "txn/s",
                    "ms_per_step": ms / steps, "steps": steps})
    elif "error" not in out:
        out["error"] = "another rank failed"
    try:
        db.close()
    except Exception:
        pass
    return out


def index_pass(args, db, b, schemes, LA, res, flag):
    """One timed submit per scheme of batch b with an index flag (untimed overall): the
    per-scheme submit / exec times and the aggregate committed txn/s over the 8 submits."""
    from paper_2406_10158_b200.gcctb import CC_FLAG_TIMING
    out = {"index": "binary (PAPER.md:344)", "per_scheme": {}}
    tot = 0.0
    for s in schemes:
        db.submit(b, s, **LA[s], flags=flag, result=res[s], watchdog_s=60, lanes=args.lanes)   # warm
        db.sync()
        db.timing(reset=True)
        db.submit(b, s, **LA[s], flags=flag | CC_FLAG_TIMING, result=res[s], watchdog_s=60, lanes=args.lanes)
        db.sync()
        pm, _ = db.timing(reset=True)
        out["per_scheme"][s] = {"submit_ms": pm[4], "exec_ms": pm[2], "txn_s": args.batch / (pm[4] / 1e3)}
        tot += pm[4]
    out["value"] = len(schemes) * args.batch / (tot / 1e3)
    out["unit"] = "txn/s"
    return out


# TPC-C launches per configuration (tile mode, a warp per transaction; profiles/r01_tpcc_launch.txt):
# (warps per block, blocks: 0 = full-occupancy grid, else blocks = SMs).  One warehouse: one
# warp per SM (the hot W row's hand-off chain decides, fewer resident transactions collide
# less); 64 warehouses: 8 warps per SM; 512 warehouses: the full grid, GaccO 16 warps per SM.
TPCC_CONFIGS = [
    {"name": "configs2_1wh_16K_50:50", "W": 1, "n": 16384, "mix": 5000, "launch": {"*": (1, True)}},
    {"name": "configs3_64wh_64K_45:43", "W": 64, "n": 65536, "mix": 5114,
     "launch": {"*": (8, True), "to": (4, True), "tpl_wd": (16, True), "gacco": (16, True)}, "meta_pad": True},
    {"name": "configs4_shape_512wh_64K_45:43_1gpu", "W": 512, "n": 65536, "mix": 5114,
     "launch": {"*": (4, False), "to": (8, False), "tictoc": (8, False), "gputx": (16, False)}},
]


def tpcc_alg_bytes(tx):
    """SURVEY.md §8(d) algorithmic bytes of a TPC-C batch: NewOrder 320 B of header rows
    (W, D, C reads, D update, O / NO slots) + 258 B per line (I 82 + S 112 RMW + OL 64);
    Payment 600 B + 1,000 B for a BC customer's c_data rewrite (10 % of customers, counted
    at that expectation: +100 B); 16 B per CC-managed access (word acquire + release);
    160 B of descriptor per transaction."""
    import numpy as np
    t = tx.reshape(-1, 40)
    no = t[:, 0] == 0
    lines = int(t[no, 8].sum())
    n_no, n_pay = int(no.sum()), int((~no).sum())
    b = n_no * 320 + lines * 258 + n_pay * 700
    b += 16 * (3 * n_no + lines + 3 * n_pay) + 160 * len(t)
    return b


def tpcc_block(args, local, schemes):
    """configs[2], configs[3] and the configs[4] shape on one GPU: per scheme, 3 submits of
    fresh seeded batches back to back after one warm-up submit (a2-a7 and the background
    a2 zeroing, CUDA events on the db stream around all three, cc_join before the closing
    event); committed txn/s, abort rate, mean exec ms and the exec kernel's algorithmic
    GB/s against the HBM peak.  Launches per config from profiles/r02_tpcc_launch_tune.jsonl."""
    import numpy as np
    import torch

    from paper_2406_10158_b200.api import DB, Result
    from paper_2406_10158_b200.gcctb import CC_FLAG_META_PAD, CC_FLAG_TIMING
    dev = torch.device("cuda", local)
    peaks = load_peaks()
    peak = peaks["hbm_gbs"] if peaks else 6650.0
    out = {}
    for cfg in TPCC_CONFIGS:
        db = DB(local)
        db.load_tpcc(cfg["W"], 1, cfg["n"])
        res = [Result.alloc(cfg["n"], 18, dev, stream=db.stream, out_words=48) for _ in range(3)]
        per = {}
        tot_ms, tot_commits = 0.0, 0
        # one control word per 32 B sector where it measured faster (profiles/r02_probe_meta_pad.jsonl;
        # at 512 warehouses the padded set's background zeroing -- 4x the words of ~70 M
        # records -- costs more than the padding saves: 63.0 vs 73.9 M txn/s, r02_tpcc_meta_pad_b2b.log)
        flags = CC_FLAG_TIMING | (CC_FLAG_META_PAD if cfg.get("meta_pad") else 0)
        for s in schemes:
            bs, per_sm = cfg["launch"].get(s, cfg["launch"]["*"])
            la = {"bs": bs, "grid": db.num_sms if per_sm else 0}
            # a warm-up submit, then NT submits of fresh batches back to back (as the YCSB
            # step runs them: each submit's background a2 zeroing overlaps the next one;
            # cc_join before the closing event makes the last one count too)
            NT = 3
            bt = [db.gen_tpcc(cfg["n"], 101 + r, cfg["mix"]) for r in range(NT + 1)]
            alg = tpcc_alg_bytes(bt[-1].export_tpcc())
            db.submit(bt[0], s, **la, lanes=32, flags=flags, result=res[0], watchdog_s=120)
            st = db.sync()
            assert st.commits == cfg["n"], (cfg["name"], s, st.commits)
            db.timing(reset=True)
            ea, eb = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            ea.record(db.stream)
            for r in range(NT):
                db.submit(bt[r + 1], s, **la, lanes=32, flags=flags, result=res[r], watchdog_s=120)
            db.join()
            eb.record(db.stream)
            db.sync()
            pm, n_sub = db.timing(reset=True)
            tot = ea.elapsed_time(eb)
            ab = cm = 0
            for r in range(NT):
                h = res[r].stats.cpu().numpy().view(np.uint64)
                assert int(h[0]) == cfg["n"], (cfg["name"], s, int(h[0]))
                cm += int(h[0])
                ab += int(h[1])
            for b in bt:
                b.free()
            sub = [tot / NT] * 3
            exe = [pm[2] / max(1, n_sub)] * 3
            gbs = alg / (exe[1] / 1e3) / 1e9
            per[s] = {"txn_s": cfg["n"] / (sub[1] / 1e3), "abort_rate": ab / max(1, cm), "submit_ms": sub[1],
                      "exec_ms": exe[1], "launch": la, "exec_alg_GBps": gbs, "exec_hbm_frac": gbs / peak}
            tot_ms += sub[1]
            tot_commits += cfg["n"]
        out[cfg["name"]] = {"value": tot_commits / (tot_ms / 1e3), "unit": "txn/s", "warehouses": cfg["W"],
                            "batch": cfg["n"], "neworder_permyriad": cfg["mix"], "lanes_per_txn": 32,
                            "meta_pad": bool(cfg.get("meta_pad")),
                            "per_scheme": per}
        db.close()
        del res
        torch.cuda.empty_cache()
    return out


def config_key(args):
    return (f"ycsb rows={args.rows} batch={args.batch} K={args.ops} theta={args.theta} W={args.write_frac} "
            f"wd={args.wd} bs={args.bs} lanes={args.lanes} index={args.index}"
            + (" launch=tuned" if args.launch == "tuned" and args.lanes > 1 and args.wd == 0 else ""))


def launches_per_step(schemes, pipelined=False, a3_passes=3):
    """Kernel launches libgcctb issues per step (memsets excluded -- the CC words are zeroed
    by a kernel on the reset stream, counted: 1 per non-deterministic scheme): 1 generator;
    per scheme a2 = one prologue kernel (ring, retry queues, control block,
    per-transaction results, batch error), the executor (1), a7 = commit positions + one
    copy-out kernel that also writes the stats: 2PL 0 (the dense ticket is the position);
    TO / MVCC / Silo bitmap 5; TicToc ticket inverse + gather + one cooperative sort +
    commit_pos = 4; GPUTx / GaccO iota + commit_pos 2 (+ 1 error merge when prepared).  a3
    (GaccO: gather, a3_passes radix passes x 4 (the access table has more than 128 tiles:
    the multi-kernel sort), marks, 3-kernel max-scan, positions; GPUTx + fill, rank pass,
    keys, one cooperative rank sort, copy, bounds, count) inline or on the prep stream when
    pipelined."""
    a3 = 1 + 4 * a3_passes + 1 + 3 + 1
    n = 1
    for s in schemes:
        n += 1 + 1 + 1
        if s in ("tpl_nw", "tpl_wd"):
            n += 1
        elif s in ("to", "mvcc", "silo"):
            n += 5 + 1
        elif s == "tictoc":
            n += 4 + 1
        else:
            n += 2 + (1 if pipelined else 0)
            n += a3 + (0 if s == "gacco" else 1 + 1 + 1 + 1 + 3)
    return n


def run_e2e(args, db, keys, ops, schemes, res, dev, stream, barrier, world, xflags=0):
    """Same metric through the public C ABI with HOST buffers at both ends, as a serving
    loop would run it: every step's batch is imported from pinned host memory
    (cc_batch_import_ycsb with CC_SRC_HOST_ASYNC: the copy of step i+1 overlaps step i) and
    every submit writes its results -- commit flags, restarts, order keys, commit positions,
    read outputs, stats -- into pinned HOST buffers (cc_result in host memory: the library
    stages them on the device and copies them out on its copy stream, overlapping the next
    submit).  Host result sets are double-buffered per step, so the host never waits inside
    the loop; the timed region ends when the last copy has landed (cc_sync)."""
    import torch
    from paper_2406_10158_b200.api import Result
    pk = [torch.from_numpy(keys).pin_memory() for _ in range(2)]   # double-buffered inputs
    po = [torch.from_numpy(ops).pin_memory() for _ in range(2)]
    H = [{s: Result.alloc_host(args.batch, args.ops) for s in schemes} for _ in range(2)]
    n_steps = max(2, args.steps)

    def run(n):
        b = db.import_ycsb(pk[0], po[0], args.ops, async_host=True)
        for i in range(n):
            nxt = db.import_ycsb(pk[(i + 1) % 2], po[(i + 1) % 2], args.ops, async_host=True) if i + 1 < n else None
            if args.pipeline:
                for s in schemes:
                    db.prepare(b, s, xflags)
            for s in schemes:
                db.submit(b, s, **launch_of(args, s, db.num_sms), result=H[i % 2][s], watchdog_s=60,
                          lanes=args.lanes, flags=xflags)
            b.free()   # asynchronous: the buffers return to the pool in stream order
            b = nxt
        db.sync()      # the last copy-out has landed in host memory

    run(2)
    barrier()
    t0 = time.perf_counter()
    run(n_steps)
    barrier()
    el = time.perf_counter() - t0
    last = H[(n_steps - 1) % 2][schemes[-1]]
    assert int(last.committed.sum()) == args.batch   # the host buffers hold the last step's results
    if world > 1:
        import torch.distributed as dist
        t = torch.tensor([el], device=dev, dtype=torch.float64)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        el = float(t.item())
    h2d = keys.nbytes + ops.nbytes
    d2h_bytes = len(schemes) * (args.batch * (1 + 4 + 8 + 8 + 4) + args.batch * args.ops * 8 + 8 * 16)
    return {"value": n_steps * args.batch * len(schemes) * world / el, "unit": "txn/s",
            "h2d_bytes_per_step": h2d, "d2h_bytes_per_step": d2h_bytes, "steps": n_steps,
            "note": "host wall clock around n steps through the C ABI with host buffers: async pinned H2D import of "
                    "each step's batch (in place of the on-device a1 generation the device-timed value includes) + "
                    "submit x schemes with cc_result in pinned host memory (library copy-out on its copy stream); "
                    "no host wait inside the loop"}


def run_tpcc_loopback(args, local):
    """configs[4] with G partitions held by G dbs on one GPU: the same phase A / pack /
    apply / finish kernels as the multi-GPU path, the all-to-alls being device copies."""
    import numpy as np
    import torch

    from paper_2406_10158_b200.api import DB, Result
    from paper_2406_10158_b200.partition import loopback_p2p, loopback_round, loopback_round_2pc

    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    G = args.loopback
    schemes = args.schemes.split(",")
    W, n = args.warehouses, args.tpcc_batch
    wpr = W // G
    dbs = []
    for r in range(G):
        db = DB(local, rank=r, world=G)
        db.load_tpcc(W, 1, n, w_first=r * wpr, w_count=wpr)
        dbs.append(db)
    res = {s: [Result.alloc(n, 18, dev, stream=db.stream, out_words=48) for db in dbs] for s in schemes}
    if args.exchange == "p2p":
        DB.part_connect_local(dbs)

    def step(i):
        bs = [db.gen_tpcc(n, 7919 * (r + 1) + i, args.tpcc_mix, w_lo=r * wpr, w_hi=(r + 1) * wpr)
              for r, db in enumerate(dbs)]
        for s in schemes:
            la = tpcc_launch(args, s, dbs[0].num_sms, True)
            if args.two_pc and s not in ("gputx", "gacco"):
                loopback_round_2pc(dbs, bs, s, results=res[s], **la, lanes=32, watchdog_s=60)
            elif args.exchange == "p2p":
                loopback_p2p(dbs, bs, s, results=res[s], **la, lanes=32, watchdog_s=60)
            else:
                loopback_round(dbs, bs, s, results=res[s], **la, lanes=32, watchdog_s=60)
        return bs

    clocks = Clocks(local)   # before the warm-up: NVML start-up stays out of the timed region
    clocks.start()
    time.sleep(0.5)
    for i in range(args.warmup):
        for b in step(i):
            b.free()
    for db in dbs:
        db.sync()
    torch.cuda.synchronize(dev)
    t0 = time.perf_counter()
    keep = [step(args.warmup + i) for i in range(args.steps)]
    for db in dbs:
        db.sync()
    torch.cuda.synchronize(dev)
    ms = (time.perf_counter() - t0) * 1e3   # G streams + host-driven exchange: host clock after full sync
    clk = clocks.stop()
    per = {}
    for s in schemes:
        c = a = 0
        for r in res[s]:
            h = r.stats.cpu().numpy().view(np.uint64)
            c += int(h[0])
            a += int(h[1])
        per[s] = {"commits": c, "aborts": a, "abort_rate": a / max(1, c)}
    for bs in keep:
        for b in bs:
            b.free()
    value = args.steps * n * G * len(schemes) / (ms / 1e3)
    print(json.dumps({
        "metric": METRIC, "value": value, "unit": "txn/s", "n_gpus": 1, "steps": args.steps, "warmup": args.warmup,
        "ms_per_step": ms / args.steps, "higher_is_better": True, "scaling": "weak", "vs_baseline": None,
        "dtype": "u64", "data": "synthetic",
        "config": {"workload": "tpcc_configs4_partitioned_loopback", "warehouses": W, "partitions": G,
                   "batch_per_partition": n, "neworder_permyriad": args.tpcc_mix, "schemes": schemes,
                   "lanes_per_txn": 32, "parallelism": f"{G} warehouse partitions on 1 GPU, device-side exchange",
                   "launch": {s: tpcc_launch(args, s, 148, True) for s in schemes} if args.launch == "tuned"
                   else "bs 8, full-occupancy grid",
                   "phase_b": "2PC rounds for the six non-deterministic schemes (f-2), deterministic for GPUTx/GaccO" if args.two_pc else "deterministic",
                   "exchange": "in-library over device memory (CC_FLAG_PART_P2P)" if args.exchange == "p2p" and not args.two_pc
                   else "host-orchestrated device copies",
                   "timing": "host clock around fully synchronised steps (G streams)"},
        "per_scheme": per, "clocks": clk}), flush=True)
    for db in dbs:
        db.close()


def run_tpcc(args, rank, world, local):
    """configs[4]: TPC-C with W warehouses partitioned by contiguous ranges over the
    ranks; each rank runs its own batch of home transactions; cross-partition
    transactions go through phase B (two NCCL all-to-alls per step)."""
    import numpy as np
    import torch
    import torch.distributed as dist

    from paper_2406_10158_b200.api import DB, Result
    from paper_2406_10158_b200.gcctb import CC_FLAG_TIMING
    from paper_2406_10158_b200.partition import dist_round, dist_round_2pc, p2p_round, p2p_setup

    torch.cuda.set_device(local)
    if world > 1:
        dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    dev = torch.device("cuda", local)
    schemes = args.schemes.split(",")
    W = args.warehouses
    wpr = W // world
    n = args.tpcc_batch
    db = DB(local, rank=rank, world=world)
    db.load_tpcc(W, 1, n, w_first=rank * wpr, w_count=wpr)
    res = {s: Result.alloc(n, 18, dev, stream=db.stream, out_words=48) for s in schemes}
    p2p = world > 1 and args.exchange == "p2p"
    if p2p:
        p2p_setup(db)   # windows mapped across the GPUs (CUDA IPC over NVLink), handles gathered once

    def step(i):
        b = db.gen_tpcc(n, 7919 * (rank + 1) + i, args.tpcc_mix, w_lo=rank * wpr, w_hi=(rank + 1) * wpr)
        for s in schemes:
            if p2p and not (args.two_pc and s not in ("gputx", "gacco")):
                p2p_round(db, b, s, result=res[s], **tpcc_launch(args, s, db.num_sms), lanes=32, watchdog_s=60)
            elif world > 1 and args.two_pc and s not in ("gputx", "gacco"):
                dist_round_2pc(db, b, s, result=res[s], **tpcc_launch(args, s, db.num_sms), lanes=32, watchdog_s=60)
            elif world > 1:
                dist_round(db, b, s, result=res[s], **tpcc_launch(args, s, db.num_sms), lanes=32, watchdog_s=60)
            else:
                db.submit(b, s, **tpcc_launch(args, s, db.num_sms), lanes=32, result=res[s], watchdog_s=60)
        return b

    def barrier():
        torch.cuda.synchronize(dev)
        if world > 1:
            dist.barrier()
        torch.cuda.synchronize(dev)

    clocks = Clocks(local)   # before the warm-up: NVML start-up stays out of the timed region
    clocks.start()
    time.sleep(0.5)
    for i in range(args.warmup):
        bb = step(i)
        db.sync()
        bb.free()
    barrier()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    bs_ = []
    barrier()
    e0.record(db.stream)
    for i in range(args.steps):
        bs_.append(step(args.warmup + i))
    e1.record(db.stream)
    barrier()
    clk = clocks.stop()
    db.sync()
    ms = e0.elapsed_time(e1)
    per = {}
    for s in schemes:
        h = res[s].stats.cpu().numpy().view(np.uint64)
        per[s] = {"commits": int(h[0]), "aborts": int(h[1]), "abort_rate": float(h[1]) / max(1, int(h[0]))}
    for bb in bs_:
        bb.free()
    t = torch.tensor([ms], device=dev, dtype=torch.float64)
    if world > 1:
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
    ms = float(t.item())
    value = args.steps * n * len(schemes) * world / (ms / 1e3)
    if rank == 0:
        print(json.dumps({
            "metric": METRIC, "value": value, "unit": "txn/s", "n_gpus": world, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": ms / args.steps, "higher_is_better": True,
            "scaling": "weak", "vs_baseline": None, "dtype": "u64", "data": "synthetic",
            "config": {"workload": "tpcc_configs4_partitioned", "warehouses": W, "batch_per_rank": n,
                       "neworder_permyriad": args.tpcc_mix, "schemes": schemes, "lanes_per_txn": 32,
                       "launch": {s: tpcc_launch(args, s, 148) for s in schemes} if args.launch == "tuned"
                       else "bs 8, full-occupancy grid",
                       "parallelism": f"warehouse-partitioned x{world}" + (
                           (" (in-library exchange over NVLink peer memory)" if p2p else " (NCCL all-to-all)")
                           if world > 1 else ""),
                       "phase_b": "2PC rounds for the six non-deterministic schemes (f-2), deterministic for GPUTx/GaccO" if args.two_pc else "deterministic"},
            "per_scheme": per, "clocks": clk,
            "gpu_launches": launches_per_step(schemes) * args.steps + (0 if world == 1 else
                                                                       6 * len(schemes) * args.steps),
            **({} if args.no_cpu_baseline else {"cpu_baseline": tpcc_cpu_baseline(args)})}), flush=True)
    db.close()
    if world > 1:
        dist.destroy_process_group()


def tpcc_cpu_baseline(args, warehouses=8):
    """The TPC-C oracle as it stands (oracle/: plain C serial NewOrder / Payment), one host
    core, replaying configs[4]-shaped batches (same mix, NURand, remote rates) over an
    8-warehouse population (per-transaction work does not depend on W; 512 warehouses of
    population do not fit a bounded CPU sample)."""
    import numpy as np
    import inputs.tpcc as IT
    from oracle import tpcc as OT
    try:
        os.sched_setaffinity(0, {sorted(os.sched_getaffinity(0))[0]})
    except Exception:
        pass
    S0 = IT.population(1, warehouses)
    n_txn = args.tpcc_batch
    tx = np.ascontiguousarray(OT.gen(5, warehouses, n_txn, args.tpcc_mix, IT.nurand_consts(1)), np.uint32)
    S = {k: np.array(S0[k], np.uint64, copy=True, order="C") for k in OT.TABLES}
    S["item"] = np.ascontiguousarray(S0["item"], np.uint64)
    S.update(OT.empty_slots(n_txn))
    order = np.arange(n_txn, dtype=np.uint32)
    out = np.zeros(n_txn * OT.OUT_WORDS, np.uint64)
    L, P = OT._lib(), OT._ptr
    args_ = [warehouses] + [P(S[k]) for k in ("warehouse", "district", "customer", "stock", "item", "order",
                                               "new_order", "order_line", "history")]
    done, n, t0 = 0, 0, time.perf_counter()
    while True:   # the same batch again on the evolving state: every transaction still executes
        st = L.orc_tpcc_replay(*args_, 20240601, n_txn, P(tx), P(order), n_txn, P(out))
        assert st == 0, st
        done += n_txn
        n += 1
        el = time.perf_counter() - t0
        if el >= min(args.cpu_seconds, 30.0):
            break
    return {"value": done / el, "unit": "txn/s", "cores": 1, "kind": "oracle",
            "sample": f"serial replay of {n} x {n_txn}-txn TPC-C batches (NewOrder {args.tpcc_mix}/10^4, "
                      f"Payment otherwise) over an {warehouses}-warehouse population, 1 core"}


def main():
    args = parse()
    rank, world, local = dist_env()
    if args.impl == "reference":
        run_reference(args, rank, world)
        return
    if args.workload == "tpcc":
        if args.loopback:
            run_tpcc_loopback(args, local)
        else:
            run_tpcc(args, rank, world, local)
        return
    run_ours(args, rank, world, local)


if __name__ == "__main__":
    main()
