"""Experiment sweeps (one JSON line per cell), the harness of SPEC.md's cli module:

  theta   Exp-1: YCSB configs[1], W=0.1, theta 0 .. 0.99, every
          scheme, in the paper's launch (thread mode wd=0 bs=32) and the
          B200 tile mode (16 lanes per transaction).
  presets RO / MC / HC, both modes.
  stages  Exp-6: per-stage time per transaction on RO/MC/HC, every
          scheme, the paper's launch (wd=0, bs=32) and tile mode.
  latch   Exp-7: latch-free vs latched, six CPU-oriented schemes, presets.
  wdbs    Exp-3/4/5-style heatmap on TPC-C configs[3] (64 warehouses, 45:43 mix):
          wd in 0..5 x bs in {1,2,4,8,16,32} per scheme, thread mode.

Cells whose median time exceeds --budget-ms are recorded and the remaining (harder)
cells of that scheme/mode are skipped."""
import argparse
import json
import os
import statistics
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402

import inputs  # noqa: E402
from paper_2406_10158_b200.api import DB  # noqa: E402
from paper_2406_10158_b200.gcctb import CC_FLAG_TIMING, SCHEMES  # noqa: E402

MODES = {"paper_wd0_bs32": dict(lanes=1, wd=0, bs=32), "tile16": dict(lanes=16, wd=0, bs=32),
         "bench_tile32": "bench"}   # the bench's launch: 32-lane tiles, bench.TUNED_BS warps, one block per SM


def mode_kw(kw, scheme, db):
    if kw == "bench":
        import bench
        return dict(lanes=32, wd=0, bs=bench.TUNED_BS[scheme], grid=db.num_sms)
    return kw


def cell(db, b, scheme, reps, watchdog, **kw):
    db.submit(b, scheme, watchdog_s=watchdog, **kw)   # warm-up
    db.sync()
    tots, ab, cm = [], 0, 0
    for _ in range(reps):
        db.timing(reset=True)
        db.submit(b, scheme, flags=CC_FLAG_TIMING, watchdog_s=watchdog, **kw)
        st = db.sync()
        ms, _ = db.timing(reset=True)
        tots.append(ms[4])
        ab += st.aborts
        cm += st.commits
    med = statistics.median(tots)
    return dict(ms_median=med, ms_min=min(tots), ms_max=max(tots), txn_s=b.n_txn / (med / 1e3),
                abort_rate=ab / max(cm, 1))


IDXF = {"dense": 0, "tree": 0x100, "binary": 0x10, "eytz": 0x1000}   # CC_FLAG_INDEX_TREE / CC_FLAG_INDEX_BINARY


def ycsb_db(rows):
    db = DB(0)
    db.load_ycsb(rows, 1)
    return db


def sweep_theta(a, out):
    db = ycsb_db(a.rows)
    A = inputs.scramble_mult(a.rows)
    thetas = [0.0, 0.1, 0.2, 0.3, 0.4, 0.5, 0.6, 0.7, 0.8, 0.9, 0.95, 0.99]
    dead = set()
    for th in thetas:
        T = torch.from_numpy(inputs.zipf_thresholds(a.rows, th).view(np.int64)).cuda()
        b = db.gen_ycsb(a.batch, 16, 0.1, 11, T, A)
        for mode, kw in MODES.items():
            for s in SCHEMES:
                if (mode, s) in dead:
                    continue
                try:
                    r = cell(db, b, s, a.reps, a.watchdog, **mode_kw(kw, s, db))
                except Exception as e:   # watchdog / overflow: recorded, not fatal
                    r = dict(error=str(e)[:120])
                    dead.add((mode, s))
                    db.close()
                    db = ycsb_db(a.rows)
                    b = db.gen_ycsb(a.batch, 16, 0.1, 11, T, A)
                r.update(exp="theta", theta=th, W=0.1, mode=mode, scheme=s)
                out.write(json.dumps(r) + "\n")
                out.flush()
                if r.get("ms_median", 0) > a.budget_ms:
                    dead.add((mode, s))
        b.free()
    db.close()


def sweep_presets(a, out):
    db = ycsb_db(a.rows)
    A = inputs.scramble_mult(a.rows)
    for name, (W, th) in {"RO": (0.0, 0.0), "MC": (0.1, 0.6), "HC": (0.5, 0.8)}.items():
        T = torch.from_numpy(inputs.zipf_thresholds(a.rows, th).view(np.int64)).cuda()
        b = db.gen_ycsb(a.batch, 16, W, 12, T, A)
        for mode, kw in MODES.items():
            for s in SCHEMES:
                try:
                    r = cell(db, b, s, a.reps, a.watchdog, **mode_kw(kw, s, db))
                except Exception as e:
                    r = dict(error=str(e)[:120])
                    db.close()
                    db = ycsb_db(a.rows)
                    b = db.gen_ycsb(a.batch, 16, W, 12, T, A)
                r.update(exp="preset", preset=name, theta=th, W=W, mode=mode, scheme=s)
                out.write(json.dumps(r) + "\n")
                out.flush()
        b.free()
    db.close()


PRESETS = {"RO": (0.0, 0.0), "MC": (0.1, 0.6), "HC": (0.5, 0.8)}


def sweep_stages(a, out):
    from paper_2406_10158_b200.gcctb import CC_FLAG_STAGES, STAGES
    db = ycsb_db(a.rows)
    A = inputs.scramble_mult(a.rows)
    for name, (W, th) in PRESETS.items():
        T = torch.from_numpy(inputs.zipf_thresholds(a.rows, th).view(np.int64)).cuda()
        b = db.gen_ycsb(a.batch, 16, W, 13, T, A)
        for mode, kw in MODES.items():
            for s in SCHEMES:
                try:
                    db.timing(reset=True)
                    db.submit(b, s, flags=CC_FLAG_STAGES | CC_FLAG_TIMING | IDXF[a.index], watchdog_s=a.watchdog,
                              **mode_kw(kw, s, db))
                    st = db.sync()
                    ms, _ = db.timing(reset=True)
                    ns_per_cycle = 1e6 / max(st.sm_clock_khz, 1)
                    per_txn = {STAGES[k]: st.stage_cycles[k] * ns_per_cycle / max(st.commits, 1) for k in range(6)}
                    r = dict(stage_ns_per_txn=per_txn, attempts=st.stage_cycles[6], prep_ms=ms[1],
                             exec_ms=ms[2], abort_rate=st.aborts / max(st.commits, 1))
                except Exception as e:
                    r = dict(error=str(e)[:120])
                    db.close()
                    db = ycsb_db(a.rows)
                    b = db.gen_ycsb(a.batch, 16, W, 13, T, A)
                r.update(exp="stages", preset=name, mode=mode, scheme=s, index=a.index)
                out.write(json.dumps(r) + "\n")
                out.flush()
        b.free()
    db.close()


def sweep_latch(a, out):
    from paper_2406_10158_b200.gcctb import CC_FLAG_LATCHED
    db = ycsb_db(a.rows)
    A = inputs.scramble_mult(a.rows)
    for name, (W, th) in PRESETS.items():
        T = torch.from_numpy(inputs.zipf_thresholds(a.rows, th).view(np.int64)).cuda()
        b = db.gen_ycsb(a.batch, 16, W, 14, T, A)
        for mode, kw in MODES.items():
            for s in SCHEMES[:6]:
                for latched in (False, True):
                    try:
                        k2 = dict(mode_kw(kw, s, db))
                        r = cell(db, b, s, a.reps, a.watchdog, **k2) if not latched else \
                            cell_flags(db, b, s, a.reps, a.watchdog, CC_FLAG_LATCHED, **k2)
                    except Exception as e:
                        r = dict(error=str(e)[:120])
                        db.close()
                        db = ycsb_db(a.rows)
                        b = db.gen_ycsb(a.batch, 16, W, 14, T, A)
                    r.update(exp="latch", preset=name, mode=mode, scheme=s, latched=latched)
                    out.write(json.dumps(r) + "\n")
                    out.flush()
        b.free()
    db.close()


def cell_flags(db, b, scheme, reps, watchdog, flags, **kw):
    db.submit(b, scheme, watchdog_s=watchdog, flags=flags, **kw)
    db.sync()
    tots, ab, cm = [], 0, 0
    for _ in range(reps):
        db.timing(reset=True)
        db.submit(b, scheme, flags=CC_FLAG_TIMING | flags, watchdog_s=watchdog, **kw)
        st = db.sync()
        ms, _ = db.timing(reset=True)
        tots.append(ms[4])
        ab += st.aborts
        cm += st.commits
    med = statistics.median(tots)
    return dict(ms_median=med, ms_min=min(tots), ms_max=max(tots), txn_s=b.n_txn / (med / 1e3),
                abort_rate=ab / max(cm, 1))


def sweep_wdbs(a, out):
    db = DB(0)
    db.load_tpcc(64, 1, 65536)
    db.snapshot(True)
    b = db.gen_tpcc(65536, 7, 5114)
    for s in SCHEMES:
        for wd in range(6):
            for bs in (1, 2, 4, 8, 16, 32):
                db.snapshot(False)
                try:
                    r = cell(db, b, s, 1, a.watchdog, lanes=1, wd=wd, bs=bs)
                except Exception as e:
                    r = dict(error=str(e)[:120])
                r.update(exp="tpcc_wdbs", W=64, mode="thread", scheme=s, wd=wd, bs=bs)
                out.write(json.dumps(r) + "\n")
                out.flush()
    db.close()


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("exp", choices=["theta", "presets", "wdbs", "stages", "latch"])
    ap.add_argument("--rows", type=int, default=10 * (1 << 20))
    ap.add_argument("--batch", type=int, default=1 << 16)
    ap.add_argument("--reps", type=int, default=3)
    ap.add_argument("--watchdog", type=float, default=20.0)
    ap.add_argument("--budget-ms", type=float, default=3000.0)
    ap.add_argument("--out", default="-")
    ap.add_argument("--index", default="dense", choices=list(IDXF),
                    help="stages: YCSB index (binary = the paper's, PAPER.md:344)")
    a = ap.parse_args()
    out = sys.stdout if a.out == "-" else open(a.out, "a")
    t0 = time.time()
    {"theta": sweep_theta, "presets": sweep_presets, "wdbs": sweep_wdbs, "stages": sweep_stages,
     "latch": sweep_latch}[a.exp](a, out)
    sys.stderr.write(f"{a.exp} done in {time.time() - t0:.1f}s\n")


if __name__ == "__main__":
    main()
