"""TPC-C perf probe: committed txn/s and abort rate per scheme (not the bench)."""
import argparse
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2406_10158_b200.api import DB  # noqa: E402
from paper_2406_10158_b200.gcctb import CC_FLAG_TIMING, SCHEMES  # noqa: E402


def fresh(a):
    db = DB(0)
    db.load_tpcc(a.W, 1, a.batch)
    db.snapshot(True)
    return db, db.gen_tpcc(a.batch, 7, a.mix)


def cell(db, b, s, a):
    kw = dict(wd=a.wd, bs=a.bs, lanes=a.lanes, watchdog_s=a.watchdog, grid=a.grid)
    db.snapshot(False)
    db.submit(b, s, flags=a.flags, **kw)
    db.sync()
    db.timing(reset=True)
    for _ in range(a.reps):
        db.snapshot(False)
        db.submit(b, s, flags=CC_FLAG_TIMING | a.flags, **kw)
    st = db.sync()
    ms, n = db.timing(reset=True)
    per = [m / n for m in ms]
    return dict(txn_s=a.batch / (per[4] / 1e3), abort_rate=st.aborts / max(1, st.commits), ms_reset=per[0],
                ms_prep=per[1], ms_exec=per[2], ms_emit=per[3], ms_total=per[4])


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--W", type=int, default=1)
    ap.add_argument("--batch", type=int, default=16384)
    ap.add_argument("--mix", type=int, default=5000, help="NewOrder share in 1/10,000")
    ap.add_argument("--schemes", default=",".join(SCHEMES))
    ap.add_argument("--lanes", type=int, default=32)
    ap.add_argument("--wd", type=int, default=0)
    ap.add_argument("--bs", type=int, default=8)
    ap.add_argument("--reps", type=int, default=3)
    ap.add_argument("--grid", type=int, default=0, help="blocks (0: resident capacity)")
    ap.add_argument("--flags", type=lambda x: int(x, 0), default=0)
    ap.add_argument("--watchdog", type=float, default=30)
    a = ap.parse_args()
    db, b = fresh(a)
    for s in a.schemes.split(","):
        row = dict(W=a.W, batch=a.batch, mix=a.mix, scheme=s, lanes=a.lanes, wd=a.wd, bs=a.bs, grid=a.grid,
                   flags=a.flags)
        try:
            row.update(cell(db, b, s, a))
        except Exception as e:   # watchdog etc.: recorded, the db is rebuilt
            row["error"] = str(e)[:200]
            db.close()
            db, b = fresh(a)
        print(json.dumps(row), flush=True)


if __name__ == "__main__":
    main()
