"""Quick perf probe (not the bench): C2-shaped YCSB, every scheme, a few thetas."""
import argparse
import json
import statistics
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402

import inputs  # noqa: E402
from paper_2406_10158_b200.api import DB  # noqa: E402
from paper_2406_10158_b200.gcctb import CC_FLAG_TIMING, SCHEMES  # noqa: E402


def cell(db, b, s, a):
    kw = dict(wd=a.wd, bs=a.bs, watchdog_s=a.watchdog, lanes=a.lanes, grid=a.grid, claim_chunk=a.chunk)
    db.submit(b, s, flags=IDXF[a.index] | a.flags, **kw)
    db.sync()
    tots, execs = [], []
    aborts = commits = 0
    for _ in range(a.reps):
        db.timing(reset=True)
        db.submit(b, s, flags=CC_FLAG_TIMING | IDXF[a.index] | a.flags, **kw)
        st = db.sync()
        ms, n = db.timing(reset=True)
        tots.append(ms[4])
        execs.append(ms[2])
        aborts += st.aborts
        commits += st.commits
    med = statistics.median(tots)
    return dict(txn_s=a.batch / (med / 1e3), abort_rate=aborts / commits, ms_total_median=med,
                max_rank=int(st.max_rank),
                ms_total_min=min(tots), ms_total_max=max(tots), ms_exec_median=statistics.median(execs))


IDXF = {"dense": 0, "tree": 0x100, "binary": 0x10, "eytz": 0x1000}


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--rows", type=int, default=10 * (1 << 20))
    ap.add_argument("--batch", type=int, default=1 << 16)
    ap.add_argument("--K", type=int, default=16)
    ap.add_argument("--W", type=float, default=0.1)
    ap.add_argument("--thetas", default="0,0.6,0.8,0.99")
    ap.add_argument("--schemes", default=",".join(SCHEMES))
    ap.add_argument("--wd", type=int, default=0)
    ap.add_argument("--bs", type=int, default=32)
    ap.add_argument("--reps", type=int, default=3)
    ap.add_argument("--lanes", type=int, default=1)
    ap.add_argument("--index", default="dense", choices=["dense", "tree", "binary", "eytz"])
    ap.add_argument("--grid", type=int, default=0)
    ap.add_argument("--seeds", default="3")
    ap.add_argument("--chunk", type=int, default=1)
    ap.add_argument("--flags", type=lambda x: int(x, 0), default=0)
    ap.add_argument("--watchdog", type=float, default=20)
    a = ap.parse_args()
    db = DB(0)
    db.load_ycsb(a.rows, 1)
    A = inputs.scramble_mult(a.rows)
    out = []
    for th, seed in [(float(x), int(sd)) for x in a.thetas.split(",") for sd in a.seeds.split(",")]:
        T = torch.from_numpy(inputs.zipf_thresholds(a.rows, th).view(np.int64)).cuda()
        b = db.gen_ycsb(a.batch, a.K, a.W, seed, T, A)
        for s in a.schemes.split(","):
            base = dict(theta=th, seed=seed, chunk=a.chunk, scheme=s, wd=a.wd, bs=a.bs, lanes=a.lanes, grid=a.grid,
                        index=a.index, flags=a.flags, reps=a.reps)
            try:
                row = dict(base, **cell(db, b, s, a))
            except Exception as e:   # watchdog etc.: recorded; the db is rebuilt
                row = dict(base, error=str(e)[:200])
                db.close()
                db = DB(0)
                db.load_ycsb(a.rows, 1)
                b = db.gen_ycsb(a.batch, a.K, a.W, seed, T, A)
            out.append(row)
            print(json.dumps(row), flush=True)
        b.free()


if __name__ == "__main__":
    main()
