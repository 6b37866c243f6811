"""High-contention probe: YCSB configs[1] (10,485,760 rows, 64K x 16, W=0.1) at the given
thetas, the given schemes, in the paper's thread launch (wd=0, bs=32, full grid) and the
bench's tile-16 launch; median of `reps` timed submits; one JSON line per cell.

  python tools/probe_hc.py --thetas 0.6,0.8,0.9,0.95,0.99 --schemes tpl_wd,to --tag base
"""
import argparse
import json
import os
import statistics
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import bench  # noqa: E402
import inputs  # noqa: E402
from paper_2406_10158_b200.api import DB  # noqa: E402
from paper_2406_10158_b200.gcctb import CC_FLAG_TIMING  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--thetas", default="0.6,0.8,0.9,0.95,0.99")
    ap.add_argument("--schemes", default="tpl_nw,tpl_wd,to,mvcc,silo,tictoc")
    ap.add_argument("--modes", default="thread,tile")
    ap.add_argument("--reps", type=int, default=2)
    ap.add_argument("--tag", default="")
    ap.add_argument("--flags", type=lambda x: int(x, 0), default=0)
    a = ap.parse_args()
    n = 10 * (1 << 20)
    db = DB(0)
    db.load_ycsb(n, 1)
    A = inputs.scramble_mult(n)
    for th in [float(x) for x in a.thetas.split(",")]:
        T = inputs.zipf_thresholds(n, th)
        b = db.gen_ycsb(1 << 16, 16, 0.1, 3, T, A)
        for s in a.schemes.split(","):
            for mode in a.modes.split(","):
                la = dict(lanes=1, wd=0, bs=32) if mode == "thread" else dict(lanes=32, wd=0, bs=bench.TUNED_BS[s],
                                                                              grid=db.num_sms)
                db.submit(b, s, watchdog_s=120, flags=a.flags, **la)
                db.sync()
                tots, ab, cm = [], 0, 0
                for _ in range(a.reps):
                    db.timing(reset=True)
                    db.submit(b, s, watchdog_s=120, flags=a.flags | CC_FLAG_TIMING, **la)
                    st = db.sync()
                    ms, _ = db.timing(reset=True)
                    tots.append(ms[4])
                    ab += st.aborts
                    cm += st.commits
                med = statistics.median(tots)
                print(json.dumps({"tag": a.tag, "theta": th, "scheme": s, "mode": mode, "txn_s": (1 << 16) / (med / 1e3),
                                  "abort_rate": ab / max(cm, 1), "ms": med}), flush=True)
        b.free()
    db.close()


if __name__ == "__main__":
    main()
