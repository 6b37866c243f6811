"""Packed vs padded control words (CC_FLAG_META_PAD, f-3) per workload: YCSB configs[1]
at theta 0 and 0.6 in the bench's tile launch, and TPC-C configs[3] / the configs[4] shape
in the bench's TPC-C-block launches; median of 3 submits; one JSON line per cell."""
import json
import os
import statistics
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import bench  # noqa: E402
import inputs  # noqa: E402
from paper_2406_10158_b200.api import DB  # noqa: E402
from paper_2406_10158_b200.gcctb import CC_FLAG_META_PAD, CC_FLAG_TIMING  # noqa: E402

SCHEMES = ["tpl_nw", "tpl_wd", "to", "silo", "tictoc"]   # the single-word schemes


def timed(db, b, s, flags, reps=3, **la):
    db.submit(b, s, flags=flags, watchdog_s=120, **la)
    db.sync()
    t = []
    for _ in range(reps):
        db.timing(reset=True)
        db.submit(b, s, flags=flags | CC_FLAG_TIMING, watchdog_s=120, **la)
        db.sync()
        t.append(db.timing(reset=True)[0][2])   # exec ms
    return statistics.median(t)


def main():
    n = 10 * (1 << 20)
    db = DB(0)
    db.load_ycsb(n, 1)
    A = inputs.scramble_mult(n)
    for th in (0.0, 0.6):
        b = db.gen_ycsb(1 << 16, 16, 0.1, 3, inputs.zipf_thresholds(n, th), A)
        for s in SCHEMES:
            la = dict(lanes=32, wd=0, bs=bench.TUNED_BS[s], grid=db.num_sms)
            for pad in (0, 1):
                ms = timed(db, b, s, CC_FLAG_META_PAD if pad else 0, **la)
                print(json.dumps({"workload": f"ycsb theta={th}", "scheme": s, "pad": pad, "exec_ms": ms}), flush=True)
        b.free()
    db.close()
    for cfg in bench.TPCC_CONFIGS[1:]:
        db = DB(0)
        db.load_tpcc(cfg["W"], 1, cfg["n"])
        b = db.gen_tpcc(cfg["n"], 5, cfg["mix"])
        for s in SCHEMES:
            bs, per_sm = cfg["launch"].get(s, cfg["launch"]["*"])
            for pad in (0, 1):
                ms = timed(db, b, s, CC_FLAG_META_PAD if pad else 0, lanes=32, bs=bs, grid=db.num_sms if per_sm else 0)
                print(json.dumps({"workload": cfg["name"], "scheme": s, "pad": pad, "exec_ms": ms}), flush=True)
        b.free()
        db.close()


if __name__ == "__main__":
    main()
