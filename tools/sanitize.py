"""configs[0] (1,024 rows, 1,024 x 4 ops, W=0.5, theta=0.8) under every scheme in thread
and tile mode, and a 2-warehouse TPC-C batch in tile mode, each checked against the oracle
-- the workload `compute-sanitizer --tool memcheck|racecheck|synccheck` runs (SURVEY.md
§4, §5; the results go to profiles/r02_sanitize_*.txt):

  compute-sanitizer --tool memcheck python tools/sanitize.py
"""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import numpy as np  # noqa: E402

import inputs  # noqa: E402
import oracle  # noqa: E402
from paper_2406_10158_b200.api import DB  # noqa: E402

SCHEMES = ["tpl_nw", "tpl_wd", "to", "mvcc", "silo", "tictoc", "gputx", "gacco"]


def main():
    args = [a for a in sys.argv[1:] if not a.startswith("--")]
    small = "--small" in sys.argv   # racecheck: a quarter of the batch (its instrumentation is slow)
    only = args[0].split(",") if args else SCHEMES
    n_rows, B, K, W, theta = 1024, 256 if small else 1024, 4, 0.5, 0.8
    db = DB(0)
    db.load_ycsb(n_rows, 11)
    S0 = db.read_table(0)
    db.snapshot(True)
    T = inputs.zipf_thresholds(n_rows, theta)
    A = inputs.scramble_mult(n_rows)
    b = db.gen_ycsb(B, K, W, 5, T, A)
    keys, ops = oracle.ycsb_gen(5, n_rows, B, K, W, T, A)
    for scheme in only:
        for lanes, wd, bs in ((1, 5, 8), (1, 5, 32), (1, 0, 32), (4, 0, 8), (16, 0, 4), (32, 0, 4)):
            db.snapshot(False)
            db.prepare(b, scheme)
            res = db.submit(b, scheme, wd=wd, bs=bs, lanes=lanes, watchdog_s=600)
            st = db.sync()
            assert st.commits == B, (scheme, lanes, st.commits)
            oracle.check_ycsb(scheme, S0, keys, ops, K, res.host(db.stream), db.read_table(0))
            print(f"ycsb {scheme} lanes={lanes} wd={wd} bs={bs}: ok", flush=True)
    b.free()
    db.close()
    from inputs import tpcc as IT
    from oracle import tpcc as OT
    db = DB(0)
    NT = 128 if small else 512
    db.load_tpcc(2, 5, NT)
    P0 = IT.population(5, 2)
    db.snapshot(True)
    tb = db.gen_tpcc(NT, 3, 5114)
    tx = tb.export_tpcc()
    for scheme in only:
        for lanes in (1, 32):
            db.snapshot(False)
            res = db.submit(tb, scheme, wd=0, bs=8, lanes=lanes, watchdog_s=600)
            assert db.sync().commits == NT
            OT.check(scheme, P0, tx, 2, res.host(db.stream), db.read_tpcc(list(OT.TABLES + OT.SLOTS)))
            print(f"tpcc {scheme} lanes={lanes}: ok", flush=True)
    db.close()
    print("sanitize workload ok")


if __name__ == "__main__":
    main()
