import sys, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import inputs, oracle
from paper_2406_10158_b200.api import DB

def run(n, B, K, W, theta, scheme, lanes, seed=77):
    db = DB(0)
    db.load_ycsb(n, 5)
    S0 = inputs.ycsb_rows(5, n)
    T = inputs.zipf_thresholds(n, theta); A = inputs.scramble_mult(n)
    b = db.gen_ycsb(B, K, W, seed, T, A)
    keys, ops = oracle.ycsb_gen(seed, n, B, K, W, T, A)
    res = db.submit(b, scheme, wd=0, bs=32, lanes=lanes)
    st = db.sync()
    h = res.host(db.stream)
    out = h["read_out"].reshape(B, K)
    zero_rows = np.nonzero((out == 0).any(axis=1))[0]
    msg = f"n={n} B={B} K={K} th={theta} {scheme} lanes={lanes}: commits={st.commits} aborts={st.aborts} zero-out txns={zero_rows.size}"
    try:
        oracle.check_ycsb(scheme, S0, keys, ops, K, h, db.read_table(0))
        msg += " PARITY OK"
    except AssertionError as e:
        msg += " FAIL " + str(e)[:150]
        if zero_rows.size:
            g = zero_rows[:3]
            msg += f"\n   zero gids {g.tolist()} restarts {h['restarts'][g].tolist()} lo {h['order_lo'][g].tolist()} outs {out[g[0]].tolist()[:6]}"
    print(msg, flush=True)
    db.close()

for args in [(1 << 16, 4096, 16, 0.1, 0.6), (1 << 20, 8192, 16, 0.1, 0.6), (10 << 20, 1 << 16, 16, 0.1, 0.6),
             (1024, 1024, 4, 0.5, 0.8), (1 << 16, 4096, 4, 0.1, 0.6)]:
    for scheme in ["to", "mvcc", "silo", "tpl_nw"]:
        for lanes in [16, 4] if args[2] <= 4 else [16]:
            run(*args, scheme, lanes)
