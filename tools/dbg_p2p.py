import os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from paper_2406_10158_b200.api import DB
from paper_2406_10158_b200.partition import p2p_round
G_ = int(sys.argv[1]) if len(sys.argv) > 1 else 2
W, n = 8, 2048
wpr = W // G_
dbs, bs = [], []
for r in range(G_):
    db = DB(0, rank=r, world=G_)
    db.load_tpcc(W, 17, n, w_first=r * wpr, w_count=wpr)
    dbs.append(db)
    bs.append(db.gen_tpcc(n, 100 + r, 5114, w_lo=r * wpr, w_hi=(r + 1) * wpr))
DB.part_connect_local(dbs)
torch.cuda.synchronize()
for s in sys.argv[2].split(","):
    t = time.time()
    for db, b in zip(dbs, bs):
        t0 = time.time()
        p2p_round(db, b, s, bs=8, lanes=32, watchdog_s=8)
        print(s, "enqueue rank", db.rank, round(time.time() - t0, 3), flush=True)
    for db in dbs:
        try:
            print(s, "rank", db.rank, "commits", db.sync().commits, round(time.time() - t, 2), flush=True)
        except Exception as e:
            print(s, "rank", db.rank, "ERR", e, flush=True)
