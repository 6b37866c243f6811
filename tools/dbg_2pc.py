"""Repeat the G=4 loopback 2PC check (tests/test_gpu_partition.py::test_loopback_2pc) until
a mismatch, then print what differs: which words of which transactions, whether they
were local (phase A) or distributed (2PC rounds), their rounds and restarts."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402

from inputs import tpcc as IT  # noqa: E402
from oracle import tpcc as OT  # noqa: E402
from oracle import order_from_result  # noqa: E402
from paper_2406_10158_b200.api import DB  # noqa: E402
from paper_2406_10158_b200.partition import loopback_round_2pc  # noqa: E402

POP = ["warehouse", "district", "customer", "stock"]


def once(scheme, G_, it):
    W, n = 8, 2048
    wpr = W // G_
    dbs, batches = [], []
    for r in range(G_):
        db = DB(0, rank=r, world=G_)
        db.load_tpcc(W, 17, n, w_first=r * wpr, w_count=wpr)
        dbs.append(db)
        batches.append(db.gen_tpcc(n, 300 + r, 5114, w_lo=r * wpr, w_hi=(r + 1) * wpr))
    S0 = IT.population(17, W)
    res, rounds = loopback_round_2pc(dbs, batches, scheme, bs=8, lanes=32)
    for db in dbs:
        assert db.sync().commits == n
    txs = [b.export_tpcc() for b in batches]
    hs = [r.host(db.stream) for r, db in zip(res, dbs)]
    m = {k: np.concatenate([h[k] for h in hs]) for k in ("committed", "order_hi", "order_lo", "restarts")}
    m["read_out"] = np.concatenate([h["read_out"] for h in hs])
    pos = np.empty(len(m["committed"]), np.uint32)
    pos[np.lexsort((m["order_lo"], m["order_hi"]))] = np.arange(len(pos))
    tx = np.concatenate(txs)
    pi = order_from_result(m["committed"], pos, m["order_hi"], m["order_lo"])
    S, out = OT.replay(S0, tx, pi, W)
    og = np.asarray(m["read_out"], np.uint64).reshape(-1, OT.OUT_WORDS)
    oe = out.reshape(-1, OT.OUT_WORDS)
    bad = np.nonzero((og != oe).any(axis=1))[0]
    if bad.size:
        print(f"iter {it}: {scheme} G={G_} rounds={rounds}: {bad.size} txns differ")
        T = tx.reshape(-1, OT.TX_WORDS)
        for t in bad[:6]:
            w = np.nonzero(og[t] != oe[t])[0]
            hi = int(m["order_hi"][t])
            print(f"  txn {t} (rank {t // n}, type {T[t][0]}): words {w.tolist()} gpu {og[t][w].tolist()} exp {oe[t][w].tolist()}"
                  f" phase {'B(2PC) round ' + str(hi & 0xFFFFFFFF) if hi >> 63 else 'A'} lo {int(m['order_lo'][t])}"
                  f" restarts {int(m['restarts'][t])} pos {int(pos[t])}")
            print(f"    tx words {T[t][:24].tolist()}")
    for db in dbs:
        db.close()
    return bad.size


def main():
    scheme = sys.argv[1] if len(sys.argv) > 1 else "silo"
    iters = int(sys.argv[2]) if len(sys.argv) > 2 else 50
    fails = 0
    for it in range(iters):
        fails += once(scheme, 4, it) > 0
    print(f"{scheme}: {fails} of {iters} iterations differ")


if __name__ == "__main__":
    main()
