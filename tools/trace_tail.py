"""Commit-time profile of one executor launch (experiment; needs a -DGC_TRACE_COMMIT=1
variant build loaded with GCCTB_LIB): when, after the kernel starts, the batch's
commits and aborts happen -- is the time a throughput phase or a hot-record tail?

  python paper_2406_10158_b200/build.py --out variants/trace.so "-DGC_TRACE_COMMIT=1"
  GCCTB_LIB=variants/trace.so python tools/trace_tail.py --schemes tpl_nw,to --thetas 0.6
"""
import argparse
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402

import inputs  # noqa: E402
from paper_2406_10158_b200.api import DB  # noqa: E402
from paper_2406_10158_b200.gcctb import CC_FLAG_TIMING  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--rows", type=int, default=10 * (1 << 20))
    ap.add_argument("--batch", type=int, default=1 << 16)
    ap.add_argument("--K", type=int, default=16)
    ap.add_argument("--W", type=float, default=0.1)
    ap.add_argument("--thetas", default="0.6")
    ap.add_argument("--schemes", default="tpl_nw,tpl_wd,to,mvcc,silo,tictoc")
    ap.add_argument("--lanes", type=int, default=16)
    ap.add_argument("--bs", type=int, default=16)
    ap.add_argument("--grid", type=int, default=148)
    ap.add_argument("--bucket_ns", type=int, default=5000)
    ap.add_argument("--flags", type=lambda x: int(x, 0), default=0)
    a = ap.parse_args()
    assert os.environ.get("GCCTB_LIB"), "load a GC_TRACE_COMMIT variant with GCCTB_LIB"
    db = DB(0)
    db.load_ycsb(a.rows, 1)
    dev = torch.device("cuda", 0)
    A = inputs.scramble_mult(a.rows)
    for th in [float(x) for x in a.thetas.split(",")]:
        T = torch.from_numpy(inputs.zipf_thresholds(a.rows, th).view(np.int64)).to(dev)
        b = db.gen_ycsb(a.batch, a.K, a.W, 3, T, A)
        for s in a.schemes.split(","):
            kw = dict(wd=0, bs=a.bs, lanes=a.lanes, grid=a.grid, watchdog_s=30)
            db.submit(b, s, flags=a.flags, **kw)
            db.sync()
            tr = torch.zeros(2050, dtype=torch.int64, device=dev)
            tr[1] = a.bucket_ns
            torch.cuda.synchronize()
            os.environ["GCCTB_TRACE_PTR"] = str(tr.data_ptr())
            db.timing(reset=True)
            db.submit(b, s, flags=CC_FLAG_TIMING | a.flags, **kw)
            st = db.sync()
            del os.environ["GCCTB_TRACE_PTR"]
            ms, _ = db.timing(reset=True)
            h = tr.cpu().numpy()
            c, ab = h[2:1026], h[1026:2050]
            cum = np.cumsum(c)
            n = int(cum[-1])
            q = {f"t{int(f * 100)}_us": float((np.searchsorted(cum, f * n) + 1) * a.bucket_ns / 1e3) for f in (0.5, 0.9, 0.99, 1.0)}
            last = int(np.nonzero(c + ab)[0].max()) + 1
            print(json.dumps(dict(theta=th, scheme=s, flags=a.flags, commits=n, aborts=int(st.aborts), exec_ms=ms[2],
                                  bucket_us=a.bucket_ns / 1e3, **q, commits_hist=c[:last].tolist(),
                                  aborts_hist=ab[:last].tolist())), flush=True)
        b.free()
    db.close()


if __name__ == "__main__":
    main()
