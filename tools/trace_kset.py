"""Per-K-set timeline of one GPUTx executor launch (experiment; needs a
-DGC_TRACE_COMMIT=1 variant loaded with GCCTB_LIB): when each K-set completed and when its
first member passed the gate -- the hand-off (detection) and the work of every K-set.

  GCCTB_LIB=variants/trace.so python tools/trace_kset.py --thetas 0.6
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
    ap.add_argument("--thetas", default="0.6")
    ap.add_argument("--bs", type=int, default=8)
    a = ap.parse_args()
    assert os.environ.get("GCCTB_LIB"), "load a GC_TRACE_COMMIT variant with GCCTB_LIB"
    db = DB(0)
    db.load_ycsb(a.rows, 1)
    dev = torch.device("cuda", 0)
    A = inputs.scramble_mult(a.rows)
    for th in [float(x) for x in a.thetas.split(",")]:
        T = torch.from_numpy(inputs.zipf_thresholds(a.rows, th).view(np.int64)).to(dev)
        b = db.gen_ycsb(1 << 16, 16, 0.1, 3, T, A)
        kw = dict(wd=0, bs=a.bs, lanes=32, grid=db.num_sms, watchdog_s=30)
        db.submit(b, "gputx", **kw)
        db.sync()
        tr = torch.zeros(6146, dtype=torch.int64, device=dev)
        tr[1] = 5000
        tr[4098:] = np.iinfo(np.int64).max
        torch.cuda.synchronize()
        os.environ["GCCTB_TRACE_PTR"] = str(tr.data_ptr())
        db.timing(reset=True)
        db.submit(b, "gputx", flags=CC_FLAG_TIMING, **kw)
        st = db.sync()
        del os.environ["GCCTB_TRACE_PTR"]
        ms, _ = db.timing(reset=True)
        h = tr.cpu().numpy()
        t0, K = h[0], min(int(st.max_rank) + 1, 2048)
        done = (h[2050:2050 + K] - t0) / 1e3
        first = (h[4098:4098 + K] - t0) / 1e3
        first[0] = 0.0
        detect = first[1:] - done[:-1]        # K-set k-1 complete -> first member of k past the gate
        work = done[1:] - first[1:]           # first member of k past the gate -> k complete
        print(json.dumps(dict(theta=th, ksets=K, exec_ms=ms[2], done0_us=float(done[0]),
                              detect_med_us=float(np.median(detect)), work_med_us=float(np.median(work)),
                              detect_p90_us=float(np.percentile(detect, 90)), work_p90_us=float(np.percentile(work, 90)),
                              tail_from_us=float(done[0]), end_us=float(done[-1]),
                              done_us=[round(float(x), 2) for x in done], first_us=[round(float(x), 2) for x in first])),
              flush=True)
        b.free()
    db.close()


if __name__ == "__main__":
    main()
