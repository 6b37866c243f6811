"""The gather ceiling against access size (cc_gather_sweep): GB/s and accesses/s of random
32 / 64 / 128 / 256 B reads over 1 GiB; run under `ncu --metrics dram__bytes_read.sum,
gpu__time_duration.sum -k regex:roof_gather_sweep` to check the GB/s against DRAM bytes."""
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2406_10158_b200.api import DB  # noqa: E402

db = DB(0)
r = db.gather_sweep()
print(json.dumps({"gather_gbs": r, "accesses_per_s": {k: v * 1e9 / k for k, v in r.items()}}))
db.close()
