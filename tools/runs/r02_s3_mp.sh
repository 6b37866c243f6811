export PYTHONUNBUFFERED=1
python - <<'P'
import sys, json, types
sys.path.insert(0, '.')
import bench
base = [c for c in bench.TPCC_CONFIGS if c["W"] in (64, 512)]
for mp in (True, False):
    bench.TPCC_CONFIGS = [dict(c, meta_pad=mp) for c in base]
    out = bench.tpcc_block(types.SimpleNamespace(), 0, ["tpl_nw", "to", "silo", "tictoc", "gacco"])
    for k, v in out.items():
        print("meta_pad", mp, k, round(v["value"] / 1e6, 2), {s: (round(x["txn_s"] / 1e6, 2), round(x["exec_ms"], 3)) for s, x in v["per_scheme"].items()}, flush=True)
P
