"""Summarise a bench.py JSON line: value, step, roofline, per-scheme exec / submit / median step ms."""
import json
import sys

for f in sys.argv[1:]:
    d = json.loads(open(f).read().strip().splitlines()[-1])
    print(f, "value %.1f M" % (d["value"] / 1e6), "step %.3f ms" % d["ms_per_step"], "frac %.4f" % d["roofline"]["frac"],
          "e2e %.1f M" % (d["e2e"]["value"] / 1e6), "max/med %.2f" % d["step_ms_max_over_median"])
    med = {s: sorted(v)[len(v) // 2] for s, v in d["step_scheme_ms"].items()}
    for s, v in d["per_scheme"].items():
        print("  %-7s exec %.3f submit %.3f step-med %.3f abort %.3f" % (s, v["exec_ms"], v["submit_ms"], med[s], v["abort_rate"]))
