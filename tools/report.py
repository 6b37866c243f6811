"""Render sweep JSONL files (tools/sweep.py) as markdown tables."""
import json
import sys
from collections import defaultdict

SCHEMES = ["tpl_nw", "tpl_wd", "to", "mvcc", "silo", "tictoc", "gputx", "gacco"]


def load(path):
    return [json.loads(l) for l in open(path) if l.startswith("{")]


def fmt(v):
    if v is None:
        return "—"
    if v >= 1e6:
        return f"{v / 1e6:.1f}M"
    return f"{v / 1e3:.0f}K"


def theta_table(rows):
    out = []
    for mode in sorted({r["mode"] for r in rows}):
        th = sorted({r["theta"] for r in rows if r["mode"] == mode})
        out.append(f"\n**{mode}** — committed txn/s (abort rate)\n")
        out.append("| θ | " + " | ".join(SCHEMES) + " |")
        out.append("|---|" + "---|" * len(SCHEMES))
        cell = {(r["theta"], r["scheme"]): r for r in rows if r["mode"] == mode}
        for t in th:
            vals = []
            for s in SCHEMES:
                r = cell.get((t, s))
                if r is None:
                    vals.append("skipped")
                elif "error" in r:
                    vals.append("err")
                else:
                    vals.append(f"{fmt(r['txn_s'])} ({r['abort_rate']:.2f})")
            out.append(f"| {t} | " + " | ".join(vals) + " |")
    return "\n".join(out)


def preset_table(rows):
    out = ["| preset | mode | " + " | ".join(SCHEMES) + " |", "|---|---|" + "---|" * len(SCHEMES)]
    cell = {(r["preset"], r["mode"], r["scheme"]): r for r in rows}
    for p in ("RO", "MC", "HC"):
        for m in sorted({r["mode"] for r in rows}):
            vals = []
            for s in SCHEMES:
                r = cell.get((p, m, s))
                vals.append("—" if r is None else ("err" if "error" in r else f"{fmt(r['txn_s'])} ({r['abort_rate']:.2f})"))
            out.append(f"| {p} | {m} | " + " | ".join(vals) + " |")
    return "\n".join(out)


def wdbs_table(rows):
    out = []
    for s in SCHEMES:
        rs = [r for r in rows if r["scheme"] == s and "txn_s" in r]
        if not rs:
            continue
        grid = defaultdict(dict)
        for r in rs:
            grid[r["wd"]][r["bs"]] = r["txn_s"]
        best = max(rs, key=lambda r: r["txn_s"])
        out.append(f"\n**{s}** — best wd={best['wd']} bs={best['bs']}: {fmt(best['txn_s'])}\n")
        bss = sorted({r["bs"] for r in rs})
        out.append("| wd \\ bs | " + " | ".join(str(b) for b in bss) + " |")
        out.append("|---|" + "---|" * len(bss))
        for wd in sorted(grid):
            out.append(f"| {wd} | " + " | ".join(fmt(grid[wd].get(b)) for b in bss) + " |")
    return "\n".join(out)


def stages_table(rows):
    st = ["index", "ts_alloc", "wait", "cc_manager", "abort", "useful"]
    out = ["| preset | mode | lookup | scheme | " + " | ".join(st) + " | (ns per committed txn) |",
           "|---|---|---|---|" + "---|" * len(st) + "---|"]
    for r in rows:
        if "stage_ns_per_txn" not in r:
            continue
        d = r["stage_ns_per_txn"]
        out.append(f"| {r['preset']} | {r['mode']} | {r.get('index', 'tree')} | {r['scheme']} | "
                   + " | ".join(f"{d[k]:.0f}" for k in st) + " | |")
    return "\n".join(out)


def latch_table(rows):
    out = ["| preset | mode | scheme | latch-free | latched | ratio |", "|---|---|---|---|---|---|"]
    cell = {(r["preset"], r["mode"], r["scheme"], r["latched"]): r for r in rows if "txn_s" in r}
    for (p, m, s, lt), r in sorted(cell.items()):
        if lt:
            continue
        l2 = cell.get((p, m, s, True))
        if l2:
            out.append(f"| {p} | {m} | {s} | {fmt(r['txn_s'])} | {fmt(l2['txn_s'])} | {r['txn_s'] / l2['txn_s']:.2f} |")
    return "\n".join(out)


def main():
    for path in sys.argv[1:]:
        rows = load(path)
        if not rows:
            continue
        exp = rows[0].get("exp")
        print(f"\n### {path}\n")
        print({"theta": theta_table, "preset": preset_table, "tpcc_wdbs": wdbs_table, "stages": stages_table,
               "latch": latch_table}[exp](rows))


if __name__ == "__main__":
    main()
